"""Multi-process (gloo, world_size 2) tests of the snapshot-sharding host logic.

The GPU path needs one B200 per rank; here each rank runs the CPU oracle on its
shard and the single post-loop gather is checked against a single-process run
(independent shards => identical arithmetic => bitwise equal results).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_13592_b200.distributed import gather_rows, max_over_ranks, shard_bounds, workload_shard


def test_shard_bounds_partition():
    for total in (1, 7, 32, 64, 1024):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_bounds(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _solve_shard(lo, hi):
    from oracle import bccb_oracle as orc
    rng = np.random.default_rng(42)
    occ = np.zeros((4, 4), dtype=bool)
    occ[[0, 3, 1, 2], [1, 2, 0, 3]] = True
    l1, l2 = 8, 8
    eig_t = np.ascontiguousarray(orc.gram_eigenvalues_exact(occ, l1, l2).T)
    m1, m2 = orc.occupied_coordinates(occ)
    ys = rng.standard_normal((7, 4)) + 1j * rng.standard_normal((7, 4))
    out = []
    for s in range(lo, hi):
        b = orc.adjoint_fft(m1, m2, l1, l2, ys[s])
        out.append(orc.fista(eig_t, b, 0.1 * np.abs(b).max(), 1.0 / (l1 * l2), 25))
    return np.array(out).reshape(hi - lo, l1 * l2)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        total = 7
        # bench.py's own shard choice (strong scaling of a fixed global batch, configs 4/5)
        lo, hi = workload_shard(total, rank, world, strong=True)
        local = torch.from_numpy(_solve_shard(lo, hi))
        # bench.py's e2e gather: spectra (complex) and peak lists (int32) into rank 0's output only
        out = torch.empty((total, local.shape[1]), dtype=local.dtype) if rank == 0 else None
        full = gather_rows(local, total, out=out)
        idx = torch.arange(lo * 3, hi * 3, dtype=torch.int32).reshape(hi - lo, 3)
        idx_full = gather_rows(idx, total)
        m = max_over_ranks(float(rank + 1))
        if rank == 0:
            assert full is out
            q.put((full.numpy(), idx_full.numpy(), m))
        else:
            assert full is None and idx_full is None
    finally:
        dist.destroy_process_group()


def test_gloo_two_rank_gather_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, idx, m = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_array_equal(full, _solve_shard(0, 7))
    np.testing.assert_array_equal(idx, np.arange(21, dtype=np.int32).reshape(7, 3))
    assert m == 2.0


def test_workload_shard_strong_and_weak():
    # strong: BASELINE configs 4/5 split the fixed global batch; weak: every rank its own batch
    assert [workload_shard(32, r, 8, True) for r in range(8)] == [(4 * r, 4 * r + 4) for r in range(8)]
    assert [workload_shard(1024, r, 3, True) for r in range(3)] == [(0, 342), (342, 683), (683, 1024)]
    assert [workload_shard(64, r, 2, False) for r in range(2)] == [(0, 64), (64, 128)]
