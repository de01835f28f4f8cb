"""Snapshot sharding across GPUs: one process per GPU, no per-iteration communication.

Snapshots are independent (same geometry, Lambda and mu; per-snapshot tau), so
rank r solves the contiguous slice [r*B/P, (r+1)*B/P) and the only collective is
one gather to rank 0 after the loop: recovered spectra and peak
lists, as grouped point-to-point sends into rank 0's output (NCCL over
NVLink/NVSwitch on GPUs, gloo in the CPU tests).  This replaces the reference's
sequential per-trial sweep (pkg/src/bccblasso/experiments.py:330-349).
"""

import os

import torch
import torch.distributed as dist


def shard_bounds(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of `total` items for `rank` of `world` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def env_rank_world() -> tuple[int, int, int]:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def init(backend: str | None = None) -> tuple[int, int, int]:
    """Initialise torch.distributed from the torchrun environment (no-op for world 1)."""
    rank, world, local = env_rank_world()
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return rank, world, local


def workload_shard(batch: int, rank: int, world: int, strong: bool) -> tuple[int, int]:
    """Snapshot slice [lo, hi) this rank solves.

    strong=True : the global batch `batch` is split over the ranks (BASELINE configs 4/5:
                  "batch 1024 / 32 sharded across 1/2/4/8 GPUs");
    strong=False: every rank solves its own `batch` snapshots (weak scaling).
    """
    if strong:
        return shard_bounds(batch, rank, world)
    return rank * batch, (rank + 1) * batch


def _flat(t: torch.Tensor) -> torch.Tensor:
    # NCCL moves real dtypes; complex rows travel as interleaved (re, im) pairs
    return torch.view_as_real(t) if t.is_complex() else t


def gather_rows(local: torch.Tensor, total_rows: int, root: int = 0, out: torch.Tensor | None = None):
    """Gather row-sharded tensors (dim 0 split by shard_bounds) to `root` only.

    One grouped point-to-point exchange (NCCL send/recv over NVLink, or gloo on CPU):
    every other rank sends its rows straight into its slice of root's (total_rows, ...)
    output, so nothing is padded, concatenated or received by the non-root ranks
    (the only collective of the path).  Returns the full tensor on root
    (`out` if given) and None elsewhere.
    """
    if not dist.is_initialized() or dist.get_world_size() == 1:
        if out is None:
            return local
        out.copy_(local)
        return out
    world, rank = dist.get_world_size(), dist.get_rank()
    bounds = [shard_bounds(total_rows, r, world) for r in range(world)]
    lo, hi = bounds[rank]
    if local.shape[0] != hi - lo:
        raise ValueError(f"rank {rank} holds {local.shape[0]} rows, its shard is {hi - lo}")
    if rank != root:
        if hi > lo:
            for req in dist.batch_isend_irecv([dist.P2POp(dist.isend, _flat(local.contiguous()), root)]):
                req.wait()
        return None
    if out is None:
        out = torch.empty((total_rows,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    ops = []
    for r, (a, b) in enumerate(bounds):
        if r == root:
            out[a:b].copy_(local)
        elif b > a:
            ops.append(dist.P2POp(dist.irecv, _flat(out[a:b]), r))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return out


def max_over_ranks(value: float) -> float:
    """Max of a host scalar over ranks (multi-GPU timings are reported as the max)."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
