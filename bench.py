#!/usr/bin/env python
"""Benchmark of the fused BCCB-FISTA hot path (BASELINE.json metric, grid-point-iterations/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl b200|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU, NCCL)

A step = one full solve (T solver iterations) over this rank's batch of snapshots.
Default workload = BASELINE config 2 (configs[1], the metric's configuration):
FISTA, 64 snapshots per GPU, L1 = L2 = 256, T = 1000 (weak scaling: every rank
solves its own 64 snapshots).  `value` times the device-resident solve loop with
CUDA events (max over ranks); `e2e` times the public API end to end with host
(pinned) buffers: H2D of y, GPU adjoint, solve, top-K, D2H of spectra + peaks.
--impl reference times the reference algorithm (the pinned CPU oracle port,
oracle/bccb_oracle.py) on this host's cores.
"""

import argparse
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FISTA grid-point-iters/s (batch·L1·L2·iters/s); HBM GB/s vs B200 peak"
UNIT = "gpi/s"
# algorithmic bytes per grid-point-iteration ("FFT sweeps x 8 B")
B_ALG = {"ista": 64, "fista": 80, "admm": 80}
# share of the rows pass (K4+K2: 8 sweeps) and the column pass (K3: 2 sweeps) for FISTA
B_ALG_ROWS = {"ista": 48, "fista": 64, "admm": 64}
B_ALG_COLS = 16


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--iterations", type=int, default=None, help="override T (debug only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


# ----------------------------------------------------------------------------- CPU leg

def _cpu_worker(args):
    cfg, snap, iters = args
    import numpy as np
    from oracle import bccb_oracle as orc
    from paper_2509_13592_b200 import scenes
    w = scenes.workload(cfg)
    geom, ys, _ = scenes.make_scene(w, [snap])
    m1, m2 = geom.occupied_coordinates()
    eig = orc.gram_eigenvalues_exact(geom.occupancy, w.l1, w.l2)
    b = orc.adjoint_fft(m1, m2, w.l1, w.l2, ys[0])
    tau = w.tau_fraction * float(np.max(np.abs(b)))
    t0 = time.perf_counter()
    if w.solver == "admm":
        orc.admm(eig, b, tau, w.rho, iters)
    else:
        eig_t = np.ascontiguousarray(eig.T)
        (orc.ista if w.solver == "ista" else orc.fista)(eig_t, b, tau, 1.0 / (w.l1 * w.l2), iters)
    return time.perf_counter() - t0


def cpu_sample(cfg: int, workers: int, iters: int, pool):
    """Run `workers` snapshots x `iters` iterations concurrently; return (gpi/s, wall, loop secs)."""
    from paper_2509_13592_b200 import scenes
    w = scenes.workload(cfg)
    t0 = time.perf_counter()
    loops = pool.map(_cpu_worker, [(cfg, s, iters) for s in range(workers)])
    wall = time.perf_counter() - t0
    # loop-only time like SolverResult.total_seconds (solvers.py:271-278): slowest worker
    return workers * w.grid_points * iters / max(loops), wall, loops


def _cpu_pool(workers):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("MKL_NUM_THREADS", "1")
    return mp.get_context("spawn").Pool(workers)


def cpu_iters_for(cfg: int, workers: int, budget_cpu_s: float = 15.0) -> int:
    # survey single-core ms/iteration/snapshot
    ms = {1: 0.34, 2: 7.11, 3: 37.8, 4: 80.9, 5: 3371.0}[cfg]
    from paper_2509_13592_b200 import scenes
    t = int(budget_cpu_s * 1e3 / (ms * workers))
    return max(2, min(t, scenes.workload(cfg).iterations))


DENSE_BUDGET = 8 << 30   # the reference's dictionary / DenseGram budget (dictionary.py:17, 163-166)


def dense_sample(cfg: int, budget_s: float = 10.0):
    """The reference's dense O((L1L2)^2) "regular" ISTA (oracle.ista_dense, pinned bitwise to
    the reference by tests/golden/dense.npz) on snapshot 0, where the DenseGram fits the
    reference's memory budget (config 1 only).  The Gram build is untimed precompute, as in
    the reference (SolverResult.total_seconds times the loop only, solvers.py:271-278).
    OpenBLAS runs with its default threads (the reference's `@`)."""
    import numpy as np
    from oracle import bccb_oracle as orc
    from paper_2509_13592_b200 import scenes
    w = scenes.workload(cfg)
    need = w.grid_points ** 2 * 16
    if need > DENSE_BUDGET:
        return {"value": None, "unavailable": f"DenseGram needs {need / 2**30:.0f} GiB > the reference's 8 GiB "
                                              f"budget (MemoryBudgetError, dictionary.py:163-166)"}
    geom, ys, _ = scenes.make_scene(w, [0])
    m1, m2 = geom.occupied_coordinates()
    g = orc.dense_gram(m1, m2, w.l1, w.l2)
    b = orc.adjoint_fft(m1, m2, w.l1, w.l2, ys[0])
    tau = w.tau_fraction * float(np.max(np.abs(b)))
    mu = 1.0 / w.grid_points
    orc.ista_dense(g, b, tau, mu, 2)                    # warm-up
    t0 = time.perf_counter()
    iters = 0
    while time.perf_counter() - t0 < budget_s and iters < w.iterations:
        orc.ista_dense(g, b, tau, mu, 5)
        iters += 5
    dt = time.perf_counter() - t0
    try:
        from threadpoolctl import threadpool_info
        threads = max(i["num_threads"] for i in threadpool_info() if i.get("user_api") == "blas")
    except Exception:
        threads = len(os.sched_getaffinity(0))
    return {"value": w.grid_points * iters / dt, "unit": UNIT, "cores": int(threads), "kind": "port",
            "ms_per_iteration": dt * 1e3 / iters,
            "sample": f"dense regular-backend ISTA (DenseGram @ c, complex128) on 1 snapshot x {iters} iterations"}


def run_reference(args, rank):
    if rank != 0:
        return
    from paper_2509_13592_b200 import scenes
    w = scenes.workload(args.config)
    cores = len(os.sched_getaffinity(0))
    workers = min(cores, max(w.batch, 1))
    iters = cpu_iters_for(args.config, workers, budget_cpu_s=2.0 * workers)
    pool = _cpu_pool(workers)
    vals = []
    try:
        for i in range(args.warmup + args.steps):
            v, wall, _ = cpu_sample(args.config, workers, iters, pool)
            if i >= args.warmup:
                vals.append((v, wall))
    finally:
        pool.close()
    value = statistics.mean(v for v, _ in vals)
    ms = statistics.mean(t for _, t in vals) * 1e3
    sample = f"{workers} snapshots x {iters} iterations per step (of B={w.batch}, T={w.iterations}); loop time of the slowest worker"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": workload_config(w, args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(w, n):
    return {
        "workload": (f"cfg{w.cfg}: {w.solver.upper()}, {w.batch} snapshots/GPU, {w.m1}x{w.m2} URA with "
                     f"{w.elements} elements, L1={w.l1} L2={w.l2}, T={w.iterations}, K={w.targets} targets, "
                     f"{w.snr_db:g} dB, tau={w.tau_fraction:g} max|A^H y|"),
        "batch_per_gpu": w.batch, "global_batch": w.batch * n, "l1": w.l1, "l2": w.l2,
        "iterations": w.iterations, "parallelism": f"dp{n} (snapshot shards, no per-iteration comm)",
        "l2_cache": "flushed between steps (256 MiB write)",
    }


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile(mode="w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(gpu_index)], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait(timeout=10)
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        if not rows:
            # timed region shorter than the 100 ms sampling period (config 1): one query at its end
            try:
                q = subprocess.run(self.p.args[:3] + ["-i", self.p.args[-1]],
                                   capture_output=True, text=True, timeout=10).stdout
                rows = [r.split(",") for r in q.strip().splitlines() if r.strip()]
            except Exception:
                rows = []
        if not rows:
            return None
        sm = [float(r[1]) for r in rows]
        smax = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip().lower() == "active"})
        loaded = [s for s in sm if s >= 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows)}


# ----------------------------------------------------------------------------- GPU leg

def main():
    args = parse()
    from paper_2509_13592_b200 import distributed as bdist
    rank, world, local = bdist.init()
    if args.impl == "reference":
        run_reference(args, rank)
        return
    import numpy as np
    import torch
    import paper_2509_13592_b200 as bb
    from paper_2509_13592_b200 import _lib, scenes
    from paper_2509_13592_b200.bccb import _stream_ptr

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    w = scenes.workload(args.config)
    T = args.iterations or w.iterations
    B = w.batch
    snaps = range(rank * B, (rank + 1) * B)            # weak scaling: own 64 snapshots per rank
    geom, y_np, _ = scenes.make_scene(w, snaps)
    op = bb.gram_operator(geom, w.l1, w.l2, device=dev)
    L = op.dimension
    mu = 1.0 / op.max_eigenvalue()
    y_dev = torch.from_numpy(y_np.astype(np.complex64)).to(dev)
    prob = bb.LassoProblem.from_measurements(op, y_dev, tau_fraction=w.tau_fraction)
    bhat, extra, tau_dev = prob.device_data()
    stream = torch.cuda.current_stream(dev)
    sptr = _stream_ptr(local)
    ws = op.workspace(B)
    fb = torch.empty(B, dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    if w.solver == "admm":
        s1 = torch.zeros((B, L), dtype=torch.complex128, device=dev)    # z
        s2 = torch.zeros((B, L), dtype=torch.complex128, device=dev)    # v (float64 dual)
        run = lambda: _lib.check(_lib.lib.bccb_admm_run(  # noqa: E731
            op._plan, B, 0, T, float(w.rho), tau_dev.data_ptr(), bhat.data_ptr(), None, s1.data_ptr(),
            s2.data_ptr(), None, fb.data_ptr(), ws.data_ptr(), sptr))
    else:
        s1 = torch.zeros((B, L), dtype=torch.complex128, device=dev)
        s2 = torch.zeros((B, L), dtype=torch.complex64, device=dev) if w.solver == "fista" else None
        run = lambda: _lib.check(_lib.lib.bccb_fista_run(  # noqa: E731
            op._plan, B, 0, T, mu, tau_dev.data_ptr(), bhat.data_ptr(), None, s1.data_ptr(),
            s2.data_ptr() if s2 is not None else None, fb.data_ptr(), ws.data_ptr(), sptr))

    def reset():
        flush.fill_(1)                     # evict L2 (126 MB) between timed steps
        s1.zero_()
        if s2 is not None:
            s2.zero_()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        reset()
        run()
    torch.cuda.synchronize(dev)
    assert int(fb.min()) == 2**31 - 1, "non-finite iterate in warm-up"

    # ---- timed region: K steps, CUDA events on the launching stream
    clocks = ClockSampler(local if "CUDA_VISIBLE_DEVICES" not in os.environ else
                          int(os.environ["CUDA_VISIBLE_DEVICES"].split(",")[local]))
    times = []
    launches0 = _lib.lib.bccb_launch_count()
    for _ in range(args.steps):
        reset()
        barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        times.append(e0.elapsed_time(e1))
    launches = _lib.lib.bccb_launch_count() - launches0
    clk = clocks.stop()
    ms_local = statistics.mean(times)
    ms_step = bdist.max_over_ranks(ms_local)
    gpi_step = B * L * T
    value = world * gpi_step / (ms_step / 1e3)

    # ---- per-kernel live timing: one extra profiled step, single stream (one launch = the whole
    # batch, no concurrent-stream overlap inside the event brackets), events around every launch
    reset()
    torch.cuda.synchronize(dev)
    _lib.check(_lib.lib.bccb_set_substreams(1))
    _lib.lib.bccb_profile_begin()
    run()
    import ctypes
    ms_k = (ctypes.c_double * 3)()
    n_k = (ctypes.c_longlong * 3)()
    _lib.check(_lib.lib.bccb_profile_end(ms_k, n_k))
    _lib.check(_lib.lib.bccb_set_substreams(0))        # back to the library default
    rows_ms = ms_k[0] / max(n_k[0], 1)
    cols_ms = ms_k[1] / max(n_k[1], 1)
    step_kernel_ms = ms_k[0] + ms_k[1] + ms_k[2]

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json copy test)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    fused_cols = n_k[1] == 0
    # algorithmic bytes of one launch: the per-iteration model x the iterations the launch
    # covers (T / launches: ~1 for the per-pass kernels, T for the whole-solve small-grid and
    # cluster kernels)
    iters_per_launch = T / max(n_k[0], 1)
    rows_bytes = (B_ALG_ROWS[w.solver] + (B_ALG_COLS if fused_cols else 0)) * B * L * iters_per_launch
    achieved = rows_bytes / (rows_ms / 1e3) / 1e9
    traffic = None
    ncu_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(ncu_path):
        try:
            per_gpi = json.load(open(ncu_path)).get(f"cfg{w.cfg}", {}).get("rows_dram_bytes_per_gpi")
            traffic = None if per_gpi is None else per_gpi * B * L   # DRAM bytes per (full-batch) launch
        except Exception:
            traffic = None
    iter_achieved = B_ALG[w.solver] * (value / world) / 1e9
    roofline = {
        "bound": "hbm", "kernel": f"rows_{w.solver}_kernel (band IFFT + fused epilogue + band FFT)",
        "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
        "traffic": traffic, "traffic_source": "profiles/ncu_summary.json (ncu dram__bytes_read+write, solve average)",
        "peak_source": peak_src,
        "algorithmic_bytes_per_launch": rows_bytes,
        "bytes_model": (f"{B_ALG_ROWS[w.solver]}{' + 16 (fused K3)' if fused_cols else ''} B/gpi x {B}x{L} gpi "
                        f"x {iters_per_launch:.4g} iterations per launch (SURVEY 8(d) K4+K2 share)"),
        "avg_launch_ms": rows_ms, "share_of_step": ms_k[0] / step_kernel_ms,
        "launch_timing": "profiled extra step, single stream, CUDA events on the launch stream",
        "cols_kernel": ({"avg_launch_ms": cols_ms, "achieved": B_ALG_COLS * B * L / (cols_ms / 1e3) / 1e9,
                         "share_of_step": ms_k[1] / step_kernel_ms} if n_k[1] else
                        {"fused": "column pass runs inside the rows kernel (last CTA per snapshot)"}),
        "iteration": {"bytes_per_gpi": B_ALG[w.solver], "achieved": iter_achieved,
                      "frac": iter_achieved / hbm_peak, "frac_vs_8TBs_spec": iter_achieved / 8000.0},
    }

    # ---- end to end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        y_host = torch.from_numpy(y_np.astype(np.complex64)).pin_memory()
        k = min(w.targets, 64)
        # rank 0 receives every rank's spectra and peak lists (one NCCL all-gather after the loop)
        rows_out = B * world if rank == 0 else B
        out_host = torch.empty((rows_out, L), dtype=torch.complex64).pin_memory()
        idx_host = torch.empty((rows_out, k), dtype=torch.int32).pin_memory()
        cfg = bb.SolverConfig(iterations=T, step_size_mu=mu, rho=w.rho)
        solve = {"ista": bb.ista_solve, "fista": bb.fista_solve, "admm": bb.admm_solve}[w.solver]

        def e2e_step():
            yd = y_host.to(dev, non_blocking=True)
            p = bb.LassoProblem.from_measurements(op, yd, tau_fraction=w.tau_fraction)
            r = solve(p, cfg)
            est = r.estimate.to(torch.complex64)
            idx, _ = bb.topk_peaks(est, k)
            if world > 1:
                est = bdist.gather_rows(est, B * world)
                idx = bdist.gather_rows(idx, B * world)
            if est is not None:
                out_host.copy_(est, non_blocking=True)
                idx_host.copy_(idx, non_blocking=True)
            torch.cuda.synchronize(dev)

        for _ in range(max(1, args.warmup)):
            e2e_step()
        et = []
        for _ in range(args.steps):
            flush.fill_(1)
            barrier()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            e2e_step()
            et.append(time.perf_counter() - t0)
            barrier()
        e_s = bdist.max_over_ranks(statistics.mean(et))
        e2e = {"value": world * gpi_step / e_s, "unit": UNIT, "ms_per_step": e_s * 1e3,
               "h2d_bytes_per_step": int(world * y_host.numel() * 8),
               "d2h_bytes_per_step": int(world * B * L * 8 + world * B * k * 4),
               "path": ("LassoProblem.from_measurements (GPU A^H y) -> solve -> topk_peaks"
                        + (" -> NCCL all-gather of spectra + peaks to rank 0" if world > 1 else "")
                        + "; pinned host y in (every rank), complex64 spectra + peak indices out (rank 0)")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = len(os.sched_getaffinity(0))
        workers = min(cores, B)
        iters = cpu_iters_for(w.cfg, workers)
        pool = _cpu_pool(workers)
        try:
            v, wall, _ = cpu_sample(w.cfg, workers, iters, pool)
        finally:
            pool.close()
        cpu = {"value": v, "unit": UNIT, "cores": workers, "kind": "port",
               "sample": f"oracle {w.solver.upper()} (numpy pocketfft, float64) on {workers} snapshots x {iters} "
                         f"iterations, one process per core; {wall:.1f} s wall",
               "dense": dense_sample(w.cfg)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c64 FFT + f64 iterate", "data": "synthetic (seeded scenes, SURVEY 8(d))",
            "config": workload_config(w, world) | ({"iterations": T} if args.iterations else {}),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches), "gpu_launches_per_step": int(launches) // max(args.steps, 1),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
