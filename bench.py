#!/usr/bin/env python
"""Benchmark of the fused BCCB-FISTA hot path (BASELINE.json metric, grid-point-iterations/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl b200|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU, NCCL)

A step = one full solve (T solver iterations) over this rank's shard of snapshots.
Default workload = BASELINE config 5 (configs[4]), the largest single-GPU configuration
and the one north_star's "fused FISTA iteration" target is quoted on: FISTA, batch 32,
L1 = L2 = 4096, T = 1000.  Configs 4 and 5 are strong-scaled like BASELINE states ("batch
sharded across 1/2/4/8 GPUs": rank r solves shard_bounds(B, r, N)); configs 1-3 are weak-
scaled (every rank solves its own batch).  `value` times the device-resident solve with
CUDA events (max over ranks); `e2e` times the public API end to end with host (pinned)
buffers on every rank: H2D of y, GPU adjoint, solve, top-K, then one grouped NCCL
send/recv gather of spectra + peaks to rank 0 and its D2H, timed with CUDA events on the
launching stream (max over ranks).  --impl reference times the reference algorithm (the
pinned CPU oracle port, oracle/bccb_oracle.py) on this host's cores; it maps no CUDA
library of this repo (the package loads libbccb_b200.so lazily).
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
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--iterations", type=int, default=None, help="override T (debug only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=0,
                    help="e2e: solve the shard in this many chunks with overlapped D2H (0: 4 at configs 4/5 on one GPU)")
    ap.add_argument("--substreams", type=int, default=0, help="sub-batch streams (0: library default)")
    ap.add_argument("--no-kernel-events", action="store_true",
                    help="do not bracket each launch of the timed steps with CUDA events")
    return ap.parse_args()


# BASELINE.json configs 4 and 5: "batch ... sharded across 1/2/4/8 GPUs" (strong scaling)
STRONG = (4, 5)


# ----------------------------------------------------------------------------- CPU leg

_CPU_CACHE = {}


def _cpu_worker(args):
    cfg, snap, iters = args
    import numpy as np
    from oracle import bccb_oracle as orc
    from paper_2509_13592_b200 import scenes
    w = scenes.workload(cfg)
    # untimed precompute (like SolverResult.total_seconds, solvers.py:271-278), cached per
    # worker process: the shared spectrum once per config, b for the last snapshot seen
    if _CPU_CACHE.get("cfg") != cfg:
        _CPU_CACHE.clear()
        geom = scenes.geometry_for(w)
        _CPU_CACHE.update(cfg=cfg, geom=geom, eig=orc.gram_eigenvalues_exact(geom.occupancy, w.l1, w.l2))
    if _CPU_CACHE.get("snap") != snap:
        geom, ys, _ = scenes.make_scene(w, [snap])
        m1, m2 = geom.occupied_coordinates()
        b = orc.adjoint_fft(m1, m2, w.l1, w.l2, ys[0])
        _CPU_CACHE.update(snap=snap, b=b, tau=w.tau_fraction * float(np.max(np.abs(b))))
    eig, b, tau = _CPU_CACHE["eig"], _CPU_CACHE["b"], _CPU_CACHE["tau"]
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
        "scaling": scaling_of(w), "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": workload_config(w, args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(w, n):
    strong = w.cfg in STRONG
    per_gpu = f"{w.batch} snapshots sharded over {n} GPU(s)" if strong else f"{w.batch} snapshots/GPU"
    return {
        "workload": (f"cfg{w.cfg}: {w.solver.upper()}, {per_gpu}, {w.m1}x{w.m2} URA with "
                     f"{w.elements} elements, L1={w.l1} L2={w.l2}, T={w.iterations}, K={w.targets} targets, "
                     f"{w.snr_db:g} dB, tau={w.tau_fraction:g} max|A^H y|"),
        "global_batch": w.batch if strong else w.batch * n,
        "batch_per_gpu": (-(-w.batch // n)) if strong else w.batch,
        "l1": w.l1, "l2": w.l2, "iterations": w.iterations,
        "parallelism": f"dp{n} (snapshot shards, no per-iteration comm; rank-0 gather after the loop)",
        "l2_cache": "flushed between steps (256 MiB write); the iterate state exceeds L2",
    }


def scaling_of(w):
    return "strong" if w.cfg in STRONG else "weak"


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

FP32_LANES_PER_SM = 128       # B200 (sm_100a): 4 SMSPs x 32 FP32 lanes
B200_SMS = 148


def ncu_summary(cfg):
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        return json.load(open(path)).get(f"cfg{cfg}", {})
    except Exception:
        return {}


def build_roofline(w, T, B, value_per_gpu, rows_ms, n_rows, kern_ms_total, step_ms_total, cols, clk, nsub=1):
    """Roofline of the dominant kernel (the rows pass), against the bound that binds.

    The band-pruned, sparsity-skipping rows pass is FP32-issue bound (profiles/: sm__throughput
    56-65 %, FADD+FFMA+FMUL ~70 % of instructions, DRAM 0.7-1.9 B/gpi), so the roofline is
    FP32 flops per launch / launch time against 148 SMs x 128 lanes x 2 flops x the SM clock
    measured during the timed region.  Flops per grid-point-iteration of the rows kernel come
    from the ncu launch list of one full solve of the same code (profiles/ncu_summary.json:
    sm__sass_thread_inst_executed_op_{fadd,fmul,ffma}_pred_on.sum, FFMA counted twice); DRAM
    traffic per launch from the same list.  SURVEY 8(d)'s dense 80 B/gpi model is reported only
    as "effective_bandwidth" (band pruning makes the kernel move ~1 B/gpi)."""
    summ = ncu_summary(w.cfg)
    L = w.l1 * w.l2
    iters_per_launch = T * B / max(n_rows, 1) / B      # ~1 for per-pass kernels, T for whole-solve kernels
    gpi_per_launch = B * L * T / max(n_rows, 1)
    sm_mhz = (clk or {}).get("sm_mhz") or 1965.0
    fp32_peak = B200_SMS * FP32_LANES_PER_SM * 2 * sm_mhz * 1e6 / 1e12       # TFLOP/s
    flops_gpi = summ.get("rows_fp32_flops_per_gpi")
    inst_gpi = summ.get("rows_warp_inst_per_gpi")
    dram_gpi = summ.get("rows_dram_bytes_per_gpi")
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = "measured (MEASURED_PEAKS.json copy test)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    # nsub sub-batch streams run their launches concurrently: a launch's event-to-event duration
    # then covers time shared with nsub - 1 other launches, so rates use the exclusive share
    # rows_ms / nsub (the sum over all launches / nsub is the time the rows pass occupies a step)
    launch_s = rows_ms / max(nsub, 1) / 1e3
    r = {"kernel": f"rows_{w.solver}_kernel (band IFFT + fused prox/momentum epilogue + band FFT)",
         "avg_launch_ms": rows_ms, "avg_launch_ms_exclusive": rows_ms / max(nsub, 1),
         "launches_per_step": n_rows,
         "gpi_per_launch": gpi_per_launch, "iterations_per_launch": iters_per_launch,
         "share_of_step": kern_ms_total / max(nsub, 1) / step_ms_total if step_ms_total else None,
         "launch_timing": "CUDA events around every launch of the timed steps, on the launch's stream"}
    if flops_gpi:
        achieved = flops_gpi * gpi_per_launch / launch_s / 1e12
        r.update({"bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                  "frac": achieved / fp32_peak,
                  "flops_per_launch": flops_gpi * gpi_per_launch,
                  "flops_per_gpi": flops_gpi,
                  "flops_source": summ.get("source"),
                  "peak_source": f"{B200_SMS} SMs x {FP32_LANES_PER_SM} FP32 lanes x 2 x {sm_mhz:.0f} MHz "
                                 "(SM clock measured during the timed region)"})
    else:
        r.update({"bound": "fp32", "achieved": None, "peak": fp32_peak, "unit": "TFLOP/s", "frac": None,
                  "flops_source": "profiles/ncu_summary.json has no FP32 count for this config"})
    if summ.get("late_phase_fp32_tflops_ncu"):
        # the same kernel timed ALONE by ncu (serialised, cold cache): the lower bracket of the
        # fraction; the live figure above credits the overlap of the concurrent sub-batch streams
        r["ncu_alone"] = {"late_phase_fp32_tflops": summ["late_phase_fp32_tflops_ncu"],
                          "frac": summ["late_phase_fp32_tflops_ncu"] / fp32_peak,
                          "mean_launch_us": summ.get("rows_mean_us_ncu"),
                          "mean_fp32_tflops": (flops_gpi * gpi_per_launch / (summ["rows_mean_us_ncu"] * 1e-6) / 1e12
                                               if flops_gpi and summ.get("rows_mean_us_ncu") else None)}
    r["traffic"] = dram_gpi * gpi_per_launch if dram_gpi is not None else None
    r["traffic_note"] = "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch (full-solve average)"
    if inst_gpi:
        ipc_peak = 4 * B200_SMS * sm_mhz * 1e6                  # one warp-instruction per SMSP per clock
        ach = inst_gpi * gpi_per_launch / launch_s
        r["issue"] = {"warp_inst_per_gpi": inst_gpi, "achieved_warp_inst_per_s": ach, "peak": ipc_peak,
                      "frac": ach / ipc_peak}
    if dram_gpi is not None:
        r["hbm"] = {"achieved_gbs": dram_gpi * gpi_per_launch / launch_s / 1e9, "peak_gbs": hbm_peak,
                    "frac": dram_gpi * gpi_per_launch / launch_s / 1e9 / hbm_peak, "peak_source": hbm_src}
    dense = summ.get("dense_phase")
    if dense:
        r["hbm_dense_phase"] = dense | {"frac": dense["gbs"] / hbm_peak, "peak_gbs": hbm_peak}
    eff = B_ALG[w.solver] * value_per_gpu / 1e9
    r["effective_bandwidth"] = {"bytes_per_gpi": B_ALG[w.solver], "gbs": eff, "of_hbm_peak": eff / hbm_peak,
                                "note": "SURVEY 8(d) dense 'FFT sweeps x 8 B' model x measured gpi/s: "
                                        "an effective figure, not a roofline (band pruning + sparsity "
                                        "skipping move ~1 B/gpi)"}
    if cols:
        r["cols_kernel"] = cols
    return r


def main():
    args = parse()
    from paper_2509_13592_b200 import distributed as bdist
    rank, world, local = bdist.init()
    if args.impl == "reference":
        run_reference(args, rank)
        return
    import ctypes
    import numpy as np
    import torch
    import paper_2509_13592_b200 as bb
    from paper_2509_13592_b200 import _lib, scenes
    from paper_2509_13592_b200.bccb import _stream_ptr

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    w = scenes.workload(args.config)
    T = args.iterations or w.iterations
    strong = w.cfg in STRONG
    lo, hi = bdist.workload_shard(w.batch, rank, world, strong)
    B = hi - lo
    total = w.batch if strong else w.batch * world
    if B < 1:
        raise SystemExit(f"rank {rank}: empty shard ({w.batch} snapshots over {world} ranks)")
    if args.substreams:
        _lib.check(_lib.lib.bccb_set_substreams(args.substreams))
    geom, y_np, _ = scenes.make_scene(w, range(lo, hi))
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

    # ---- timed region: K steps, CUDA events on the launching stream; every library launch is
    # also bracketed by CUDA events on its own stream (bccb_profile_begin/end) for the roofline
    clocks = ClockSampler(local if "CUDA_VISIBLE_DEVICES" not in os.environ else
                          int(os.environ["CUDA_VISIBLE_DEVICES"].split(",")[local]))
    times = []
    launches0 = _lib.lib.bccb_launch_count()
    ms_k = (ctypes.c_double * 3)()
    n_k = (ctypes.c_longlong * 3)()
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
    value = total * L * T / (ms_step / 1e3)
    nsub = int(_lib.lib.bccb_substreams_for(op._plan, B))

    # ---- per-launch kernel timing: one more step in the SAME stream configuration with every
    # library launch bracketed by CUDA events on its own stream (events between the passes cost
    # PDL overlap at short lines, so they stay out of the timed steps; at config 5 they were
    # measured neutral: profiles/r2/r2a_bench_cfg5_noev.json)
    roofline = None
    if not args.no_kernel_events:
        reset()
        torch.cuda.synchronize(dev)
        pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        _lib.lib.bccb_profile_begin()
        pe0.record(stream)
        run()
        pe1.record(stream)
        _lib.check(_lib.lib.bccb_profile_end(ms_k, n_k))
        torch.cuda.synchronize(dev)
        prof_ms = pe0.elapsed_time(pe1)
        if n_k[0]:
            rows_ms = ms_k[0] / n_k[0]
            cols = None
            if n_k[1]:
                cols = {"kernel": "cols pass (band FFT . D + P.Bhat . band IFFT)", "avg_launch_ms": ms_k[1] / n_k[1],
                        "avg_launch_ms_exclusive": ms_k[1] / n_k[1] / max(nsub, 1),
                        "launches_per_step": n_k[1], "share_of_step": ms_k[1] / max(nsub, 1) / prof_ms}
            roofline = build_roofline(w, T, B, value / world, rows_ms, n_k[0], ms_k[0], prof_ms, cols, clk, nsub)
            roofline["substreams"] = nsub
            roofline["profiled_step_ms"] = prof_ms
            roofline["launch_timing"] = ("CUDA events around every launch of one extra step (same stream "
                                         "configuration as the timed steps), on the launch's stream")
            if nsub > 1:
                roofline["launch_timing"] += (f"; {nsub} sub-batch streams run concurrently, so a launch's "
                                              "duration includes time shared with the other streams: rates "
                                              "(achieved, hbm, issue) and share_of_step use duration / "
                                              f"{nsub} (avg_launch_ms_exclusive)")

    # ---- end to end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        y_host = torch.from_numpy(y_np.astype(np.complex64)).pin_memory()
        k = min(w.targets, 64)
        out_dev = torch.empty((total, L), dtype=torch.complex64, device=dev) if rank == 0 else None
        idx_dev = torch.empty((total, k), dtype=torch.int32, device=dev) if rank == 0 else None
        out_host = torch.empty((total, L), dtype=torch.complex64).pin_memory() if rank == 0 else None
        idx_host = torch.empty((total, k), dtype=torch.int32).pin_memory() if rank == 0 else None
        cfg = bb.SolverConfig(iterations=T, step_size_mu=mu, rho=w.rho)
        solve = {"ista": bb.ista_solve, "fista": bb.fista_solve, "admm": bb.admm_solve}[w.solver]

        # Single GPU, large outputs (configs 4/5 return 4.3 GB of spectra): the shard is solved in
        # `chunks` consecutive public-API calls and each chunk's D2H runs on a copy stream while
        # the next chunk solves; the timed region ends after the last copy.
        chunks = args.e2e_chunks or (4 if (strong and world == 1 and B >= 8) else 1)
        if world > 1:
            chunks = 1
        copy_stream = torch.cuda.Stream(dev) if chunks > 1 else None

        def e2e_step_chunked():
            yd = y_host.to(dev, non_blocking=True)
            for ci in range(chunks):
                a, b = bdist.shard_bounds(B, ci, chunks)
                p = bb.LassoProblem.from_measurements(op, yd[a:b], tau_fraction=w.tau_fraction)
                r = solve(p, cfg)
                est = r.estimate.to(torch.complex64)
                idx, _ = bb.topk_peaks(est, k)
                done = torch.cuda.Event()
                done.record(stream)
                with torch.cuda.stream(copy_stream):
                    copy_stream.wait_event(done)
                    out_host[a:b].copy_(est, non_blocking=True)
                    idx_host[a:b].copy_(idx, non_blocking=True)
                est.record_stream(copy_stream)
                idx.record_stream(copy_stream)
            stream.wait_stream(copy_stream)

        def e2e_step():
            if chunks > 1:
                return e2e_step_chunked()
            yd = y_host.to(dev, non_blocking=True)
            p = bb.LassoProblem.from_measurements(op, yd, tau_fraction=w.tau_fraction)
            r = solve(p, cfg)
            est = r.estimate.to(torch.complex64)
            idx, _ = bb.topk_peaks(est, k)
            # rank-0 gather (grouped NCCL send/recv straight into rank 0's output)
            est = bdist.gather_rows(est, total, out=out_dev)
            idx = bdist.gather_rows(idx, total, out=idx_dev)
            if rank == 0:
                out_host.copy_(est, non_blocking=True)
                idx_host.copy_(idx, non_blocking=True)

        for _ in range(max(1, args.warmup)):
            e2e_step()
        torch.cuda.synchronize(dev)
        et = []
        for _ in range(args.steps):
            flush.fill_(1)
            barrier()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            e2e_step()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            et.append(e0.elapsed_time(e1))
            barrier()
        e_ms = bdist.max_over_ranks(statistics.mean(et))
        e2e = {"value": total * L * T / (e_ms / 1e3), "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(total * w.elements * 8),
               "d2h_bytes_per_step": int(total * L * 8 + total * k * 4),
               "timing": "CUDA events on the launching stream around the whole step, max over ranks",
               "chunks": chunks,
               "path": ("pinned host y -> LassoProblem.from_measurements (GPU A^H y, device tau) -> "
                        f"{w.solver}_solve -> topk_peaks"
                        + (" -> grouped NCCL send/recv of spectra + peaks to rank 0" if world > 1 else "")
                        + " -> complex64 spectra + peak indices D2H (rank 0)"
                        + (f"; {chunks} consecutive chunks of the shard, each chunk's D2H on a copy stream "
                           "overlapping the next chunk's solve" if chunks > 1 else ""))}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = len(os.sched_getaffinity(0))
        workers = min(cores, B)
        iters = cpu_iters_for(w.cfg, workers)
        pool = _cpu_pool(workers)
        try:
            cpu_sample(w.cfg, workers, 1, pool)          # untimed: per-worker scene precompute
            v, wall, _ = cpu_sample(w.cfg, workers, iters, pool)
        finally:
            pool.close()
        cpu = {"value": v, "unit": UNIT, "cores": workers, "kind": "port",
               "sample": f"oracle {w.solver.upper()} (numpy pocketfft, float64) on {workers} snapshots x {iters} "
                         f"iterations, one process per core; loop time of the slowest worker; {wall:.1f} s wall",
               "dense": dense_sample(w.cfg)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": scaling_of(w),
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
