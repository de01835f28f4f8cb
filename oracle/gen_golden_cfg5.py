"""Config-5 golden at its BASELINE iteration count, from the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden_cfg5.py [--snapshots 8] [--iters 1000]

SURVEY.md 8(d) parity subset for config 5: 8 snapshots x 1000 FISTA iterations of the
reference's own `fista_solve` (/root/reference/pkg/src/bccblasso/solvers.py:311-355) on its own
`gram_operator` (bccb.py:108), one snapshot per worker process (numpy's FFT is single-threaded),
~1-2 h on 8 host cores.  Inputs are the reference's `subsample_preserving_aperture` geometry
and `synthesize_snapshot` measurements with the seeds of scenes.snapshot_seeds; b = A^H y comes
from the float64 FFT identity (SURVEY finding 9: the dense dictionary is 1.1 TB at L = 4096^2,
beyond the reference's MemoryBudgetError budget), tau = 0.02 max|b| in float64, mu = 1/max Re(Omega).

Output tests/golden/cfg5_t1000.npz (sparse estimates: the iterate is ~99.9 % exactly zero):
  y (S, M) complex128, tau (S,), mu, occupancy, snapshots, iterations,
  est_b / est_i / est_v (nonzeros of the reference estimates), est_norm (S,),
  topk (S, 32) = stable argsort(-|c|)[:32] (solvers.py:499), ynorm (S,).
The fixture is test infrastructure; the GPU test (tests/test_gpu_cfg5.py) solves the same y through
the production path (device A^H y and device tau) and compares.
"""

import argparse
import multiprocessing as mp
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

CFG = 5


def _scene(s):
    import bccblasso as ref
    from oracle import bccb_oracle as orc
    from paper_2509_13592_b200 import scenes

    w = scenes.workload(CFG)
    geom = ref.subsample_preserving_aperture(ref.make_ura(w.m1, w.m2), w.elements,
                                             seed=scenes.BASE_SEED + CFG)
    words = scenes.snapshot_seeds(CFG, s)
    targets = [ref.Target(t.f1, t.f2, t.amplitude)
               for t in scenes.draw_scene_targets(w, np.random.default_rng(int(words[2])))]
    nv = ref.snr_to_noise_variance(targets, w.snr_db)
    y = ref.synthesize_snapshot(geom, targets, nv, seed=int(words[3])).values
    m1, m2 = geom.occupied_coordinates()
    b = orc.adjoint_fft(m1, m2, w.l1, w.l2, y)
    return w, geom, y, b


def _worker(args):
    s, iters = args
    import bccblasso as ref
    from bccblasso.solvers import LassoProblem, SolverConfig
    from oracle import bccb_oracle as orc

    w, geom, y, b = _scene(s)
    op = ref.gram_operator(geom, w.l1, w.l2)
    mu = 1.0 / float(np.max(op.eigenvalues.real))
    tau = w.tau_fraction * float(np.max(np.abs(b)))
    t0 = time.time()
    res = ref.fista_solve(LassoProblem(op, b, tau), SolverConfig(iterations=iters, step_size_mu=mu))
    est = res.estimate
    nz = np.flatnonzero(est)
    print(f"cfg5 snapshot {s}: {time.time() - t0:.0f}s, loop {res.total_seconds:.0f}s, nnz={nz.size}",
          flush=True)
    return dict(s=s, y=y, tau=tau, mu=mu, nz=nz, vals=est[nz], norm=float(np.linalg.norm(est)),
                topk=orc.topk(est, w.targets), ynorm=float(np.real(np.vdot(y, y))),
                occupancy=geom.occupancy)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--snapshots", type=int, default=8)
    ap.add_argument("--iters", type=int, default=1000)
    ap.add_argument("--procs", type=int, default=len(os.sched_getaffinity(0)))
    ap.add_argument("--out", default=os.path.join(OUT, "cfg5_t1000.npz"))
    a = ap.parse_args()
    t0 = time.time()
    jobs = [(s, a.iters) for s in range(a.snapshots)]
    with mp.get_context("spawn").Pool(min(a.procs, len(jobs))) as pool:
        res = sorted(pool.map(_worker, jobs, chunksize=1), key=lambda r: r["s"])
    mus = {r["mu"] for r in res}
    assert len(mus) == 1
    out = {
        "occupancy": res[0]["occupancy"],
        "mu": res[0]["mu"],
        "iterations": a.iters,
        "snapshots": np.array([r["s"] for r in res]),
        "y": np.stack([r["y"] for r in res]),
        "tau": np.array([r["tau"] for r in res]),
        "ynorm": np.array([r["ynorm"] for r in res]),
        "topk": np.stack([r["topk"] for r in res]),
        "est_b": np.concatenate([np.full(r["nz"].size, k) for k, r in enumerate(res)]),
        "est_i": np.concatenate([r["nz"] for r in res]),
        "est_v": np.concatenate([r["vals"] for r in res]),
        "est_norm": np.array([r["norm"] for r in res]),
    }
    np.savez_compressed(a.out, **out)
    print(f"cfg5 T={a.iters}: {len(res)} snapshots in {time.time() - t0:.0f}s -> {a.out}", flush=True)


if __name__ == "__main__":
    main()
