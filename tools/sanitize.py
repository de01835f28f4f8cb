"""Exercise every kernel family once at small shapes (for compute-sanitizer).

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize.py

One gpurun call per tool (B200_PROFILING.md: at most one compute-sanitizer tool per call).
Families: rows pass (CUDA-core engine at config-2 shape, tensor-core engine at config-4/5
line lengths), column pass (warp and shared-memory), fused column pass (L1 = 64 with the
cluster and small-grid solvers off), 64 x 64 cluster solver, small-grid persistent solver,
split ADMM and the complex128 ADMM engine, adjoint scatter, spectrum / synthesis (complex64
and complex128), matvec, top-K, fused objective trace.  Small batches and few iterations keep
the instrumented run short; results are checked for finiteness only (parity is pytest's job).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2509_13592_b200 as bb  # noqa: E402
from paper_2509_13592_b200 import scenes  # noqa: E402


def adjoint(m1, m2, l1, l2, y):
    """b = A^H y as L1 L2 ifft2 of the signed scatter of y (host numpy; inputs only)."""
    e = np.zeros((l2, l1), dtype=np.complex128)
    np.add.at(e, (np.asarray(m2) % l2, np.asarray(m1) % l1), y * (-1.0) ** (np.asarray(m1) + np.asarray(m2)))
    return np.fft.ifft2(e).ravel() * (l1 * l2)


def problem(cfg, nsnap, l1=None, l2=None):
    w = scenes.workload(cfg)
    geom, ys, _ = scenes.make_scene(w, range(nsnap))
    l1, l2 = l1 or w.l1, l2 or w.l2
    op = bb.gram_operator(geom, l1, l2)
    m1, m2 = geom.occupied_coordinates()
    bs = np.stack([adjoint(m1, m2, l1, l2, y) for y in ys])
    taus = np.array([w.tau_fraction * np.abs(b).max() for b in bs])
    return w, op, ys, bs, taus


def finite(x):
    x = x if isinstance(x, np.ndarray) else x.cpu().numpy()
    assert np.isfinite(x).all()


def main():
    which = set(sys.argv[1:]) or {"all"}
    run = lambda name: "all" in which or name in which  # noqa: E731
    if run("fista"):
        # CUDA-core rows engine + warp column pass (config-2 shape), sub-batch streams
        w, op, ys, bs, taus = problem(2, 6)
        finite(bb.fista_solve(bb.LassoProblem(op, bs, taus), bb.SolverConfig(iterations=6, step_size_mu=1 / op.dimension)).estimate)
        finite(bb.ista_solve(bb.LassoProblem(op, bs, taus), bb.SolverConfig(iterations=4, step_size_mu=1 / op.dimension)).estimate)
    if run("tc"):
        # tensor-core rows engine at L1 = 1024 (KP 8) and 4096 (KP 32) on short column lines
        for cfg, l2 in ((4, 64), (5, 32)):
            w, op, ys, bs, taus = problem(cfg, 1, l2=l2)
            finite(bb.fista_solve(bb.LassoProblem(op, bs, taus), bb.SolverConfig(iterations=3, step_size_mu=1 / op.dimension)).estimate)
    if run("trace"):
        w, op, ys, bs, taus = problem(2, 2)
        yn = np.real(np.einsum("ij,ij->i", ys.conj(), ys))
        finite(bb.fista_solve(bb.LassoProblem(op, bs, taus, y_norm_sq=yn),
                              bb.SolverConfig(iterations=4, step_size_mu=1 / op.dimension, record_objective=True)).objective_trace)
    if run("fused"):      # run with BCCB_CLUSTER=0 BCCB_SMALL_GRID=0 (read once per process)
        w, op, ys, bs, taus = problem(1, 3)
        finite(bb.fista_solve(bb.LassoProblem(op, bs, taus), bb.SolverConfig(iterations=5, step_size_mu=1 / op.dimension)).estimate)
    if run("cluster"):
        w, op, ys, bs, taus = problem(1, 1)
        finite(bb.ista_solve(bb.LassoProblem(op, bs[0], taus[0]), bb.SolverConfig(iterations=5, step_size_mu=1 / op.dimension)).estimate)
    if run("small"):
        geom = bb.subsample_preserving_aperture(bb.make_ura(6, 4), 14, seed=4)
        op = bb.gram_operator(geom, 8, 4)
        b = np.random.default_rng(0).standard_normal(32) + 0j
        finite(bb.fista_solve(bb.LassoProblem(op, b, 0.5), bb.SolverConfig(iterations=5, step_size_mu=1 / 32)).estimate)
    if run("admm"):
        w, op, ys, bs, taus = problem(3, 2)
        finite(bb.admm_solve(bb.LassoProblem(op, bs, taus * 0.01), bb.SolverConfig(iterations=4, rho=1.0)).estimate)
    if run("operator"):
        w, op, ys, bs, taus = problem(2, 2)
        p = bb.LassoProblem.from_measurements(op, ys, tau_fraction=0.05, keep_b=True)
        finite(p.adjoint_rhs)
        x = torch.randn(2, op.dimension, dtype=torch.complex64, device="cuda")
        finite(bb.bccb_matvec(op, x))
        finite(bb.bccb_matvec(op, x.to(torch.complex128)))
        finite(bb.bccb_spectrum(op, x))
        col = np.random.default_rng(1).standard_normal(48) + 1j
        g = bb.bccb_from_first_column(col, 8, 6)
        finite(bb.bccb_first_column(g).values)
        idx, mag = bb.topk_peaks(x, 8)
        finite(mag)
    torch.cuda.synchronize()
    print("sanitize workload done:", sorted(which))


if __name__ == "__main__":
    main()
