"""Generate tests/golden/*.npz from the REAL reference package (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden.py

Inputs come from the reference's own functions (subsample_preserving_aperture,
synthesize_snapshot, apply_adjoint, gram_operator) and outputs from its own
solvers (ista_solve / fista_solve / admm_solve with an explicit step size, SURVEY
finding 8).  The fixtures pin (a) oracle/bccb_oracle.py, (b) the package's seeded
scene generator, and (c) the GPU path.  /root/reference is NOT available on the
GPU box; only these committed fixtures travel.
"""

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import bccblasso as ref  # noqa: E402
from bccblasso.experiments import draw_targets  # noqa: E402
from bccblasso.solvers import LassoProblem, SolverConfig  # noqa: E402

from oracle import bccb_oracle as orc  # noqa: E402
from paper_2509_13592_b200 import scenes  # noqa: E402


def to_ref_targets(targets):
    return [ref.Target(t.f1, t.f2, t.amplitude) for t in targets]


def small_fixture():
    """Mirrors pkg/tests/test_solvers.py:75-97 (make_problem) and test_bccb.py:56-60."""
    out = {}
    for seed in (3, 4, 5, 6, 8, 13):
        geom = ref.subsample_preserving_aperture(ref.make_ura(6, 4), 14, seed=seed)
        l1, l2 = 8, 4
        g1, g2 = ref.make_uniform_grid(l1), ref.make_uniform_grid(l2)
        dic = ref.build_subsampled_dictionary(geom, g1, g2)
        targets = [ref.Target(-0.25, 0.0, 1.5 - 0.5j), ref.Target(0.125, -0.25, 1.0j)]
        snap = ref.synthesize_snapshot(geom, targets, 0.05, seed=seed + 100)
        b = ref.apply_adjoint(dic, snap.values)
        tau = 0.1 * float(np.max(np.abs(b)))
        op = ref.gram_operator(geom, l1, l2)
        lam = ref.max_gram_eigenvalue(lambda v: ref.bccb_matvec(op, v), op.dimension)
        mu = 1.0 / (lam * (1.0 + 1e-6))
        p = f"s{seed}_"
        out[p + "occupancy"] = geom.occupancy
        out[p + "y"] = snap.values
        out[p + "b"] = b
        out[p + "tau"] = tau
        out[p + "mu"] = mu
        out[p + "eig"] = op.eigenvalues
        out[p + "ynorm"] = float(np.real(np.vdot(snap.values, snap.values)))
        prob = LassoProblem(op, b, tau)
        for T in (1, 7, 40):
            out[p + f"ista{T}"] = ref.ista_solve(prob, SolverConfig(iterations=T, step_size_mu=mu)).estimate
            out[p + f"fista{T}"] = ref.fista_solve(prob, SolverConfig(iterations=T, step_size_mu=mu)).estimate
        for rho in (1.0, 2.5):
            cap = []
            res = ref.admm_solve(prob, SolverConfig(iterations=60, rho=rho),
                                 iterate_callback=lambda t, c, z, v: cap.append((c.copy(), v.copy())))
            out[p + f"admm_z_{rho}"] = res.estimate
            out[p + f"admm_c_{rho}"] = cap[-1][0]
            out[p + f"admm_v_{rho}"] = cap[-1][1]
        # oracle pin (bitwise) at generation time
        assert np.array_equal(orc.fista(op._eig_t, b, tau, mu, 40), out[p + "fista40"])
        assert np.array_equal(orc.ista(op._eig_t, b, tau, mu, 40), out[p + "ista40"])
        assert np.array_equal(orc.admm(op.eigenvalues, b, tau, 2.5, 60)[0], out[p + "admm_z_2.5"])
    rng = np.random.default_rng(11)
    shapes = [(8, 4), (7, 5), (9, 6), (1, 6), (5, 1), (16, 16), (64, 32), (12, 10)]
    out["generic_shapes"] = np.array(shapes)
    for l1, l2 in shapes:
        col = rng.standard_normal(l1 * l2) + 1j * rng.standard_normal(l1 * l2)
        op = ref.bccb_from_first_column(col, l1, l2)
        c = rng.standard_normal(l1 * l2) + 1j * rng.standard_normal(l1 * l2)
        out[f"g{l1}x{l2}_col"] = col
        out[f"g{l1}x{l2}_eig"] = op.eigenvalues
        out[f"g{l1}x{l2}_c"] = c
        out[f"g{l1}x{l2}_matvec"] = ref.bccb_matvec(op, c)
        assert np.array_equal(orc.matvec(op._eig_t, c), out[f"g{l1}x{l2}_matvec"])
    # extract_support table (test_solvers.py:401-413 style) on a random sparse vector
    c = np.zeros(64, dtype=complex)
    c[[3, 17, 40, 41]] = [2.0 - 1j, -5j, 0.2, 1.0 + 1.0j]
    out["support_c"] = c
    sup = ref.extract_support(c, ref.make_uniform_grid(8), ref.make_uniform_grid(8), 0.1)
    out["support_ref"] = np.array([[a, b_, v.real, v.imag] for a, b_, v in sup])
    np.savez_compressed(os.path.join(OUT, "small.npz"), **out)


def config_fixture(cfg: int, snapshots, iterations: int, use_dense_adjoint: bool, store="dense"):
    w = scenes.workload(cfg)
    t0 = time.time()
    geom = ref.subsample_preserving_aperture(ref.make_ura(w.m1, w.m2), w.elements, seed=scenes.BASE_SEED + cfg)
    ours = scenes.geometry_for(w)
    assert np.array_equal(geom.occupancy, ours.occupancy), "scene geometry differs from the reference"
    op = ref.gram_operator(geom, w.l1, w.l2)
    mu = 1.0 / float(np.max(op.eigenvalues.real))
    m1, m2 = geom.occupied_coordinates()
    dic = None
    if use_dense_adjoint:
        dic = ref.build_subsampled_dictionary(geom, ref.make_uniform_grid(w.l1), ref.make_uniform_grid(w.l2))
    out = {"occupancy": geom.occupancy, "mu": mu, "iterations": iterations, "snapshots": np.array(snapshots)}
    ys, taus, ests, cs, vs, tops = [], [], [], [], [], []
    for s in snapshots:
        words = scenes.snapshot_seeds(cfg, s)
        rng = np.random.default_rng(int(words[2]))
        if w.amplitudes == "unit":
            targets = draw_targets(rng, (w.targets, w.targets))  # the reference's own draw
            mine = scenes.draw_scene_targets(w, np.random.default_rng(int(words[2])))
            assert [(t.f1, t.f2, t.amplitude) for t in targets] == [(t.f1, t.f2, t.amplitude) for t in mine]
        else:
            targets = to_ref_targets(scenes.draw_scene_targets(w, rng))
        nv = ref.snr_to_noise_variance(targets, w.snr_db)
        y = ref.synthesize_snapshot(geom, targets, nv, seed=int(words[3])).values
        if dic is not None:
            b = ref.apply_adjoint(dic, y)
            bf = orc.adjoint_fft(m1, m2, w.l1, w.l2, y)
            assert orc.rel_l2(bf, b) < 1e-13
        else:
            b = orc.adjoint_fft(m1, m2, w.l1, w.l2, y)   # dense dictionary exceeds the budget (finding 9)
        tau = w.tau_fraction * float(np.max(np.abs(b)))
        prob = LassoProblem(op, b, tau)
        if w.solver == "admm":
            cap = []
            res = ref.admm_solve(prob, SolverConfig(iterations=iterations, rho=w.rho),
                                 iterate_callback=lambda t, c, z, v: (cap.clear(), cap.append((c.copy(), v.copy()))))
            cs.append(cap[-1][0].astype(np.complex64))
            vs.append(cap[-1][1].astype(np.complex64))
        else:
            solve = ref.ista_solve if w.solver == "ista" else ref.fista_solve
            res = solve(prob, SolverConfig(iterations=iterations, step_size_mu=mu))
        est = res.estimate
        ys.append(y)
        taus.append(tau)
        ests.append(est)
        tops.append(orc.topk(est, w.targets))
        print(f"cfg{cfg} snapshot {s}: {res.total_seconds:.1f}s loop, nnz={np.count_nonzero(est)}", flush=True)
    out["y"] = np.stack(ys)
    out["tau"] = np.array(taus)
    out["topk"] = np.stack(tops)
    E = np.stack(ests)
    if store == "sparse":
        nzb, nzi = np.nonzero(E)
        out["est_b"], out["est_i"], out["est_v"] = nzb, nzi, E[nzb, nzi]
        out["est_norm"] = np.linalg.norm(E, axis=1)
    elif store == "sample":
        rng = np.random.default_rng(1234)
        sample = np.sort(rng.choice(E.shape[1], size=200_000, replace=False))
        big = np.unique(np.concatenate([orc.topk(e, 4096) for e in E]))
        sample = np.union1d(sample, big)
        out["est_sample_idx"] = sample
        out["est_sample"] = E[:, sample]
        out["est_norm"] = np.linalg.norm(E, axis=1)
    else:
        out["est"] = E
    if cs:
        out["admm_c"] = np.stack(cs)
        out["admm_v"] = np.stack(vs)
    np.savez_compressed(os.path.join(OUT, f"cfg{cfg}.npz"), **out)
    print(f"cfg{cfg}: done in {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    which = sys.argv[1:] or ["small", "1", "2", "3", "4", "5"]
    if "small" in which:
        small_fixture()
        print("small: done", flush=True)
    if "1" in which:
        config_fixture(1, [0], 500, True)
    if "2" in which:
        config_fixture(2, [0, 1], 1000, True, store="sparse")
    if "3" in which:
        config_fixture(3, [0], 500, True, store="sparse")
    if "4" in which:
        config_fixture(4, [0], 500, True, store="sparse")
    if "5" in which:
        config_fixture(5, [0], 20, False, store="sparse")
