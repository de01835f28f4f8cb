"""Generate tests/golden/dense.npz from the REAL reference's dense "regular" backend
(run in the build container):

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden_dense.py

It pins oracle.dense_gram / oracle.ista_dense (the O((L1L2)^2) CPU baseline that bench.py
times beside the FFT path at config 1, BASELINE north_star) against
DenseGram = dense_gram(build_subsampled_dictionary(...)) (dictionary.py:155-168) and
ista_solve / fista_solve with backend "regular" (solvers.py:186-202, 252-355).
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import bccblasso as ref  # noqa: E402
from bccblasso.dictionary import dense_gram  # noqa: E402
from bccblasso.solvers import LassoProblem, SolverConfig  # noqa: E402

from oracle import bccb_oracle as orc  # noqa: E402
from paper_2509_13592_b200 import scenes  # noqa: E402


def main():
    out = {}
    # reference-test geometry (pkg/tests/test_solvers.py:75-97), L = 8 x 4
    for seed in (3, 4):
        geom = ref.subsample_preserving_aperture(ref.make_ura(6, 4), 14, seed=seed)
        dic = ref.build_subsampled_dictionary(geom, ref.make_uniform_grid(8), ref.make_uniform_grid(4))
        g = dense_gram(dic)
        snap = ref.synthesize_snapshot(geom, [ref.Target(-0.25, 0.0, 1.5 - 0.5j)], 0.05, seed=seed + 100)
        b = ref.apply_adjoint(dic, snap.values)
        tau = 0.1 * float(np.max(np.abs(b)))
        mu = 1.0 / 32.0
        prob = LassoProblem(g, b, tau)
        p = f"s{seed}_"
        out[p + "occupancy"] = geom.occupancy
        out[p + "gram"] = g.entries
        out[p + "b"] = b
        out[p + "tau"] = tau
        out[p + "mu"] = mu
        out[p + "ista40"] = ref.ista_solve(prob, SolverConfig(iterations=40, step_size_mu=mu, backend="regular")).estimate
        m1, m2 = geom.occupied_coordinates()
        assert np.array_equal(orc.dense_gram(m1, m2, 8, 4), g.entries)
        assert np.array_equal(orc.ista_dense(g.entries, b, tau, mu, 40), out[p + "ista40"])
    # config 1 (16x16 URA, 64 elements, L = 64 x 64): the size at which bench.py times the dense path
    w = scenes.workload(1)
    geom = ref.subsample_preserving_aperture(ref.make_ura(w.m1, w.m2), w.elements, seed=scenes.BASE_SEED + 1)
    dic = ref.build_subsampled_dictionary(geom, ref.make_uniform_grid(w.l1), ref.make_uniform_grid(w.l2))
    g = dense_gram(dic)
    _, ys, _ = scenes.make_scene(w, [0])
    b = ref.apply_adjoint(dic, ys[0])
    tau = w.tau_fraction * float(np.max(np.abs(b)))
    mu = 1.0 / (w.l1 * w.l2)
    T = 25
    res = ref.ista_solve(LassoProblem(g, b, tau), SolverConfig(iterations=T, step_size_mu=mu, backend="regular"))
    m1, m2 = geom.occupied_coordinates()
    mine = orc.dense_gram(m1, m2, w.l1, w.l2)
    out["cfg1_gram_diag"] = np.diag(g.entries).copy()
    out["cfg1_gram_row0"] = g.entries[0].copy()
    out["cfg1_gram_rowsum"] = g.entries.sum(axis=1)
    out["cfg1_b"] = b
    out["cfg1_tau"] = tau
    out["cfg1_mu"] = mu
    out["cfg1_iterations"] = T
    out["cfg1_ista"] = res.estimate
    assert np.array_equal(mine, g.entries)
    assert np.array_equal(orc.ista_dense(mine, b, tau, mu, T), res.estimate)
    np.savez_compressed(os.path.join(OUT, "dense.npz"), **out)
    print("dense: done")


if __name__ == "__main__":
    main()
