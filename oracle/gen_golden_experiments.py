"""Generate tests/golden/experiments.npz by running the REAL reference harness
(bccblasso.experiments.run_grid) on the reference CLI test's sweep (pkg/tests/test_cli.py:236-258):

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden_experiments.py

Stores each record's cell, seed and epsilon_r, plus the fast-backend estimate of every trial
(re-solved with the reference's own seeds and fast solvers), so the package's GPU harness can
be checked cell by cell.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
sys.path.insert(0, REF)

import bccblasso as ref  # noqa: E402
from bccblasso import experiments as ex  # noqa: E402
from bccblasso.solvers import LassoProblem, SolverConfig  # noqa: E402

CFG = dict(m1_count=10, m2_count=6, element_count=24, l2=8, l1_values=[8, 16], iteration_values=[10, 40],
           trials=2, base_seed=7, solvers=["ista", "fista", "admm"])


def main():
    config = ex.ExperimentConfig(**CFG)
    records, _ = ex.run_grid(config)
    out = {"config": np.array(repr(CFG)),
           "cells": np.array([[ex.SOLVER_IDS[r.solver], r.l1, r.n_iter, r.trial_index] for r in records]),
           "seeds": np.array([r.seed for r in records], dtype=np.int64),
           "epsilon_r": np.array([r.epsilon_r for r in records])}
    for i, r in enumerate(records):
        words = np.random.SeedSequence((config.base_seed, ex.SOLVER_IDS[r.solver], r.l1, r.n_iter,
                                        r.trial_index)).generate_state(4)
        geom = ref.subsample_preserving_aperture(ref.make_ura(config.m1_count, config.m2_count),
                                                 config.element_count, seed=int(words[1]))
        targets = ex.draw_targets(np.random.default_rng(int(words[2])), config.k_range)
        snap = ref.synthesize_snapshot(geom, targets, ref.snr_to_noise_variance(targets, config.snr_db),
                                       seed=int(words[3]))
        dic = ref.build_subsampled_dictionary(geom, ref.make_uniform_grid(r.l1), ref.make_uniform_grid(config.l2))
        b = ref.apply_adjoint(dic, snap.values)
        tau = config.tau_fraction * float(np.max(np.abs(b)))
        op = ref.gram_operator(geom, r.l1, config.l2)
        mu = None
        if r.solver != "admm":
            lam = ref.max_gram_eigenvalue(lambda v: ref.bccb_matvec(op, v), op.dimension, seed=int(words[0]))
            mu = 1.0 / (lam * (1.0 + 1e-6))
        solve = {"ista": ref.ista_solve, "fista": ref.fista_solve, "admm": ref.admm_solve}[r.solver]
        est = solve(LassoProblem(op, b, tau), SolverConfig(iterations=r.n_iter, step_size_mu=mu)).estimate
        out[f"est{i}"] = est
    np.savez_compressed(os.path.join(OUT, "experiments.npz"), **out)
    print("experiments: done", len(records))


if __name__ == "__main__":
    main()
