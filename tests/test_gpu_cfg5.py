"""Config 5 at its BASELINE iteration count through the production path.

Fixture tests/golden/cfg5_t1000.npz: the REAL reference's fista_solve (pkg/src/bccblasso/
solvers.py:311-355) on 8 config-5 snapshots x 1000 iterations (oracle/gen_golden_cfg5.py).
Here the same measurements y go through the drop-in exactly as a user runs it: the GPU adjoint
A^H y and the device tau = 0.02 max|A^H y| (LassoProblem.from_measurements), the fused FISTA
solve, and the device top-K.  Bar (BASELINE north_star): rel-L2 <= 1e-4 against the float64
reference estimate and identical top-32 peak index sets.
"""

import json
import os

import numpy as np
import pytest
import torch

import paper_2509_13592_b200 as bb
from conftest import load_golden
from paper_2509_13592_b200 import scenes

pytestmark = pytest.mark.gpu


def test_config5_fista_t1000_production_path():
    g = load_golden("cfg5_t1000")
    w = scenes.workload(5)
    geom = scenes.geometry_for(w)
    assert np.array_equal(geom.occupancy, g["occupancy"])
    op = bb.gram_operator(geom, w.l1, w.l2)
    L = op.dimension
    n = len(g["snapshots"])
    prob = bb.LassoProblem.from_measurements(op, torch.as_tensor(g["y"]).cuda(), tau_fraction=w.tau_fraction)
    tau_dev = prob.tau.cpu().numpy()
    tau_err = np.abs(tau_dev - g["tau"]) / g["tau"]
    assert tau_err.max() < 1e-6, tau_err
    res = bb.fista_solve(prob, bb.SolverConfig(iterations=int(g["iterations"]), step_size_mu=float(g["mu"])))
    est = res.estimate
    assert est.shape == (n, L) and est.dtype == torch.complex128
    idx, _ = bb.topk_peaks(est, w.targets)
    idx = idx.cpu().numpy()
    report = []
    for s in range(n):
        sel = g["est_b"] == s
        ref = torch.zeros(L, dtype=torch.complex128, device="cuda")
        ref[torch.as_tensor(g["est_i"][sel]).cuda()] = torch.as_tensor(g["est_v"][sel]).cuda()
        err = float(torch.linalg.vector_norm(est[s] - ref) / torch.linalg.vector_norm(ref))
        nnz = int(torch.count_nonzero(est[s]))
        ordered = int(np.sum(idx[s] == g["topk"][s]))
        report.append({"snapshot": int(g["snapshots"][s]), "rel_l2": err, "nnz_gpu": nnz,
                       "nnz_ref": int(sel.sum()), "top32_same_set": bool(set(idx[s]) == set(g["topk"][s])),
                       "top32_same_position": ordered, "tau_rel_err": float(tau_err[s])})
    out = os.environ.get("BCCB_PARITY_OUT")
    if out:
        with open(out, "w") as f:
            json.dump({"config": 5, "iterations": int(g["iterations"]), "snapshots": report,
                       "path": "from_measurements (GPU A^H y, device tau) -> fista_solve -> topk_peaks"}, f, indent=1)
    for r in report:
        assert r["rel_l2"] <= 1e-4, r
        assert r["top32_same_set"], r
