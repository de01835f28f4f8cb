"""Exactly one full device-resident solve of a BASELINE config (for ncu launch lists and
captures): setup (operator, GPU adjoint), then one bccb_fista_run / bccb_admm_run of T
iterations over the config's batch.   usage: python tools/one_solve.py CFG [T]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_13592_b200 as bb
from paper_2509_13592_b200 import _lib, scenes
from paper_2509_13592_b200.bccb import _stream_ptr

cfg = int(sys.argv[1])
w = scenes.workload(cfg)
T = int(sys.argv[2]) if len(sys.argv) > 2 else w.iterations
B = w.batch
geom, y, _ = scenes.make_scene(w, range(B))
op = bb.gram_operator(geom, w.l1, w.l2)
prob = bb.LassoProblem.from_measurements(op, y, tau_fraction=w.tau_fraction)
bhat, extra, tau = prob.device_data()
L = op.dimension
fb = torch.empty(B, dtype=torch.int32, device="cuda")
ws = op.workspace(B)
s1 = torch.zeros((B, L), dtype=torch.complex128, device="cuda")
if w.solver == "admm":
    s2 = torch.zeros((B, L), dtype=torch.complex128, device="cuda")
    _lib.check(_lib.lib.bccb_admm_run(op._plan, B, 0, T, float(w.rho), tau.data_ptr(), bhat.data_ptr(), None,
                                      s1.data_ptr(), s2.data_ptr(), None, fb.data_ptr(), ws.data_ptr(), _stream_ptr(0)))
else:
    s2 = torch.zeros((B, L), dtype=torch.complex64, device="cuda") if w.solver == "fista" else None
    _lib.check(_lib.lib.bccb_fista_run(op._plan, B, 0, T, 1.0 / L, tau.data_ptr(), bhat.data_ptr(), None,
                                       s1.data_ptr(), s2.data_ptr() if s2 is not None else None, fb.data_ptr(),
                                       ws.data_ptr(), _stream_ptr(0)))
torch.cuda.synchronize()
print(f"cfg{cfg}: one solve of {B} x {w.l1}x{w.l2} x {T} iterations, {_lib.lib.bccb_launch_count()} library launches")
