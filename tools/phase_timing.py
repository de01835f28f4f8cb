"""Per-phase timing of a FISTA solve: iterations [a, b) timed separately via chunked
continuation (bccb_fista_run first_iteration), reporting us/iteration per phase."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_13592_b200 as bb
from paper_2509_13592_b200 import _lib, scenes
from paper_2509_13592_b200.bccb import _stream_ptr

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = scenes.workload(cfg)
B = w.batch
geom, y, _ = scenes.make_scene(w, range(B))
op = bb.gram_operator(geom, w.l1, w.l2)
prob = bb.LassoProblem.from_measurements(op, y, tau_fraction=w.tau_fraction)
bhat, extra, tau = prob.device_data()
L = op.dimension
c = torch.zeros((B, L), dtype=torch.complex128, device="cuda")
d = torch.zeros((B, L), dtype=torch.complex64, device="cuda")
fb = torch.empty(B, dtype=torch.int32, device="cuda")
ws = op.workspace(B)
edges = sorted({e for e in [0, 5, 20, 50, 100, 200, 500, w.iterations] if e <= w.iterations})
def run(first, n):
    _lib.check(_lib.lib.bccb_fista_run(op._plan, B, first, n, 1.0 / L, tau.data_ptr(), bhat.data_ptr(), None,
                                       c.data_ptr(), d.data_ptr(), fb.data_ptr(), ws.data_ptr(), _stream_ptr(0)))
for rep in range(2):
    c.zero_(); d.zero_()
    out = []
    for a, b2 in zip(edges, edges[1:]):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(a, b2 - a); e1.record(); e1.synchronize()
        nnz = float((c != 0).float().mean())
        out.append((a, b2, round(e0.elapsed_time(e1) * 1e3 / (b2 - a), 2), round(nnz, 5)))
print(json.dumps({"cfg": cfg, "phases [a,b,us_per_iter,c_density]": out}))
# device time of the kernels alone over a late window (launch gaps = event time - kernel sum)
import ctypes
c.zero_(); d.zero_(); run(0, 400)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); run(400, 100); e1.record(); e1.synchronize()
ev_us = e0.elapsed_time(e1) * 1e3 / 100
_lib.lib.bccb_profile_begin(); run(400, 100)
ms = (ctypes.c_double * 3)(); n = (ctypes.c_longlong * 3)()
_lib.check(_lib.lib.bccb_profile_end(ms, n))
print(json.dumps({"cfg": cfg, "late_event_us_per_iter": round(ev_us, 2), "rows_us": round(ms[0] * 1e3 / max(n[0], 1), 2),
                  "cols_us": round(ms[1] * 1e3 / max(n[1], 1), 2), "cols_launches": n[1],
                  "kernel_sum_us_per_iter": round((ms[0] + ms[1]) * 1e3 / 100, 2)}))
