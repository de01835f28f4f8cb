"""Time the fused FISTA iteration for one rows-kernel variant (BCCB_ROWS_VARIANT env)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import numpy as np
import torch
import paper_2509_13592_b200 as bb
from paper_2509_13592_b200 import _lib, scenes
from paper_2509_13592_b200.bccb import _stream_ptr

cfg = int(sys.argv[1]); T = int(sys.argv[2]) if len(sys.argv) > 2 else 200
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
run = lambda: _lib.check(_lib.lib.bccb_fista_run(op._plan, B, 0, T, 1.0 / L, tau.data_ptr(), bhat.data_ptr(), None,
                                                 c.data_ptr(), d.data_ptr(), fb.data_ptr(), ws.data_ptr(), _stream_ptr(0)))
for _ in range(2):
    c.zero_(); d.zero_(); run()
torch.cuda.synchronize()
c.zero_(); d.zero_()
_lib.lib.bccb_profile_begin()
run()
ms = (ctypes.c_double * 3)(); n = (ctypes.c_longlong * 3)()
_lib.check(_lib.lib.bccb_profile_end(ms, n))
rows = ms[0] / max(n[0], 1); cols = ms[1] / max(n[1], 1)
gbs = 48 * B * L / (rows / 1e3) / 1e9
print(json.dumps({"cfg": cfg, "variant": os.environ.get("BCCB_ROWS_VARIANT", "1"), "rows_ms": round(rows, 4),
                  "cols_ms": round(cols, 4), "rows_actual_GBs": round(gbs), "iter_ms": round((ms[0] + ms[1]) / T, 4)}))
