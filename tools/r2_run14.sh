# Round 2, GPU call 14: timing probes of the tensor-core tile (BCCB_DEBUG bits 8/16/32/64: parts of
# the tile removed, results invalid) -- where the per-tile time goes.
set -x
OUT=gpurun_out/r2o
mkdir -p $OUT
for D in 0 8 16 32 64 72 104; do
  BCCB_DEBUG=$D timeout 300 python - > $OUT/probe_$D.txt 2>&1 <<'P'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2509_13592_b200 as bb
from paper_2509_13592_b200 import _lib, scenes
from paper_2509_13592_b200.bccb import _stream_ptr
w = scenes.workload(5)
B = 32
geom, y, _ = scenes.make_scene(w, range(B))
op = bb.gram_operator(geom, w.l1, w.l2)
prob = bb.LassoProblem.from_measurements(op, torch.as_tensor(y).cuda(), tau_fraction=w.tau_fraction)
bhat, extra, tau = prob.device_data()
L = op.dimension
c = torch.zeros((B, L), dtype=torch.complex128, device="cuda")
d = torch.zeros((B, L), dtype=torch.complex64, device="cuda")
fb = torch.empty(B, dtype=torch.int32, device="cuda")
ws = op.workspace(B)
sp = _stream_ptr(0)
# warm start from a converged iterate computed WITHOUT probes is not available in one process (the
# debug mask is read once), so time iterations 0..T of a cold solve for two T and difference them:
# the late phase is iterations 300..600
def run(T):
    c.zero_(); d.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.check(_lib.lib.bccb_fista_run(op._plan, B, 0, T, 1.0 / L, tau.data_ptr(), bhat.data_ptr(), None,
                                       c.data_ptr(), d.data_ptr(), fb.data_ptr(), ws.data_ptr(), sp))
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)
run(50)
t300, t600 = run(300), run(600)
print("BCCB_DEBUG", os.environ.get("BCCB_DEBUG"), "ms(300)", t300, "ms(600)", t600, "ms per iteration 300..600", (t600 - t300) / 300)
P
done
cat $OUT/probe_*.txt
echo done
