"""Is the per-pass solve host-launch bound?  Times one full FISTA solve three ways:
(1) plain enqueue (host wall time of the enqueue vs device time), (2) replay of a CUDA
graph captured around the same call (torch.cuda.graph), (3) env-selected variants."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_13592_b200 as bb
from paper_2509_13592_b200 import _lib, scenes
from paper_2509_13592_b200.bccb import _stream_ptr

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
T = int(sys.argv[2]) if len(sys.argv) > 2 else 0
w = scenes.workload(cfg)
T = T or w.iterations
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


def run(stream_ptr):
    _lib.check(_lib.lib.bccb_fista_run(op._plan, B, 0, T, 1.0 / L, tau.data_ptr(), bhat.data_ptr(), None,
                                       c.data_ptr(), d.data_ptr(), fb.data_ptr(), ws.data_ptr(), stream_ptr))


def timed(fn, reps=3):
    out = []
    for _ in range(reps):
        c.zero_(); d.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0 = time.perf_counter()
        e0.record(); fn(); e1.record()
        h1 = time.perf_counter()
        e1.synchronize()
        out.append((round(e0.elapsed_time(e1), 3), round((h1 - h0) * 1e3, 3)))
    return out


run(_stream_ptr(0)); torch.cuda.synchronize()
res = {"cfg": cfg, "T": T, "plain [device_ms, host_enqueue_ms]": timed(lambda: run(_stream_ptr(0)))}
ref = c.clone()
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
c.zero_(); d.zero_()
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.graph(g, stream=s):
    run(s.cuda_stream)
t1 = time.perf_counter()
res["capture_ms"] = round((t1 - t0) * 1e3, 2)
res["graph [device_ms, host_ms]"] = timed(g.replay)
res["graph_bitwise_equal"] = bool(torch.equal(c, ref))
print(json.dumps(res))
