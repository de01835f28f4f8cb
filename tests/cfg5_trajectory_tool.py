"""Config-5 snapshot trajectory: GPU FISTA after T iterations against float64 oracle iterates
(tests/golden/cfg5_trajectory.npz, made in the build container by running oracle.fista on the golden
measurements of tests/golden/cfg5_t1000.npz) — where along the 1000 iterations the fp32 engine
drifts from the float64 trajectory."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2509_13592_b200 as bb
from paper_2509_13592_b200 import scenes

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
g = np.load(os.path.join(root, "tests/golden/cfg5_t1000.npz"))
sn = np.load(os.path.join(root, "tests/golden/cfg5_trajectory.npz"))
w = scenes.workload(5)
geom = scenes.geometry_for(w)
op = bb.gram_operator(geom, w.l1, w.l2)
L = op.dimension
y = torch.as_tensor(g["y"][:1]).cuda()
prob = bb.LassoProblem.from_measurements(op, y, tau_fraction=w.tau_fraction)
out = []
for T in sorted(int(k[1:]) for k in sn.files if k.startswith("i")):
    res = bb.fista_solve(prob, bb.SolverConfig(iterations=T, step_size_mu=float(g["mu"])))
    ref = torch.zeros(L, dtype=torch.complex128, device="cuda")
    ref[torch.as_tensor(sn[f"i{T}"]).cuda()] = torch.as_tensor(sn[f"v{T}"]).cuda()
    est = res.estimate[0]
    err = float(torch.linalg.vector_norm(est - ref) / torch.linalg.vector_norm(ref))
    out.append({"T": T, "rel_l2": err, "nnz_gpu": int(torch.count_nonzero(est)), "nnz_ref": int(len(sn[f"i{T}"]))})
    print(out[-1], flush=True)
json.dump(out, open(sys.argv[1], "w"), indent=1) if len(sys.argv) > 1 else None
