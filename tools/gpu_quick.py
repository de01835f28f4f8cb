"""Quick GPU sanity check of the band-FFT operator and solvers against numpy fp64."""
import sys, time
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np
import torch
import paper_2509_13592_b200 as bb
from paper_2509_13592_b200 import scenes

rng = np.random.default_rng(0)

def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))

# 1. generic operators (full box) incl. non-pow2
for (l1, l2) in [(8, 4), (7, 5), (9, 6), (16, 16), (64, 32), (1, 6), (6, 1), (256, 256), (1024, 512)]:
    eig = rng.standard_normal((l1, l2)) + 1j * rng.standard_normal((l1, l2))
    op = bb.BccbOperator(l1, l2, eig)
    c = rng.standard_normal(l1 * l2) + 1j * rng.standard_normal(l1 * l2)
    ref = np.fft.ifft2(np.fft.fft2(c.reshape(l2, l1)) * eig.T).ravel()
    got = bb.bccb_matvec(op, c)
    print(f"generic matvec {l1}x{l2}: box=({op.k1},{op.k2}) rel={rel(got, ref):.2e}")

# 2. gram operators at config sizes
for cfg in (1, 2, 3, 4, 5):
    w = scenes.workload(cfg)
    geom = scenes.geometry_for(w)
    op = bb.gram_operator(geom, w.l1, w.l2)
    m1, m2 = geom.occupied_coordinates()
    eig_t = np.zeros((w.l2, w.l1)); np.add.at(eig_t, (m2 % w.l2, m1 % w.l1), w.l1 * w.l2)
    c = rng.standard_normal(w.l1 * w.l2) + 1j * rng.standard_normal(w.l1 * w.l2)
    ref = np.fft.ifft2(np.fft.fft2(c.reshape(w.l2, w.l1)) * eig_t).ravel()
    got = bb.bccb_matvec(op, c)
    print(f"gram matvec cfg{cfg} {w.l1}x{w.l2}: box=({op.k1},{op.k2}) rel={rel(got, ref):.2e}")
    # adjoint
    y = rng.standard_normal(op.element_count) + 1j * rng.standard_normal(op.element_count)
    E = np.zeros((w.l2, w.l1), complex)
    np.add.at(E, (m2 % w.l2, m1 % w.l1), y * (-1.0) ** (m1 + m2))
    bref = np.fft.ifft2(E).ravel() * (w.l1 * w.l2)
    bgot = bb.apply_adjoint(op, y)
    print(f"   adjoint rel={rel(bgot, bref):.2e}")

# 3. FISTA config-2 single snapshot vs numpy fp64 emulation
w = scenes.workload(2)
geom, ys, _ = scenes.make_scene(w, [0])
op = bb.gram_operator(geom, w.l1, w.l2)
m1, m2 = geom.occupied_coordinates()
E = np.zeros((w.l2, w.l1), complex); np.add.at(E, (m2, m1), ys[0] * (-1.0) ** (m1 + m2))
b = np.fft.ifft2(E).ravel() * (w.l1 * w.l2)
tau = w.tau_fraction * np.abs(b).max()
mu = 1.0 / (w.l1 * w.l2)
eig_t = np.zeros((w.l2, w.l1)); eig_t[m2, m1] = w.l1 * w.l2
def mv(x): return np.fft.ifft2(np.fft.fft2(x.reshape(w.l2, w.l1)) * eig_t).ravel()
def soft(z, k):
    m = np.abs(z)
    with np.errstate(divide="ignore", invalid="ignore"):
        f = np.maximum(1 - k / m, 0)
    return z * np.nan_to_num(f)
for T in (1, 10, 1000):
    cp = np.zeros(w.l1 * w.l2, complex); z = cp.copy(); a = 1.0
    t0 = time.time()
    for it in range(T):
        c = soft(z - mu * mv(z) + mu * b, mu * tau)
        an = 0.5 * (np.sqrt(1 + 4 * a * a) + 1)
        z = c + ((a - 1) / an) * (c - cp); cp = c; a = an
    tcpu = time.time() - t0
    prob = bb.LassoProblem(op, b, tau)
    r = bb.fista_solve(prob, bb.SolverConfig(iterations=T, step_size_mu=mu))
    print(f"FISTA cfg2 T={T}: rel={rel(r.estimate, cp):.2e} gpu {r.total_seconds*1e3:.2f} ms cpu {tcpu*1e3:.1f} ms")
    prob2 = bb.LassoProblem.from_measurements(op, ys[0], tau=tau)
    r2 = bb.fista_solve(prob2, bb.SolverConfig(iterations=T, step_size_mu=mu))
    print(f"   from_measurements rel={rel(r2.estimate, cp):.2e}")

# 4. batched throughput quick look (cfg2 batch 64, 100 its)
geom, ys, _ = scenes.make_scene(w)
prob = bb.LassoProblem.from_measurements(op, ys, tau_fraction=w.tau_fraction)
for T in (100, 1000):
    r = bb.fista_solve(prob, bb.SolverConfig(iterations=T, step_size_mu=mu))
    r = bb.fista_solve(prob, bb.SolverConfig(iterations=T, step_size_mu=mu))
    gpi = w.batch * w.l1 * w.l2 * T / r.total_seconds
    print(f"cfg2 batch64 T={T}: {r.total_seconds*1e3:.2f} ms  {gpi/1e9:.1f} G gpi/s  {gpi*80/6.455e12:.3f} of HBM roofline (80 B/gpi)")
idx, mag = bb.topk_peaks(r.estimate[:2], 8)
print("topk", idx.cpu().numpy()[0], mag.cpu().numpy()[0])
