"""Float64 FISTA trajectory of config-5 snapshot 0 (build container; ~45 min on one core).

    python oracle/gen_golden_cfg5_trajectory.py [--complex64-operator]

Runs the pinned oracle (oracle/bccb_oracle.py fista = the loop of the reference's fista_solve,
/root/reference/pkg/src/bccblasso/solvers.py:322-343) on the measurements of
tests/golden/cfg5_t1000.npz (snapshot 0: the real reference's y, tau, mu) and stores the sparse
iterates after T = 50, 100, 200, 300, 400, 600, 800, 1000 iterations in
tests/golden/cfg5_trajectory.npz (i<T> indices, v<T> values).  The T = 1000 iterate is checked
against the REAL reference's estimate in the same fixture (est_b/est_i/est_v): they agree to
6.1e-7 relative L2 -- not to rounding, because the oracle uses the closed-form spectrum
L * occupancy while the reference FFTs a zgemm first column (1e-13 relative differences): FISTA's
momentum amplifies perturbations along the near-null directions of the restricted Gram roughly
like T^2.

--complex64-operator: the conditioning experiment.  Same float64 loop, but the operator output
G z is rounded to complex64 once per iteration (the least any complex64 engine does); prints the
relative L2 distance to the float64 trajectory at the stored T (profiles/parity/
cfg5_conditioning.txt).  Test infrastructure only.
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
from oracle import bccb_oracle as orc  # noqa: E402

AT = (50, 100, 200, 300, 400, 600, 800, 1000)
L = 4096


def inputs():
    d = np.load(os.path.join(ROOT, "tests", "golden", "cfg5_t1000.npz"))
    m1, m2 = orc.occupied_coordinates(d["occupancy"])
    eig_t = np.ascontiguousarray(orc.gram_eigenvalues_exact(d["occupancy"], L, L).T)
    b = orc.adjoint_fft(m1, m2, L, L, d["y"][0])
    return d, eig_t, b, float(d["mu"]), float(d["tau"][0])


def main():
    d, eig_t, b, mu, tau = inputs()
    out_path = os.path.join(ROOT, "tests", "golden", "cfg5_trajectory.npz")
    t0 = time.time()
    if "--complex64-operator" in sys.argv:
        sn = np.load(out_path)
        kappa = mu * tau
        c_prev = np.zeros(L * L, complex)
        z = c_prev.copy()
        alpha = 1.0
        for it in range(max(AT)):
            gz = orc.matvec(eig_t, z).astype(np.complex64).astype(np.complex128)
            c = orc.prox_step(z, gz, b, mu, kappa)
            an = orc.next_alpha(alpha)
            z = c + ((alpha - 1.0) / an) * (c - c_prev)
            c_prev, alpha = c, an
            if it + 1 in AT:
                ref = np.zeros(L * L, complex)
                ref[sn[f"i{it + 1}"]] = sn[f"v{it + 1}"]
                print(it + 1, np.linalg.norm(c - ref) / np.linalg.norm(ref), np.count_nonzero(c), flush=True)
        return
    c, snaps = orc.fista(eig_t, b, tau, mu, max(AT), snapshots_at=AT)
    out = {}
    for k, v in snaps.items():
        nz = np.flatnonzero(v)
        out[f"i{k}"] = nz
        out[f"v{k}"] = v[nz]
    np.savez(out_path, **out)
    sel = d["est_b"] == 0
    ref = np.zeros(L * L, complex)
    ref[d["est_i"][sel]] = d["est_v"][sel]
    print("seconds", time.time() - t0, "oracle vs reference at T=1000:", np.linalg.norm(c - ref) / np.linalg.norm(ref))


if __name__ == "__main__":
    main()
