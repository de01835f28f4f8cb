"""CPU oracle for the BCCB Gram hot path — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference leg may import it.  The GPU product
path (paper_2509_13592_b200) never calls into oracle/.

It restates, in float64 numpy, the reference algorithm of
/root/reference/pkg/src/bccblasso (arXiv 2509.13592) for the hot path, keeping
the reference's operation order so results match it bitwise where the same
numpy kernels run (pinned by tests/test_oracle_golden.py against fixtures made
from the real reference by oracle/gen_golden.py).  The FFT arithmetic is numpy's
pocketfft, exactly the third-party code the reference calls (numpy>=1.24,
pkg/pyproject.toml:11; 2.3.5 installed).
"""

import numpy as np

SINGULAR_GUARD = 1e-12       # bccb.py:22
STEP_SIZE_INFLATION = 1e-6   # solvers.py:24
POWER_TOL = 1e-10            # solvers.py:25
POWER_MAX_ITER = 5000        # solvers.py:26


class OracleDivergence(Exception):
    def __init__(self, iteration):
        self.iteration = iteration
        super().__init__(f"non-finite iterate at iteration {iteration}")


# ------------------------------------------------------------------ operator

def occupied_coordinates(occupancy: np.ndarray):
    """(m1, m2) in scan order m2 outer, m1 inner — arrays.py:55-62."""
    m2, m1 = np.nonzero(np.asarray(occupancy, dtype=bool).T)
    return m1, m2


def gram_first_column(m1, m2, l1: int, l2: int) -> np.ndarray:
    """r[q1 + q2*L1] = sum_m exp(+2j pi (m1 q1/L1 + m2 q2/L2)) — bccb.py:77-90."""
    p1 = np.exp(2j * np.pi * np.outer(np.arange(l1), m1) / l1)
    p2 = np.exp(2j * np.pi * np.outer(np.arange(l2), m2) / l2)
    return (p1 @ p2.T).ravel(order="F")


def eigenvalues_from_first_column(col: np.ndarray, l1: int, l2: int) -> np.ndarray:
    """(L1, L2) eigenvalues = fft2 of the (L2, L1) view, transposed — bccb.py:93-105."""
    return np.fft.fft2(np.asarray(col, dtype=np.complex128).reshape(l2, l1)).T


def gram_eigenvalues(occupancy, l1: int, l2: int) -> np.ndarray:
    """gram_operator(geometry, l1, l2).eigenvalues — bccb.py:108-110."""
    m1, m2 = occupied_coordinates(occupancy)
    return eigenvalues_from_first_column(gram_first_column(m1, m2, l1, l2), l1, l2)


def gram_eigenvalues_exact(occupancy, l1: int, l2: int) -> np.ndarray:
    """Closed form L1*L2 * (aliased occupancy count) — SURVEY finding 3, pinned by
    pkg/tests/test_bccb.py:116-125.  Used where the first column is too costly."""
    m1, m2 = occupied_coordinates(occupancy)
    eig = np.zeros((l1, l2), dtype=np.complex128)
    np.add.at(eig, (m1 % l1, m2 % l2), float(l1 * l2))
    return eig


def matvec(eig_t: np.ndarray, c: np.ndarray) -> np.ndarray:
    """ifft2(eig_t * fft2(c.reshape(L2, L1))).ravel() — bccb.py:113-125."""
    l2, l1 = eig_t.shape
    spectrum = np.fft.fft2(np.asarray(c).reshape(l2, l1))
    spectrum *= eig_t
    return np.fft.ifft2(spectrum).ravel()


# ------------------------------------------------------------------ adjoint

def adjoint_dense(m1, m2, l1: int, l2: int, y: np.ndarray) -> np.ndarray:
    """D_s^H y with the explicit dictionary on f = -1/2 + l/L — dictionary.py:41-45, 83-97, 129-136."""
    f1 = -0.5 + np.arange(l1) / l1
    f2 = -0.5 + np.arange(l2) / l2
    r1 = np.exp(-2j * np.pi * np.outer(m1, f1))
    r2 = np.exp(-2j * np.pi * np.outer(m2, f2))
    mat = (r2[:, :, None] * r1[:, None, :]).reshape(len(m1), l1 * l2)
    return mat.conj().T @ y


def dictionary_matrix(m1, m2, l1: int, l2: int) -> np.ndarray:
    """Explicit M x L1L2 dictionary, row (m1, m2), column l1 + l2*L1 — dictionary.py:83-97."""
    f1 = -0.5 + np.arange(l1) / l1
    f2 = -0.5 + np.arange(l2) / l2
    r1 = np.exp(-2j * np.pi * np.outer(m1, f1))
    r2 = np.exp(-2j * np.pi * np.outer(m2, f2))
    return (r2[:, :, None] * r1[:, None, :]).reshape(len(m1), l1 * l2)


def dense_gram(m1, m2, l1: int, l2: int) -> np.ndarray:
    """D_s^H D_s (the regular backend's DenseGram) — dictionary.py:155-168."""
    mat = dictionary_matrix(m1, m2, l1, l2)
    return mat.conj().T @ mat


def adjoint_fft(m1, m2, l1: int, l2: int, y: np.ndarray) -> np.ndarray:
    """Same b via L1*L2*ifft2 of the signed scatter E[m2, m1] = (-1)^(m1+m2) y_m
    (SURVEY finding 4; matches adjoint_dense to ~1e-15, tests/test_oracle_golden.py)."""
    e = np.zeros((l2, l1), dtype=np.complex128)
    np.add.at(e, (np.asarray(m2) % l2, np.asarray(m1) % l1), y * (-1.0) ** (np.asarray(m1) + np.asarray(m2)))
    return np.fft.ifft2(e).ravel() * (l1 * l2)


# ------------------------------------------------------------------ solvers

def soft_threshold(z: np.ndarray, kappa: float) -> np.ndarray:
    """z * max(1 - kappa/|z|, 0) — solvers.py:131-145."""
    z = np.asarray(z, dtype=np.complex128)
    if kappa == 0:
        return z.copy()
    magnitude = np.abs(z)
    with np.errstate(divide="ignore"):
        factor = np.maximum(1.0 - kappa / magnitude, 0.0)
    return z * factor


def prox_step(point, gz, b, mu: float, kappa: float) -> np.ndarray:
    """S_kappa(point - mu*G point + mu*b), this evaluation order — solvers.py:245-249."""
    return soft_threshold(point - mu * gz + mu * b, kappa)


def _finite(c, it):
    if not np.all(np.isfinite(c)):
        raise OracleDivergence(it)


def ista(eig_t, b, tau: float, mu: float, iterations: int, c0=None) -> np.ndarray:
    """Loop of ista_solve — solvers.py:264-278."""
    kappa = mu * tau
    c = np.zeros(b.size, dtype=np.complex128) if c0 is None else np.array(c0, dtype=np.complex128)
    for it in range(iterations):
        c = prox_step(c, matvec(eig_t, c), b, mu, kappa)
        _finite(c, it)
    return c


def ista_dense(gram: np.ndarray, b, tau: float, mu: float, iterations: int, c0=None) -> np.ndarray:
    """ista_solve on the regular backend: G c as a dense O(L^2) product (solvers.py:73-77,
    264-278) — the reference's dense baseline path."""
    kappa = mu * tau
    c = np.zeros(b.size, dtype=np.complex128) if c0 is None else np.array(c0, dtype=np.complex128)
    for it in range(iterations):
        c = prox_step(c, gram @ c, b, mu, kappa)
        _finite(c, it)
    return c


def next_alpha(alpha: float) -> float:
    """alpha' = (sqrt(1 + 4 alpha^2) + 1)/2 — solvers.py:294-296."""
    return 0.5 * (np.sqrt(1.0 + 4.0 * alpha * alpha) + 1.0)


def fista(eig_t, b, tau: float, mu: float, iterations: int, c0=None, snapshots_at=()):
    """Loop of fista_solve — solvers.py:322-343.  Returns the last c (= c_prev);
    with `snapshots_at`, also {t: c after t iterations}."""
    kappa = mu * tau
    c_prev = np.zeros(b.size, dtype=np.complex128) if c0 is None else np.array(c0, dtype=np.complex128)
    z = c_prev.copy()
    alpha = 1.0
    snaps = {}
    for it in range(iterations):
        c = prox_step(z, matvec(eig_t, z), b, mu, kappa)
        _finite(c, it)
        alpha_next = next_alpha(alpha)
        z = c + ((alpha - 1.0) / alpha_next) * (c - c_prev)
        c_prev = c
        alpha = alpha_next
        if it + 1 in snapshots_at:
            snaps[it + 1] = c_prev.copy()
    return (c_prev, snaps) if snapshots_at else c_prev


def admm(eig: np.ndarray, b, tau: float, rho: float, iterations: int, z0=None):
    """admm_solve fast backend — solvers.py:403-436.  Returns (z, c, v) of the last iteration."""
    shifted = eig + rho                                   # bccb_scale_add_identity(., 1, rho)
    mags = np.abs(shifted)
    if mags.min() <= SINGULAR_GUARD * mags.max():         # bccb_inverse guard, bccb.py:142-147
        raise ZeroDivisionError("singular shifted operator")
    inv_t = np.ascontiguousarray((1.0 / shifted).T)
    q = matvec(inv_t, b)
    kappa2 = rho * tau
    z = np.zeros(b.size, dtype=np.complex128) if z0 is None else np.array(z0, dtype=np.complex128)
    v = np.zeros(b.size, dtype=np.complex128)
    c = None
    for it in range(iterations):
        c = q + rho * matvec(inv_t, z - v)
        _finite(c, it)
        z = soft_threshold(c + v, kappa2)
        v = v + (c - z)
    return z, c, v


def power_max_eigenvalue(apply, dimension: int, seed: int = 0, tol: float = POWER_TOL,
                         max_iter: int = POWER_MAX_ITER) -> float:
    """Rayleigh-quotient power iteration — solvers.py:148-183."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(dimension) + 1j * rng.standard_normal(dimension)
    x /= np.linalg.norm(x)
    est = 0.0
    for k in range(max_iter):
        y = apply(x)
        val = float(np.real(np.vdot(x, y)))
        ny = float(np.linalg.norm(y))
        if ny == 0.0:
            return 0.0
        if k > 0 and abs(val - est) <= tol * max(abs(val), np.finfo(float).tiny):
            return val
        est = val
        x = y / ny
    raise RuntimeError("power iteration did not settle")


# ------------------------------------------------------------------ peaks

def topk(c: np.ndarray, k: int) -> np.ndarray:
    """First k of the stable argsort of -|c| (extract_support order, solvers.py:494-499)."""
    return np.argsort(-np.abs(c), kind="stable")[:k]


def extract_support(c, f1, f2, threshold_fraction: float):
    """solvers.py:476-507 (grids given as frequency vectors)."""
    mags = np.abs(c)
    peak = float(mags.max())
    if peak == 0.0:
        return []
    kept = np.flatnonzero(mags >= threshold_fraction * peak)
    kept = kept[np.argsort(-mags[kept], kind="stable")]
    l1 = len(f1)
    return [(float(f1[i % l1]), float(f2[i // l1]), complex(c[i])) for i in kept]


def rel_l2(est, ref) -> float:
    """||est - ref|| / ||ref|| (the experiments.relative_error convention, experiments.py:173-182)."""
    ref = np.asarray(ref)
    den = float(np.linalg.norm(ref))
    if den == 0.0:
        raise ZeroDivisionError("zero reference")
    return float(np.linalg.norm(np.asarray(est) - ref)) / den
