"""ISTA / FISTA / ADMM on the GPU, behind the reference's solver signatures.

Drop-in for pkg/src/bccblasso/solvers.py: `LassoProblem`, `SolverConfig`,
`SolverResult`, `ista_solve`, `fista_solve`, `admm_solve`, `soft_threshold`,
`max_gram_eigenvalue`, `fista_alpha_sequence`, `extract_support`.  The whole
iteration loop runs as fused sm_100a kernels (include/bccb_b200.h:
bccb_fista_run / bccb_admm_run); Python only prepares device buffers, launches
one C call per solve and maps status codes onto the reference exceptions.

Extensions over the reference (which is single-snapshot): `adjoint_rhs` may be
(B, L) and `tau` a length-B vector; `LassoProblem.from_measurements` builds b and
tau = frac*max|b| on the GPU from raw snapshots (the A^H y of dictionary.py:129-136
as scatter + inverse FFT).
"""

import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .bccb import BccbOperator, _as_device_c64, _stream_ptr, bccb_matvec
from .errors import ConvergenceError, DivergenceError, InvalidArgumentError

BACKEND_REGULAR = "regular"
BACKEND_FAST = "fast"
STEP_SIZE_INFLATION = 1e-6   # solvers.py:24
POWER_TOL = 1e-10            # solvers.py:25
POWER_MAX_ITER = 5000        # solvers.py:26
POWER_SEED = 0               # solvers.py:27
INT_MAX = 2**31 - 1
# Out-of-band part of a user-supplied b below this fraction of max|b| is complex64
# round-off of an in-range b (b = A^H y has no off-box spectrum, SURVEY finding 4).
EXTRA_RHS_TOL = 1e-5


def _to_operator(gram) -> BccbOperator:
    if isinstance(gram, BccbOperator):
        return gram
    # the reference's BccbOperator (duck-typed): l1, l2, eigenvalues
    if all(hasattr(gram, a) for a in ("l1", "l2", "eigenvalues")):
        cached = getattr(gram, "_b200_operator", None)
        if cached is None:
            cached = BccbOperator(gram.l1, gram.l2, np.asarray(gram.eigenvalues))
            try:
                object.__setattr__(gram, "_b200_operator", cached)
            except (AttributeError, TypeError):
                pass
        return cached
    raise InvalidArgumentError("gram must be a BccbOperator (the dense regular backend is not "
                               "part of the GPU path)")


class LassoProblem:
    """One LASSO instance (or a batch sharing one operator) — solvers.py:30-77.

    gram        : BccbOperator (this package's or the reference's)
    adjoint_rhs : b = D_s^H y, shape (L,) or (B, L); numpy or CUDA tensor
    tau         : positive float or length-B vector
    """

    def __init__(self, gram, adjoint_rhs, tau, y_norm_sq=None, dictionary_matrix=None):
        self.gram = _to_operator(gram)
        tau_arr = tau.detach().cpu().numpy() if isinstance(tau, torch.Tensor) else np.asarray(tau, dtype=np.float64)
        if np.any(~(tau_arr > 0)):
            raise InvalidArgumentError("tau must be positive")
        self.tau = tau
        self.y_norm_sq = y_norm_sq
        self.dictionary_matrix = dictionary_matrix
        self._bhat = None
        self._extra = None
        self._tau_dev = None
        self._b_dense = None
        if adjoint_rhs is None:
            self.adjoint_rhs = None
            return
        rhs = adjoint_rhs
        self._was_numpy = not isinstance(rhs, torch.Tensor)
        shape = tuple(rhs.shape) if not self._was_numpy else np.shape(rhs)
        if len(shape) not in (1, 2):
            raise InvalidArgumentError("adjoint right-hand side must be 1D (or 2D for a batch)")
        if shape[-1] != self.gram.dimension:
            raise InvalidArgumentError(
                f"adjoint right-hand side length {shape[-1]} does not match the gram dimension "
                f"{self.gram.dimension}")
        self._squeeze = len(shape) == 1
        self.batch = 1 if self._squeeze else int(shape[0])
        if tau_arr.ndim == 1 and tau_arr.size not in (1, self.batch):
            raise InvalidArgumentError("tau vector length does not match the batch")
        self.adjoint_rhs = rhs

    # -- native batched constructor (GPU adjoint)
    @classmethod
    def from_measurements(cls, gram: BccbOperator, y, tau_fraction: float | None = None,
                          tau=None, keep_b: bool = False) -> "LassoProblem":
        """b = A^H y and tau = frac * max|b| per snapshot, all on the GPU.

        y: (M,) or (B, M) measurements in occupancy scan order (arrays.py:55-62).
        """
        op = _to_operator(gram)
        if op.element_count < 1:
            raise InvalidArgumentError("from_measurements needs a Gram operator (gram_operator)")
        was_numpy = not isinstance(y, torch.Tensor)
        yt = _as_device_c64(y, op.device)
        squeeze = yt.dim() == 1
        yt = yt.reshape(-1, op.element_count)
        batch = yt.shape[0]
        dev = yt.device
        bhat = torch.empty((batch, op.k1, op.k2), dtype=torch.complex64, device=dev)
        maxabs = torch.zeros(batch, dtype=torch.float32, device=dev)
        b = torch.empty((batch, op.dimension), dtype=torch.complex64, device=dev) if keep_b else None
        _lib.check(_lib.lib.bccb_adjoint(op._plan, batch, yt.data_ptr(), bhat.data_ptr(),
                                         b.data_ptr() if b is not None else None, maxabs.data_ptr(),
                                         op.workspace(batch).data_ptr(), _stream_ptr(op.device)))
        if tau is None:
            if tau_fraction is None or not tau_fraction > 0:
                raise InvalidArgumentError("give tau or a positive tau_fraction")
            tau_dev = maxabs.to(torch.float64) * float(tau_fraction)
        else:
            tau_dev = torch.as_tensor(np.broadcast_to(np.asarray(tau, dtype=np.float64), (batch,)).copy(),
                                      device=dev)
        self = cls.__new__(cls)
        self.gram = op
        self.tau = tau_dev
        self.y_norm_sq = (yt.abs() ** 2).sum(dim=1).to(torch.float64)
        self.dictionary_matrix = None
        self.adjoint_rhs = b
        self._was_numpy = was_numpy
        self._squeeze = squeeze
        self.batch = batch
        self._bhat = bhat
        self._extra = None
        self._tau_dev = tau_dev
        self._b_dense = b
        self.maxabs_b = maxabs
        return self

    @property
    def dimension(self) -> int:
        return self.gram.dimension

    def device_data(self):
        """(bhat box, extra-or-None, tau (B,) float64) on the operator's device."""
        if self._bhat is None:
            op = self.gram
            batch = self.batch
            b = _as_device_c64(self.adjoint_rhs, op.device).reshape(batch, op.dimension)
            stream = _stream_ptr(op.device)
            ws = op.workspace(batch).data_ptr()
            bhat = torch.empty((batch, op.k1, op.k2), dtype=torch.complex64, device=b.device)
            _lib.check(_lib.lib.bccb_spectrum_box(op._plan, batch, b.data_ptr(), bhat.data_ptr(), ws, stream))
            extra = None
            if not op.is_full_box:
                # residual b - ifft2(box part): nonzero only for a b outside range(A^H)
                resid = torch.empty_like(b)
                rmax = torch.zeros(batch, dtype=torch.float32, device=b.device)
                _lib.check(_lib.lib.bccb_synthesize(op._plan, batch, bhat.data_ptr(), -1.0 / op.dimension,
                                                    b.data_ptr(), 1.0, resid.data_ptr(), rmax.data_ptr(), ws,
                                                    stream))
                bmax = b.abs().amax(dim=1)
                if bool((rmax > EXTRA_RHS_TOL * bmax).any()):
                    extra = resid
            self._bhat, self._extra, self._b_dense = bhat, extra, b
        if self._tau_dev is None:
            t = self.tau
            if isinstance(t, torch.Tensor):
                t = t.detach().to(device=self._bhat.device, dtype=torch.float64).reshape(-1)
            else:
                t = torch.as_tensor(np.asarray(t, dtype=np.float64).reshape(-1), device=self._bhat.device)
            if t.numel() == 1:
                t = t.expand(self.batch).contiguous()
            self._tau_dev = t
        return self._bhat, self._extra, self._tau_dev


@dataclass(frozen=True, eq=False)
class SolverConfig:
    """Iterations, hyper-parameters, backend (solvers.py:88-114)."""

    iterations: int
    step_size_mu: float | None = None
    rho: float = 1.0
    initial_c: object = None
    backend: str | None = None
    record_objective: bool = False
    power_seed: int = POWER_SEED

    def __post_init__(self) -> None:
        if self.iterations < 1:
            raise InvalidArgumentError("iteration count must be positive")
        if self.step_size_mu is not None and self.step_size_mu <= 0:
            raise InvalidArgumentError("step size must be positive")
        if self.rho <= 0:
            raise InvalidArgumentError("rho must be positive")
        if self.backend not in (None, BACKEND_REGULAR, BACKEND_FAST):
            raise InvalidArgumentError(f"unknown backend {self.backend!r}")


@dataclass(frozen=True, eq=False)
class SolverResult:
    """Estimate plus loop timing (solvers.py:117-128); timing is CUDA-event device time."""

    estimate: object
    objective_trace: np.ndarray
    per_iteration_seconds: float
    total_seconds: float
    backend: str
    iterations: int
    precompute_seconds: float
    step_size_mu: float | None = None


def soft_threshold(z, kappa: float):
    """Phase-preserving shrinkage z * max(1 - kappa/|z|, 0) (solvers.py:131-145)."""
    if kappa < 0:
        raise InvalidArgumentError("threshold must be nonnegative")
    if isinstance(z, torch.Tensor):
        if kappa == 0:
            return z.clone()
        mag = z.abs()
        scale = torch.clamp(1.0 - kappa / mag, min=0.0)
        scale = torch.where(mag == 0, torch.zeros_like(scale), scale)
        return z * scale
    z = np.asarray(z, dtype=np.complex128)
    if kappa == 0:
        return z.copy()
    mag = np.abs(z)
    with np.errstate(divide="ignore"):
        scale = np.maximum(1.0 - kappa / mag, 0.0)
    return z * scale


def fista_alpha_sequence(count: int) -> np.ndarray:
    """alpha_0 = 1, alpha_{t+1} = (sqrt(1 + 4 alpha_t^2) + 1)/2 (solvers.py:294-308)."""
    if count < 1:
        raise InvalidArgumentError("sequence length must be positive")
    out = np.empty(count)
    a = 1.0
    for i in range(count):
        out[i] = a
        a = 0.5 * (np.sqrt(1.0 + 4.0 * a * a) + 1.0)
    return out


def max_gram_eigenvalue(gram_apply, dimension: int, tol: float = POWER_TOL,
                        max_iter: int = POWER_MAX_ITER, seed: int = POWER_SEED) -> float:
    """Largest eigenvalue of a Hermitian PSD operator (solvers.py:148-183).

    `gram_apply` may be a callable on numpy vectors (as in the reference) or a
    BccbOperator, whose spectrum gives the answer exactly (SURVEY finding 3).
    """
    if dimension < 1:
        raise InvalidArgumentError("operator dimension must be positive")
    if isinstance(gram_apply, BccbOperator) and gram_apply.is_hermitian_psd():
        return gram_apply.max_eigenvalue()
    apply = (lambda v: bccb_matvec(gram_apply, v)) if isinstance(gram_apply, BccbOperator) else gram_apply
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(dimension) + 1j * rng.standard_normal(dimension)
    x /= np.linalg.norm(x)
    previous = 0.0
    for k in range(max_iter):
        y = np.asarray(apply(x))
        rq = float(np.real(np.vdot(x, y)))
        ny = float(np.linalg.norm(y))
        if ny == 0.0:
            return 0.0
        if k > 0 and abs(rq - previous) <= tol * max(abs(rq), np.finfo(float).tiny):
            return rq
        previous = rq
        x = y / ny
    raise ConvergenceError(f"power iteration did not settle within {max_iter} iterations", previous)


def _resolve_backend(problem: LassoProblem, config: SolverConfig) -> str:
    if config.backend == BACKEND_REGULAR:
        raise InvalidArgumentError("the regular (dense) backend is not part of the GPU path; "
                                   "use the reference package for it")
    return BACKEND_FAST


def _auto_mu(problem: LassoProblem, config: SolverConfig) -> float:
    op = problem.gram
    if op.is_hermitian_psd():
        lam = op.max_eigenvalue()
    else:
        lam = max_gram_eigenvalue(op, op.dimension, tol=1e-6, seed=config.power_seed)
    if lam <= 0:
        raise InvalidArgumentError("cannot derive a step size from a zero operator")
    return 1.0 / (lam * (1.0 + STEP_SIZE_INFLATION))


def _initial_state(problem: LassoProblem, config: SolverConfig, dtype) -> torch.Tensor:
    op = problem.gram
    shape = (problem.batch, op.dimension)
    dev = f"cuda:{op.device}"
    if config.initial_c is None:
        return torch.zeros(shape, dtype=dtype, device=dev)
    init = config.initial_c
    if isinstance(init, torch.Tensor):
        t = init.to(device=dev, dtype=dtype)
    else:
        t = torch.from_numpy(np.array(init, dtype=np.complex128)).to(dev).to(dtype)
    if t.shape[-1] != op.dimension or t.numel() not in (op.dimension, problem.batch * op.dimension):
        raise InvalidArgumentError("initial vector length does not match the problem")
    return t.reshape(1, -1).expand(shape).contiguous() if t.numel() == op.dimension else t.reshape(shape).contiguous()


def _require_y_norm(problem: LassoProblem):
    if problem.y_norm_sq is None:
        raise InvalidArgumentError("recording the objective trace requires y_norm_sq")
    return problem.y_norm_sq


def _finish(problem: LassoProblem, est: torch.Tensor):
    out = est.reshape(problem.batch, problem.gram.dimension)
    if problem._squeeze:
        out = out[0]
    if problem._was_numpy:
        return out.cpu().numpy().astype(np.complex128)
    return out


def _check_divergence(first_bad: torch.Tensor) -> None:
    fb = first_bad.cpu().numpy()
    bad = fb < INT_MAX
    if bad.any():
        per = np.where(bad, fb, -1)
        raise DivergenceError(int(fb[bad].min()), per_snapshot=per)


def _objective(problem: LassoProblem, c: torch.Tensor, tau_dev: torch.Tensor, y_norm) -> np.ndarray:
    """||y||^2 - 2 Re<b,c> + Re<c,Gc> + tau ||c||_1 per snapshot (solvers.py:233-242), on device."""
    op = problem.gram
    b = problem._b_dense.to(torch.complex128)
    c128 = c.to(torch.complex128)
    gc = bccb_matvec(op, c.to(torch.complex64)).to(torch.complex128)
    yn = torch.as_tensor(y_norm, dtype=torch.float64, device=c.device).reshape(-1)
    val = (yn - 2.0 * (b.conj() * c128).sum(dim=1).real + (c128.conj() * gc).sum(dim=1).real
           + tau_dev * c128.abs().sum(dim=1))
    return val.cpu().numpy()


def _fista_like(problem: LassoProblem, config: SolverConfig, momentum: bool) -> SolverResult:
    backend = _resolve_backend(problem, config)
    op = problem.gram
    t0 = time.perf_counter()
    mu = config.step_size_mu if config.step_size_mu is not None else _auto_mu(problem, config)
    bhat, extra, tau_dev = problem.device_data()
    c = _initial_state(problem, config, torch.complex128)
    d = torch.zeros((problem.batch, op.dimension), dtype=torch.complex64, device=c.device) if momentum else None
    first_bad = torch.empty(problem.batch, dtype=torch.int32, device=c.device)
    ws = op.workspace(problem.batch)
    stream = _stream_ptr(op.device)
    record = config.record_objective
    y_norm = _require_y_norm(problem) if record else None
    precompute = time.perf_counter() - t0
    T = config.iterations
    trace = np.zeros((problem.batch, T if record else 0))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    args = lambda first, n: (op._plan, problem.batch, first, n, float(mu), tau_dev.data_ptr(),  # noqa: E731
                             bhat.data_ptr(), extra.data_ptr() if extra is not None else None,
                             c.data_ptr(), d.data_ptr() if d is not None else None,
                             first_bad.data_ptr(), ws.data_ptr(), stream)
    ev0.record()
    fused = False
    if record and extra is None and config.initial_c is None:
        # objective trace fused into the pass kernels (device reductions, one call)
        tr = torch.empty((problem.batch, T), dtype=torch.float64, device=c.device)
        rc = _lib.lib.bccb_fista_run_traced(op._plan, problem.batch, T, float(mu), tau_dev.data_ptr(),
                                            bhat.data_ptr(), c.data_ptr(), d.data_ptr() if d is not None else None,
                                            first_bad.data_ptr(), tr.data_ptr(), ws.data_ptr(), stream)
        if rc != _lib.ERR_UNSUPPORTED:
            _lib.check(rc)
            fused = True
    if not record:
        _lib.check(_lib.lib.bccb_fista_run(*args(0, T)))
    elif not fused:
        # per-iteration slow path (generic operators, b off the box, small grids)
        if problem._b_dense is None:
            raise InvalidArgumentError("recording the objective trace needs the dense b (keep_b=True)")
        for t in range(T):
            _lib.check(_lib.lib.bccb_fista_run(*args(t, 1)))
            trace[:, t] = _objective(problem, c, tau_dev, y_norm)
    ev1.record()
    ev1.synchronize()
    elapsed = ev0.elapsed_time(ev1) / 1e3
    _check_divergence(first_bad)
    if fused:
        yn = torch.as_tensor(y_norm, dtype=torch.float64, device=c.device).reshape(-1, 1)
        trace = (tr + yn).cpu().numpy()
    return SolverResult(
        estimate=_finish(problem, c),
        objective_trace=trace[0] if problem._squeeze else trace,
        per_iteration_seconds=elapsed / T,
        total_seconds=elapsed,
        backend=backend,
        iterations=T,
        precompute_seconds=precompute,
        step_size_mu=mu,
    )


def ista_solve(problem: LassoProblem, config: SolverConfig) -> SolverResult:
    """c <- S_{mu tau}(c - mu G c + mu b), fused on the GPU (solvers.py:252-291)."""
    return _fista_like(problem, config, momentum=False)


def fista_solve(problem: LassoProblem, config: SolverConfig) -> SolverResult:
    """ISTA with Nesterov momentum (solvers.py:311-355); step 1 equals one ISTA step bitwise."""
    return _fista_like(problem, config, momentum=True)


def admm_solve(problem: LassoProblem, config: SolverConfig, iterate_callback=None) -> SolverResult:
    """Three-step ADMM; the estimate is the final z (solvers.py:385-448).

    `iterate_callback(iteration, c, z, v)` runs on a per-iteration slow path
    (arrays handed over as host complex128 numpy for numpy problems).
    """
    backend = _resolve_backend(problem, config)
    op = problem.gram
    t0 = time.perf_counter()
    bhat, extra, tau_dev = problem.device_data()
    z = _initial_state(problem, config, torch.complex128)
    v = torch.zeros(z.shape, dtype=torch.complex128, device=z.device)
    first_bad = torch.empty(problem.batch, dtype=torch.int32, device=z.device)
    ws = op.workspace(problem.batch)
    stream = _stream_ptr(op.device)
    record = config.record_objective
    y_norm = _require_y_norm(problem) if record else None
    slow = record or iterate_callback is not None
    c_last = torch.empty_like(v) if slow else None
    precompute = time.perf_counter() - t0
    T = config.iterations
    trace = np.zeros((problem.batch, T if record else 0))
    args = lambda first, n: (op._plan, problem.batch, first, n, float(config.rho), tau_dev.data_ptr(),  # noqa: E731
                             bhat.data_ptr(), extra.data_ptr() if extra is not None else None,
                             z.data_ptr(), v.data_ptr(), c_last.data_ptr() if c_last is not None else None,
                             first_bad.data_ptr(), ws.data_ptr(), stream)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    if not slow:
        _lib.check(_lib.lib.bccb_admm_run(*args(0, T)))
    else:
        for t in range(T):
            _lib.check(_lib.lib.bccb_admm_run(*args(t, 1)))
            if iterate_callback is not None:
                iterate_callback(t, _finish(problem, c_last), _finish(problem, z), _finish(problem, v))
            if record:
                trace[:, t] = _objective(problem, z, tau_dev, y_norm)
    ev1.record()
    ev1.synchronize()
    elapsed = ev0.elapsed_time(ev1) / 1e3
    _check_divergence(first_bad)
    return SolverResult(
        estimate=_finish(problem, z),
        objective_trace=trace[0] if problem._squeeze else trace,
        per_iteration_seconds=elapsed / T,
        total_seconds=elapsed,
        backend=backend,
        iterations=T,
        precompute_seconds=precompute,
        step_size_mu=config.step_size_mu,
    )


def admm_solve_with_c(problem: LassoProblem, config: SolverConfig):
    """ADMM returning (result, c of the last iteration) — the parity hook for config 3,
    where the reference's z is identically zero (SURVEY finding 7)."""
    op = problem.gram
    bhat, extra, tau_dev = problem.device_data()
    z = _initial_state(problem, config, torch.complex128)
    v = torch.zeros(z.shape, dtype=torch.complex128, device=z.device)
    c_last = torch.empty_like(v)
    first_bad = torch.empty(problem.batch, dtype=torch.int32, device=z.device)
    _lib.check(_lib.lib.bccb_admm_run(op._plan, problem.batch, 0, config.iterations, float(config.rho),
                                      tau_dev.data_ptr(), bhat.data_ptr(),
                                      extra.data_ptr() if extra is not None else None, z.data_ptr(),
                                      v.data_ptr(), c_last.data_ptr(), first_bad.data_ptr(),
                                      op.workspace(problem.batch).data_ptr(), _stream_ptr(op.device)))
    torch.cuda.synchronize(op.device)
    _check_divergence(first_bad)
    return z, v, c_last


# ----------------------------------------------------------------------------- peaks

def topk_peaks(values, k: int):
    """Per-snapshot top-k of |values| in extract_support order (solvers.py:494-499).

    values: (L,) or (B, L) complex, numpy or CUDA tensor.  Returns (idx int32 (B, k),
    mag float32 (B, k)) device tensors.
    """
    if isinstance(values, torch.Tensor):
        t = values
    else:
        t = torch.from_numpy(np.ascontiguousarray(values)).cuda()
    if t.dtype not in (torch.complex64, torch.complex128):
        t = t.to(torch.complex128)
    t = t.reshape(-1, t.shape[-1]).contiguous()
    batch, length = t.shape
    is_double = 1 if t.dtype == torch.complex128 else 0
    idx = torch.empty((batch, k), dtype=torch.int32, device=t.device)
    mag = torch.empty((batch, k), dtype=torch.float32, device=t.device)
    nbytes = int(_lib.lib.bccb_topk_workspace_bytes(batch, length, k))
    ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=t.device)
    _lib.check(_lib.lib.bccb_topk(batch, length, t.data_ptr(), is_double, k, idx.data_ptr(),
                                  mag.data_ptr(), ws.data_ptr(), torch.cuda.current_stream(t.device).cuda_stream))
    return idx, mag


def extract_support(c_hat, grid1, grid2, threshold_fraction: float):
    """Entries with |c| >= frac * max|c|, by descending magnitude (solvers.py:476-507).

    Selection runs on the GPU through the top-k kernel (float64 magnitudes, ties to the lower
    index); the threshold is applied to float64 magnitudes exactly as the reference does.  When
    more than 64 entries clear the threshold the ordering falls back to a device-side stable sort.
    """
    if not 0.0 < threshold_fraction < 1.0:
        raise InvalidArgumentError("threshold fraction must lie strictly between 0 and 1")
    n = grid1.length * grid2.length
    shape = tuple(c_hat.shape) if isinstance(c_hat, torch.Tensor) else np.shape(c_hat)
    if shape != (n,):
        raise InvalidArgumentError("coefficient length does not match the grids")
    host = c_hat.detach().cpu().numpy() if isinstance(c_hat, torch.Tensor) else np.asarray(c_hat)
    host = host.astype(np.complex128, copy=False)
    k = min(64, n)
    idx, _ = topk_peaks(c_hat if isinstance(c_hat, torch.Tensor) else host, k)
    idx = idx[0].cpu().numpy().astype(np.int64)
    mag = np.abs(host[idx])                       # float64, as np.abs in the reference
    peak = float(mag[0])
    if peak == 0.0:
        return []
    thr = threshold_fraction * peak
    if k < n and mag[-1] >= thr:
        dev = torch.as_tensor(np.abs(host)).cuda()
        order = torch.sort(-dev, stable=True).indices
        keep = (dev[order] >= thr).cpu().numpy()
        kept = order.cpu().numpy()[keep]
    else:
        kept = idx[mag >= thr]
    l1 = grid1.length
    return [(float(grid1.frequencies[i % l1]), float(grid2.frequencies[i // l1]), complex(host[i]))
            for i in kept]
