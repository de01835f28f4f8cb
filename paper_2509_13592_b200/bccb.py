"""Device-resident BCCB operators (drop-in for pkg/src/bccblasso/bccb.py).

A `BccbOperator` here owns a C-ABI plan (include/bccb_b200.h) holding the
eigenvalues on the GPU as a spectral BOX [0,K1) x [0,K2) plus one constant value
outside it.  For the Gram of a sparse array the box is the occupied corner
(reference pin: pkg/tests/test_bccb.py:116-125) and every pass is band-limited;
for a generic operator the box is the whole grid.

Vectors follow the reference convention l = l1 + l2*L1 (bccb.py:10-11).  All
functions accept numpy arrays (returned as complex128 numpy, like the reference)
or CUDA torch tensors (returned as CUDA tensors), with an optional leading batch
dimension.  Arithmetic is complex64 on the GPU (BASELINE.json north_star).
"""

import ctypes
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import InvalidArgumentError, SingularOperatorError

SINGULAR_GUARD = 1e-12    # bccb.py:22


def _device_index(device) -> int:
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("the BCCB GPU path needs a CUDA device (no CPU fallback)")
        return torch.cuda.current_device()
    d = torch.device(device)
    if d.type != "cuda":
        raise InvalidArgumentError("BCCB operators live on a CUDA device")
    return d.index if d.index is not None else torch.cuda.current_device()


def _stream_ptr(device: int) -> int:
    return torch.cuda.current_stream(device).cuda_stream


@dataclass(frozen=True, eq=False)
class FirstColumn:
    """Characterising first column of a BCCB matrix (bccb.py:26-37)."""

    values: np.ndarray

    def __post_init__(self) -> None:
        v = np.ascontiguousarray(self.values, dtype=np.complex128)
        if v.ndim != 1 or v.size < 1:
            raise InvalidArgumentError("first column must be a nonempty 1D vector")
        v.setflags(write=False)
        object.__setattr__(self, "values", v)


class BccbOperator:
    """BCCB matrix stored as eigenvalues on the GPU (reference: bccb.py:50-74).

    `BccbOperator(l1, l2, eigenvalues)` accepts the reference's (L1, L2) eigenvalue
    matrix; a zero region outside a corner box [0,K1) x [0,K2) is detected and
    pruned.  The host `eigenvalues` matrix is materialised lazily on access.
    """

    def __init__(self, l1: int, l2: int, eigenvalues=None, *, device=None, _box=None,
                 _lam_out=0.0, _gram=None):
        if l1 < 1 or l2 < 1:
            raise InvalidArgumentError("block sizes must be positive")
        self.l1, self.l2 = int(l1), int(l2)
        self.device = _device_index(device)
        self._eig_host = None
        self._ws = threading.local()    # scratch per calling thread
        handle = ctypes.c_void_p()
        if _gram is not None:
            m1c, m2c, occ = _gram
            occ_u8 = np.ascontiguousarray(occ, dtype=np.uint8)
            _lib.check(_lib.lib.bccb_plan_create_gram(
                self.l1, self.l2, m1c, m2c, occ_u8.ctypes.data, self.device, ctypes.byref(handle)))
        else:
            if _box is None:
                eig = np.asarray(eigenvalues, dtype=np.complex128)
                if eig.shape != (self.l1, self.l2):
                    raise InvalidArgumentError(
                        f"eigenvalue matrix shape {eig.shape} does not match ({self.l1}, {self.l2})")
                self._eig_host = eig
                _box, _lam_out = _detect_box(eig)
            box = np.ascontiguousarray(_box, dtype=np.complex128)
            k1, k2 = box.shape
            lo = complex(_lam_out)
            _lib.check(_lib.lib.bccb_plan_create(
                self.l1, self.l2, k1, k2, box.ctypes.data, lo.real, lo.imag, self.device,
                ctypes.byref(handle)))
        self._plan = handle
        l1c, l2c, k1c, k2c, mc = (ctypes.c_int() for _ in range(5))
        _lib.check(_lib.lib.bccb_plan_info(self._plan, *(ctypes.byref(v) for v in (l1c, l2c, k1c, k2c, mc))))
        self.k1, self.k2, self.element_count = k1c.value, k2c.value, mc.value
        box = np.empty((self.k1, self.k2), dtype=np.complex128)
        re, im = ctypes.c_double(), ctypes.c_double()
        _lib.check(_lib.lib.bccb_plan_eigen_box(self._plan, box.ctypes.data, ctypes.byref(re), ctypes.byref(im)))
        self.box = box                       # eigenvalues[k1, k2] on the box (host copy)
        self.lam_out = complex(re.value, im.value)

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan is not None and plan.value:
            try:
                _lib.lib.bccb_plan_destroy(plan)
            except Exception:
                pass
            self._plan = None

    # -- reference-compatible surface
    @property
    def dimension(self) -> int:
        return self.l1 * self.l2

    @property
    def is_full_box(self) -> bool:
        return self.k1 == self.l1 and self.k2 == self.l2

    @property
    def eigenvalues(self) -> np.ndarray:
        """(L1, L2) complex128 eigenvalue matrix (bccb.py:56), built on first access."""
        if self._eig_host is None:
            eig = np.full((self.l1, self.l2), self.lam_out, dtype=np.complex128)
            eig[: self.k1, : self.k2] = self.box
            eig.setflags(write=False)
            self._eig_host = eig
        return self._eig_host

    @property
    def _eig_t(self) -> np.ndarray:
        return np.ascontiguousarray(self.eigenvalues.T)

    def all_eigen_magnitudes(self) -> tuple[float, float]:
        """(min |eig|, max |eig|) over the whole grid without materialising it."""
        mags = np.abs(self.box)
        lo, hi = float(mags.min()), float(mags.max())
        if not self.is_full_box:
            o = abs(self.lam_out)
            lo, hi = min(lo, o), max(hi, o)
        return lo, hi

    def is_hermitian_psd(self) -> bool:
        ok = bool(np.all(np.abs(self.box.imag) <= 1e-9 * max(1.0, np.abs(self.box).max()))
                  and np.all(self.box.real >= -1e-9 * max(1.0, np.abs(self.box).max())))
        if not self.is_full_box:
            ok = ok and self.lam_out.imag == 0 and self.lam_out.real >= 0
        return ok

    def max_eigenvalue(self) -> float:
        """max Re(eig) for a Hermitian PSD operator (= the Gram's L1*L2, SURVEY finding 3)."""
        m = float(self.box.real.max())
        if not self.is_full_box:
            m = max(m, self.lam_out.real)
        return m

    def workspace(self, batch: int) -> torch.Tensor:
        """Scratch for one call of `batch` snapshots.  Cached per calling thread and CUDA
        stream, so concurrent matvecs / solves on one operator never share intermediates
        (reference contract SPEC.md:325: scratch per call or per thread)."""
        stream = torch.cuda.current_stream(self.device).cuda_stream
        cache = getattr(self._ws, "cache", None)
        if cache is None:
            cache = self._ws.cache = {}
        ws = cache.get((batch, stream))
        if ws is None:
            nbytes = int(_lib.lib.bccb_workspace_bytes(self._plan, batch))
            ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=f"cuda:{self.device}")
            cache.clear()                  # keep one size per thread
            cache[(batch, stream)] = ws
        return ws

    def __repr__(self) -> str:
        return (f"BccbOperator(l1={self.l1}, l2={self.l2}, box=({self.k1}, {self.k2}), "
                f"device=cuda:{self.device})")


def _detect_box(eig: np.ndarray):
    """Smallest corner box [0,K1) x [0,K2) outside which the eigenvalues are exactly zero."""
    nz = eig != 0
    if not nz.any():
        return eig[:1, :1].copy(), 0.0
    rows = np.flatnonzero(nz.any(axis=1))
    cols = np.flatnonzero(nz.any(axis=0))
    k1, k2 = int(rows[-1]) + 1, int(cols[-1]) + 1
    return eig[:k1, :k2].copy(), 0.0


def _occupancy_of(geometry):
    occ = np.asarray(geometry.occupancy, dtype=bool)
    return int(geometry.m1_count), int(geometry.m2_count), occ


# ----------------------------------------------------------------------------- construction

def gram_operator(geometry, l1: int, l2: int, device=None) -> BccbOperator:
    """Gram D_s^H D_s of `geometry` on the uniform L1 x L2 grid (bccb.py:108-110).

    Built directly from the occupancy (eigenvalues = L1*L2 on occupied cells; no
    O(M L) first column, no zgemm).  Accepts this package's ArrayGeometry or the
    reference's (duck-typed: m1_count, m2_count, occupancy).
    """
    if l1 < 1 or l2 < 1:
        raise InvalidArgumentError("grid lengths must be positive")
    op = BccbOperator(l1, l2, device=device, _gram=_occupancy_of(geometry))
    op.geometry = geometry
    return op


def _as_device_c64(x, device: int) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=f"cuda:{device}", dtype=torch.complex64).contiguous()
    arr = np.ascontiguousarray(x, dtype=np.complex64)
    return torch.from_numpy(arr).to(f"cuda:{device}")


def bccb_from_first_column(col, l1: int, l2: int, device=None) -> BccbOperator:
    """Operator whose dense form has first column `col` (bccb.py:93-105).

    The eigenvalues fft2(col.reshape(L2, L1)) are computed on the GPU.
    """
    values = col.values if isinstance(col, FirstColumn) else np.ascontiguousarray(col, dtype=np.complex128)
    if values.ndim != 1:
        raise InvalidArgumentError("first column must be a 1D vector")
    if values.size != l1 * l2:
        raise InvalidArgumentError(f"first column length {values.size} does not match L1*L2 = {l1 * l2}")
    dev = _device_index(device)
    probe = BccbOperator(l1, l2, device=dev, _box=np.ones((l1, l2)), _lam_out=0.0)
    x = torch.from_numpy(np.ascontiguousarray(values, dtype=np.complex128)).to(f"cuda:{dev}")
    box = torch.empty((1, probe.k1, probe.k2), dtype=torch.complex128, device=x.device)
    # float64 band engine: the reference computes fft2 in float64 (bccb.py:104)
    _lib.check(_lib.lib.bccb_spectrum_box_z(probe._plan, 1, x.data_ptr(), box.data_ptr(),
                                            probe.workspace(1).data_ptr(), _stream_ptr(dev)))
    eig = box[0].cpu().numpy()  # [k1][k2] = eigenvalues[k1, k2]
    return BccbOperator(l1, l2, eig, device=dev)


def bccb_scale_add_identity(op: BccbOperator, alpha: complex, beta: complex) -> BccbOperator:
    """alpha * R + beta * I as an eigenvalue shift (bccb.py:128-130)."""
    return BccbOperator(op.l1, op.l2, device=op.device, _box=alpha * op.box + beta,
                        _lam_out=alpha * op.lam_out + beta)


def bccb_inverse(op: BccbOperator) -> BccbOperator:
    """Entrywise eigenvalue inversion with the reference guard (bccb.py:133-148)."""
    lo, hi = op.all_eigen_magnitudes()
    threshold = SINGULAR_GUARD * hi
    if lo <= threshold:
        raise SingularOperatorError(lo, threshold)
    lam_out = 0.0 if op.is_full_box else 1.0 / op.lam_out
    return BccbOperator(op.l1, op.l2, device=op.device, _box=1.0 / op.box, _lam_out=lam_out)


# ----------------------------------------------------------------------------- application

def _batched_view(c, dim: int, l2: int = 0, l1: int = 0):
    """Validate (..., L) or (..., L2, L1); return (array, batch, was_numpy, batch_shape)."""
    was_numpy = not isinstance(c, torch.Tensor)
    t = np.asarray(c) if was_numpy else c
    shape = tuple(t.shape)
    if len(shape) >= 1 and shape[-1] == dim:
        batch_shape = shape[:-1]
    elif len(shape) >= 2 and l1 and shape[-2:] == (l2, l1):
        batch_shape = shape[:-2]
    else:
        raise InvalidArgumentError(f"vector length {shape} does not match L = {dim}")
    batch = int(np.prod(batch_shape)) if batch_shape else 1
    return t, batch, was_numpy, batch_shape


def bccb_matvec(op: BccbOperator, c):
    """Apply the operator: band FFT, eigenvalue multiply, band IFFT (bccb.py:113-125).

    c: (L,) / (B, L) / (B, L2, L1), numpy or CUDA tensor.  float64 inputs (numpy, or
    complex128 tensors) run the complex128 band engine and return complex128; complex64
    tensors run the complex64 engine.
    """
    t, batch, was_numpy, batch_shape = _batched_view(c, op.dimension, op.l2, op.l1)
    wide = was_numpy or t.dtype in (torch.complex128, torch.float64)
    dtype = torch.complex128 if wide else torch.complex64
    if isinstance(t, torch.Tensor):
        x = t.to(device=f"cuda:{op.device}", dtype=dtype).contiguous()
    else:
        x = torch.from_numpy(np.ascontiguousarray(t, dtype=np.complex128)).to(f"cuda:{op.device}")
    x = x.reshape(batch, op.dimension)
    y = torch.empty_like(x)
    fn = _lib.lib.bccb_matvec_z if wide else _lib.lib.bccb_matvec
    _lib.check(fn(op._plan, batch, x.data_ptr(), y.data_ptr(), op.workspace(batch).data_ptr(),
                  _stream_ptr(op.device)))
    y = y.reshape(tuple(t.shape))
    if was_numpy:
        return y.cpu().numpy()
    return y


def bccb_spectrum(op: BccbOperator, c) -> torch.Tensor:
    """fft2 of each snapshot restricted to the operator's box: (B, K1, K2) complex64 on device."""
    t, batch, _, _ = _batched_view(c, op.dimension, op.l2, op.l1)
    x = _as_device_c64(t, op.device).reshape(batch, op.dimension)
    box = torch.empty((batch, op.k1, op.k2), dtype=torch.complex64, device=x.device)
    _lib.check(_lib.lib.bccb_spectrum_box(op._plan, batch, x.data_ptr(), box.data_ptr(),
                                          op.workspace(batch).data_ptr(), _stream_ptr(op.device)))
    return box


def bccb_first_column(op: BccbOperator) -> FirstColumn:
    """Recover the first column by inverse 2D DFT on the GPU (bccb.py:151-153)."""
    dev = op.device
    lo = op.lam_out if not op.is_full_box else 0.0
    box = torch.from_numpy(np.ascontiguousarray((op.box - lo)[None], dtype=np.complex128)).to(f"cuda:{dev}")
    out = torch.empty((1, op.dimension), dtype=torch.complex128, device=box.device)
    scale = 1.0 / op.dimension
    # float64 band engine (the reference's ifft2, bccb.py:153)
    _lib.check(_lib.lib.bccb_synthesize_z(op._plan, 1, box.data_ptr(), scale, out.data_ptr(),
                                          op.workspace(1).data_ptr(), _stream_ptr(dev)))
    values = out[0].cpu().numpy()
    values[0] += lo
    return FirstColumn(values)
