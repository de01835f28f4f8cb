"""Uniform harmonic grids and the GPU adjoint A^H y (drop-in for dictionary.py).

The reference materialises the M x L dictionary to apply its adjoint
(pkg/src/bccblasso/dictionary.py:83-97, 129-136), which cannot fit at config 5
(1.1 TB).  On the grid f = -1/2 + l/L (dictionary.py:41-45),
    b[l] = sum_m conj(D[m, l]) y_m = IFFT2_unnorm(E),  E[m2, m1] = (-1)^(m1+m2) y_m,
so b is a signed scatter plus one band-limited inverse FFT (SURVEY finding 4).
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .bccb import BccbOperator, _as_device_c64, _stream_ptr
from .errors import InvalidArgumentError


@dataclass(frozen=True, eq=False)
class UniformGrid:
    """length points f[l] = -1/2 + l/length (dictionary.py:21-38)."""

    length: int
    frequencies: np.ndarray
    gamma: float = 0.5

    def __post_init__(self) -> None:
        if self.length < 1:
            raise InvalidArgumentError("grid length must be positive")
        if self.gamma != 0.5:
            raise InvalidArgumentError("only half-wavelength spacing (gamma = 1/2) is supported")
        f = np.ascontiguousarray(self.frequencies, dtype=np.float64)
        if f.shape != (self.length,):
            raise InvalidArgumentError("frequency vector length does not match the grid length")
        f.setflags(write=False)
        object.__setattr__(self, "frequencies", f)


def make_uniform_grid(length: int) -> UniformGrid:
    if length < 1:
        raise InvalidArgumentError("grid length must be positive")
    return UniformGrid(length, -0.5 + np.arange(length) / length)


def apply_adjoint(gram: BccbOperator, y):
    """b = D_s^H y for the Gram operator's geometry and grid (dictionary.py:129-136).

    y: (M,) or (B, M).  Numpy in -> complex128 numpy out; tensor in -> complex64 tensor.
    """
    if gram.element_count < 1:
        raise InvalidArgumentError("apply_adjoint needs a Gram operator (gram_operator)")
    was_numpy = not isinstance(y, torch.Tensor)
    shape = np.shape(y) if was_numpy else tuple(y.shape)
    if len(shape) == 0 or shape[-1] != gram.element_count:
        raise InvalidArgumentError(f"measurement length {shape} does not match M = {gram.element_count}")
    yt = _as_device_c64(y, gram.device).reshape(-1, gram.element_count)
    batch = yt.shape[0]
    bhat = torch.empty((batch, gram.k1, gram.k2), dtype=torch.complex64, device=yt.device)
    b = torch.empty((batch, gram.dimension), dtype=torch.complex64, device=yt.device)
    _lib.check(_lib.lib.bccb_adjoint(gram._plan, batch, yt.data_ptr(), bhat.data_ptr(), b.data_ptr(),
                                     None, gram.workspace(batch).data_ptr(), _stream_ptr(gram.device)))
    out = b.reshape(*shape[:-1], gram.dimension)
    return out.cpu().numpy().astype(np.complex128) if was_numpy else out
