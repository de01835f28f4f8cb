"""ctypes binding of the C ABI declared in include/bccb_b200.h.

The library is mapped lazily, on the first access to `lib` (PEP 562 module
`__getattr__`), so host-only modules of the package (scenes, arrays, errors,
textio) import without mapping the CUDA library: the CPU reference arm of
bench.py and the oracle workers stay free of it.  The product path has no CPU
fallback: the first GPU call raises ImportError if the shared library is
missing, and every call checks the C status code and raises the reference's
exception class (pkg/src/bccblasso/errors.py:4-65).
"""

import ctypes
import os

from .errors import (
    BccbLassoError,
    DivergenceError,
    InvalidArgumentError,
    SingularOperatorError,
)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BCCB_LIB_PATH") or os.path.join(_HERE, "libbccb_b200.so")   # override: A/B of builds

OK, ERR_INVALID, ERR_DIVERGENCE, ERR_SINGULAR, ERR_CUDA, ERR_UNSUPPORTED = range(6)

_vp = ctypes.c_void_p
_i = ctypes.c_int
_ll = ctypes.c_longlong
_d = ctypes.c_double
_f = ctypes.c_float
_sz = ctypes.c_size_t

# name -> (restype, argtypes); must match include/bccb_b200.h exactly
SIGNATURES = {
    "bccb_last_error": (ctypes.c_char_p, []),
    "bccb_version": (ctypes.c_char_p, []),
    "bccb_plan_create": (_i, [_i, _i, _i, _i, _vp, _d, _d, _i, ctypes.POINTER(_vp)]),
    "bccb_plan_create_gram": (_i, [_i, _i, _i, _i, _vp, _i, ctypes.POINTER(_vp)]),
    "bccb_plan_destroy": (_i, [_vp]),
    "bccb_plan_info": (_i, [_vp] + [ctypes.POINTER(_i)] * 5),
    "bccb_plan_eigen_box": (_i, [_vp, _vp, ctypes.POINTER(_d), ctypes.POINTER(_d)]),
    "bccb_workspace_bytes": (_sz, [_vp, _i]),
    "bccb_matvec": (_i, [_vp, _i, _vp, _vp, _vp, _vp]),
    "bccb_matvec_z": (_i, [_vp, _i, _vp, _vp, _vp, _vp]),
    "bccb_spectrum_box": (_i, [_vp, _i, _vp, _vp, _vp, _vp]),
    "bccb_synthesize": (_i, [_vp, _i, _vp, _f, _vp, _f, _vp, _vp, _vp, _vp]),
    "bccb_spectrum_box_z": (_i, [_vp, _i, _vp, _vp, _vp, _vp]),
    "bccb_synthesize_z": (_i, [_vp, _i, _vp, _d, _vp, _vp, _vp]),
    "bccb_adjoint": (_i, [_vp, _i, _vp, _vp, _vp, _vp, _vp, _vp]),
    "bccb_fista_run": (_i, [_vp, _i, _i, _i, _d] + [_vp] * 8),
    "bccb_fista_run_traced": (_i, [_vp, _i, _i, _d] + [_vp] * 8),
    "bccb_admm_run": (_i, [_vp, _i, _i, _i, _d] + [_vp] * 9),
    "bccb_topk_workspace_bytes": (_sz, [_i, _ll, _i]),
    "bccb_topk": (_i, [_i, _ll, _vp, _i, _i, _vp, _vp, _vp, _vp]),
    "bccb_launch_count": (_ll, []),
    "bccb_profile_begin": (_i, []),
    "bccb_profile_end": (_i, [_vp, _vp]),
    "bccb_set_substreams": (_i, [_i]),
    "bccb_substreams_for": (_i, [_vp, _i]),
    "bccb_set_path": (_i, [_i]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_2509_13592_b200/_build.py` "
            "(there is no CPU fallback for the BCCB GPU path)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_loaded = None


def __getattr__(name):
    global _loaded
    if name == "lib":
        if _loaded is None:
            _loaded = _load()
        return _loaded
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")


def is_loaded() -> bool:
    """True once the CUDA library has been mapped into this process."""
    return _loaded is not None


class CudaError(BccbLassoError, RuntimeError):
    """The CUDA runtime reported a failure inside the library."""


class UnsupportedSizeError(InvalidArgumentError):
    """The requested size is outside the GPU engine's supported range."""


def last_error() -> str:
    return __getattr__("lib").bccb_last_error().decode(errors="replace")


def check(status: int, iteration: int | None = None) -> None:
    """Map a C status code onto the reference exception hierarchy."""
    if status == OK:
        return
    msg = last_error()
    if status == ERR_INVALID:
        raise InvalidArgumentError(msg)
    if status == ERR_SINGULAR:
        parts = msg.split("|")
        try:
            raise SingularOperatorError(float(parts[1]), float(parts[2]))
        except (IndexError, ValueError):
            raise SingularOperatorError(0.0, 0.0) from None
    if status == ERR_DIVERGENCE:
        raise DivergenceError(iteration if iteration is not None else -1)
    if status == ERR_UNSUPPORTED:
        raise UnsupportedSizeError(msg)
    raise CudaError(msg)
