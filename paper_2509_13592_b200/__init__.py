"""B200-native BCCB Gram operator and fused ISTA/FISTA/ADMM (sm_100a).

Drop-in for the hot path of the reference package `bccblasso`
(arXiv 2509.13592): operator construction (gram_operator, bccb_matvec, ...) and
the ista/fista/admm solver entry points, batched over snapshots and executed by
hand-written CUDA through the C ABI in include/bccb_b200.h.

The first GPU call requires the built shared library (no CPU fallback);
build it with `python paper_2509_13592_b200/_build.py`.
"""

from .arrays import (
    ArrayGeometry,
    Target,
    make_ura,
    snr_to_noise_variance,
    steering_vector,
    subsample_preserving_aperture,
    synthesize_snapshot,
)
from .bccb import (
    BccbOperator,
    FirstColumn,
    bccb_first_column,
    bccb_from_first_column,
    bccb_inverse,
    bccb_matvec,
    bccb_scale_add_identity,
    bccb_spectrum,
    gram_operator,
)
from .dictionary import UniformGrid, apply_adjoint, make_uniform_grid
from .errors import (
    BccbLassoError,
    ConfigError,
    ConvergenceError,
    DivergenceError,
    DomainError,
    InvalidArgumentError,
    MemoryBudgetError,
    SingularOperatorError,
    ZeroReferenceError,
)
from .solvers import (
    BACKEND_FAST,
    BACKEND_REGULAR,
    LassoProblem,
    SolverConfig,
    SolverResult,
    admm_solve,
    extract_support,
    fista_alpha_sequence,
    fista_solve,
    ista_solve,
    max_gram_eigenvalue,
    soft_threshold,
    topk_peaks,
)

__version__ = "0.1.0"
