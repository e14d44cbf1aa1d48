"""B200-native (sm_100a) mixed-precision Gram-based thin SVD (arXiv 2603.11953).

Drop-in for the reference's ``mp_thin_svd`` / ``mpsvd_thin_svd`` path: the
C-ABI library ``libmpsvd_b200.so`` (include/mpsvd.h) runs the Gram (DMMA /
double-double SYRK), the two-sided Jacobi, and U = A V Sigma^-1 on the GPU.
"""
from .api import (  # noqa: F401
    BackwardErrorReport,
    CastOverflowError,
    Comm,
    EigensolverChoice,
    InternalError,
    InvalidArgument,
    Matrix,
    MpsvdError,
    NoConvergenceError,
    NotPositiveDefiniteError,
    PhaseTimes,
    Plan,
    Precision,
    ThinSvdResult,
    TinySingularValueError,
    ZeroColumnError,
    ZeroDivisorError,
    backward_error_device,
    device_available,
    fp64_peak_tflops,
    gram,
    gram_schedule,
    gram32_schedule,
    max_rel_sv_error,
    mp_cholesky_qr,
    mp_thin_svd,
    mp_thin_svd_f64,
    onesided_spectral,
    orth_error,
    format_shortest,
    rank_combine,
    rowwise_backward_error,
    twosided_jacobi_eig,
)
from ._lib import LIB_PATH  # noqa: F401
