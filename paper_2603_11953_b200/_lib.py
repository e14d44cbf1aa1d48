"""ctypes binding of the C ABI declared in include/mpsvd.h.

Loads the in-tree ``libmpsvd_b200.so`` (built by ``build.py`` /
``__graft_entry__.build()``). There is deliberately no fallback: if the
library is missing, importing the package fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmpsvd_b200.so")

i64 = C.c_int64
dp = C.POINTER(C.c_double)
vp = C.c_void_p


class ExecInfo(C.Structure):
    _fields_ = [
        ("status", C.c_int),
        ("error_index", i64),
        ("error_value", C.c_double),
        ("sweeps", C.c_int),
        ("rotations", i64),
        ("ms_gram", C.c_double),
        ("ms_eigen", C.c_double),
        ("ms_compute_u", C.c_double),
        ("kernel_launches", C.c_int),
        ("rounds", i64),
        ("gram_kernel", C.c_int),
        ("av_kernel", C.c_int),
    ]


# (name, restype, argtypes) for every symbol include/mpsvd.h declares
SIGNATURES = [
    ("mpsvd_last_error_message", C.c_char_p, []),
    ("mpsvd_last_error_index", i64, []),
    ("mpsvd_matrix_create", C.c_int, [i64, i64, C.c_int, C.POINTER(vp)]),
    ("mpsvd_matrix_destroy", None, [vp]),
    ("mpsvd_matrix_rows", i64, [vp]),
    ("mpsvd_matrix_cols", i64, [vp]),
    ("mpsvd_matrix_precision", C.c_int, [vp]),
    ("mpsvd_matrix_set", C.c_int, [vp, i64, i64, C.c_double]),
    ("mpsvd_matrix_get", C.c_int, [vp, i64, i64, dp]),
    ("mpsvd_matrix_bitwise_equal", C.c_int, [vp, vp]),
    ("mpsvd_matrix_data", vp, [vp]),
    ("mpsvd_orth_error", C.c_int, [vp, dp]),
    ("mpsvd_max_rel_sv_error", C.c_int, [dp, dp, i64, dp]),
    ("mpsvd_rowwise_backward_error", C.c_int, [vp, vp, dp, i64, vp, dp, C.POINTER(i64)]),
    ("mpsvd_backward_error_device", C.c_int, [C.c_int, vp, i64, vp, i64, vp, vp, i64, i64, i64, vp, dp,
                                              C.POINTER(i64)]),
    ("mpsvd_thin_svd", C.c_int, [vp, C.c_int, C.c_int, C.POINTER(vp)]),
    ("mpsvd_thin_svd_f64", C.c_int, [vp, C.c_int, C.POINTER(vp)]),
    ("mpsvd_cholesky_qr", C.c_int, [vp, C.POINTER(vp), C.POINTER(vp)]),
    ("mpsvd_plan_cholesky_qr", C.c_int, [vp, vp, i64, vp, i64, vp, vp]),
    ("mpsvd_svd_destroy", None, [vp]),
    ("mpsvd_svd_u", vp, [vp]),
    ("mpsvd_svd_v", vp, [vp]),
    ("mpsvd_svd_sigma", dp, [vp, C.POINTER(i64)]),
    ("mpsvd_svd_times", None, [vp, dp]),
    ("mpsvd_svd_sync_events", C.c_int, [vp]),
    ("mpsvd_svd_gram_blocks", i64, [vp]),
    ("mpsvd_svd_is_qr_baseline", C.c_int, [vp]),
    ("mpsvd_svd_jacobi_stats", None, [vp, C.POINTER(C.c_int), C.POINTER(i64)]),
    ("mpsvd_comm_unique_id", C.c_int, [C.c_char_p]),
    ("mpsvd_comm_init", C.c_int, [C.c_char_p, C.c_int, C.c_int, C.POINTER(vp)]),
    ("mpsvd_comm_destroy", None, [vp]),
    ("mpsvd_plan_create", C.c_int, [i64, i64, C.c_int, vp, C.POINTER(vp)]),
    ("mpsvd_plan_execute", C.c_int, [vp, vp, i64, vp, i64, vp, vp, vp]),
    ("mpsvd_plan_orth_error", C.c_int, [vp, vp, i64, vp, dp]),
    ("mpsvd_plan_wait", C.c_int, [vp, C.POINTER(ExecInfo)]),
    ("mpsvd_plan_destroy", None, [vp]),
    ("mpsvd_matrix_write_file", C.c_int, [C.c_char_p, vp]),
    ("mpsvd_matrix_read_file", C.c_int, [C.c_char_p, C.POINTER(vp)]),
    ("mpsvd_stage_gram", C.c_int, [C.c_int, vp, i64, i64, dp, dp]),
    ("mpsvd_stage_gram_schedule", C.c_int, [i64, i64, C.c_int] + [C.POINTER(C.c_int)] * 5),
    ("mpsvd_stage_gram32_schedule", C.c_int, [i64, i64, C.c_int] + [C.POINTER(C.c_int)] * 3 + [C.POINTER(i64)]),
    ("mpsvd_stage_jacobi", C.c_int, [C.c_int, dp, dp, i64, C.c_double, C.c_int, dp, dp, dp, dp,
                                     C.POINTER(C.c_int), C.POINTER(i64)]),
    ("mpsvd_stage_onesided", C.c_int, [C.c_int, dp, i64, C.c_double, C.c_int, dp, C.POINTER(C.c_float),
                                       C.POINTER(C.c_int), C.POINTER(i64)]),
    ("mpsvd_plan_set_eigensolver", C.c_int, [vp, C.c_int]),
    ("mpsvd_stage_rank_combine", C.c_int, [C.c_int, dp, dp, C.c_int, i64, dp, dp]),
    ("mpsvd_format_shortest", C.c_size_t, [C.c_double, C.c_char_p, C.c_size_t]),
    ("mpsvd_fp64_peak_tflops", C.c_double, [C.c_int]),
    ("mpsvd_device_available", C.c_int, []),
]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a). The package has no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()
