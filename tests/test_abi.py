"""The C-ABI library loads and exports every symbol include/mpsvd.h declares;
host-side behaviour that needs no GPU (matrix handles, validation order,
error mapping, thread-local diagnostics). CPU only."""
from __future__ import annotations

import ctypes as C
import os
import re
import threading

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M = pytest.importorskip("paper_2603_11953_b200")
from paper_2603_11953_b200._lib import LIB_PATH, SIGNATURES, lib  # noqa: E402


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "mpsvd.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mpsvd_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported_and_bound():
    raw = C.CDLL(LIB_PATH)
    names = declared_symbols()
    assert "mpsvd_thin_svd" in names and len(names) >= 30
    for name in names:
        assert hasattr(raw, name), name
    assert {s[0] for s in SIGNATURES} == set(names)


def test_status_values_match_reference_header():
    # proj/include/mpsvd.h:25-37
    text = open(os.path.join(ROOT, "include", "mpsvd.h")).read()
    want = {"MPSVD_OK": 0, "MPSVD_ERR_INVALID_ARGUMENT": 1, "MPSVD_ERR_NOT_POSITIVE_DEFINITE": 2,
            "MPSVD_ERR_NO_CONVERGENCE": 3, "MPSVD_ERR_ZERO_COLUMN": 4, "MPSVD_ERR_ZERO_DIVISOR": 5,
            "MPSVD_ERR_CAST_OVERFLOW": 6, "MPSVD_ERR_TINY_SINGULAR_VALUE": 7, "MPSVD_ERR_INFEASIBLE": 8,
            "MPSVD_ERR_IO": 9, "MPSVD_ERR_INTERNAL": 10}
    for k, v in want.items():
        assert re.search(rf"{k} = {v}\b", text), k


def test_matrix_lifecycle_and_rounding():
    # proj/tests/test_capi.cpp:125-142
    a = M.Matrix(3, 2, M.Precision.WORKING)
    assert (a.rows, a.cols, a.precision) == (3, 2, M.Precision.WORKING)
    a.set(0, 0, 0.1)
    assert a.get(0, 0) == float(np.float32(0.1))
    with pytest.raises(M.InvalidArgument):
        a.get(3, 0)
    assert len(lib.mpsvd_last_error_message()) > 0
    st = lib.mpsvd_matrix_set(None, 0, 0, 1.0)
    assert st == 1
    b = M.Matrix.from_numpy(a.numpy())
    assert a.bitwise_equal(b)
    b.set(2, 1, 1.0)
    assert not a.bitwise_equal(b)
    big = M.Matrix(1 << 18, 2, M.Precision.HIGHER)  # pinned-or-heap storage, zeroed
    assert big.numpy().shape == (1 << 18, 2) and not big.numpy().any()


def test_validation_precedes_device_use():
    # proj/src/thinsvd.cpp:52-56 order: precision, shape, threads
    with pytest.raises(M.InvalidArgument, match="Working-precision"):
        M.mp_thin_svd(np.eye(3))
    with pytest.raises(M.InvalidArgument):
        M.mp_thin_svd(np.zeros((2, 3), np.float32))
    with pytest.raises(M.InvalidArgument):
        M.mp_thin_svd(np.eye(2, dtype=np.float32), threads=0)
    r = C.c_void_p()
    assert lib.mpsvd_thin_svd(M.Matrix(4, 2, M.Precision.WORKING).handle, 9, 1, C.byref(r)) == 1


@pytest.mark.skipif(M.device_available(), reason="checks the no-GPU failure mode")
def test_compute_fails_loudly_without_gpu():
    with pytest.raises(M.InternalError, match="no CUDA device"):
        M.mp_thin_svd(np.eye(4, 2, dtype=np.float32))
    with pytest.raises(M.InternalError):
        M.gram(np.ones((4, 2), np.float32))
    assert M.fp64_peak_tflops(0) == 0.0


def test_diagnostics_are_thread_local():
    errs = {}

    def worker(i):
        try:
            M.mp_thin_svd(np.eye(2), threads=1) if i == 0 else None
        except M.MpsvdError:
            pass
        errs[i] = lib.mpsvd_last_error_message().decode()

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert "Working-precision" in errs[0] and errs[1] == ""
