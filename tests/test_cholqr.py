"""Mixed-precision Cholesky QR (proj/src/thinsvd.cpp:125-154,
C ABI proj/include/mpsvd.h:136-139).

CPU: the C restatement is bit-identical to the reference compiled in place
(Q and R), reproduces the reference's known answers
(proj/tests/test_thinsvd.cpp:188-215) and its NotPositiveDefinite pivot.

GPU: R from the device equals fl32(chol(M)) of the device Gram bit for bit
(K8 follows the reference's operation order); Q equals the restated row
solve with the device R bit for bit (K10); the known answers and the error
payload of proj/tests/test_capi.cpp:107-117 hold through the C ABI; the
acceptance criterion 5 grid (proj/tests/acceptance.cpp:279-305:
orth(Q) <= 100 n u kappa(B), m = 1024, n = 64) passes; the device-pointer
plan path equals the host path.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from helpers import orth_err, stacked_diag

M = pytest.importorskip("paper_2603_11953_b200")
import workloads as inputs  # noqa: E402
from paper_2603_11953_b200._lib import lib  # noqa: E402

import pyoracle  # noqa: E402

U32 = 2.0 ** -24


def _known_3x2():
    a = np.zeros((3, 2), np.float32)
    a[0, 0] = a[0, 1] = a[1, 1] = 1.0
    return a


# ---------------------------------------------------------------- CPU

@pytest.mark.parametrize("m,n", [(4, 4), (3, 2), (1000, 32), (5000, 17), (3000, 64), (2100, 1)])
def test_port_bitwise_vs_reference(ref, port, m, n):
    a = inputs.graded(m, n, 4.0, seed=n) if m > 4 else np.eye(m, n, dtype=np.float32)
    if (m, n) == (3, 2):
        a = _known_3x2()
    q_r, r_r = ref.cholesky_qr(a)
    q_p, r_p = port.cholesky_qr(a)
    assert np.array_equal(q_r, q_p) and np.array_equal(r_r, r_p)


def test_port_known_answers(port):
    q, r = port.cholesky_qr(np.eye(4, dtype=np.float32))
    assert np.array_equal(q, np.eye(4)) and np.array_equal(r, np.eye(4))
    q, r = port.cholesky_qr(_known_3x2())
    assert np.array_equal(r, [[1.0, 1.0], [0.0, 1.0]])
    assert np.array_equal(q, stacked_diag(3, [1.0, 1.0]))


def test_port_npd_pivot_matches_reference(ref, port):
    a = np.array([[1.0, 1.0], [0.0, 0.0]], np.float32)  # duplicated column
    with pytest.raises(pyoracle.OracleError) as er:
        ref.cholesky_qr(a)
    with pytest.raises(pyoracle.OracleError) as ep:
        port.cholesky_qr(a)
    assert er.value.status == ep.value.status == 2
    assert er.value.index == ep.value.index == 2


def test_cholqr_validation_order():
    with pytest.raises(M.InvalidArgument, match="Working-precision"):
        M.mp_cholesky_qr(np.eye(3))
    with pytest.raises(M.InvalidArgument):
        M.mp_cholesky_qr(np.zeros((2, 3), np.float32))


# ---------------------------------------------------------------- GPU

@pytest.mark.gpu
def test_gpu_known_answers():
    q, r = M.mp_cholesky_qr(np.eye(4, dtype=np.float32))
    assert np.array_equal(q, np.eye(4)) and np.array_equal(r, np.eye(4))
    q, r = M.mp_cholesky_qr(_known_3x2())
    assert np.array_equal(r, [[1.0, 1.0], [0.0, 1.0]])
    assert np.array_equal(q, stacked_diag(3, [1.0, 1.0]))


@pytest.mark.gpu
def test_gpu_npd_payload_like_capi_test():
    # proj/tests/test_capi.cpp:107-117
    a = M.Matrix(2, 2, M.Precision.WORKING)
    a.set(0, 0, 1.0)
    a.set(0, 1, 1.0)
    q, r = C.c_void_p(), C.c_void_p()
    assert lib.mpsvd_cholesky_qr(a.handle, C.byref(q), C.byref(r)) == 2
    assert lib.mpsvd_last_error_index() == 2
    assert len(lib.mpsvd_last_error_message()) > 0


@pytest.mark.gpu
@pytest.mark.parametrize("m,n", [(1000, 1), (4096, 32), (20000, 64), (3001, 100), (10000, 128), (2000, 200)])
def test_gpu_factors_bitwise_vs_restatement(port, m, n):
    a = inputs.graded(m, n, 4.0, seed=3 + n)
    q, r = M.mp_cholesky_qr(a)
    g = M.gram(a)  # the device Gram the factor was built from
    r_want = port.cholesky(g).astype(np.float32)
    assert np.array_equal(r, r_want)
    assert np.array_equal(q, port.cholqr_solve(a, r))


@pytest.mark.gpu
def test_gpu_acceptance_criterion_5(ref):
    worst = 0.0
    i = 0
    for kb in (1e1, 1e3, 1e5):
        for kd in (1.0, 1e4, 1e8):
            i += 1
            a, _, kb_real = ref.build_problem(1024, 64, kd, kb, 3, 42 + i)
            q, _ = M.mp_cholesky_qr(a)
            gate = 100.0 * 64 * U32 * kb_real
            worst = max(worst, orth_err(q) / gate)
    assert worst <= 1.0, worst


@pytest.mark.gpu
def test_gpu_as_orthogonal_as_reference_and_plan_path(ref):
    import torch

    a = inputs.graded(1 << 16, 64, 4.0, seed=21)
    q, r = M.mp_cholesky_qr(a)
    q_ref, _ = ref.cholesky_qr(a)
    assert orth_err(q) <= max(4.0 * orth_err(q_ref), 64 * U32)
    dev = torch.device("cuda", 0)
    m, n = a.shape
    a_t = torch.from_numpy(np.ascontiguousarray(a.T)).to(dev)
    q_t = torch.empty_like(a_t)
    r_t = torch.empty((n, n), dtype=torch.float32, device=dev)
    plan = M.Plan(m, n, M.Precision.WORKING)
    plan.cholesky_qr(a_t.data_ptr(), m, q_t.data_ptr(), m, r_t.data_ptr())
    assert plan.wait().status == 0
    assert np.array_equal(q_t.cpu().numpy().T, q)
    assert np.array_equal(r_t.cpu().numpy().T, r)
