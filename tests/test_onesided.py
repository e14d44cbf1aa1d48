"""The GramCholSvd and OneSidedJacobiOnGram branches of mp_thin_svd
(proj/src/thinsvd.cpp:37-47,90-104).

CPU: the C restatement (oracle/mpsvd_port.c) with the reference's semantics
is bit-identical to the reference compiled in place (sigma, V and U), for
both branches, on the success and the error paths. Its device semantics
(round-robin pairs, fma partials + butterfly, closed-form rotation) stay
within the reference's accuracy.

GPU: the device spectral phase (Cholesky K8 + one-sided Jacobi K9, through
mpsvd_stage_onesided) is bit-identical to the device-semantics restatement
on the same Gram, in both the shared-memory and the grid-wide solver; the
full mp_thin_svd per branch is as accurate as the reference's own result
(singular values against the double-double oracle, orthogonality of U and
V, row-wise backward error), and the error paths report what the reference
reports.
"""
from __future__ import annotations

import numpy as np
import pytest

from helpers import kappa_b, orth_err, rowwise_backward

M = pytest.importorskip("paper_2603_11953_b200")
import workloads as inputs  # noqa: E402

import pyoracle  # noqa: E402

GRAM_CHOL, ONESIDED = 1, 2
U32 = 2.0 ** -24


def _dup_column(m, n, seed):
    a = inputs.graded(m, n, 3.0, seed=seed)
    a[:, 1] = a[:, 0]  # exactly rank deficient: Cholesky breaks down
    return a


# ---------------------------------------------------------------- CPU

@pytest.mark.parametrize("choice", [GRAM_CHOL, ONESIDED])
@pytest.mark.parametrize("m,n,kd", [(1, 1, 1.0), (5, 2, 2.0), (200, 8, 3.0), (501, 17, 8.0), (3000, 64, 4.0)])
def test_port_reference_semantics_bitwise(ref, port, choice, m, n, kd):
    a = inputs.graded(m, n, kd, seed=n + choice)
    r = ref.thin_svd(a, choice=choice)
    p = port.thin_svd(a, choice=choice, sem=pyoracle.SEM_REFERENCE)
    assert np.array_equal(r.sigma, p.sigma)
    assert np.array_equal(r.v, p.v)
    assert np.array_equal(r.u, p.u)


@pytest.mark.parametrize("choice", [GRAM_CHOL, ONESIDED])
def test_port_device_semantics_accuracy(ref, port, choice):
    a = inputs.graded(2000, 48, 5.0, seed=3)
    r = ref.thin_svd(a, choice=choice)
    d = port.thin_svd(a, choice=choice, sem=pyoracle.SEM_DEVICE)
    kb = kappa_b(a)
    assert np.max(np.abs(d.sigma - r.sigma) / r.sigma) <= 10 * 48 * U32 * kb
    assert orth_err(d.v) <= 10 * 48 * U32


@pytest.mark.parametrize("m,n,kd", [(1024, 128, 2.0), (2000, 100, 3.0), (4096, 32, 6.0)])
def test_port_device_semantics_v_orthogonality_like_reference(ref, port, m, n, kd):
    # GramCholSvd runs the one-sided Jacobi in binary32: the rotation's cosine
    # must be as accurate as the reference's 1 / hypotf(1, t) (jacobi.cpp:37);
    # the binary32 closed form sqrt((|x| + r) / 2r) left V 4-5x less orthogonal
    a = inputs.graded(m, n, kd, seed=7 + n)
    r = ref.thin_svd(a, choice=GRAM_CHOL)
    d = port.thin_svd(a, choice=GRAM_CHOL, sem=pyoracle.SEM_DEVICE)
    assert orth_err(d.v) <= 2.0 * orth_err(r.v)


def test_port_npd_matches_reference(ref, port):
    a = _dup_column(300, 6, 1)
    with pytest.raises(pyoracle.OracleError) as er:
        ref.thin_svd(a, choice=GRAM_CHOL)
    with pytest.raises(pyoracle.OracleError) as ep:
        port.thin_svd(a, choice=GRAM_CHOL, sem=pyoracle.SEM_REFERENCE)
    assert er.value.status == ep.value.status == 2
    assert er.value.index == ep.value.index
    assert er.value.value == ep.value.value


def test_port_cholesky_is_the_reference_factor(port):
    # proj/tests/test_dense.cpp:99-105: [[10,14],[14,20]] = R^T R
    r = port.cholesky(np.array([[10.0, 14.0], [14.0, 20.0]]))
    assert r[1, 0] == 0.0
    assert r[0, 0] == np.sqrt(10.0) and r[0, 1] == 14.0 / np.sqrt(10.0)
    assert np.allclose(r.T @ r, [[10.0, 14.0], [14.0, 20.0]], rtol=1e-15)


# ---------------------------------------------------------------- GPU

def _gram(port, a):
    return port.partitioned_gram_f32(a, blocks=16)


@pytest.mark.gpu
@pytest.mark.parametrize("choice", [GRAM_CHOL, ONESIDED])
@pytest.mark.parametrize("n", [1, 2, 7, 32, 64, 65, 100, 128, 200, 256])
def test_gpu_spectral_bitwise_vs_device_restatement(port, choice, n):
    a = inputs.graded(max(4 * n, 64), n, 5.0, seed=100 + n)
    g = _gram(port, a)
    s_gpu, v_gpu, sw_gpu, rot_gpu = M.onesided_spectral(choice, g)
    s_p, v_p, sw_p, rot_p = port.onesided_spectral(choice, g, sem=pyoracle.SEM_DEVICE)
    assert np.array_equal(s_gpu, s_p)
    assert np.array_equal(v_gpu, v_p)
    assert (sw_gpu, rot_gpu) == (sw_p, rot_p)


@pytest.mark.gpu
@pytest.mark.parametrize("choice", [GRAM_CHOL, ONESIDED])
@pytest.mark.parametrize("m,n,kd", [(4096, 32, 6.0), (1 << 15, 64, 4.0), (2000, 100, 3.0), (1024, 128, 2.0)])
def test_gpu_thin_svd_as_accurate_as_reference(ref, choice, m, n, kd):
    a = inputs.graded(m, n, kd, seed=7 + n)
    r = M.mp_thin_svd(a, choice=choice)
    assert r.eigensolver == choice
    w = ref.thin_svd(a, choice=choice)
    exact = ref.dd_oracle_singular_values(a)
    err_gpu = np.max(np.abs(r.sigma - exact) / exact)
    err_ref = np.max(np.abs(w.sigma - exact) / exact)
    assert err_gpu <= max(4.0 * err_ref, 10 * n * U32), (err_gpu, err_ref)
    assert orth_err(r.v) <= max(4.0 * orth_err(w.v), 10 * n * U32)
    assert orth_err(r.u) <= max(4.0 * orth_err(w.u), 10 * n * U32 * kappa_b(a))
    assert rowwise_backward(a, r.u, r.sigma, r.v) <= max(4.0 * rowwise_backward(a, w.u, w.sigma, w.v), 100 * n * U32)


@pytest.mark.gpu
def test_gpu_gram_chol_npd_like_reference(ref):
    a = _dup_column(300, 6, 1)
    with pytest.raises(pyoracle.OracleError) as er:
        ref.thin_svd(a, choice=GRAM_CHOL)
    with pytest.raises(M.NotPositiveDefiniteError) as eg:
        M.mp_thin_svd(a, choice=M.EigensolverChoice.GRAM_CHOL_SVD)
    assert eg.value.pivot == er.value.index == 2


@pytest.mark.gpu
def test_gpu_branches_share_plans_and_switch_back(port):
    a = inputs.graded(1 << 14, 64, 4.0, seed=5)
    r0 = M.mp_thin_svd(a)
    r1 = M.mp_thin_svd(a, choice=M.EigensolverChoice.GRAM_CHOL_SVD)
    r2 = M.mp_thin_svd(a, choice=M.EigensolverChoice.ONESIDED_JACOBI_GRAM)
    again = M.mp_thin_svd(a)
    assert np.array_equal(r0.sigma, again.sigma) and np.array_equal(r0.u, again.u)
    assert np.max(np.abs(r1.sigma - r0.sigma) / r0.sigma) < 1e-4
    assert np.max(np.abs(r2.sigma - r0.sigma) / r0.sigma) < 1e-5


@pytest.mark.gpu
def test_gpu_plan_eigensolver_device_path_matches_host_path():
    import torch

    a = inputs.graded(1 << 15, 32, 4.0, seed=9)
    host = M.mp_thin_svd(a, choice=M.EigensolverChoice.ONESIDED_JACOBI_GRAM)
    dev = torch.device("cuda", 0)
    m, n = a.shape
    a_t = torch.from_numpy(np.ascontiguousarray(a.T)).to(dev)  # (n, m): column-major m x n
    u_t = torch.empty_like(a_t)
    s_t = torch.empty(n, dtype=torch.float64, device=dev)
    v_t = torch.empty((n, n), dtype=torch.float32, device=dev)
    plan = M.Plan(m, n, M.Precision.WORKING)
    plan.set_eigensolver(M.EigensolverChoice.ONESIDED_JACOBI_GRAM)
    plan.execute(a_t.data_ptr(), m, u_t.data_ptr(), m, s_t.data_ptr(), v_t.data_ptr())
    info = plan.wait()
    assert info.status == 0
    assert np.array_equal(s_t.cpu().numpy(), host.sigma)
    assert np.array_equal(v_t.cpu().numpy().T, host.v)
    assert np.array_equal(u_t.cpu().numpy().T, host.u)


def _huge_stacked(scale=3.0e38):
    # A = scale * [e1; e1; e2; e2]: M = 2 scale^2 I, R = sqrt(2) scale I > FLT_MAX
    a = np.zeros((4, 2), dtype=np.float32, order="F")
    a[0, 0] = a[1, 0] = a[2, 1] = a[3, 1] = np.float32(scale)
    return a


def test_ref_gram_chol_cast_overflow():
    """cast(R, Working) of the GramCholSvd branch (thinsvd.cpp:44, dense.cpp:172):
    the reference reports CastOverflowError(1, 1, R_11)."""
    if not pyoracle.ref_available():
        pytest.skip("oracle/_ref not built")
    with pytest.raises(pyoracle.OracleError) as er:
        pyoracle.Ref().thin_svd(_huge_stacked(), choice=GRAM_CHOL)
    assert er.value.status == 6  # MPSVD_ERR_CAST_OVERFLOW


@pytest.mark.gpu
def test_gpu_gram_chol_cast_overflow_like_reference(ref):
    a = _huge_stacked()
    with pytest.raises(pyoracle.OracleError) as er:
        ref.thin_svd(a, choice=GRAM_CHOL)
    with pytest.raises(M.CastOverflowError):
        M.mp_thin_svd(a, choice=M.EigensolverChoice.GRAM_CHOL_SVD)
    assert er.value.status == M.CastOverflowError.status
    # the default branch has no checked cast (thinsvd.cpp:81-89): sigma = fl32(sqrt(lambda)) = inf
    # passes check_sigma_normal, W = V / inf = 0, U = 0 - same on both sides
    w = ref.thin_svd(a)
    r = M.mp_thin_svd(a)
    assert np.array_equal(np.asarray(r.sigma), np.asarray(w.sigma)) and np.all(np.isinf(np.asarray(r.sigma)))
    assert np.array_equal(np.asarray(r.u), np.asarray(w.u))
