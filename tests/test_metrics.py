"""Error metrics: max_rel_sv_error on the host and the
row-wise backward error on the GPU, checked against the reference compiled
in place (oracle/_ref, proj/src/metrics.cpp:26-70) and against the numpy
restatement in tests/helpers.py.

Tolerances: the GPU forms W = U diag(sigma) exactly like the reference
(binary64 products, rounded once) but accumulates W V^T in a different
order (DMMA k-steps), so each entry of the product differs by at most
~n * 2^-53 * |W||V| from the reference's; against residuals >= 2^-30 |A| the
relative change of the metric is below 1e-6, the tolerance used here.
Zero-row counts are exact.
"""
from __future__ import annotations

import numpy as np
import pytest

from helpers import rowwise_backward

M = pytest.importorskip("paper_2603_11953_b200")

RTOL = 1e-6


def _factors(m, n, seed, dtype=np.float32, zero_rows=()):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, n)).astype(dtype)
    for r in zero_rows:
        a[r, :] = 0
    a64 = a.astype(np.float64)
    u, s, vt = np.linalg.svd(a64, full_matrices=False)
    # perturb like a working-precision factorisation would
    return np.asfortranarray(a), np.asfortranarray(u.astype(dtype)), s, np.asfortranarray(vt.T.astype(dtype))


# ---------------------------------------------------------------- CPU (oracle pin, host function)

@pytest.mark.parametrize("m,n,zeros", [(40, 7, ()), (33, 5, (0, 17, 32)), (5, 5, (2,)), (1, 1, ())])
def test_restatement_matches_reference(ref, m, n, zeros):
    a, u, s, v = _factors(m, n, 3 + m, zero_rows=zeros)
    got, skipped = ref.rowwise_backward_error(a, u, s, v)
    assert skipped == len(zeros)
    assert rowwise_backward(a, u, s, v) == pytest.approx(got, rel=1e-12)


def test_reference_all_zero_rows(ref):
    a = np.zeros((4, 2), np.float32, order="F")
    u = np.zeros((4, 2), np.float32, order="F")
    assert ref.rowwise_backward_error(a, u, np.ones(2), np.eye(2, dtype=np.float32)) == (0.0, 4)


def test_max_rel_sv_error_matches_reference(ref):
    rng = np.random.default_rng(5)
    want = rng.uniform(0.1, 10.0, 37)
    got = want * (1 + rng.uniform(-1e-6, 1e-6, 37))
    assert M.max_rel_sv_error(got, want) == ref.max_rel_sv_error(got, want)
    assert M.max_rel_sv_error([], []) == 0.0


@pytest.mark.parametrize("bad", [0.0, -1.0, float("nan")])
def test_max_rel_sv_error_rejects_nonpositive_reference(ref, bad):
    want = np.array([1.0, bad, 2.0])
    with pytest.raises(M.InvalidArgument) as e:
        M.max_rel_sv_error(np.ones(3), want)
    assert "2" in str(e.value)  # 1-based index, like metrics.cpp:33-35
    import pyoracle

    with pytest.raises(pyoracle.OracleError) as er:
        ref.max_rel_sv_error(np.ones(3), want)
    assert er.value.status == 1


def test_max_rel_sv_error_length_mismatch():
    with pytest.raises(M.InvalidArgument):
        M.max_rel_sv_error([1.0, 2.0], [1.0])


def test_backward_error_needs_device_or_checks_shapes():
    a = np.ones((4, 2), np.float32)
    with pytest.raises(M.InvalidArgument):  # shape check precedes the device check
        M.rowwise_backward_error(a, a, np.ones(3), np.eye(2, dtype=np.float32))
    if not M.device_available():
        with pytest.raises(M.MpsvdError):
            M.rowwise_backward_error(a, a, np.ones(2), np.eye(2, dtype=np.float32))


# ---------------------------------------------------------------- GPU

@pytest.mark.gpu
@pytest.mark.parametrize("m,n,zeros", [(1, 1, ()), (128, 64, ()), (1000, 37, (0, 999)), (4099, 65, (5,)),
                                       (777, 130, (1, 2, 3)), (20000, 128, ()), (300, 257, ())])
def test_gpu_backward_error_f32_matches_reference(ref, m, n, zeros):
    a, u, s, v = _factors(m, n, 11 + n, zero_rows=zeros)
    want, wsk = ref.rowwise_backward_error(a, u, s, v)
    got = M.rowwise_backward_error(a, u, s, v)
    assert got.skipped_rows == wsk == len(zeros)
    assert got.max_rel == pytest.approx(want, rel=RTOL)


@pytest.mark.gpu
@pytest.mark.parametrize("m,n", [(513, 17), (3000, 64), (2048, 200)])
def test_gpu_backward_error_f64_matches_reference(ref, m, n):
    a, u, s, v = _factors(m, n, 29 + n, dtype=np.float64, zero_rows=(7,))
    want, wsk = ref.rowwise_backward_error(a, u, s, v)
    got = M.rowwise_backward_error(a, u, s, v)
    assert got.skipped_rows == wsk == 1
    assert got.max_rel == pytest.approx(want, rel=RTOL)


@pytest.mark.gpu
def test_gpu_backward_error_mixed_precision_widens_exactly():
    a, u, s, v = _factors(900, 48, 3)
    got = M.rowwise_backward_error(a, u.astype(np.float64), s, v)
    same = M.rowwise_backward_error(a.astype(np.float64), u.astype(np.float64), s, v.astype(np.float64))
    assert got == same
    assert got.max_rel == pytest.approx(rowwise_backward(a, u, s, v), rel=RTOL)


@pytest.mark.gpu
def test_gpu_backward_error_of_thin_svd_and_device_variant():
    import torch

    import workloads as inputs

    a = inputs.graded(1 << 16, 64, 5.0, seed=3)
    r = M.mp_thin_svd(a)
    host = M.rowwise_backward_error(a, r.u, r.sigma, r.v)
    assert host.max_rel == pytest.approx(rowwise_backward(a, r.u, r.sigma, r.v), rel=RTOL)
    assert host.max_rel <= 100.0 * 8.0 * 2.0 ** -24
    dev = torch.device("cuda", 0)
    col = lambda x: torch.from_numpy(np.asarray(x).T.copy()).to(dev).T  # column-major on device
    d = M.backward_error_device(col(a), col(r.u), torch.from_numpy(r.sigma).to(dev), col(r.v))
    assert d == host  # same kernels, same order: identical


@pytest.mark.gpu
def test_gpu_backward_error_detects_a_wrong_factor():
    a, u, s, v = _factors(2000, 32, 9)
    s_bad = s.copy()
    s_bad[3] *= 1.01
    good = M.rowwise_backward_error(a, u, s, v).max_rel
    bad = M.rowwise_backward_error(a, u, s_bad, v).max_rel
    assert good < 1e-5 < bad
