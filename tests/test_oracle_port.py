"""Pins the C restatement (oracle/_port) to the UNMODIFIED reference
(oracle/_ref, compiled in place from /root/reference by oracle/Makefile):
bit-for-bit on the fp32 path, and on the reference's own double-double test
oracle (proj/tests/support/dd.cpp). CPU only."""
from __future__ import annotations

import numpy as np
import pytest

import pyoracle
from helpers import U64, stacked_diag


def graded(m, n, decades, seed, dtype=np.float32):
    r = np.random.default_rng(seed)
    b = r.standard_normal((n, m))
    b /= np.linalg.norm(b, axis=1)[:, None]
    d = 10.0 ** (-decades * np.arange(n) / max(n - 1, 1))
    return np.asfortranarray((b * d[:, None]).T.astype(dtype))


@pytest.mark.parametrize("m,n,workers", [(1, 1, 1), (9, 3, 1), (37, 5, 3), (257, 6, 16), (1024, 64, 8),
                                         (3001, 24, 4)])
def test_partitioned_gram_bitwise(ref, port, m, n, workers):
    a = graded(m, n, 4.0, seed=m)
    blocks = min(16, m)
    g_ref, sync, nb = ref.partitioned_gram_f32(a, workers=min(workers, m), blocks=blocks)
    assert sync == 1 and nb == blocks  # parallel_gram.cpp:110
    assert np.array_equal(port.partitioned_gram_f32(a, blocks=blocks), g_ref)


def test_partition_plan_matches_reference_tests(port):
    # proj/tests/test_parallel_gram.cpp:30-46
    assert port.partition_plan(10, 3, 4) == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert len(port.partition_plan(100, 1)) == 1
    assert len(port.partition_plan(100, 3)) == 8
    assert len(port.partition_plan(4, 4)) == 4
    for bad in [(8, 0, 0), (8, 9, 0), (8, 2, 16)]:
        with pytest.raises(pyoracle.OracleError):
            port.partition_plan(*bad)


@pytest.mark.parametrize("n,seed", [(2, 1), (5, 2), (24, 3), (64, 4), (100, 5)])
def test_twosided_jacobi_bitwise(ref, port, n, seed):
    a = graded(3 * n + 7, n, 6.0, seed, np.float64)
    g = a.T @ a
    g = (g + g.T) / 2
    lr, vr, sr, rr = ref.twosided_jacobi(g)
    lp, vp, sp, rp = port.twosided_jacobi(g)
    assert np.array_equal(lr, lp) and np.array_equal(vr, vp) and (sr, rr) == (sp, rp)


@pytest.mark.parametrize("m,n,seed", [(4, 2, 0), (300, 24, 9), (1024, 64, 5), (5000, 32, 7)])
def test_thin_svd_bitwise(ref, port, m, n, seed):
    a = graded(m, n, 6.0, seed)
    r = ref.thin_svd(a, threads=4)
    p = port.thin_svd(a, threads=4)
    assert np.array_equal(r.u, p.u) and np.array_equal(r.v, p.v) and np.array_equal(r.sigma, p.sigma)
    assert r.sync_events == 1 and r.gram_blocks == min(16, m)


def test_thin_svd_reference_suite_instance(ref, port):
    # the build_problem instance of proj/tests/test_thinsvd.cpp:103-132
    a, _, kb = ref.build_problem(1024, 64, 1e8, 1e3, 3, 5)
    assert kb == pytest.approx(1e3, rel=1e-10)
    r = ref.thin_svd(a)
    p = port.thin_svd(a)
    assert np.array_equal(r.u, p.u) and np.array_equal(r.sigma, p.sigma)


def test_stacked_diagonal_golden(port):
    # proj/tests/test_thinsvd.cpp:70-84
    p = port.thin_svd(stacked_diag(4, [5.0, 3.0]))
    assert list(p.sigma) == [5.0, 3.0]
    assert np.array_equal(p.v, np.eye(2, dtype=np.float32))
    assert np.array_equal(p.u, stacked_diag(4, [1.0, 1.0]))


def test_jacobi_golden_2x2(port):
    # proj/tests/test_jacobi.cpp:193-206: lambda (3, 1), sign tie at the lowest row
    for sem in (pyoracle.SEM_REFERENCE, pyoracle.SEM_DEVICE):
        lam, v, _, _ = port.twosided_jacobi(np.array([[2.0, 1.0], [1.0, 2.0]]), sem=sem)
        isq = 1 / np.sqrt(2.0)
        assert lam == pytest.approx([3.0, 1.0], rel=1e-15)
        assert v[:, 0] == pytest.approx([isq, isq], rel=1e-15)
        assert v[:, 1] == pytest.approx([isq, -isq], rel=1e-15)


def test_tiny_sigma_and_validation(port, ref):
    # proj/tests/test_thinsvd.cpp:244-276
    for lib in (port, ref):
        with pytest.raises(pyoracle.OracleError) as e:
            lib.thin_svd(stacked_diag(2, [1.0, 1e-39]))
        assert e.value.status == 7 and e.value.index == 2
    with pytest.raises(pyoracle.OracleError) as e:
        ref.thin_svd_f64_input(np.eye(2))
    assert e.value.status == 1


def test_dd_gram_bitwise_vs_reference_dd_oracle(ref, port):
    a = graded(500, 12, 8.0, seed=3, dtype=np.float64)
    hr, lr = ref.dd_gram(a)
    hp, lp = port.dd_gram(a, threads=3)
    assert np.array_equal(hr, hp) and np.array_equal(lr, lp)


def test_dd_primitives_are_error_free(port):
    rng = np.random.default_rng(0)
    for _ in range(200):
        x, y = rng.standard_normal(2) * 10.0 ** rng.integers(-20, 20, 2)
        h, l = port.dd_op("add", (x, 0.0), (y, 0.0))
        assert h == x + y and abs(l) <= abs(h) * 2.0 ** -53
        h, l = port.dd_op("mul", (x, 0.0), (y, 0.0))
        assert h == x * y
        # (h + l) == x*y exactly: check with the exact rational product
        from fractions import Fraction
        assert Fraction(h) + Fraction(l) == Fraction(x) * Fraction(y)


@pytest.mark.parametrize("sem", [pyoracle.SEM_REFERENCE, pyoracle.SEM_DEVICE])
def test_dd_jacobi_vs_reference_bisection(ref, port, sem):
    # the reference's dd LDL^T bisection oracle (proj/tests/support/dd.cpp:96-153), n <= 16
    h = np.array([[1.0 / (i + j + 1) for j in range(8)] for i in range(8)])
    (lh, ll), _, _, _ = port.twosided_jacobi_dd(h, sem=sem)
    oracle = ref.dd_oracle_eigenvalues(h)
    assert np.max(np.abs(lh - oracle) / oracle) <= 64 * U64


@pytest.mark.parametrize("sem", [pyoracle.SEM_REFERENCE, pyoracle.SEM_DEVICE])
def test_dd_jacobi_prescribed_sigma_needs_more_than_30_sweeps(port, sem):
    # C5-shaped Gram (sigma over 10 decades, Haar V0), n = 128: both
    # orderings need ~30 sweeps; the dd path's cap is 100 (kDdMaxSweeps)
    import sys, os
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
    import workloads as inputs
    n = 128
    a, sigma = inputs.prescribed(2 * n, n, 10.0, seed=500 + n)
    hi, lo = port.dd_gram(a, threads=8)
    with pytest.raises(pyoracle.OracleError):
        port.twosided_jacobi_dd(hi, lo, max_sweeps=25, sem=sem)
    (lh, _), _, sw, _ = port.twosided_jacobi_dd(hi, lo, max_sweeps=100, sem=sem)
    assert 25 < sw <= 40
    assert np.all(np.abs(np.sqrt(lh) - sigma) <= 64 * U64 * n + 1e-12 * sigma)


def test_dd_thin_svd_vs_reference_dd_oracle(ref, port):
    # f64 working: sigma from dd Gram + dd Jacobi vs the reference dd oracle
    a = graded(64, 8, 10.0, seed=4, dtype=np.float64)
    o = port.thin_svd_f64dd(a, threads=2)
    want = ref.dd_oracle_singular_values(a)
    assert np.max(np.abs(o.sigma - want) / want) <= 8 * U64
