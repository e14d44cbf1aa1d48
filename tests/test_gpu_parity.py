"""GPU parity tests: every call goes through the C-ABI library
(libmpsvd_b200.so) on the B200 and is checked against the CPU oracles
(oracle/_port restatement, pinned to the reference; oracle/_ref, the
reference itself, when present)."""
from __future__ import annotations

import numpy as np
import pytest

from helpers import U32, U64, UDD, dd_diff, kappa_b, max_rel, north_star_gates, orth_err, rowwise_backward, stacked_diag

pytestmark = pytest.mark.gpu

M = pytest.importorskip("paper_2603_11953_b200")
import workloads as inputs  # noqa: E402

if not M.device_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import pyoracle  # noqa: E402

SEM_DEVICE = pyoracle.SEM_DEVICE


def rng_matrix(m, n, seed, dtype=np.float32, scale_decades=0.0):
    r = np.random.default_rng(seed)
    a = r.uniform(-1.0, 1.0, size=(n, m))
    if scale_decades:
        a *= 10.0 ** (-scale_decades * np.arange(n) / max(n - 1, 1))[:, None]
    return np.asfortranarray(a.T.astype(dtype))


# ---------------------------------------------------------------------------
# K1: fp32 -> fp64 Gram
@pytest.mark.parametrize("m,n", [(1, 1), (7, 3), (37, 5), (300, 24), (1024, 64), (5000, 100), (4096, 128),
                                 (2000, 200), (65, 65)])
def test_gram_f32_matches_reference(port, m, n):
    a = rng_matrix(m, n, seed=m + n)
    g = M.gram(a)
    ref = port.partitioned_gram_f32(a, blocks=min(16, m))
    # exact symmetry by construction (parallel_gram.cpp:28-29)
    assert np.array_equal(g, g.T)
    # test_parallel_gram.cpp:74-86 criterion
    assert np.linalg.norm(g - ref) / np.linalg.norm(ref) <= 10.0 * m * U64
    # entrywise: both sums are within m*u_h*||a_i|| ||a_j|| of the exact one
    d = np.sqrt(np.diag(ref))
    assert np.all(np.abs(g - ref) <= 2.0 * m * U64 * np.outer(d, d) + 1e-300)


def test_gram_f32_large_rows(port):
    a = inputs.make(inputs.CONFIGS["c1"], seed=3)  # 20000 x 32 graded
    g = M.gram(a)
    ref = port.partitioned_gram_f32(a, blocks=16)
    d = np.sqrt(np.diag(ref))
    assert np.all(np.abs(g - ref) <= 2.0 * a.shape[0] * U64 * np.outer(d, d))
    assert np.array_equal(g, g.T)


# K2: fp64 -> double-double Gram
@pytest.mark.parametrize("m,n", [(1, 1), (9, 4), (300, 24), (2048, 64), (3000, 130)])
def test_gram_dd_matches_oracle(port, m, n):
    a = rng_matrix(m, n, seed=7 * m + n, dtype=np.float64, scale_decades=6.0)
    hi, lo = M.gram(a)
    rh, rl = port.dd_gram(a)
    assert np.array_equal(hi, hi.T) and np.array_equal(lo, lo.T)
    an = np.sqrt(np.einsum("ij,ij->j", a, a))
    # Dot2 / dd_add accumulation: error <= ~(m u)^2 * sum|a_i a_j| <= (m u)^2 ||a_i|| ||a_j||
    bound = 4.0 * (m * U64) ** 2 * np.outer(an, an) + 8.0 * UDD * np.abs(rh)
    assert np.all(dd_diff(hi, lo, rh, rl) <= bound)


# ---------------------------------------------------------------------------
# K4: fp64 Jacobi — bitwise against the device-semantics restatement
@pytest.mark.parametrize("n", [1, 2, 3, 5, 24, 64, 101, 128, 129, 200, 201, 256])
def test_jacobi_f64_bitwise_vs_restatement(port, n):
    a = rng_matrix(3 * n + 5, n, seed=n, dtype=np.float64, scale_decades=3.0)
    g = a.T @ a
    g = (g + g.T) / 2
    lam, v, sw, rot = M.twosided_jacobi_eig(g)
    plam, pv, psw, prot = port.twosided_jacobi(g, sem=SEM_DEVICE)
    assert (sw, rot) == (psw, prot)
    assert np.array_equal(lam, plam)
    assert np.array_equal(v, pv)
    # and within rounding of the reference's cyclic order
    rlam, rv, _, _ = port.twosided_jacobi(g)
    assert max_rel(lam, rlam) <= 1e3 * n * U64 * np.linalg.cond(a) ** 2


def test_jacobi_golden_examples():
    # proj/tests/test_jacobi.cpp:184-207
    lam, v, _, _ = M.twosided_jacobi_eig(np.diag([4.0, 1.0]))
    assert list(lam) == [4.0, 1.0] and v[0, 0] == 1.0 and v[1, 1] == 1.0
    lam, v, _, _ = M.twosided_jacobi_eig(np.array([[2.0, 1.0], [1.0, 2.0]]))
    isq = 1.0 / np.sqrt(2.0)
    assert lam[0] == pytest.approx(3.0, rel=1e-15) and lam[1] == pytest.approx(1.0, rel=1e-15)
    assert v[0, 0] == pytest.approx(isq, rel=1e-15) and v[1, 0] == pytest.approx(isq, rel=1e-15)
    assert v[0, 1] == pytest.approx(isq, rel=1e-15) and v[1, 1] == pytest.approx(-isq, rel=1e-15)


def test_jacobi_hilbert_vs_dd_bisection(ref):
    # proj/tests/test_jacobi.cpp:209-227
    h = np.array([[1.0 / (i + j + 1) for j in range(4)] for i in range(4)])
    lam, _, _, _ = M.twosided_jacobi_eig(h)
    oracle = ref.dd_oracle_eigenvalues(h)
    bh = h / np.sqrt(np.outer(np.diag(h), np.diag(h)))
    bl = ref.dd_oracle_eigenvalues(bh)
    assert max_rel(lam, oracle) <= 1e3 * U64 * bl[0] / bl[-1]


def test_jacobi_errors():
    # NPD paths (test_jacobi.cpp:245-262)
    with pytest.raises(M.NotPositiveDefiniteError) as e:
        M.twosided_jacobi_eig(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert e.value.index == 1
    with pytest.raises(M.NotPositiveDefiniteError):
        M.twosided_jacobi_eig(np.array([[-1.0]]))
    with pytest.raises(M.NoConvergenceError):
        g = rng_matrix(40, 20, 1, np.float64)
        M.twosided_jacobi_eig(g.T @ g, max_sweeps=1)


def _indefinite(n, seed):
    # positive diagonal, one slightly negative eigenvalue: the pivot check fails inside a round
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.linspace(1.0, 2.0, n)
    lam[-1] = -1e-3
    g = (q * lam) @ q.T
    return (g + g.T) / 2


@pytest.mark.parametrize("n", [40, 200, 201])
def test_jacobi_f64_error_paths_like_restatement(port, n):
    """NotPositiveDefinite raised inside a round and NoConvergence, on the single-CTA
    (n = 40) and multi-CTA solvers: same pivot / value / payload as the restatement."""
    g = _indefinite(n, seed=n)
    with pytest.raises(pyoracle.OracleError) as ep:
        port.twosided_jacobi(g, sem=SEM_DEVICE)
    with pytest.raises(M.NotPositiveDefiniteError) as eg:
        M.twosided_jacobi_eig(g)
    assert eg.value.index == ep.value.index
    a = rng_matrix(2 * n, n, seed=7 + n, dtype=np.float64, scale_decades=3.0)
    g = a.T @ a
    g = (g + g.T) / 2
    with pytest.raises(pyoracle.OracleError) as ep:
        port.twosided_jacobi(g, max_sweeps=2, sem=SEM_DEVICE)
    with pytest.raises(M.NoConvergenceError) as eg:
        M.twosided_jacobi_eig(g, max_sweeps=2)
    assert ep.value.index == 2 and "2 sweeps" in str(eg.value)
    worst = float(str(eg.value).rsplit(" ", 1)[1])
    assert abs(worst - ep.value.value) <= 1e-5 * ep.value.value


# K5: double-double Jacobi — bitwise against the restatement
@pytest.mark.parametrize("n", [2, 7, 32, 90, 111, 120])
def test_jacobi_dd_bitwise_vs_restatement(port, n):
    a = rng_matrix(2 * n + 3, n, seed=100 + n, dtype=np.float64, scale_decades=8.0)
    hi, lo = port.dd_gram(a)
    (lh, ll), (vh, vl), sw, rot = M.twosided_jacobi_eig(hi, lo, dd=True)
    (plh, pll), (pvh, pvl), psw, prot = port.twosided_jacobi_dd(hi, lo, sem=SEM_DEVICE)
    assert (sw, rot) == (psw, prot)
    assert np.array_equal(lh, plh) and np.array_equal(ll, pll)
    assert np.array_equal(vh, pvh) and np.array_equal(vl, pvl)


# K5 on the C5 distribution (prescribed sigma over 10 decades, Haar V0): the
# non-graded, ill-conditioned Gram needs more than the fp64 path's 30 sweeps
# (kDdMaxSweeps = 100), still bit-identical to the restatement.
@pytest.mark.parametrize("n", [64, 128])
def test_jacobi_dd_prescribed_sigma_bitwise(port, n):
    a, sigma = inputs.prescribed(2 * n, n, 10.0, seed=500 + n)
    hi, lo = port.dd_gram(a, threads=8)
    (lh, ll), (vh, vl), sw, rot = M.twosided_jacobi_eig(hi, lo, dd=True)
    (plh, pll), (pvh, pvl), psw, prot = port.twosided_jacobi_dd(hi, lo, max_sweeps=100, sem=SEM_DEVICE)
    assert (sw, rot) == (psw, prot)
    if n == 128:
        assert sw > 30
    assert np.array_equal(lh, plh) and np.array_equal(ll, pll)
    assert np.array_equal(vh, pvh) and np.array_equal(vl, pvl)
    # sigma against the prescribed values: A formed in fp64 perturbs sigma_i
    # by ~ u * ||A|| / sigma_i relative
    s = np.sqrt(lh)
    assert np.all(np.abs(s - sigma) <= 64 * U64 * n * sigma[0] + 1e-12 * sigma)


def test_thin_svd_f64_prescribed_sigma_c5_shape(port):
    n = 96
    a, sigma = inputs.prescribed(4096, n, 10.0, seed=7)
    r = M.mp_thin_svd_f64(a)
    o = port.thin_svd_f64dd(a, threads=8, sem=SEM_DEVICE)
    assert r.jacobi_sweeps > 0
    # sigma^2 = lambda(M) with kappa(M) = kappa(B)^2 = 1e20: the device and
    # the restatement sum the dd Gram in different orders (2^-104-level
    # differences), amplified by kappa(M) in the smallest sigma
    assert max_rel(r.sigma, o.sigma) <= 10 * n * UDD * 1e20 + 4 * U64
    assert orth_err(r.v) <= 10 * n * U64
    # U = A V Sigma^-1 loses orthogonality ~ u * kappa(B) (1e-6 here) by
    # construction; the restatement shows the same loss
    assert orth_err(r.u) <= 2 * orth_err(o.u) + 10 * n * U64


# ---------------------------------------------------------------------------
# Full pipeline through mpsvd_thin_svd
def test_thin_svd_stacked_diagonal_exact():
    # proj/tests/test_thinsvd.cpp:70-84, proj/tests/test_capi.cpp:164-188
    a = stacked_diag(4, [5.0, 3.0])
    r = M.mp_thin_svd(a)
    assert list(r.sigma) == [5.0, 3.0]
    assert np.array_equal(r.v, np.eye(2, dtype=np.float32))
    assert np.array_equal(r.u, stacked_diag(4, [1.0, 1.0]))
    assert r.gram_sync_events == 1
    t = r.times
    assert min(t.gram, t.eigen, t.compute_u, t.overlap) >= 0.0
    assert abs(t.gram + t.eigen + t.compute_u + t.overlap - t.total) <= 1e-9 + 1e-6 * t.total


def test_thin_svd_graded_suite_instance(ref):
    # proj/tests/test_thinsvd.cpp:103-132 (build_problem {1024,64,1e8,1e3,3,5})
    a, _, kb = ref.build_problem(1024, 64, 1e8, 1e3, 3, 5)
    oracle = ref.reference_svd(a)
    r = M.mp_thin_svd(a)
    high_acc = 100.0 * (U32 + U64 * kb * kb)
    assert max_rel(r.sigma, oracle) <= high_acc
    assert rowwise_backward(a, r.u, r.sigma, r.v) <= 100.0 * 8.0 * U32
    assert orth_err(r.u) <= 100.0 * (8.0 * U32 + 64.0 * high_acc)
    assert orth_err(r.v) <= 100.0 * 64.0 * U64 + 64.0 * U32


@pytest.mark.parametrize("seed", [1, 2])
def test_thin_svd_config_c1(port, seed):
    cfg = inputs.CONFIGS["c1"]
    a = inputs.make(cfg, seed=seed)
    r = M.mp_thin_svd(a)
    o = port.thin_svd(a, threads=8)
    kb = kappa_b(a)
    g_sigma, g_orth = north_star_gates(cfg.n, U32, kb)
    assert max_rel(r.sigma, o.sigma) <= g_sigma
    assert orth_err(r.v) <= g_orth
    assert orth_err(r.u) <= g_orth
    assert rowwise_backward(a, r.u, r.sigma, r.v) <= 100.0 * np.sqrt(cfg.n) * U32


# Shape sweep over every kernel-selection boundary: n in {1, ..} around the
# 64-column tile, the shared-memory Jacobi limit (n <= 128 fp64 / np <= 64),
# the tensor-core K7 limit (n <= 128) and beyond (multi-CTA Jacobi, SIMT U);
# m ragged with respect to the 128-row tiles and the 16 logical blocks.
@pytest.mark.parametrize("m,n", [(1, 1), (17, 16), (200, 63), (515, 65), (1000, 127), (1024, 128), (1300, 129),
                                 (3001, 200), (4096, 256), (2048, 300)])
def test_thin_svd_shape_sweep_f32(port, m, n):
    a = inputs.graded(m, n, 3.0, seed=m * 7 + n)
    r = M.mp_thin_svd(a)
    o = port.thin_svd(a, threads=8)
    kb = kappa_b(a)
    g_sigma, g_orth = north_star_gates(n, U32, kb)
    assert max_rel(r.sigma, o.sigma) <= g_sigma
    assert orth_err(r.v) <= g_orth
    if m >= n:
        assert orth_err(r.u) <= max(g_orth, 4 * orth_err(o.u))
    w = r.v.astype(np.float32) / r.sigma.astype(np.float32)[None, :]
    assert_av_bound(a, w, r.u)


@pytest.mark.parametrize("m,n", [(5, 3), (640, 64), (900, 129), (2000, 200)])
def test_thin_svd_shape_sweep_f64(port, m, n):
    a = inputs.graded(m, n, 8.0, seed=m + n, dtype=np.float64)
    r = M.mp_thin_svd_f64(a)
    o = port.thin_svd_f64dd(a, threads=8, sem=SEM_DEVICE)
    kb = kappa_b(a)
    g_sigma, g_orth = north_star_gates(n, U64, kb)
    assert max_rel(r.sigma, o.sigma) <= g_sigma
    assert orth_err(r.v) <= g_orth
    assert orth_err(r.u) <= max(g_orth, 4 * orth_err(o.u))


def test_thin_svd_tiny_sigma():
    # proj/tests/test_thinsvd.cpp:244-264; test_capi.cpp:118-126
    a = stacked_diag(2, [1.0, 1e-39])
    with pytest.raises(M.TinySingularValueError) as e:
        M.mp_thin_svd(a)
    assert e.value.index == 2


def test_thin_svd_argument_validation():
    # proj/tests/test_thinsvd.cpp:266-276
    with pytest.raises(M.InvalidArgument):
        M.mp_thin_svd(np.eye(2))  # f64 input rejected
    with pytest.raises(M.InvalidArgument):
        M.mp_thin_svd(np.zeros((2, 3), np.float32))
    with pytest.raises(M.InvalidArgument):
        M.mp_thin_svd(np.eye(2, dtype=np.float32), threads=0)


def test_thin_svd_device_semantics_bitwise(port):
    """Given the device's own Gram, the downstream pipeline (Jacobi, sort/sign,
    sigma, W) is bit-identical to the restatement; U = A W from the tensor-core
    K7 (bf16x3 split, fp32 accumulation) is within the working-precision
    bound of the restatement's fp32 fma chain."""
    a = inputs.make(inputs.CONFIGS["c1"], seed=5, m=4096)
    r = M.mp_thin_svd(a)
    g = M.gram(a)
    lam, v, _, _ = port.twosided_jacobi(g, sem=SEM_DEVICE)
    sigma = np.sqrt(lam).astype(np.float32).astype(np.float64)
    assert np.array_equal(r.sigma, sigma)
    assert np.array_equal(r.v, v.astype(np.float32))
    w = v.astype(np.float32) / sigma.astype(np.float32)[None, :]
    assert_av_bound(a, w, r.u)
    assert_av_bound(a, w, port.av_f32(a, w))


def assert_av_bound(a, w, u, c=2.0, unit=U32):
    """|U - A W| <= c * n * unit * (|A| |W|) elementwise, A W in fp64
    (for fp64 operands the reference product carries its own ~n u64 error,
    inside the same bound)."""
    a64, w64 = a.astype(np.float64), w.astype(np.float64)
    exact = a64 @ w64
    bound = c * a.shape[1] * unit * (np.abs(a64) @ np.abs(w64)) + 1e-300
    err = np.abs(u.astype(np.float64) - exact)
    assert np.all(err <= bound), float(np.max(err / bound))


# K7 fp64 on the DMMA pipe: ragged tiles, odd m (unaligned columns), n = 1
@pytest.mark.parametrize("m,n", [(3, 1), (129, 7), (1001, 64), (4096, 100), (2050, 130)])
def test_compute_u_f64_dmma_bound(m, n):
    a = inputs.graded(m, n, 4.0, seed=m + 3 * n, dtype=np.float64)
    r = M.mp_thin_svd_f64(a)
    w = r.v / r.sigma[None, :]
    assert_av_bound(a, w, r.u, c=4.0, unit=U64)


# K7 on tcgen05: ragged tiles (m % 128 != 0), n not a multiple of 16, n = 1
@pytest.mark.parametrize("m,n", [(4, 1), (128, 16), (300, 17), (301, 7), (1028, 40), (4100, 64), (20000, 100), (8192, 128)])
def test_compute_u_tensor_core_bound(m, n):
    a = inputs.graded(m, n, 3.0, seed=m + n)
    r = M.mp_thin_svd(a)
    w = r.v.astype(np.float32) / r.sigma.astype(np.float32)[None, :]
    assert_av_bound(a, w, r.u)
    kb = kappa_b(a)
    g_sigma, g_orth = north_star_gates(n, U32, kb)
    assert orth_err(r.u) <= g_orth


def test_thin_svd_f64_dd_small(port):
    cfg = inputs.CONFIGS["c3"]
    a = inputs.make(cfg, seed=2, m=4096)[:, :64].copy(order="F")
    r = M.mp_thin_svd_f64(a)
    o = port.thin_svd_f64dd(a, threads=8)
    kb = kappa_b(a)
    g_sigma, g_orth = north_star_gates(64, U64, kb)
    assert max_rel(r.sigma, o.sigma) <= g_sigma
    assert orth_err(r.v) <= g_orth
    assert orth_err(r.u) <= g_orth


# ---------------------------------------------------------------------------
# Device-resident plan API (bench path) and the NCCL exchange with one rank
@pytest.mark.parametrize("working", ["f32", "f64"])
def test_plan_api_matches_host_api_and_single_rank_nccl(working):
    torch = pytest.importorskip("torch")
    m, n = 8192, 40
    if working == "f32":
        a = inputs.graded(m, n, 4.0, seed=3)
        prec = M.Precision.WORKING
        host = M.mp_thin_svd(a)
    else:
        a = inputs.graded(m, n, 10.0, seed=3, dtype=np.float64)
        prec = M.Precision.HIGHER
        host = M.mp_thin_svd_f64(a)
    dev = torch.device("cuda", 0)
    a_t = torch.from_numpy(np.ascontiguousarray(a.T)).to(dev)  # (n, m) row-major = column-major m x n
    outs = []
    comm = M.Comm(M.Comm.unique_id(), 1, 0)
    for c in (None, comm):
        plan = M.Plan(m, n, prec, c)
        u = torch.empty_like(a_t)
        s = torch.empty(n, dtype=torch.float64, device=dev)
        v = torch.empty((n, n), dtype=a_t.dtype, device=dev)
        plan.execute(a_t.data_ptr(), m, u.data_ptr(), m, s.data_ptr(), v.data_ptr(), 0)
        info = plan.wait()
        assert info.status == 0 and info.kernel_launches >= 7
        outs.append((u.T.cpu().numpy(), s.cpu().numpy(), v.T.cpu().numpy()))
    for u, s, v in outs:
        assert np.array_equal(s, host.sigma)
        assert np.array_equal(v, host.v)
        assert np.array_equal(u, host.u)
