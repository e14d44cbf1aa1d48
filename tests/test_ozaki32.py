"""K1z: the binary64 Gram of a binary32 A on the int8 tensor cores
(csrc/gram_ozaki32.cu), the default Gram of the binary32 path for
64 < n <= 128 and m >= 2^20 (C4).

CPU: the C restatement (oracle/mpsvd_port.c port_gram_f32_ozaki) against the
reference's own criterion ||dM||_F / ||M||_F <= 10 m u_h
(proj/tests/test_parallel_gram.cpp:74-86), an entrywise column-scaled
bound, exact symmetry, and the non-finite handling.
GPU: the kernel bit for bit against the restatement on the plan's own
schedule (mpsvd_stage_gram32_schedule), and the whole thin SVD through it
against the oracle's gates."""
from __future__ import annotations

import numpy as np
import pytest

from helpers import U32, U64, kappa_b, max_rel, north_star_gates, orth_err


def _a(m, n, seed, decades=0.0, dist="normal"):
    r = np.random.default_rng(seed)
    x = r.standard_normal((m, n)) if dist == "normal" else r.uniform(-1, 1, (m, n))
    x *= 10.0 ** (-decades * np.arange(n) / max(n - 1, 1))[None, :]
    return np.asfortranarray(x.astype(np.float32))


def _bounds(m, nranges):
    nch = (m + 31) // 32
    return np.linspace(0, nch, nranges + 1).astype(np.int64)


def _exact(a):
    al = a.astype(np.longdouble)
    return (al.T @ al).astype(np.float64)


@pytest.mark.parametrize("m,n,decades", [(4096, 100, 0), (3000, 128, 6), (5000, 70, 3), (20000, 128, 4),
                                         (33, 1, 0), (4099, 65, 2)])
def test_port_ozaki32_accuracy(port, m, n, decades):
    a = _a(m, n, seed=m + n, decades=decades)
    g = port.gram_f32_ozaki(a, 3, _bounds(m, 4))
    assert np.array_equal(g, g.T)
    ex = _exact(a)
    d = np.sqrt(np.diag(ex))
    ref = port.partitioned_gram_f32(a, blocks=16)
    # the reference's criterion (test_parallel_gram.cpp:83) against its own Gram
    assert np.linalg.norm(g - ref) / np.linalg.norm(ref) <= 10 * max(m, 1024) * U64
    # column-scaled entrywise: dropped digit products are zero-mean noise of
    # ~2^-39 colmax_i colmax_j per row, rounding to the
    # 47-bit grid is unbiased, the biased D8 diagonal is carried exactly
    cm = np.max(np.abs(a.astype(np.float64)), axis=0)
    bound = 2.0 ** -36 * np.sqrt(m) * np.outer(cm, cm) + 4 * U64 * np.abs(ex)
    assert np.all(np.abs(g - ex) <= bound)
    # diagonal: no systematic bias - within a few u_h of the exact value
    assert np.all(np.abs(np.diag(g) - np.diag(ex)) <= 2.0 ** -40 * np.diag(ex) + 1e-300)


def test_port_ozaki32_nonfinite_column(port):
    a = _a(2048, 40, seed=3)
    a[100, 7] = np.inf
    a[5, 11] = np.nan
    g = port.gram_f32_ozaki(a, 2, _bounds(2048, 2))
    bad = {7, 11}
    for i in range(40):
        for j in range(40):
            assert np.isnan(g[i, j]) == (i in bad or j in bad)


def test_port_ozaki32_span_breaks_and_zero_columns(port):
    # magnitudes growing along the rows force exponent-driven span breaks;
    # a zero column and a column that turns on late
    m, n = 8192, 33
    a = _a(m, n, seed=4)
    a *= np.exp(np.linspace(0, 12, m))[:, None].astype(np.float32)
    a[:, 3] = 0.0
    a[: m // 2, 5] = 0.0
    g = port.gram_f32_ozaki(a, 2, _bounds(m, 3), span_max=7)
    ex = _exact(a)
    cm = np.max(np.abs(a.astype(np.float64)), axis=0)
    assert np.all(np.abs(g - ex) <= 2.0 ** -36 * np.sqrt(m) * np.outer(cm, cm) + 4 * U64 * np.abs(ex))
    assert np.all(g[3, :] == 0) and np.all(g[:, 3] == 0)


# ---------------------------------------------------------------- GPU
M = None


def _gpu():
    global M
    M = pytest.importorskip("paper_2603_11953_b200")
    if not M.device_available():
        pytest.skip("no CUDA device")
    return M


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,decades,span", [(4096, 100, 0, 0), (3000, 128, 6, 0), (5000, 70, 3, 0),
                                              (20000, 128, 4, 0), (64, 1, 0, 0), (4100, 65, 2, 0),
                                              (65536, 128, 0, 5), (1 << 20, 128, 0, 0)])
def test_gpu_ozaki32_bitwise_vs_restatement(port, monkeypatch, m, n, decades, span):
    M = _gpu()
    monkeypatch.setenv("MPSVD_F32_GRAM", "ozaki")
    if span:
        monkeypatch.setenv("MPSVD_OZAKI32_SPAN", str(span))
    a = _a(m, n, seed=7 + n, decades=decades)
    oz, npairs, bounds = M.gram32_schedule(m, n)
    assert oz and npairs >= 1 and bounds[0] == 0 and bounds[-1] == (m + 31) // 32
    g = M.gram(a)
    want = port.gram_f32_ozaki(a, npairs, bounds, span_max=span or 512, threads=16)
    assert np.array_equal(g, want)


@pytest.mark.gpu
def test_gpu_ozaki32_nonfinite_and_span_breaks(port, monkeypatch):
    M = _gpu()
    monkeypatch.setenv("MPSVD_F32_GRAM", "ozaki")
    monkeypatch.setenv("MPSVD_OZAKI32_SPAN", "7")
    m, n = 8192, 33
    a = _a(m, n, seed=4)
    a *= np.exp(np.linspace(0, 12, m))[:, None].astype(np.float32)
    a[:, 3] = 0.0
    a[: m // 2, 5] = 0.0
    a[100, 7] = np.inf
    oz, npairs, bounds = M.gram32_schedule(m, n)
    g = M.gram(a)
    want = port.gram_f32_ozaki(a, npairs, bounds, span_max=7)
    assert np.array_equal(np.isnan(g), np.isnan(want))
    ok = ~np.isnan(want)
    assert np.array_equal(g[ok], want[ok])


@pytest.mark.gpu
def test_gpu_ozaki32_default_choice_and_fallback(monkeypatch):
    M = _gpu()
    monkeypatch.delenv("MPSVD_F32_GRAM", raising=False)
    assert M.gram32_schedule(1 << 20, 128)[0]          # C4-shaped: K1z
    assert not M.gram32_schedule(1 << 20, 64)[0]       # C2-shaped: K1 (n <= 64)
    assert not M.gram32_schedule(1 << 16, 128)[0]      # short: K1
    monkeypatch.setenv("MPSVD_F32_GRAM", "dmma")
    assert not M.gram32_schedule(1 << 22, 128)[0]


@pytest.mark.gpu
@pytest.mark.parametrize("m,n", [(1 << 20, 128), (1 << 20, 100)])
def test_gpu_thin_svd_through_ozaki32(port, m, n):
    """The default path for these shapes: the whole SVD against the
    restatement (reference semantics) with the north_star gates."""
    M = _gpu()
    a = _a(m, n, seed=11, decades=4.0)
    assert M.gram32_schedule(m, n)[0]
    r = M.mp_thin_svd(a)
    o = port.thin_svd(a, threads=16)
    kb = kappa_b(a)
    g_sigma, g_orth = north_star_gates(n, U32, kb)
    assert max_rel(r.sigma, o.sigma) <= g_sigma
    assert orth_err(r.v) <= g_orth and orth_err(r.u) <= g_orth


@pytest.mark.gpu
def test_gpu_ozaki32_deterministic_at_scale(monkeypatch):
    """Repeated device Grams of one 2^22 x 128 A are bit-identical: the ring
    race that a lane-0 slot release after __syncwarp allowed (a converter's
    load returning the next occupant of the slot) showed up at
    this size as run-to-run differences; with every ring shape the result is
    the same bits."""
    M = _gpu()
    monkeypatch.setenv("MPSVD_F32_GRAM", "ozaki")
    a = _a(1 << 22, 128, seed=21)
    g0 = M.gram(a)
    for _ in range(3):
        assert np.array_equal(M.gram(a), g0)
    assert np.all(np.isfinite(g0)) and np.array_equal(g0, g0.T)
