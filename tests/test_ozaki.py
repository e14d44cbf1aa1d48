"""K2z: the double-double Gram on the int8 tensor cores (Ozaki scheme,
csrc/gram_ozaki.cu).

CPU: the restatement (oracle/mpsvd_port.c port_gram_dd_ozaki) against the
reference's double-double Gram oracle dd_gram (proj/tests/support/dd.cpp:75-88):
column-scaled error |dM_ij| / (||a_i|| ||a_j||) far below the Dot2 bound
4 (m u_h)^2 the K2 tests use (tests/test_gpu_parity.py), for ragged shapes,
graded columns, short exact-accumulation spans, empty splits, zero columns;
a non-finite column yields NaN in its row and column of M.

GPU: the device Gram is bit-identical to the restatement replayed on the
plan's own split schedule (mpsvd_stage_gram_schedule), across the tile,
chunk and span boundaries.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

M = pytest.importorskip("paper_2603_11953_b200")

import pyoracle  # noqa: E402

U_H = 2.0 ** -53


def _graded(m, n, decades, seed):
    rng = np.random.default_rng(seed)
    b = rng.standard_normal((m, n))
    b /= np.linalg.norm(b, axis=0)
    return np.asfortranarray(b * np.logspace(0, -decades, n))


def _scaled_err(hi, lo, rh, rl, a):
    nrm = np.linalg.norm(a, axis=0)
    nrm[nrm == 0] = 1.0
    return np.max(np.abs((hi - rh) + (lo - rl)) / np.outer(nrm, nrm))


def _schedule(m, nsplit, nblocks):
    nch = (m + 31) // 32
    scb = np.linspace(0, nch, nsplit + 1).astype(np.int32)
    bsb = np.linspace(0, nsplit, nblocks + 1).astype(np.int32)
    return scb, bsb


# ---------------------------------------------------------------- CPU

@pytest.mark.parametrize("m,n,decades,nsplit,nblocks,span", [
    (1, 1, 0, 1, 1, 1 << 20),
    (33, 3, 2, 1, 1, 1 << 20),
    (700, 17, 12, 4, 2, 3),
    (2000, 40, 16, 8, 4, 5),
    (3001, 65, 6, 16, 16, 1 << 20),
    (5000, 20, 12, 16, 16, 7),
])
def test_port_ozaki_matches_dd_gram(port, m, n, decades, nsplit, nblocks, span):
    a = _graded(m, n, decades, seed=m + n)
    scb, bsb = _schedule(m, nsplit, nblocks)
    hi, lo = port.gram_dd_ozaki(a, scb, bsb, span_cap=span)
    rh, rl = port.dd_gram(a)
    assert np.array_equal(hi, hi.T) and np.array_equal(lo, lo.T)
    # the digit-truncation level, 2^-80 relative to ||a_i|| ||a_j|| whatever
    # m; from m = 4096 rows (the engine's K2z threshold) it is
    # also inside the Dot2 bound 4 (m u_h)^2 the K2 tests use
    err = _scaled_err(hi, lo, rh, rl, a)
    assert err <= 2.0 ** -80
    if m >= 4096:
        assert err <= 4 * (m * U_H) ** 2


def test_port_ozaki_empty_split_zero_column_and_nonfinite(port):
    a = _graded(500, 9, 8, seed=3)
    a[:, 4] = 0.0
    scb = np.array([0, 0, 7, 7, 16], np.int32)  # splits 0 and 2 hold no chunk
    bsb = np.array([0, 2, 4], np.int32)
    hi, lo = port.gram_dd_ozaki(a, scb, bsb)
    rh, rl = port.dd_gram(a)
    assert np.all(hi[4] == 0.0) and np.all(lo[4] == 0.0)
    assert _scaled_err(hi, lo, rh, rl, a) <= 2.0 ** -80
    a[17, 6] = np.inf
    hi, _ = port.gram_dd_ozaki(a, scb, bsb)
    assert np.all(np.isnan(hi[6])) and np.all(np.isnan(hi[:, 6]))
    assert np.isfinite(np.delete(np.delete(hi, 6, 0), 6, 1)).all()


def test_port_ozaki_scale_invariance(port):
    # power-of-two column scaling commutes with the digit split exactly (the
    # column exponents absorb it); sign flips change the digits, not the accuracy
    a = _graded(640, 12, 10, seed=5)
    scb, bsb = _schedule(640, 4, 2)
    hi, lo = port.gram_dd_ozaki(a, scb, bsb)
    s = 2.0 ** np.arange(-6, 6)
    h2, l2 = port.gram_dd_ozaki(a * s, scb, bsb)
    f = np.outer(s, s)
    assert np.array_equal(h2, hi * f) and np.array_equal(l2, lo * f)
    sg = np.where(np.arange(12) % 3 == 0, -1.0, 1.0)
    h3, l3 = port.gram_dd_ozaki(a * sg, scb, bsb)
    rh, rl = port.dd_gram(a * sg)
    assert _scaled_err(h3, l3, rh, rl, a) <= 2.0 ** -80


def test_sub_groups_cover_every_digit_product_once(port):
    # the 6 sub-groups' products (p - k, w_hi - p), k < nw, p in [pa, pb],
    # p - k >= 1, are exactly the 66 digit pairs (a, b) with a + b <= 12
    seen = {}
    for i in range(6):
        whi, nw, pa, pb = port.oz_sub_group(i)
        assert 1 <= pa <= pb <= whi - 1 and pb - pa + 1 <= 4 and nw in (3, 4)
        for p in range(pa, pb + 1):
            for k in range(nw):
                if p - k >= 1:
                    pair = (p - k, whi - p)
                    assert pair not in seen
                    seen[pair] = i
    want = {(a, b) for a in range(1, 12) for b in range(1, 12) if a + b <= 12}
    assert set(seen) == want and len(want) == 66
    assert port.oz_sub_group(6) == (0, 0, 0, 0)


# ---------------------------------------------------------------- GPU

@pytest.mark.gpu
@pytest.mark.parametrize("m,n,decades", [
    (32, 1, 0), (100, 7, 3), (4096, 64, 12), (5000, 129, 8), (2048, 256, 12), (1999, 300, 4),
])
def test_gpu_ozaki_gram_bitwise_vs_restatement(port, m, n, decades, monkeypatch):
    monkeypatch.setenv("MPSVD_DD_GRAM", "ozaki")  # below 4096 rows the engine picks K2
    a = _graded(m, n, decades, seed=11 + n)
    oz, scb, bsb = M.gram_schedule(m, n)
    assert oz
    hi, lo = M.gram(a)
    rh, rl = port.gram_dd_ozaki(a, scb, bsb)
    assert np.array_equal(hi, rh)
    assert np.array_equal(lo, rl)


@pytest.mark.gpu
def test_gpu_ozaki_short_spans_bitwise(port, monkeypatch):
    # several drains per CTA (MPSVD_OZAKI_SPAN: chunks per exact span)
    monkeypatch.setenv("MPSVD_OZAKI_SPAN", "3")
    monkeypatch.setenv("MPSVD_DD_GRAM", "ozaki")  # the engine picks K2z itself only from n = 128
    m, n = 6000, 70
    a = _graded(m, n, 10, seed=2)
    oz, scb, bsb = M.gram_schedule(m, n)
    assert oz
    hi, lo = M.gram(a)
    rh, rl = port.gram_dd_ozaki(a, scb, bsb, span_cap=3)
    assert np.array_equal(hi, rh) and np.array_equal(lo, rl)


@pytest.mark.gpu
def test_gpu_ozaki_matches_dot2_kernel(port, monkeypatch):
    # K2z against K2 (MPSVD_DD_GRAM=dot2) and the reference oracle
    m, n = 20000, 96
    a = _graded(m, n, 12, seed=9)
    monkeypatch.setenv("MPSVD_DD_GRAM", "ozaki")
    hi, lo = M.gram(a)
    monkeypatch.setenv("MPSVD_DD_GRAM", "dot2")
    dh, dl = M.gram(a)
    rh, rl = port.dd_gram(a)
    assert _scaled_err(hi, lo, rh, rl, a) <= 2.0 ** -80
    assert _scaled_err(dh, dl, rh, rl, a) <= 4 * (m * U_H) ** 2
