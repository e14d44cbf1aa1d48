"""Shared test helpers: tolerances and metrics written out next to the gates
they implement (BASELINE.json north_star; proj/tests/* citations inline)."""
from __future__ import annotations

import numpy as np

U32 = 2.0 ** -24   # working unit roundoff, fp32 (proj/include/mpsvd/types.hpp:23-25)
U64 = 2.0 ** -53   # higher unit roundoff, fp64
UDD = 2.0 ** -104  # double-double unit roundoff used for the dd Jacobi tolerance


def kappa_b(a: np.ndarray) -> float:
    """kappa(B) for A = B*D, D the column norms: from the equilibrated Gram."""
    a64 = np.asarray(a, dtype=np.float64)
    g = a64.T @ a64
    d = np.sqrt(np.diag(g))
    lam = np.linalg.eigvalsh(g / np.outer(d, d))
    return float(np.sqrt(lam[-1] / lam[0]))


def orth_err(q: np.ndarray) -> float:
    """||Q^T Q - I||_F accumulated in binary64 (proj/src/dense.cpp:250-272)."""
    q64 = np.asarray(q, dtype=np.float64)
    g = q64.T @ q64
    return float(np.linalg.norm(g - np.eye(q.shape[1])))


def max_rel(got, want) -> float:
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    return float(np.max(np.abs(got - want) / np.abs(want))) if want.size else 0.0


def north_star_gates(n: int, u: float, kb: float):
    """sigma: 10*n*u*kappa(B); ||V^T V - I||, ||U^T U - I||: 10*n*u."""
    return 10.0 * n * u * kb, 10.0 * n * u


def rowwise_backward(a, u, sigma, v) -> float:
    """max_i ||(U diag(sigma) V^T - A)(i,:)|| / ||A(i,:)|| at binary64
    (proj/src/metrics.cpp:40-70)."""
    a = np.asarray(a, dtype=np.float64)
    p = (np.asarray(u, dtype=np.float64) * np.asarray(sigma)[None, :]) @ np.asarray(v, dtype=np.float64).T
    res = np.linalg.norm(p - a, axis=1)
    row = np.linalg.norm(a, axis=1)
    ok = row > 0
    return float(np.max(res[ok] / row[ok])) if ok.any() else 0.0


def dd_diff(h1, l1, h2, l2):
    """|(h1 + l1) - (h2 + l2)| for double-double pairs, exact enough for
    comparing two accurate sums (hi difference is exact by Sterbenz)."""
    return np.abs((np.asarray(h1) - np.asarray(h2)) + (np.asarray(l1) - np.asarray(l2)))


def stacked_diag(m: int, d, dtype=np.float32) -> np.ndarray:
    a = np.zeros((m, len(d)), dtype=dtype, order="F")
    for j, x in enumerate(d):
        a[j, j] = x
    return a


def rank_tree(parts, add):
    """The fixed reduction tree of proj/src/parallel_gram.cpp:93-102 over a
    list (rank order): (0,1),(2,3),... then doubling widths. Plan::exchange
    applies it to the all-gathered per-rank partial Grams."""
    slots = list(parts)
    width = 1
    while width < len(slots):
        for b in range(0, len(slots) - width, 2 * width):
            slots[b] = add(slots[b], slots[b + width])
        width *= 2
    return slots[0]


def dd_add_elementwise(port, x, y):
    """Elementwise dd_add (proj/tests/support/dd.cpp:32-38, via the restatement)
    of two (hi, lo) array pairs."""
    (xh, xl), (yh, yl) = x, y
    oh, ol = np.empty_like(xh), np.empty_like(xl)
    for idx in np.ndindex(xh.shape):
        oh[idx], ol[idx] = port.dd_op("add", (xh[idx], xl[idx]), (yh[idx], yl[idx]))
    return oh, ol
