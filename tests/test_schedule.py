"""Host-side schedule logic: the parallel round-robin Jacobi schedule (shared
by the CUDA kernels and the restatement), the fixed priority-block set the
warp-specialised Jacobi relies on, and the row sharding of A. CPU only."""
from __future__ import annotations

import itertools

import pytest

from paper_2603_11953_b200 import sharding


def rr_pair(n, r, k):
    # independent Python model of mpsvd::dev::rr_pair (csrc/common.cuh)
    N = n + (n & 1)
    M = N - 1
    a, b = (M, r) if k == 0 else ((r + k) % M, (r - k) % M)
    return min(a, b), max(a, b)


@pytest.mark.parametrize("n", list(range(1, 40)) + [64, 65, 128, 255, 256])
def test_round_robin_covers_every_pair_once(port, n):
    N = n + (n & 1)
    seen = set()
    for r in range(N - 1):
        used = set()
        for k in range(N // 2):
            p, q = port.rr_pair(n, r, k)
            assert (p, q) == rr_pair(n, r, k)
            assert p not in used and q not in used  # disjoint within a round
            used |= {p, q}
            if q < n:
                assert (p, q) not in seen
                seen.add((p, q))
    assert seen == set(itertools.combinations(range(n), 2))


@pytest.mark.parametrize("n", range(2, 140))
def test_priority_blocks_are_round_invariant(n):
    """The blocks holding round r+1's (p', q') in round r's pair slots are
    {(k, k+2)} + {(np-2, np-1)} + {(0, 1) for even n} for every r
    (assumption of jacobi_smem in csrc/jacobi.cu)."""
    N = n + (n & 1)
    np_ = N // 2
    fixed = {(a, a + 2) for a in range(np_ - 2)}
    if np_ >= 2:
        fixed.add((np_ - 2, np_ - 1))
        if n % 2 == 0:
            fixed.add((0, 1))

    def slot(r, x):
        return next(k for k in range(np_) if x in rr_pair(n, r, k))

    for r in range(N - 2):
        pri = []
        for k in range(np_):
            p, q = rr_pair(n, r + 1, k)
            if q < n:
                a, b = slot(r, p), slot(r, q)
                pri.append((min(a, b), max(a, b)))
        if np_ >= 3:
            assert len(pri) == len(set(pri))  # one next-round pair per block
        assert set(pri) == fixed


def test_row_sharding():
    assert sharding.row_ranges(10, 4) == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert sharding.row_ranges(1 << 26, 8)[7] == (7 << 23, 1 << 26)
    for m, p in [(0, 3), (5, 8), (1 << 20, 3)]:
        rr = sharding.row_ranges(m, p)
        assert rr[0][0] == 0 and rr[-1][1] == m
        assert all(a[1] == b[0] for a, b in zip(rr, rr[1:]))
        sizes = [b - a for a, b in rr]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        sharding.local_rows(10, 2, 2)
