"""Row sharding of A across ranks (one process per GPU).

Contiguous, balanced row ranges whose sizes differ by at most one, the first
``m % nranks`` ranks one row longer — the partition rule of the reference's
make_partition_plan (proj/src/parallel_gram.cpp:57-77) applied to ranks
instead of thread blocks. Each rank keeps its rows of every column
(column-major with leading dimension = its own row count), computes the
partial Gram of those rows, and the partial Grams meet in ONE collective
inside the library.
"""
from __future__ import annotations


def row_ranges(m: int, nranks: int) -> list[tuple[int, int]]:
    if m < 0 or nranks < 1:
        raise ValueError("need m >= 0 and nranks >= 1")
    base, extra = divmod(m, nranks)
    out, row = [], 0
    for r in range(nranks):
        ln = base + (1 if r < extra else 0)
        out.append((row, row + ln))
        row += ln
    return out


def local_rows(m: int, nranks: int, rank: int) -> tuple[int, int]:
    if not 0 <= rank < nranks:
        raise ValueError("rank out of range")
    return row_ranges(m, nranks)[rank]
