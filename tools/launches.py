"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: count,
mean duration and share per kernel (only this library's kernels by default)."""
import collections
import csv
import sys


def main(path, pattern=""):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi = h.index("Kernel Name"), h.index("Metric Value")
    d = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > mi and pattern in r[ki]:
            d[r[ki].split("(")[0][:60]].append(float(r[mi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):5d} {sum(v) / len(v) / 1e3:10.1f} us {100 * sum(v) / tot:5.1f}%  {k}")


if __name__ == "__main__":
    main(*sys.argv[1:])
