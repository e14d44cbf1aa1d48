"""Per-instruction-class stall breakdown from an ncu source page CSV:
`ncu -i r.ncu-rep --page source --csv --print-source sass > s.csv;
 python tools/ncu_source.py s.csv`."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
by_op = collections.defaultdict(lambda: collections.Counter())
tot = collections.Counter()
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    op = r[ix["Source"]].split()
    if not op:
        continue
    mnem = op[1] if op[0].startswith("@") else op[0]
    mnem = mnem.split(".")[0]
    for h in reasons:
        try:
            v = int(r[ix[h]])
        except ValueError:
            continue
        by_op[mnem][h] += v
        tot[h] += v
print("total", sum(tot.values()), dict(tot.most_common(8)))
for mnem, c in sorted(by_op.items(), key=lambda kv: -sum(kv[1].values()))[:12]:
    print(f"{mnem:10s} {sum(c.values()):7d}", dict(c.most_common(4)))
