"""K1z vs its restatement on one shape, with the mismatching entries listed
(diagnostics): `python tools/oz32_diag.py m n [span]`."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
os.environ["MPSVD_F32_GRAM"] = "ozaki"
import paper_2603_11953_b200 as M  # noqa: E402
import pyoracle  # noqa: E402

m, n = int(sys.argv[1]), int(sys.argv[2])
span = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
if span != 1024:
    os.environ["MPSVD_OZAKI32_SPAN"] = str(span)
r = np.random.default_rng(7 + n)
a = np.asfortranarray(r.standard_normal((m, n)).astype(np.float32))
oz, npairs, bounds = M.gram32_schedule(m, n)
g1 = M.gram(a)
g2 = M.gram(a)
want = pyoracle.Port().gram_f32_ozaki(a, npairs, bounds, span_max=span, threads=16)
print("npairs", npairs, "deterministic", np.array_equal(g1, g2))
d = g1 != want
print("mismatches", int(d.sum()), "of", d.size, "diag", int(np.diag(d).sum()))
idx = np.argwhere(d)[:20]
for i, j in idx:
    print(i, j, g1[i, j], want[i, j], (g1[i, j] - want[i, j]) / abs(want[i, j]))
al = a.astype(np.longdouble)
ex = (al.T @ al).astype(np.float64)
dd = np.sqrt(np.diag(ex))
print("max scaled err dev %.3e port %.3e" % ((np.abs(g1 - ex) / np.outer(dd, dd)).max(),
                                           (np.abs(want - ex) / np.outer(dd, dd)).max()))
