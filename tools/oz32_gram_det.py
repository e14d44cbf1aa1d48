"""K1z Gram determinism at moderate size: the device Gram of the same A
`reps` times (bitwise comparison) and its error against numpy's binary64 Gram.

    MPSVD_F32_GRAM=ozaki python tools/oz32_gram_det.py 22 4
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2603_11953_b200 as M  # noqa: E402
import workloads  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 22
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
m, n = 1 << lg, 128
a = workloads.gaussian(m, n, seed=5)
a64 = np.asarray(a, dtype=np.float64)
ref = a64.T @ a64
d = np.sqrt(np.diag(ref))
gs = [M.gram(a) for _ in range(reps)]
for k, g in enumerate(gs):
    same = np.array_equal(g, gs[0])
    ndiff = int(np.sum(g != gs[0]))
    err = float(np.max(np.abs(g - ref) / np.outer(d, d)))
    print(f"rep {k}: same_as_0 {same} ndiff {ndiff} max scaled err vs fp64 {err:.3e}", flush=True)
