"""Localise a K1z Gram race: repeat the device Gram of one A until a result
differs from the first, then find the wrong column c and the aligned 8-row
group(s) whose products x_kc x_kj explain the difference."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2603_11953_b200 as M  # noqa: E402
import workloads  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 22
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
m, n = 1 << lg, 128
a = workloads.gaussian(m, n, seed=5)
a64 = np.asarray(a, dtype=np.float64)
ref = a64.T @ a64
g0 = M.gram(a)
e0 = np.abs(g0 - ref).max()
print("first: max abs err vs fp64", e0, flush=True)
for r in range(reps):
    g = M.gram(a)
    if np.array_equal(g, g0):
        continue
    dif = g - g0
    bad = np.argwhere(dif != 0)
    cols = np.unique(bad[:, 1])
    e1 = np.abs(g - ref).max()
    print(f"rep {r}: {len(bad)} entries differ, err vs fp64 {e1:.3e} (first {e0:.3e}); columns {cols[:10]}", flush=True)
    # the wrong column: the one present in every differing pair
    cnt = np.bincount(bad.ravel(), minlength=n)
    c = int(np.argmax(cnt))
    d = (g if np.abs(g - ref).max() > e0 else g0) - ref
    delta = d[:, c]
    print(f"  column {c}: |delta| max {np.abs(delta).max():.3e}, delta[c] {delta[c]:.4e}", flush=True)
    # per 8-row group contributions x_kc * x_kj
    prod = (a64[:, c][:, None] * a64).reshape(m // 8, 8, n).sum(axis=1)  # (groups, n)
    # best single group explaining +/- delta (excluding the diagonal entry)
    mask = np.ones(n, bool)
    mask[c] = False
    for sgn in (1, -1):
        res = np.linalg.norm(prod[:, mask] - sgn * delta[mask], axis=1)
        k = int(np.argmin(res))
        print(f"  sign {sgn:+d}: best 8-row group {k} (rows {8 * k}..{8 * k + 7}, chunk {8 * k // 32}, half {(8 * k % 32) // 16}, "
              f"q {(8 * k % 16) // 8}) residual {res[k]:.3e} vs |delta| {np.linalg.norm(delta[mask]):.3e}", flush=True)
    prod16 = prod.reshape(m // 16, 2, n).sum(axis=1)
    for sgn in (1, -1):
        res = np.linalg.norm(prod16[:, mask] - sgn * delta[mask], axis=1)
        k = int(np.argmin(res))
        print(f"  sign {sgn:+d}: best 16-row group {k} (chunk {k // 2}, half {k % 2}) residual {res[k]:.3e}", flush=True)
    break
else:
    print("no difference in", reps, "repetitions")
