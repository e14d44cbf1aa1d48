"""K2z spot check on the GPU for a given shape: device Gram vs K2 (Dot2).
python tools/oz_check.py m n"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_11953_b200 as M  # noqa: E402

m, n = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(1)
a = np.asfortranarray(rng.standard_normal((m, n)) * np.logspace(0, -8, n))
os.environ["MPSVD_DD_GRAM"] = "ozaki"
hi, lo = M.gram(a)
os.environ["MPSVD_DD_GRAM"] = "dot2"
dh, dl = M.gram(a)
nrm = np.linalg.norm(a, axis=0)
err = np.max(np.abs((hi - dh) + (lo - dl)) / np.outer(nrm, nrm))
print(f"m={m} n={n}: max scaled |ozaki - dot2| = {err:.3e}")
