"""Regenerate tests/golden/*.npz from the UNMODIFIED reference
(oracle/_ref/libmpsvd_ref.so, built in place from /root/reference by
oracle/Makefile). Run in the build container: `python tests/golden/make_golden.py`.

Each fixture stores the inputs (or the seed recipe that rebuilds them
bit-exactly) and the reference's outputs for one known-answer case of the
hot path (citations: proj/tests/*.cpp lines in each entry's `source`)."""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import pyoracle  # noqa: E402
import workloads as inputs  # noqa: E402


def main():
    ref = pyoracle.Ref()
    out = {}

    a = np.zeros((4, 2), np.float32, order="F")
    a[0, 0], a[1, 1] = 5.0, 3.0
    r = ref.thin_svd(a)
    out["stacked_diag"] = dict(a=a, u=r.u, v=r.v, sigma=r.sigma, source="proj/tests/test_thinsvd.cpp:70-84")

    a, sref, kb = ref.build_problem(1024, 64, 1e8, 1e3, 3, 5)
    r = ref.thin_svd(a)
    out["graded_suite"] = dict(a=a, u=r.u, v=r.v, sigma=r.sigma, sigma_oracle=ref.reference_svd(a),
                               kappa_b=np.float64(kb), source="proj/tests/test_thinsvd.cpp:103-132")

    a, _, kb = ref.build_problem(300, 24, 1e4, 1e2, 7, 9)
    r1 = ref.thin_svd(a, threads=1)
    r4 = ref.thin_svd(a, threads=4)
    assert np.array_equal(r1.u, r4.u) and np.array_equal(r1.sigma, r4.sigma)
    out["thread_invariance"] = dict(a=a, u=r1.u, v=r1.v, sigma=r1.sigma, gram_blocks=np.int64(r1.gram_blocks),
                                    sync_events=np.int64(r1.sync_events),
                                    source="proj/tests/test_thinsvd.cpp:134-149")

    m2 = np.array([[2.0, 1.0], [1.0, 2.0]])
    lam, v, sw, rot = ref.twosided_jacobi(m2)
    out["jacobi_2x2"] = dict(m=m2, lam=lam, v=v, source="proj/tests/test_jacobi.cpp:193-206")

    for k in (4, 8):
        h = np.array([[1.0 / (i + j + 1) for j in range(k)] for i in range(k)])
        out[f"hilbert{k}"] = dict(m=h, lam_dd=ref.dd_oracle_eigenvalues(h), lam=ref.twosided_jacobi(h)[0],
                                  source="proj/tests/test_jacobi.cpp:209-227 (dd LDL^T bisection oracle)")

    rng = np.random.default_rng(17)
    a64 = np.asfortranarray(rng.uniform(-1, 1, (40, 6)) * 10.0 ** -np.arange(6)[None, :])
    hi, lo = ref.dd_gram(a64)
    out["dd_gram"] = dict(a=a64, hi=hi, lo=lo, sigma_dd=ref.dd_oracle_singular_values(a64),
                          source="proj/tests/support/dd.cpp:75-88,155-163")

    cfg = inputs.CONFIGS["c1"]
    a = inputs.make(cfg, seed=1)
    r = ref.thin_svd(a, threads=8)
    out["config_c1"] = dict(seed=np.int64(1), v=r.v, sigma=r.sigma, u_head=r.u[:64].copy(order="F"),
                            u_colsum=r.u.astype(np.float64).sum(axis=0), a_colsum=a.astype(np.float64).sum(axis=0),
                            source="BASELINE.json configs[0] (seeded numpy PCG64 input, paper_2603_11953_b200.inputs)")

    for name, d in out.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
        print(name, {k: getattr(v, "shape", v) for k, v in d.items() if k != "source"})


if __name__ == "__main__":
    main()
