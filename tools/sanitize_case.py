"""One small thin SVD per case, for compute-sanitizer (racecheck / synccheck /
memcheck) runs of the persistent and warp-specialised kernels:

    compute-sanitizer --tool racecheck python tools/sanitize_case.py <case>

cases (each forces the kernel it names through the public API):
    jacobi_smem   fp32 thin SVD, n = 64   (K4 single-CTA Jacobi, K1 Gram, K7 av_tc_tmem_f32)
    jacobi_grid   fp64 thin SVD, n = 160  (K5 cooperative-grid dd Jacobi, av_dmma_f64)
    k2z           fp64 thin SVD, m = 8192, n = 128, MPSVD_DD_GRAM=ozaki (gram_dd_ozaki)
    k1z           fp32 thin SVD, m = 8192, n = 128, MPSVD_F32_GRAM=ozaki (gram_f32_ozaki)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads  # noqa: E402

CASES = {
    "jacobi_smem": (4096, 64, "f32", {}),
    "jacobi_grid": (4096, 160, "f64", {"MPSVD_DD_GRAM": "dot2"}),
    "k2z": (8192, 128, "f64", {"MPSVD_DD_GRAM": "ozaki"}),
    "k1z": (8192, 128, "f32", {"MPSVD_F32_GRAM": "ozaki"}),
}


def main():
    case = sys.argv[1]
    m, n, working, env = CASES[case]
    os.environ.update(env)
    import paper_2603_11953_b200 as M

    if working == "f32":
        a = workloads.graded(m, n, 4.0, seed=3)
        r = M.mp_thin_svd(a)
    else:
        a = workloads.graded(m, n, 8.0, seed=3, dtype=np.float64)
        r = M.mp_thin_svd_f64(a)
    u = r.u.astype(np.float64)
    print(f"{case}: m={m} n={n} sweeps={r.jacobi_sweeps} sigma[0]={r.sigma[0]:.6e} "
          f"orth_u={np.linalg.norm(u.T @ u - np.eye(n)):.3e}")


if __name__ == "__main__":
    main()
