"""Small driver for ncu captures of one stage (gram | jacobi | av) on a
BASELINE-shaped input: `python tools/prof_stage.py jacobi c2 [reps]`."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_11953_b200 as M  # noqa: E402
import workloads as inputs  # noqa: E402


def main():
    stage = sys.argv[1]
    cfg = inputs.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c2"]
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    m = min(cfg.m, int(os.environ.get("PROF_M", 1 << 16)))
    a = inputs.make(cfg, seed=1, m=m)
    if stage == "jacobi":
        if cfg.working == "f32":
            g = M.gram(a)
            for _ in range(reps):
                lam, v, sw, rot = M.twosided_jacobi_eig(g)
        else:
            hi, lo = M.gram(a)
            for _ in range(reps):
                lam, v, sw, rot = M.twosided_jacobi_eig(hi, lo, dd=True)
        print("sweeps", sw, "rotations", rot)
    elif stage == "gram":
        for _ in range(reps):
            M.gram(a)
    else:
        for _ in range(reps):
            r = M.mp_thin_svd(a) if cfg.working == "f32" else M.mp_thin_svd_f64(a)
        print("sweeps", r.jacobi_sweeps)


if __name__ == "__main__":
    main()
