"""Device time of the mixed-precision Cholesky QR (Plan.cholesky_qr) and its
phases on BASELINE-shaped binary32 inputs; prints one JSON line per config."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_11953_b200 as M  # noqa: E402
import workloads as inputs  # noqa: E402

for name in sys.argv[1:] or ["c2", "c4"]:
    cfg = inputs.CONFIGS[name]
    dev = torch.device("cuda", 0)
    a = inputs.device_make(cfg, seed=1, m=cfg.m, device=dev)
    q = torch.empty_like(a)
    r = torch.empty((cfg.n, cfg.n), dtype=torch.float32, device=dev)
    plan = M.Plan(cfg.m, cfg.n, M.Precision.WORKING)
    st = torch.cuda.Stream(dev)
    for _ in range(3):
        plan.cholesky_qr(a.data_ptr(), cfg.m, q.data_ptr(), cfg.m, r.data_ptr(), st.cuda_stream)
    info = plan.wait()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 5
    e0.record(st)
    for _ in range(steps):
        plan.cholesky_qr(a.data_ptr(), cfg.m, q.data_ptr(), cfg.m, r.data_ptr(), st.cuda_stream)
    e1.record(st)
    info = plan.wait()
    ms = e0.elapsed_time(e1) / steps
    m, n = cfg.m, cfg.n
    solve_flops = m * n * (n - 1)  # one multiply + one subtract per (row, j, k < j)
    print(json.dumps({"config": name, "m": m, "n": n, "status": info.status, "ms": ms,
                      "phase_ms": {"gram": info.ms_gram, "chol": info.ms_eigen, "row_solve": info.ms_compute_u},
                      "row_solve_gflops": solve_flops / (info.ms_compute_u * 1e-3) / 1e9,
                      "row_solve_hbm_gbs": 2 * m * n * 4 / (info.ms_compute_u * 1e-3) / 1e9}), flush=True)
    del a, q, r, plan
    torch.cuda.empty_cache()
