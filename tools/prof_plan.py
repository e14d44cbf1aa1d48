"""Device-resident pipeline driver for ncu captures at full config size:
`python tools/prof_plan.py c4 [reps]` (A generated on the GPU, one plan,
`reps` executes; pick kernels with ncu -k / -s / -c)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2603_11953_b200 as M  # noqa: E402
import workloads as inputs  # noqa: E402

cfg = inputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
m = int(os.environ.get("PROF_M", cfg.m))
dev = torch.device("cuda", 0)
a = inputs.device_make(cfg, seed=1, m=m, device=dev)
u = torch.empty_like(a)
s = torch.empty(cfg.n, dtype=torch.float64, device=dev)
v = torch.empty((cfg.n, cfg.n), dtype=a.dtype, device=dev)
plan = M.Plan(m, cfg.n, M.Precision.WORKING if cfg.working == "f32" else M.Precision.HIGHER)
for _ in range(reps):
    plan.execute(a.data_ptr(), m, u.data_ptr(), m, s.data_ptr(), v.data_ptr(), 0)
    info = plan.wait()
print("ms gram %.3f eigen %.3f u %.3f sweeps %d" % (info.ms_gram, info.ms_eigen, info.ms_compute_u, info.sweeps))
