"""Determinism check of the device pipeline at full size: the same A through
one plan `reps` times; prints sweeps and a hash of sigma per run (they must
all agree), and of M when MPSVD stage access is available.

    python tools/oz32_det.py c4 3
"""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2603_11953_b200 as M  # noqa: E402
import workloads as inputs  # noqa: E402

cfg = inputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
m = int(os.environ.get("PROF_M", cfg.m))
dev = torch.device("cuda", 0)
a = inputs.device_make(cfg, seed=1, m=m, device=dev)
u = torch.empty_like(a)
s = torch.empty(cfg.n, dtype=torch.float64, device=dev)
v = torch.empty((cfg.n, cfg.n), dtype=a.dtype, device=dev)
plan = M.Plan(m, cfg.n, M.Precision.WORKING if cfg.working == "f32" else M.Precision.HIGHER)
hs = []
for _ in range(reps):
    plan.execute(a.data_ptr(), m, u.data_ptr(), m, s.data_ptr(), v.data_ptr(), 0)
    info = plan.wait()
    h = hashlib.sha1(s.cpu().numpy().tobytes()).hexdigest()[:12]
    hs.append(h)
    print(f"sweeps {info.sweeps} rotations {info.rotations} sigma {h} gram_ms {info.ms_gram:.3f}", flush=True)
print("DETERMINISTIC" if len(set(hs)) == 1 else "NONDETERMINISTIC")
