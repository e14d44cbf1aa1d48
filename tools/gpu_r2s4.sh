#!/bin/bash
# Session pass: smoke, GPU suite, default bench (driver's invocation), reference arm, K1z ncu source capture
d=gpurun_out/${1:-s4}; mkdir -p $d
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $d/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $d/smoke.log 2>&1; echo "smoke rc=$?" >> $d/smoke.log
( time timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider ) > $d/gputests.log 2>&1; echo "pytest rc=$?" >> $d/gputests.log
( time timeout 900 python bench.py ) > $d/bench_default.json 2> $d/bench_default.err
( time timeout 900 python bench.py --impl reference --steps 3 --warmup 1 ) > $d/bench_reference.json 2> $d/bench_reference.err
PROF_M=4194304 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_f32_ozaki -s 1 -c 1 \
  -o $d/k1z python tools/prof_plan.py c4 2 > $d/ncu_k1z.log 2>&1
ncu -i $d/k1z.ncu-rep --page source --csv --print-source sass > $d/k1z_sass.csv 2>/dev/null
ncu -i $d/k1z.ncu-rep --page raw --csv > $d/k1z_raw.csv 2>/dev/null
