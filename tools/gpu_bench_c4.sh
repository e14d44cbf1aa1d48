#!/bin/bash
# c4 bench line + ncu launch list (per-kernel share of the step) into gpurun_out/$1
d=gpurun_out/${1:-c4run}; mkdir -p $d
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $d/smi.txt 2>&1
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 > $d/bench_c4.json 2> $d/bench_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $d/launches_c4.csv \
  python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline > $d/ncu_c4.log 2>&1
timeout 900 python bench.py --config c2 --steps 20 --warmup 3 > $d/bench_c2.json 2> $d/bench_c2.err
