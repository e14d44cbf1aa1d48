#!/bin/bash
# Full evidence pass into gpurun_out/$1: GPU suite, smoke, bench lines for every config, c4 launch list
d=gpurun_out/${1:-final}; mkdir -p $d
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $d/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $d/smoke.log 2>&1; echo "smoke rc=$?" >> $d/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $d/gputests.log 2>&1; echo "pytest rc=$?" >> $d/gputests.log
cp gpurun_out/config_parity.jsonl $d/ 2>/dev/null
for c in c4 c2 c3 c5; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 > $d/bench_$c.json 2> $d/bench_$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $d/launches_c4.csv \
  python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline > $d/ncu_c4.log 2>&1
