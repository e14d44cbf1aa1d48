#!/bin/bash
# One GPU-box session: smoke, the -m gpu suite (or a subset), bench lines
# and (NCU=1) the launch list of the first bench config; logs land in gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1500 python -m pytest ${TESTS:-tests} -m gpu -x -q -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests.log
fi
for c in ${BENCH_CONFIGS:-c4}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup ${WARMUP:-3} ${BENCH_ARGS} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?" >> gpurun_out/bench_rc.txt
done
if [ "${NCU:-0}" = 1 ]; then
  c=${BENCH_CONFIGS%% *}; c=${c:-c4}
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_$c.log 2>&1; echo "ncu rc=$?" >> gpurun_out/bench_rc.txt
fi
