#!/bin/bash
# One GPU-box session: smoke, the -m gpu suite (or a subset), the latency
# probe and a bench line; logs land in gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
./tools/microbench/rot_latency > gpurun_out/rot_latency.txt 2>&1
timeout 1500 python -m pytest ${TESTS:-tests} -m gpu -x -q -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests.log
for c in ${BENCH_CONFIGS:-c4}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup ${WARMUP:-3} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?" >> gpurun_out/bench_rc.txt
done
