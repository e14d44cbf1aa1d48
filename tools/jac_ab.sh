#!/bin/bash
# Jacobi timing after a change: eigen phase ms per config, traces, then the Jacobi-related GPU tests
mkdir -p gpurun_out; o=gpurun_out/jac_ab.txt; : > $o
for c in c5 c3; do
  echo "$c $(timeout 600 python tools/prof_plan.py $c 3 2>&1 | tail -1)" >> $o
done
for c in c5 c3; do
MPSVD_JACOBI_TRACE=1 timeout 600 python tools/prof_plan.py $c 1 2>&1 | grep -i "trace" >> $o
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "jacobi or config or c5 or c3 or grid or dd or scal" > gpurun_out/jac_tests.log 2>&1; echo "rc=$?" >> gpurun_out/jac_tests.log
