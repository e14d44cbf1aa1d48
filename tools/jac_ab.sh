#!/bin/bash
# Jacobi timing after a change: V split variants, latency probe, Jacobi-related GPU tests
mkdir -p gpurun_out; o=gpurun_out/jac_ab.txt; : > $o
for v in 0 50 100 30 70; do
  echo "c5 vsplit=$v $(MPSVD_JACOBI_VSPLIT=$v timeout 600 python tools/prof_plan.py c5 2 2>&1 | tail -1)" >> $o
done
for v in 0 50 100; do
  echo "c3 vsplit=$v $(MPSVD_JACOBI_VSPLIT=$v timeout 600 python tools/prof_plan.py c3 3 2>&1 | tail -1)" >> $o
done
for v in 0 50 100; do
MPSVD_JACOBI_VSPLIT=$v MPSVD_JACOBI_TRACE=1 timeout 600 python tools/prof_plan.py c5 1 2>&1 | grep -i "trace" >> $o
done
./tools/microbench/rot_latency > gpurun_out/rot_latency.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "jacobi or config or c5 or c3 or grid or dd or scal" > gpurun_out/jac_tests.log 2>&1; echo "rc=$?" >> gpurun_out/jac_tests.log
