#!/bin/bash
# A/B of two builds of the library on one box: tools/_ab/libmpsvd_{old,new}.so
# (built here from two trees), c4 phase times per build, alternating; then
# the K1z parity tests on the new build
mkdir -p gpurun_out; out=gpurun_out/k1z_ab.txt; : > $out
L=paper_2603_11953_b200/libmpsvd_b200.so
for rep in 1 2 3; do for v in old new; do
  cp tools/_ab/libmpsvd_$v.so $L
  echo "$v $(python tools/prof_plan.py ${CFG:-c4} 4 2>&1 | tail -1)" >> $out
done; done
cp tools/_ab/libmpsvd_new.so $L
timeout 900 python -m pytest tests/test_ozaki32.py tests/test_configs_gpu.py -m gpu -q -p no:cacheprovider > gpurun_out/k1z_tests.log 2>&1; echo "rc=$?" >> gpurun_out/k1z_tests.log
