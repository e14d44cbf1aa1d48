#!/bin/bash
# Bench lines of the three mp_thin_svd spectral branches (c2, c4) plus the
# reference arm for the one-sided ones; output under gpurun_out/eig/.
mkdir -p gpurun_out/eig
for cfg in c2 c4; do
  for eig in twosided gramchol onesided; do
    timeout 600 python bench.py --config $cfg --eig $eig --steps 5 --warmup 3 --no-cpu-baseline \
      > gpurun_out/eig/${cfg}_${eig}.json 2> gpurun_out/eig/${cfg}_${eig}.err
  done
done
for eig in gramchol onesided; do
  timeout 600 python bench.py --impl reference --config c2 --eig $eig --steps 2 --warmup 1 \
    > gpurun_out/eig/ref_c2_${eig}.json 2> gpurun_out/eig/ref_c2_${eig}.err
done
