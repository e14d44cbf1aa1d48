#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck, one tool per process,
# on small shapes of the persistent / warp-specialised kernels
# (tools/sanitize_case.py). Logs: gpurun_out/sanitize_<tool>_<case>.log
mkdir -p gpurun_out
for tool in ${TOOLS:-racecheck synccheck memcheck}; do
  for c in ${CASES:-jacobi_smem jacobi_grid k2z k1z}; do
    MPSVD_NO_GRAPH=1 timeout 900 compute-sanitizer --tool $tool --print-limit 20 \
      python tools/sanitize_case.py $c > gpurun_out/sanitize_${tool}_$c.log 2>&1
    echo "$tool $c rc=$?" >> gpurun_out/sanitize_rc.txt
  done
done
