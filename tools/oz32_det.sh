#!/bin/bash
mkdir -p gpurun_out
for st in ${STAGES:-8x3 7x3 7x4 6x4 6x3}; do for w in ${WAITS:-0}; do
  echo "== stages=$st wait=$w" >> gpurun_out/oz32_det.txt
  if [ -n "$GRAM_LG" ]; then
    MPSVD_F32_GRAM=ozaki MPSVD_OZ32_STAGES=$st MPSVD_OZ32_WAIT=$w timeout 300 python tools/oz32_gram_det.py $GRAM_LG ${REPS:-3} >> gpurun_out/oz32_det.txt 2>&1
  else
    MPSVD_OZ32_STAGES=$st MPSVD_OZ32_WAIT=$w timeout 300 python tools/oz32_det.py c4 ${REPS:-3} >> gpurun_out/oz32_det.txt 2>&1
  fi
done; done
