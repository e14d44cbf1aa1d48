#!/bin/bash
# K1z variants on c4 (MPSVD_OZ32_STAGES x MPSVD_OZ32_WAIT): gram phase ms per variant
mkdir -p gpurun_out
for st in ${STAGES:-8 7}; do for w in ${WAITS:-0 1 2}; do
  echo "stages=$st wait=$w $(MPSVD_OZ32_STAGES=$st MPSVD_OZ32_WAIT=$w python tools/prof_plan.py ${CFG:-c4} 4 2>&1 | tail -1)" >> gpurun_out/oz32_ab.txt
done; done
