#!/bin/bash
# ncu source-level capture of the multi-CTA Jacobi at c5's n (reduced rows: the solver does not depend on m)
d=gpurun_out/ncu_jac; mkdir -p $d
PROF_M=65536 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:jacobi_kernel -c 1 \
  -o $d/jac_c5 python tools/prof_plan.py c5 1 > $d/ncu.log 2>&1
ncu -i $d/jac_c5.ncu-rep --page source --csv --print-source sass > $d/jac_c5_sass.csv 2>/dev/null
ncu -i $d/jac_c5.ncu-rep --page raw --csv > $d/jac_c5_raw.csv 2>/dev/null
python tools/ncu_source.py $d/jac_c5_sass.csv > $d/jac_c5_stalls.txt 2>&1
python tools/ncu_summary.py $d/jac_c5.ncu-rep jacobi > $d/jac_c5_summary.txt 2>&1
rm -f $d/jac_c5.ncu-rep
