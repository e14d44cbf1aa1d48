#!/bin/bash
# Compile one csrc/*.cu for sm_100a with -Xptxas -v and dump its SASS
# (tools/sass_check.sh gram_ozaki32.cu [kernel-substring]) -> /tmp/<file>.sass
set -e
R=/root/repo/paper_2603_11953_b200
f=$1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC \
  --expt-relaxed-constexpr -I/root/repo/include -I$R/csrc -Xptxas -v -c $R/csrc/$f -o /tmp/${f%.cu}.o 2>&1 \
  | grep -E "registers|stack|error|warning" || true
cuobjdump -sass /tmp/${f%.cu}.o > /tmp/${f%.cu}.sass
