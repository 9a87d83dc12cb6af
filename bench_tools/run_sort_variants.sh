#!/bin/bash
# Build and run onesweep variants: "items ctas window extra-flags"
cd "$(dirname "$0")"
mkdir -p ../gpurun_out/sortbench
while read -r it ct wi fl; do
  [ -z "$it" ] && continue
  exe=/tmp/sb_${it}_${ct}_${wi}_${fl//[^A-Z]/}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DLMGS_SORT_ITEMS=$it -DLMGS_SORT_MIN_CTAS=$ct \
       -DLMGS_LOOK_WINDOW=$wi $fl -I../include sort_bench.cu -o $exe 2>/dev/null || { echo "build $it $ct $wi $fl failed"; continue; }
  echo "== $fl"
  $exe 20900000 8 2 0
  $exe 6000000 4 4 1
done
