#!/bin/bash
# K1 view groups in the current batch regime
out=gpurun_out/r10t; mkdir -p $out
bash bench_tools/variant_ab.sh ";" ";--group 3" ";--group 4" ";--group 4 --streams 3" ";--group 4 --streams 2" \
  "-DLMGS_PRE_MULTI_MIN_CTAS=4;--group 4" "-DLMGS_PRE_MULTI_MIN_CTAS=4;" ";--group 8 --streams 2" > $out/variants.txt 2>&1
cat $out/variants.txt
