#!/bin/bash
out=gpurun_out/r10j; mkdir -p $out
bash bench_tools/variant_ab.sh "-DLMGS_SORT_PERSIST_CTAS=1;--flags 32" "-DLMGS_SORT_PERSIST_CTAS=1;--flags 32 --streams 4" \
  "-DLMGS_SORT_PERSIST_CTAS=1;--flags 32 --streams 5" "-DLMGS_SORT_PERSIST_CTAS=1;--streams 4" \
  "-DLMGS_SORT_PERSIST_CTAS=1;--flags 32 --streams 6 --group 1" "-DLMGS_SORT_PERSIST_CTAS=1;--flags 32 --streams 4 --mode nosync" > $out/variants.txt 2>&1
cat $out/variants.txt
