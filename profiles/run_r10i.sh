#!/bin/bash
out=gpurun_out/r10i; mkdir -p $out
bash bench_tools/variant_ab.sh ";" ";--flags 32" "-DLMGS_SORT_PERSIST_CTAS=1;" "-DLMGS_SORT_PERSIST_CTAS=1;--flags 32" \
  "-DLMGS_SORT_PERSIST_CTAS=2;" "-DLMGS_SORT_PERSIST_CTAS=2;--flags 32" ";" ";--flags 32" > $out/variants.txt 2>&1
cat $out/variants.txt
