#!/bin/bash
out=gpurun_out/r10y; mkdir -p $out
bash bench_tools/variant_ab.sh ";" "-DLMGS_SORT_ITEMS=12 -DLMGS_SORT_MIN_CTAS=4 -DLMGS_SORT_MIN_CTAS_NARROW=5;" \
  "-DLMGS_SORT_ITEMS=20 -DLMGS_SORT_MIN_CTAS=2 -DLMGS_SORT_MIN_CTAS_NARROW=3;" "-DLMGS_SORT_MIN_CTAS=2 -DLMGS_SORT_MIN_CTAS_NARROW=3;" \
  "-DLMGS_SORT_ITEMS=12 -DLMGS_SORT_MIN_CTAS=3 -DLMGS_SORT_MIN_CTAS_NARROW=4;" > $out/variants.txt 2>&1
cat $out/variants.txt
