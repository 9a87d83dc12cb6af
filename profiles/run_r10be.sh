#!/bin/bash
out=gpurun_out/r10be; mkdir -p $out
bash bench_tools/variant_ab.sh ";" "-DLMGS_SORT_SMEM_PAD=16384;" "-DLMGS_SORT_SMEM_PAD=49152;" > $out/variants.txt 2>&1
cat $out/variants.txt
