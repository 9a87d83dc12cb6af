#!/bin/bash
out=gpurun_out/r10av; mkdir -p $out
bash bench_tools/variant_ab.sh ";" "-DLMGS_FIX_THREADS=256;" "-DLMGS_FIX_THREADS=512;" > $out/variants.txt 2>&1
cat $out/variants.txt
