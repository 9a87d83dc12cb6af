#!/bin/bash
out=gpurun_out/r10bi; mkdir -p $out
bash bench_tools/variant_ab.sh ";" "-DLMGS_BLEND_MAXREG=56;" "-DLMGS_BLEND_MAXREG=60;" ";" > $out/variants.txt 2>&1
cat $out/variants.txt
