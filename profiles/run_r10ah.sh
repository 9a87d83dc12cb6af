#!/bin/bash
out=gpurun_out/r10ah; mkdir -p $out
bash bench_tools/variant_ab.sh ";" "-DLMGS_BLEND_CTAS_PER_SM=3;" "-DLMGS_PRE_MULTI_MIN_CTAS=6;" ";--streams 5" ";--streams 3" "-DLMGS_FIX_CTAS_PER_SM=8;" > $out/variants.txt 2>&1
cat $out/variants.txt
