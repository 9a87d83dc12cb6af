#!/bin/bash
out=gpurun_out/r10bn; mkdir -p $out
bash bench_tools/variant_ab.sh ";" "-DLMGS_BLEND_CTAS_PER_SM=3;" "-DLMGS_FIX_CTAS_PER_SM=8;" "-DLMGS_DEPTH_KEYS_CTAS_PER_SM=4;" ";" "-DLMGS_BLEND_CTAS_PER_SM=3;" "-DLMGS_FIX_CTAS_PER_SM=8;" "-DLMGS_DEPTH_KEYS_CTAS_PER_SM=4;" > $out/variants.txt 2>&1
cat $out/variants.txt
