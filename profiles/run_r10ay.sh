#!/bin/bash
out=gpurun_out/r10ay; mkdir -p $out
bash bench_tools/variant_ab.sh ";" "-DLMGS_DEPTH_KEYS_CTAS_PER_SM=2;" "-DLMGS_DEPTH_KEYS_CTAS_PER_SM=4;" "-DLMGS_FIX_CTAS_PER_SM=4;" > $out/variants.txt 2>&1
cat $out/variants.txt
