#!/bin/bash
out=gpurun_out/r10bq; mkdir -p $out
bash bench_tools/variant_ab.sh ";" "-DLMGS_BLEND_CTAS_PER_SM=3;" "-DLMGS_BLEND_CTAS_PER_SM=2;" ";" "-DLMGS_BLEND_CTAS_PER_SM=3;" "-DLMGS_BLEND_CTAS_PER_SM=2;" ";" "-DLMGS_BLEND_CTAS_PER_SM=3;" > $out/variants.txt 2>&1
cat $out/variants.txt
