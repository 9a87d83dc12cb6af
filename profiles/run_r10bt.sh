#!/bin/bash
out=gpurun_out/r10bt; mkdir -p $out
bash bench_tools/variant_ab.sh ";" "-DLMGS_FIX_CTAS_PER_SM=2;" "-DLMGS_FIX_CTAS_PER_SM=1;" ";" "-DLMGS_FIX_CTAS_PER_SM=2;" "-DLMGS_FIX_CTAS_PER_SM=1;" > $out/variants.txt 2>&1
cat $out/variants.txt
