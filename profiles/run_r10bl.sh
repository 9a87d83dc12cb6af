#!/bin/bash
out=gpurun_out/r10bl; mkdir -p $out
bash bench_tools/variant_ab.sh ";" ";--streams 5" ";--streams 3" "-DLMGS_SORT_PERSIST_CTAS=2;" "-DLMGS_EMIT_PERSIST_CTAS=4;" ";" ";--streams 5" > $out/variants.txt 2>&1
cat $out/variants.txt
