#!/bin/bash
out=gpurun_out/r10bs; mkdir -p $out
bash bench_tools/variant_ab.sh ";" ";--streams 5" ";--streams 6" "-DLMGS_EMIT_PERSIST_CTAS=3;" ";" ";--streams 5" ";--streams 6" "-DLMGS_EMIT_PERSIST_CTAS=3;" > $out/variants.txt 2>&1
cat $out/variants.txt
