#!/bin/bash
out=gpurun_out/r10bo; mkdir -p $out
timeout 900 python bench_tools/stress_parity.py 22 3000 > $out/stress.txt 2>&1; tail -1 $out/stress.txt
bash bench_tools/variant_ab.sh ";" "-DLMGS_EMIT_ITEMS=2;" "-DLMGS_EMIT_ITEMS=8;" ";" "-DLMGS_EMIT_ITEMS=2;" "-DLMGS_EMIT_ITEMS=8;" > $out/variants.txt 2>&1
cat $out/variants.txt
