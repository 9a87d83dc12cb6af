#!/bin/bash
out=gpurun_out/r10at; mkdir -p $out
bash bench_tools/variant_ab.sh ";" "-DLMGS_EMIT_ITEMS=3;" "-DLMGS_EMIT_ITEMS=6;" "-DLMGS_EMIT_ITEMS=2 -DLMGS_EMIT_THREADS=512;" "-DLMGS_EMIT_ITEMS=8;" > $out/variants.txt 2>&1
cat $out/variants.txt
