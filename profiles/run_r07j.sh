#!/bin/bash
# emit ranks per thread (kEmitItems) variants
out=gpurun_out/r07j; mkdir -p $out
bash bench_tools/variant_bench.sh "-DLMGS_EMIT_ITEMS=4" "-DLMGS_EMIT_ITEMS=6" "" > $out/variants.txt 2>&1
