#!/bin/bash
# emit shape variants: ranks per thread x threads per CTA
out=gpurun_out/r07k; mkdir -p $out
bash bench_tools/variant_bench.sh "-DLMGS_EMIT_ITEMS=2" "-DLMGS_EMIT_ITEMS=3" "-DLMGS_EMIT_ITEMS=4" \
  "-DLMGS_EMIT_ITEMS=4 -DLMGS_EMIT_THREADS=128" "-DLMGS_EMIT_ITEMS=4 -DLMGS_EMIT_THREADS=512" \
  "-DLMGS_EMIT_ITEMS=2 -DLMGS_EMIT_THREADS=512" > $out/variants.txt 2>&1
