#!/bin/bash
# blend work-counter slices and colour-sector prefetch variants
out=gpurun_out/r07h; mkdir -p $out
bash bench_tools/variant_bench.sh "-DLMGS_BLEND_SLICES=1" "" "-DLMGS_BLEND_SLICES=16" "-DLMGS_BLEND_PF_COLOR=1" \
  "-DLMGS_BLEND_PF_COLOR=1 -DLMGS_BLEND_SLICES=16" > $out/variants.txt 2>&1
