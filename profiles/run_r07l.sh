#!/bin/bash
# GPU suite with emit items 4; onesweep shape variants under the 2-item ranking
out=gpurun_out/r07l; mkdir -p $out
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $out/pytest_gpu.log 2>&1
bash bench_tools/variant_bench.sh "" "-DLMGS_SORT_ITEMS=12 -DLMGS_SORT_MIN_CTAS=4" "-DLMGS_SORT_ITEMS=8 -DLMGS_SORT_MIN_CTAS=5" \
  "-DLMGS_SORT_ITEMS=16 -DLMGS_SORT_MIN_CTAS=3 -DLMGS_RANK_GROUP=1" "-DLMGS_LOOK_WINDOW=16" > $out/variants.txt 2>&1
