#!/bin/bash
# ranking A/B, repeated and interleaved: group 2 (default), group 1, original mode 0
out=gpurun_out/r07m; mkdir -p $out
bash bench_tools/variant_bench.sh "" "-DLMGS_RANK_GROUP=1" "-DLMGS_RANK_MODE=0" "" "-DLMGS_RANK_GROUP=1" "-DLMGS_RANK_MODE=0" > $out/variants.txt 2>&1
