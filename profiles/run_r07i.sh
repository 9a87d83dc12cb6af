#!/bin/bash
# K1 view pairs on separate warps (k_preprocess_pair) vs k_preprocess_tma<2>
out=gpurun_out/r07i; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_group.py tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > $out/pytest_group.log 2>&1
bash bench_tools/variant_bench.sh "" "-DLMGS_PRE_PAIR_SPLIT=0" "-DLMGS_PRE_SPLIT_MIN_CTAS=2" "-DLMGS_PRE_SPLIT_MIN_CTAS=4" > $out/variants.txt 2>&1
