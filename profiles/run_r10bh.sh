#!/bin/bash
out=gpurun_out/r10bh; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $out/pytest_gpu.log 2>&1; tail -1 $out/pytest_gpu.log
timeout 300 python bench_tools/stress_parity.py 13 60 > $out/stress.log 2>&1; tail -1 $out/stress.log
bash bench_tools/variant_ab.sh ";" "-DLMGS_BLEND_SMEM_FP64=1;" ";" "-DLMGS_BLEND_SMEM_FP64=1;" > $out/variants.txt 2>&1
cat $out/variants.txt
