#!/bin/bash
out=gpurun_out/r10ao; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $out/pytest_gpu.log 2>&1; tail -2 $out/pytest_gpu.log
bash bench_tools/variant_ab.sh ";" ";" > $out/variants.txt 2>&1
cat $out/variants.txt
