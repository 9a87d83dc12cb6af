#!/bin/bash
out=gpurun_out/r10q; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py -q -x -p no:cacheprovider 2>&1 | tail -2
bash bench_tools/variant_ab.sh ";" "-DLMGS_BLEND_PAIRS=0;" ";" "-DLMGS_BLEND_PAIRS=0;" > $out/variants.txt 2>&1
cat $out/variants.txt
