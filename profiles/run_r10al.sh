#!/bin/bash
out=gpurun_out/r10al; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_group.py tests/test_gpu_fused.py tests/test_gpu_pipeline.py -q -x -p no:cacheprovider > $out/pytest.log 2>&1; tail -3 $out/pytest.log
bash bench_tools/variant_ab.sh ";" "-DLMGS_SORT_PREFETCH=0;" ";" "-DLMGS_SORT_PREFETCH=0;" ";--mode graph" > $out/variants.txt 2>&1
cat $out/variants.txt
