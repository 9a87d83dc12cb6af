#!/bin/bash
out=gpurun_out/r10br; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py tests/test_gpu_group.py tests/test_gpu_fused.py -q -x -p no:cacheprovider > $out/pytest.log 2>&1; tail -1 $out/pytest.log
bash bench_tools/variant_ab.sh ";" "-DLMGS_BLEND_CONCURRENT_CTAS=0;" "-DLMGS_BLEND_CONCURRENT_CTAS=3;" ";" "-DLMGS_BLEND_CONCURRENT_CTAS=0;" "-DLMGS_BLEND_CONCURRENT_CTAS=3;" ";" "-DLMGS_BLEND_CONCURRENT_CTAS=0;" > $out/variants.txt 2>&1
cat $out/variants.txt
