#!/bin/bash
out=gpurun_out/r10x; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_group.py tests/test_gpu_fused.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > $out/pytest.log 2>&1; tail -1 $out/pytest.log
bash bench_tools/variant_ab.sh ";" ";--mode nosync" ";--mode graph" ";--mode graph --streams 3" ";--mode nosync --streams 5" > $out/variants.txt 2>&1
cat $out/variants.txt
