#!/bin/bash
out=gpurun_out/r10ai; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_group.py tests/test_gpu_fused.py -q -x -p no:cacheprovider > $out/pytest.log 2>&1; tail -1 $out/pytest.log
bash bench_tools/variant_ab.sh ";" "-DLMGS_SERIAL_K1=0;" ";--streams 3" ";--streams 5" ";--mode graph" > $out/variants.txt 2>&1
cat $out/variants.txt
