#!/bin/bash
out=gpurun_out/r10au; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > $out/pytest.log 2>&1; tail -1 $out/pytest.log
bash bench_tools/variant_ab.sh ";" ";" > $out/variants.txt 2>&1
cat $out/variants.txt
