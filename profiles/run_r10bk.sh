#!/bin/bash
out=gpurun_out/r10bk; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py tests/test_gpu_group.py tests/test_gpu_fused.py -q -x -p no:cacheprovider > $out/pytest.log 2>&1; tail -1 $out/pytest.log
bash bench_tools/variant_ab.sh ";" "-DLMGS_SORT_IOTA16=0;" "-DLMGS_RANK_SPLIT=2;" ";" "-DLMGS_SORT_IOTA16=0;" "-DLMGS_RANK_SPLIT=2;" > $out/variants.txt 2>&1
cat $out/variants.txt
