#!/bin/bash
out=gpurun_out/r10l; mkdir -p $out
timeout 300 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_group.py -q -x -p no:cacheprovider 2>&1 | tail -2
bash bench_tools/variant_ab.sh ";" "-DLMGS_EMIT_PERSIST_CTAS=1;" "-DLMGS_EMIT_PERSIST_CTAS=2;" "-DLMGS_EMIT_PERSIST_CTAS=3;" \
   "-DLMGS_BLEND_CTAS_PER_SM=3;" "-DLMGS_SORT_PERSIST_CTAS=2;" ";" > $out/variants.txt 2>&1
cat $out/variants.txt
