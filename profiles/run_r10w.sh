#!/bin/bash
out=gpurun_out/r10w; mkdir -p $out
LMGS_NVCC_FLAGS="-DLMGS_PRE_PERSIST_CTAS=4" python -c "from paper_2503_21364_b200 import build; build.build(force=True)" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_group.py tests/test_gpu_fused.py tests/test_gpu_batch*.py -q -x -p no:cacheprovider 2>&1 | tail -2
bash bench_tools/variant_ab.sh ";" "-DLMGS_PRE_PERSIST_CTAS=3;" "-DLMGS_PRE_PERSIST_CTAS=4;" "-DLMGS_PRE_PERSIST_CTAS=5;" "-DLMGS_PRE_PERSIST_CTAS=2;" > $out/variants.txt 2>&1
cat $out/variants.txt
