#!/bin/bash
out=gpurun_out/r10u; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_fused.py -q -x -p no:cacheprovider 2>&1 | tail -1
bash bench_tools/variant_ab.sh ";" "-DLMGS_LOOKBACK_LATE=1;" "-DLMGS_LOOK_WINDOW=16;" "-DLMGS_LOOKBACK_LATE=1 -DLMGS_LOOK_WINDOW=16;" ";" "-DLMGS_LOOKBACK_LATE=1;" > $out/variants.txt 2>&1
cat $out/variants.txt
LMGS_NVCC_FLAGS="-DLMGS_SORT_TRACE=2 -DLMGS_LOOKBACK_LATE=1" python -c "from paper_2503_21364_b200 import build; build.build(force=True)" > /dev/null 2>&1
python bench_tools/sort_trace.py 0 > $out/trace.txt 2>&1
python bench_tools/sort_trace.py 1 >> $out/trace.txt 2>&1
python -c "from paper_2503_21364_b200 import build; build.build(force=True)" > /dev/null 2>&1
cat $out/trace.txt
