#!/bin/bash
out=gpurun_out/r10aj; mkdir -p $out
LMGS_NVCC_FLAGS="-DLMGS_LOOKBACK_LATE=2" python -c "from paper_2503_21364_b200 import build; build.build(force=True)" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py tests/test_gpu_group.py -q -x -p no:cacheprovider > $out/pytest.log 2>&1; tail -1 $out/pytest.log
bash bench_tools/variant_ab.sh ";" "-DLMGS_LOOKBACK_LATE=2;" ";" "-DLMGS_LOOKBACK_LATE=2;" > $out/variants.txt 2>&1
cat $out/variants.txt
