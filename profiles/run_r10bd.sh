#!/bin/bash
out=gpurun_out/r10bd; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py tests/test_gpu_group.py tests/test_gpu_fused.py -q -x -p no:cacheprovider > $out/pytest.log 2>&1; tail -1 $out/pytest.log
sed 's#gpurun_out/r10aa#gpurun_out/r10bd#g' profiles/run_r10aa.sh > /tmp/inst.sh; bash /tmp/inst.sh | grep "onesweep\|total"
bash bench_tools/variant_ab.sh ";" "-DLMGS_RANK_PAIRS=0;" ";" "-DLMGS_RANK_PAIRS=0;" > $out/variants.txt 2>&1
cat $out/variants.txt
