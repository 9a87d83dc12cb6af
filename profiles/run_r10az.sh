#!/bin/bash
out=gpurun_out/r10az; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > $out/pytest.log 2>&1; tail -1 $out/pytest.log
sed 's#gpurun_out/r10aa#gpurun_out/r10az#g' profiles/run_r10aa.sh > /tmp/inst.sh; bash /tmp/inst.sh | grep "k_emit\|total"
bash bench_tools/variant_ab.sh ";" ";" > $out/variants.txt 2>&1
cat $out/variants.txt
