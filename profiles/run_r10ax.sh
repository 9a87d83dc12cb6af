#!/bin/bash
out=gpurun_out/r10ax; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py tests/test_gpu_group.py -q -x -p no:cacheprovider > $out/pytest.log 2>&1; tail -1 $out/pytest.log
timeout 300 python bench_tools/stress_parity.py 11 60 > $out/stress.log 2>&1; tail -2 $out/stress.log
sed 's#gpurun_out/r10aa#gpurun_out/r10ax#g' profiles/run_r10aa.sh > /tmp/inst.sh; bash /tmp/inst.sh | grep "fixup\|total"
bash bench_tools/variant_ab.sh ";" "-DLMGS_FIXUP_WARP=0;" ";" "-DLMGS_FIXUP_WARP=0;" > $out/variants.txt 2>&1
cat $out/variants.txt
