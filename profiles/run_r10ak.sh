#!/bin/bash
out=gpurun_out/r10ak; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x -p no:cacheprovider > $out/pytest.log 2>&1; tail -3 $out/pytest.log
sed 's#gpurun_out/r10aa#gpurun_out/r10ak#g' profiles/run_r10aa.sh > /tmp/inst.sh; sed -i 's#python profiles/view_probe.py 2 1920 1080 2#python profiles/view_probe.py 2 1920 1080 2 32#' /tmp/inst.sh; bash /tmp/inst.sh | grep -v "at::\|radix_plan\|nproc"
bash bench_tools/variant_ab.sh ";" ";--flags 32" ";" ";--flags 32" > $out/variants.txt 2>&1
cat $out/variants.txt
