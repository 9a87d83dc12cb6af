#!/bin/bash
out=gpurun_out/r10ba; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $out/pytest_gpu.log 2>&1; tail -1 $out/pytest_gpu.log
timeout 300 python bench_tools/stress_parity.py 12 60 > $out/stress.log 2>&1; tail -1 $out/stress.log
sed 's#gpurun_out/r10aa#gpurun_out/r10ba#g' profiles/run_r10aa.sh > /tmp/inst.sh; bash /tmp/inst.sh | grep "blend\|preprocess\|total"
bash bench_tools/variant_ab.sh ";" "-DLMGS_BLEND_REC_BAND=0;" ";" "-DLMGS_BLEND_REC_BAND=0;" > $out/variants.txt 2>&1
cat $out/variants.txt
