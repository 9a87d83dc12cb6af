#!/bin/bash
# combined {count, match} ranking: full GPU suite, bench fused / unfused, launch list
out=gpurun_out/r10h; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_pipeline.py -q -x -p no:cacheprovider > $out/pytest_gpu.log 2>&1
tail -3 $out/pytest_gpu.log
for fl in 0 32 0 32; do
timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-c5 --flags $fl > $out/bench_$fl.log 2>&1
tail -1 $out/bench_$fl.log | python -c "import json,sys; d=json.load(sys.stdin); print('flags=$fl', round(d['value'],1), round(d['e2e']['value'],1), {k: round(v,4) for k,v in d['roofline']['stage_ms_per_frame'].items()})"
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $out/launches.csv python profiles/view_probe.py 1 > /dev/null 2>&1
python profiles/launch_table.py $out/launches.csv > $out/launch_table.txt 2>&1
cat $out/launch_table.txt | grep -v "at::"
