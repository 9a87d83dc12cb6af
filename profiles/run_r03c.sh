#!/bin/bash
# Round-3 closing measurement (under gpurun, repo root): bench line, launch
# list of the bench command, K7b full capture, c5 block bench at N=1.
set -x
out=gpurun_out/r03c; mkdir -p $out
python -m pytest tests -q -m gpu > $out/pytest_gpu.log 2>&1
python bench.py > $out/bench.log 2>&1
tail -1 $out/bench.log > $out/bench.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $out/launches.csv python bench.py --steps 1 --warmup 1 --views 4 --e2e-steps 1 \
    --no-cpu-baseline > $out/launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_touched_fix -s 1 -c 1 \
    -o $out/k_touched_fix -f python profiles/view_probe.py 1 > $out/k_touched_fix.log 2>&1
python bench_configs.py --configs c2,c4,bw --out $out/configs.jsonl > $out/configs.log 2>&1
