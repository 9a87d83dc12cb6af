#!/bin/bash
# Round-3 measurement set (run under gpurun from the repo root): GPU tests,
# bench line, ncu launch list of the bench command, the other configurations
# (c2, c4, c5, training step, streaming), full ncu capture of k_backward.
set -x
out=gpurun_out/r03; mkdir -p $out
python -m pytest tests -q -m gpu > $out/pytest_gpu.log 2>&1
python bench.py > $out/bench.log 2>&1
tail -1 $out/bench.log > $out/bench.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $out/launches.csv python bench.py --steps 1 --warmup 1 --views 4 --e2e-steps 1 \
    --no-cpu-baseline > $out/launches.log 2>&1
python bench_configs.py --configs c2,c4,bw,stream,c5 --out $out/configs.jsonl > $out/configs.log 2>&1
