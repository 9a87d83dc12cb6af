#!/bin/bash
# Round measurement set r05 (run under gpurun from the repo root): GPU tests,
# bench line (group 2), ncu launch list of the bench command (time + DRAM
# bytes), full ncu capture of K1 (grouped), the other configurations.
set -x
out=gpurun_out/r05; mkdir -p $out
python -m pytest tests -q -m gpu > $out/pytest_gpu.log 2>&1
python __graft_entry__.py > $out/smoke.log 2>&1
python bench.py > $out/bench.log 2>&1
tail -1 $out/bench.log > $out/bench.json
python bench.py --impl reference > $out/bench_ref.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $out/launches.csv python bench.py --steps 1 --warmup 1 --views 4 --e2e-steps 1 \
    --no-cpu-baseline > $out/launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_preprocess_tma -s 2 -c 1 \
    -o $out/k_preprocess_tma_g2 -f python bench.py --steps 1 --warmup 1 --views 4 --e2e-steps 1 \
    --no-cpu-baseline > $out/ncu_pre.log 2>&1
python bench_configs.py --configs c2,c4,c5 --out $out/configs.jsonl > $out/configs.log 2>&1
