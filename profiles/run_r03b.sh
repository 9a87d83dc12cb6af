#!/bin/bash
# Round-3 final measurement set (under gpurun, repo root): bench line, launch
# list of the bench command, full ncu captures of the top kernels on a warm c3
# view, the other configurations.
set -x
out=gpurun_out/r03b; mkdir -p $out
python bench.py > $out/bench.log 2>&1
tail -1 $out/bench.log > $out/bench.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $out/launches.csv python bench.py --steps 1 --warmup 1 --views 4 --e2e-steps 1 \
    --no-cpu-baseline > $out/launches.log 2>&1
for spec in k_blend16w:1:1 k_preprocess_tma:1:1 "k_onesweep<unsigned long:1:2" k_emit:1:1 k_touched_fix:1:1; do
  IFS=: read k s c <<< "$spec"
  name=$(echo "$k" | tr -c 'a-zA-Z0-9_\n' '_')
  ncu --set full --clock-control none --import-source on -k "regex:$k" -s $s -c $c \
      -o $out/$name -f python profiles/view_probe.py 1 > $out/$name.log 2>&1
done
python bench_configs.py --configs c2,c4,bw,stream,c5peer --out $out/configs.jsonl > $out/configs.log 2>&1
