#!/bin/bash
# Round-2 measurement set (run under gpurun from the repo root):
#   bench line, ncu launch list of the bench command (reduced views/steps),
#   full ncu captures of the top kernels on a warm c3 view.
set -x
out=gpurun_out/r02; mkdir -p $out
python bench.py > $out/bench.log 2>&1
tail -1 $out/bench.log > $out/bench.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $out/launches.csv python bench.py --steps 1 --warmup 1 --views 4 --e2e-steps 1 \
    --no-cpu-baseline > $out/launches.log 2>&1
for spec in k_blend16w:1:1 k_onesweep:3:5 k_preprocess_tma:1:1 k_emit:1:1 k_depth_fixup:1:1 k_depth_keys:1:1; do
  IFS=: read k s c <<< "$spec"
  ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $c \
      -o $out/$k -f python profiles/view_probe.py 1 > $out/$k.log 2>&1
done
