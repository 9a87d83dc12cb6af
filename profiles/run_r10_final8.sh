#!/bin/bash
# Round-2 closing measurement set (session r10, eighth pass) (run under gpurun from the repo root): GPU tests,
# smoke, bench line, the reference arm, ncu launch list of a short bench
# (time + DRAM bytes per launch), full ncu captures of the top kernels.
set -x
out=gpurun_out/r10final8; mkdir -p $out
python -m pytest tests -q -m gpu -p no:cacheprovider > $out/pytest_gpu.log 2>&1
python __graft_entry__.py > $out/smoke.log 2>&1
python bench.py --steps 20 --warmup 5 > $out/bench.log 2>&1
tail -1 $out/bench.log > $out/bench.json
python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_ref.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $out/launches.csv python bench.py --steps 1 --warmup 1 --views 4 --e2e-steps 1 \
    --no-cpu-baseline --no-c5 > $out/launches.log 2>&1
python profiles/launch_table.py $out/launches.csv > $out/ncu_launch_table.txt
# view_probe renders views one at a time (k_preprocess_tma<1>); per view the
# launch order is 3 u32 onesweep passes then 2 u64 ones, so -s 3 picks the
# first tile-sort pass of view 0
for ks in "k_blend16w 2" "k_preprocess_tma 2" "k_onesweep 3" "k_emit 2" "k_touched_fix 2" \
          "k_depth_fixup_w 2"; do
  set -- $ks
  ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o $out/$1 -f \
      python profiles/view_probe.py 2 > $out/ncu_$1.log 2>&1
  python profiles/ncu_summary.py $out/$1.ncu-rep > $out/${1}_summary.txt 2>&1
done
