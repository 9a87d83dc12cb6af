#!/bin/bash
# Concurrency sweep: contexts/streams the view batch alternates over x views
# per K1 launch.  Run under gpurun from the repo root.
out=gpurun_out/streams; mkdir -p $out
for s in 2 3 4 6; do
  for g in 1 2; do
    timeout 300 python bench.py --streams $s --group $g --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $out/b_s${s}_g${g}.log 2>&1
    tail -1 $out/b_s${s}_g${g}.log | python -c "import json,sys; d=json.load(sys.stdin); print('streams=$s group=$g', round(d['value'],1))" >> $out/summary.txt
  done
done
