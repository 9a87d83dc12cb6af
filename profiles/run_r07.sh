#!/bin/bash
# K1 counters by REDUX: parity + bench at group 1 / 2
out=gpurun_out/r07; mkdir -p $out
timeout 900 python -m pytest tests -q -m gpu -x > $out/pytest_gpu.log 2>&1
for g in 1 2; do
  timeout 300 python bench.py --group $g --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $out/b_g$g.log 2>&1
  tail -1 $out/b_g$g.log | python -c "import json,sys; d=json.load(sys.stdin); print('group=$g', round(d['value'],1), {k: round(v,4) for k,v in d['roofline']['stage_ms_per_frame'].items()})" >> $out/summary.txt
done
