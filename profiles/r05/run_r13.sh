#!/bin/bash
# per-view scalars reset by one kernel
out=gpurun_out/r13; mkdir -p $out
timeout 900 python -m pytest tests -q -m gpu -x > $out/pytest_gpu.log 2>&1
timeout 300 python bench_tools/stress_parity.py 29 120 > $out/stress.log 2>&1
for rep in 1 2 3; do
  timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $out/b.log 2>&1
  tail -1 $out/b.log | python -c "import json,sys; d=json.load(sys.stdin); print('reset_kernel', round(d['value'],1), {k: round(v,4) for k,v in d['roofline']['stage_ms_per_frame'].items()})" >> $out/summary.txt
done
