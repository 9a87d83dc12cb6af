#!/bin/bash
out=gpurun_out/r10bb; mkdir -p $out
for c in 1 2 3 1 2; do
  LMGS_E2E_COPY_STREAMS=$c timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 5 --no-cpu-baseline --no-c5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('copy streams $c', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
done
