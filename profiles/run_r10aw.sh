#!/bin/bash
# the other configurations, the training step and streaming at the round-2 close
out=gpurun_out/r10aw; mkdir -p $out
timeout 1500 python bench_configs.py --configs c2,c4,c5,bw,stream,c5peer --out $out/configs.jsonl > $out/configs.log 2>&1
tail -3 $out/configs.log
cat $out/configs.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print({k: d[k] for k in list(d)[:6]})"
