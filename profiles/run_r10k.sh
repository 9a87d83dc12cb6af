#!/bin/bash
# defaults after the ranking rewrite + persistent sort grids + 4 streams
out=gpurun_out/r10k; mkdir -p $out
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $out/pytest_gpu.log 2>&1
tail -3 $out/pytest_gpu.log
timeout 300 python __graft_entry__.py > $out/smoke.log 2>&1; tail -2 $out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > $out/bench.log 2>&1
tail -1 $out/bench.log > $out/bench.json
python -c "import json; d=json.load(open('$out/bench.json')); print(round(d['value'],1), d['e2e']['value'], d['latency_ms_single_view'], (d.get('c5') or {}).get('value'), d['roofline']['frame'])"
