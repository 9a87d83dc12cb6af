#!/bin/bash
# Session check of the committed tree: GPU tests, smoke, bench line.
out=gpurun_out/r10; mkdir -p $out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > $out/pytest_gpu.log 2>&1
timeout 300 python __graft_entry__.py > $out/smoke.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > $out/bench.log 2>&1
tail -1 $out/bench.log > $out/bench.json
tail -3 $out/pytest_gpu.log
tail -1 $out/bench.json | head -c 600
