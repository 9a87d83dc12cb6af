#!/bin/bash
# Round-2 session-2 start check of the committed tree: GPU tests, smoke,
# bench line (shared world covariance in grouped K1 is in this tree).
out=gpurun_out/r07a; mkdir -p $out
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $out/pytest_gpu.log 2>&1
timeout 300 python __graft_entry__.py > $out/smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $out/bench.log 2>&1
tail -1 $out/bench.log > $out/bench.json
