#!/bin/bash
# Re-entry check on a fresh box: GPU tests, smoke(), bench line.
set -x
out=gpurun_out/r04; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/gpu.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
timeout 300 python __graft_entry__.py > $out/smoke.log 2>&1
timeout 600 python bench.py > $out/bench.log 2>&1
tail -1 $out/bench.log > $out/bench.json
timeout 600 python bench.py --impl reference > $out/bench_ref.log 2>&1
