#!/bin/bash
# shared-divisor fp64 division in K1: parity + bench
set -x
out=gpurun_out/r06; mkdir -p $out
timeout 900 python -m pytest tests -q -m gpu -x > $out/pytest_gpu.log 2>&1
timeout 300 python bench_tools/stress_parity.py 7 200 > $out/stress.log 2>&1
for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $out/bench_$i.log 2>&1; done
