#!/bin/bash
# tile sort with narrowing keys: stand-alone checks + timings, GPU suite, bench
out=gpurun_out/r07b; mkdir -p $out
B=bench_tools/sweep_bin
{
for args in "20700000 8160" "20700000 32400" "20700000 8160 29" "1000 8160" "5000 300" "100000 200" \
            "3000000 70000" "1 1" "7 2" "4097 257" "20700000 8160 32"; do
  timeout 60 $B/tile_sort_bench $args
done
timeout 60 $B/sort_bench 20700000 8 2
timeout 60 $B/sort_bench 6000000 4 3 1
} > $out/tile_sort.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $out/pytest_gpu.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-c5 > $out/bench.log 2>&1
tail -1 $out/bench.log > $out/bench.json
