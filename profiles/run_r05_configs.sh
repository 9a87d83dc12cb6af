#!/bin/bash
# r05 refresh of the remaining configurations (training step, streaming, c5 blocks) and a
# longer c3 bench (20 timed steps)
out=gpurun_out/r05c; mkdir -p $out
timeout 900 python bench_configs.py --configs bw,stream --out $out/configs.jsonl > $out/configs.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 --e2e-steps 5 > $out/bench_long.log 2>&1
tail -1 $out/bench_long.log > $out/bench_long.json
for ex in peer nccl; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench_blocks.py --exchange $ex > $out/blocks_$ex.log 2>&1; tail -1 $out/blocks_$ex.log >> $out/c5_blocks.jsonl; done
