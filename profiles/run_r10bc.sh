#!/bin/bash
out=gpurun_out/r10bc; mkdir -p $out
timeout 120 python bench.py --gpus 2 --steps 2 --warmup 1 > $out/gpus2.log 2>&1; echo "rc=$?"; tail -3 $out/gpus2.log
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > $out/ref.log 2>&1; echo "rc=$?"; tail -1 $out/ref.log | cut -c1-300
