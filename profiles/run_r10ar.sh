#!/bin/bash
out=gpurun_out/r10ar; mkdir -p $out
bash bench_tools/variant_ab.sh ";--group 1" ";--group 2" ";--group 3" ";--group 1 --streams 8" > $out/variants.txt 2>&1
cat $out/variants.txt
