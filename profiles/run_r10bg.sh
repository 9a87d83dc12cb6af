#!/bin/bash
out=gpurun_out/r10bg; mkdir -p $out
bash bench_tools/variant_ab.sh ";" "-DLMGS_CARVEOUT=100;" "-DLMGS_CARVEOUT=75;" "-DLMGS_CARVEOUT=50;" "-DLMGS_CARVEOUT=25;" ";" > $out/variants.txt 2>&1
cat $out/variants.txt
