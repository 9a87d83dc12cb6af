#!/bin/bash
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DLMGS_SORT_CHAINS=1 -I../include sort_bench.cu -o /tmp/sbp
ncu --set full --clock-control none --import-source on -k regex:k_onesweep -s 2 -c 1 -o ../gpurun_out/sortprof -f /tmp/sbp 20900000 8 2 0 > ../gpurun_out/sortprof.log 2>&1
