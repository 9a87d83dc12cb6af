#!/bin/bash
# full ncu captures of the onesweep passes (m2g2 build) for source-level stalls
out=gpurun_out/r07e; mkdir -p $out
B=bench_tools/sweep_bin
ncu --set full --clock-control none --import-source on -k regex:k_onesweep -s 4 -c 2 -o $out/tsb -f $B/tsb_m2g2 20700000 8160 > $out/tsb.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_onesweep -s 4 -c 1 -o $out/sb -f $B/sb_m2g2 6000000 4 3 1 > $out/sb.log 2>&1
