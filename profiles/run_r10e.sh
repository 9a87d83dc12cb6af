#!/bin/bash
# ncu captures of the fused tile sort kernels (fine warp sampling)
out=gpurun_out/r10e; mkdir -p $out
for ks in "long, .int.2" "int, .int.1, .int.0" "k_tile_plan" "k_rank_write" "k_rank_sums"; do
  nm=$(echo "$ks" | tr -c 'a-z0-9\n' '_')
  timeout 300 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on --kernel-name-base demangled -k "regex:$ks" -s 1 -c 1 -o $out/$nm -f \
      python profiles/view_probe.py 2 > $out/ncu_$nm.log 2>&1
  python profiles/ncu_summary.py $out/$nm.ncu-rep > $out/${nm}_summary.txt 2>&1
  head -12 $out/${nm}_summary.txt
done
