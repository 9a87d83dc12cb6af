#!/bin/bash
out=gpurun_out/r10o; mkdir -p $out
for ks in "long, .int.1, .int.1"; do
  nm=$(echo "$ks" | tr -c 'a-z0-9\n' '_')
  timeout 300 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on --kernel-name-base demangled -k "regex:$ks" -s 1 -c 1 -o $out/$nm -f \
      python profiles/view_probe.py 2 > $out/ncu_$nm.log 2>&1
  python profiles/ncu_summary.py $out/$nm.ncu-rep > $out/${nm}_summary.txt 2>&1
  head -12 $out/${nm}_summary.txt
done
