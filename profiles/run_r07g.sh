#!/bin/bash
# full ncu captures (source-level) of the current kernels in the c3 pipeline
out=gpurun_out/r07g; mkdir -p $out
for ks in "k_blend16w 2" "k_emit 2" "k_touched_fix 2" "k_depth_fixup 2"; do
  set -- $ks
  ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o $out/$1 -f \
      python profiles/view_probe.py 2 > $out/ncu_$1.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_preprocess_tma -s 1 -c 1 -o $out/k_preprocess_tma2 -f \
    python profiles/view_probe.py 2 1920 1080 2 > $out/ncu_k1.log 2>&1
