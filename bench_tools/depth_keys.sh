#!/bin/bash
# k_depth_keys: keys per thread per step x CTAs per SM (kernel time from ncu)
out=gpurun_out/dk; mkdir -p $out
for v in "4 8" "8 8" "4 16" "8 4"; do
  set -- $v
  LMGS_NVCC_FLAGS="-DLMGS_DEPTH_KEYS_U=$1 -DLMGS_DEPTH_KEYS_CTAS_PER_SM=$2" python -c "from paper_2503_21364_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_depth_keys \
      --log-file $out/l.csv python profiles/view_probe.py 1 > /dev/null 2>&1
  python profiles/launch_table.py $out/l.csv | grep depth_keys | sed "s/^/U=$1 ctas=$2 /" >> $out/summary.txt
done
python -c "from paper_2503_21364_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
