#!/bin/bash
# Grouped-view K1 (lmgs_render_group): bench at group 1/2/4/8 with the default
# build, then rebuilds with other LMGS_PRE_MULTI_MIN_CTAS values.  Run under
# gpurun from the repo root.
out=gpurun_out/group; mkdir -p $out
for mc in 5 4 6; do
  if [ $mc != 5 ]; then
    LMGS_NVCC_FLAGS="-DLMGS_PRE_MULTI_MIN_CTAS=$mc" python -c "from paper_2503_21364_b200 import build as b; b.build(force=True)" > $out/build_$mc.log 2>&1
  fi
  for g in 1 2 4 8; do
    [ $mc != 5 ] && [ $g = 1 ] && continue
    timeout 300 python bench.py --group $g --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $out/b_mc${mc}_g${g}.log 2>&1
    tail -1 $out/b_mc${mc}_g${g}.log | python -c "import json,sys; d=json.load(sys.stdin); print('mc=$mc g=$g', round(d['value'],1), {k: round(v,4) for k,v in d['roofline']['stage_ms_per_frame'].items()})" >> $out/summary.txt
  done
done
python -c "from paper_2503_21364_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
