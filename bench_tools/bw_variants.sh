#!/bin/bash
# usage (under gpurun): bash bench_tools/bw_variants.sh "<flags1>" "<flags2>" ...
# Rebuilds liblmgs with each flag set and times the backward (bench_configs bw).
for f in "$@"; do
  LMGS_NVCC_FLAGS="$f" python -c "from paper_2503_21364_b200 import build; build.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $f"; continue; }
  echo "== $f"
  python bench_configs.py --configs bw --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('ms_per_view_train','ms_forward_view0','ms_backward_view0')})"
done
