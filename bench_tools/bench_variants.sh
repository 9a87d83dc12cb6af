#!/bin/bash
# usage (under gpurun): bash bench_tools/bench_variants.sh "<flags>" ...  (bench value per build)
for f in "$@"; do
  LMGS_NVCC_FLAGS="$f" python -c "from paper_2503_21364_b200 import build; build.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $f"; continue; }
  v=$(python bench.py --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1))")
  echo "== $f : $v fps"
done
