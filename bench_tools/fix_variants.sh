#!/bin/bash
# usage (under gpurun): bash bench_tools/fix_variants.sh "<flags>" ...  (K7b variants)
for f in "$@"; do
  LMGS_NVCC_FLAGS="$f" python -c "from paper_2503_21364_b200 import build; build.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $f"; continue; }
  echo "== $f"
  ncu --metrics gpu__time_duration.sum -k regex:k_touched_fix --csv python bench_tools/fix_probe.py 2>/dev/null | grep k_touched | cut -d, -f15- | tr '\n' ' '; echo
  python bench.py --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1))"
done
