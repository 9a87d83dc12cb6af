#!/bin/bash
# usage (under gpurun): bash bench_tools/variant_bench.sh "<flags>" ...
# Rebuild liblmgs with each flag set (LMGS_NVCC_FLAGS), then per-stage times
# of 8 serial c3 views and a 10-step bench line (frames/s).
for f in "$@"; do
  LMGS_NVCC_FLAGS="$f" python -c "from paper_2503_21364_b200 import build; build.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $f"; continue; }
  echo "== [$f]"
  PYTHONPATH=. python profiles/view_probe.py 8 | cut -c1-150
  python bench.py --steps 10 --warmup 3 --no-c5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
done
python -c "from paper_2503_21364_b200 import build; build.build(force=True)" > /dev/null 2>&1
