#!/bin/bash
# usage (under gpurun): bash bench_tools/blend_variant.sh "<flags>" ...
# Rebuild with each flag set; touched mismatches at c2/c3/4K and stage times.
for f in "$@"; do
  LMGS_NVCC_FLAGS="$f" python -c "from paper_2503_21364_b200 import build; build.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $f"; continue; }
  echo "== $f"
  python -m pytest tests/test_gpu_parity.py -q -m gpu -s -k "c2_full or c3_view" 2>&1 | grep -i "touched_mism\|passed\|failed" | cut -c1-200
  PYTHONPATH=. python profiles/view_probe.py 4 | cut -c1-110
done
