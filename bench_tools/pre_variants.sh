#!/bin/bash
# rebuild liblmgs with each flag set and print the per-stage times of 4 c3 views
while read -r fl; do
  LMGS_NVCC_FLAGS="$fl" python -m paper_2503_21364_b200.build --force > /dev/null 2>&1 || { echo "build failed: $fl"; continue; }
  echo "== $fl"; python profiles/view_probe.py 4 2>&1 | tail -1 | cut -c1-120
done
