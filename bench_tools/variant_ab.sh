#!/bin/bash
# usage (under gpurun): bash bench_tools/variant_ab.sh "<nvcc flags>;<bench.py flags>" ...
# Rebuild liblmgs with each nvcc flag set (LMGS_NVCC_FLAGS) and print one
# 10-step bench line (frames/s, e2e, per-stage ms) per variant.
for v in "$@"; do
  f="${v%%;*}"; b="${v#*;}"; [ "$b" = "$v" ] && b=""
  LMGS_NVCC_FLAGS="$f" python -c "from paper_2503_21364_b200 import build; build.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $f"; continue; }
  python bench.py --steps 10 --warmup 3 --no-c5 --no-cpu-baseline --e2e-steps 1 $b 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('[$f | $b]', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'lat', round(d['latency_ms_single_view']['ms'],3), {k: round(x,4) for k,x in d['roofline']['stage_ms_per_frame'].items()})"
done
python -c "from paper_2503_21364_b200 import build; build.build(force=True)" > /dev/null 2>&1
