#!/bin/bash
# k_depth_fixup keys per thread (LMGS_FIXUP_PER): time per launch and bench
out=gpurun_out/fixper; mkdir -p $out
for per in 4 8 2; do
  LMGS_NVCC_FLAGS="-DLMGS_FIXUP_PER=$per" python -c "from paper_2503_21364_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  [ $per = 8 ] && timeout 300 python -m pytest tests/test_gpu_parity.py -q -x > $out/pytest_8.log 2>&1
  timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $out/b.log 2>&1
  tail -1 $out/b.log | python -c "import json,sys; d=json.load(sys.stdin); print('per=$per', round(d['value'],1), {k: round(v,4) for k,v in d['roofline']['stage_ms_per_frame'].items()})" >> $out/summary.txt
  ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_depth_fixup \
      --log-file $out/l_$per.csv python profiles/view_probe.py 1 > /dev/null 2>&1
  python profiles/launch_table.py $out/l_$per.csv | grep fixup | sed "s/^/per=$per /" >> $out/summary.txt
done
python -c "from paper_2503_21364_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
