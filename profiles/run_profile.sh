#!/bin/bash
# Profile recipe (run under gpurun): launch list + full capture of the top kernels.
# usage: bash profiles/run_profile.sh <tag>
tag=${1:-prof}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
    --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 1 --warmup 1 --views 2 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${tag}_launches.log 2>&1
for k in k_blend k_onesweep k_preprocess; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 \
      -o gpurun_out/${tag}_$k -f \
      python bench.py --steps 1 --warmup 1 --views 2 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${tag}_$k.log 2>&1
done
