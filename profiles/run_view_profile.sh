#!/bin/bash
# usage (under gpurun): bash profiles/run_view_profile.sh <tag> [regex:skip:count ...]
# Stage times of 4 views, a launch list (time + DRAM bytes) of one view rendered
# twice, then a full ncu capture of the named kernels from the second render.
tag=${1:-prof}; shift
mkdir -p gpurun_out
python profiles/view_probe.py 4 > gpurun_out/${tag}_probe.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches.csv python profiles/view_probe.py 1 > /dev/null 2>&1
for spec in "$@"; do
  IFS=: read k s c <<< "$spec"
  ncu --set full --clock-control none --import-source on -k regex:$k -s ${s:-1} -c ${c:-1} \
      -o gpurun_out/${tag}_${k} -f python profiles/view_probe.py 1 > gpurun_out/${tag}_${k}.log 2>&1
done
