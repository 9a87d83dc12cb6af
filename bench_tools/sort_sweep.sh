#!/bin/bash
# Build onesweep variants here (nvcc cross-compiles), run them on the GPU box:
#   bench_tools/sort_sweep.sh build   -> bench_tools/sweep_bin/sb_<tag>
#   bench_tools/sort_sweep.sh run     (on the box) -> gpurun_out/sortsweep.txt
# variants: "tag|flags"
cd "$(dirname "$0")"
VARIANTS=(
 "base|"
 "stream|-DLMGS_SORT_STREAMING"
 "i8c3|-DLMGS_SORT_ITEMS=8 -DLMGS_SORT_MIN_CTAS=3"
 "i8c4|-DLMGS_SORT_ITEMS=8 -DLMGS_SORT_MIN_CTAS=4"
 "i8c5|-DLMGS_SORT_ITEMS=8 -DLMGS_SORT_MIN_CTAS=5"
 "i12c3|-DLMGS_SORT_ITEMS=12 -DLMGS_SORT_MIN_CTAS=3"
 "i16c2|-DLMGS_SORT_ITEMS=16 -DLMGS_SORT_MIN_CTAS=2"
 "w16|-DLMGS_LOOK_WINDOW=16"
 "w4|-DLMGS_LOOK_WINDOW=4"
 "copy|-DLMGS_DBG_COPY"
 "i8c4s|-DLMGS_SORT_ITEMS=8 -DLMGS_SORT_MIN_CTAS=4 -DLMGS_SORT_STREAMING"
)
if [ "$1" = build ]; then
  mkdir -p sweep_bin
  for v in "${VARIANTS[@]}"; do
    tag=${v%%|*}; fl=${v#*|}
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 $fl -I../include sort_bench.cu \
      -o sweep_bin/sb_$tag 2>/dev/null || echo "build $tag failed" &
  done
  wait
  exit 0
fi
out=../gpurun_out/sortsweep.txt; : > $out
for v in "${VARIANTS[@]}"; do
  tag=${v%%|*}
  echo "== $tag" >> $out
  ./sweep_bin/sb_$tag 20700000 8 2 0 >> $out 2>&1
  ./sweep_bin/sb_$tag 6000000 4 3 1 >> $out 2>&1
done
cat $out
