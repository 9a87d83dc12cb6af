#!/bin/bash
# onesweep cost breakdown on the tile-sort shape (20.7M u64 keys, 2 passes):
# full, copy-only (load + store, no ranking), no look-back
cd "$(dirname "$0")"
for fl in "" "-DLMGS_DBG_COPY" "-DLMGS_DBG_NO_LOOKBACK"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 $fl -I../include sort_bench.cu -o /tmp/sbp 2>&1 | grep -i error
  echo "== $fl"; /tmp/sbp 20700000 8 2 0; /tmp/sbp 6000000 4 3 1
done
