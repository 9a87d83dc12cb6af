#!/bin/bash
# marginal cost of each stage in the overlapped batch (stage kernels dropped at build time)
out=gpurun_out/r10s; mkdir -p $out
bash bench_tools/variant_ab.sh ";" "-DLMGS_SKIP_STAGES=2;" "-DLMGS_SKIP_STAGES=4;" "-DLMGS_SKIP_STAGES=8;" "-DLMGS_SKIP_STAGES=16;" ";--flags 2" \
  "-DLMGS_SKIP_STAGES=30;--flags 2" "-DLMGS_SKIP_STAGES=14;" > $out/variants.txt 2>&1
cat $out/variants.txt
