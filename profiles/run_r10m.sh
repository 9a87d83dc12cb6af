#!/bin/bash
out=gpurun_out/r10m; mkdir -p $out
LMGS_NVCC_FLAGS="-DLMGS_SORT_TRACE=2" python -c "from paper_2503_21364_b200 import build; build.build(force=True)" > /dev/null 2>&1
python bench_tools/sort_trace.py 0 > $out/trace.txt 2>&1
python bench_tools/sort_trace.py 1 >> $out/trace.txt 2>&1
LMGS_NVCC_FLAGS="-DLMGS_SORT_TRACE=1" python -c "from paper_2503_21364_b200 import build; build.build(force=True)" > /dev/null 2>&1
echo "== pass index 0 (tile sort's first pass; depth pass 0 overwritten)" >> $out/trace.txt
python bench_tools/sort_trace.py 0 >> $out/trace.txt 2>&1
python -c "from paper_2503_21364_b200 import build; build.build(force=True)" > /dev/null 2>&1
cat $out/trace.txt
