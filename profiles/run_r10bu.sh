#!/bin/bash
out=gpurun_out/r10bu; mkdir -p $out
bash bench_tools/variant_ab.sh ";" "-DLMGS_SORT_PERSIST_CTAS_VALS=2;" "-DLMGS_SORT_PERSIST_CTAS_VALS=3;" ";" "-DLMGS_SORT_PERSIST_CTAS_VALS=2;" "-DLMGS_SORT_PERSIST_CTAS_VALS=3;" > $out/variants.txt 2>&1
cat $out/variants.txt
