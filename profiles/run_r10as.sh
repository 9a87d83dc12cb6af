#!/bin/bash
out=gpurun_out/r10as; mkdir -p $out
bash bench_tools/variant_ab.sh ";" "-DLMGS_BLEND_MINB=5;" "-DLMGS_BLEND_MINB=3;" "-DLMGS_BLEND_MINB=5;" > $out/variants.txt 2>&1
cat $out/variants.txt
