#!/bin/bash
out=gpurun_out/r10bm; mkdir -p $out
bash bench_tools/variant_ab.sh ";" "-DLMGS_EMIT_PERSIST_CTAS=4;" "-DLMGS_EMIT_PERSIST_CTAS=3;" "-DLMGS_EMIT_PERSIST_CTAS=6;" ";" "-DLMGS_EMIT_PERSIST_CTAS=4;" "-DLMGS_EMIT_PERSIST_CTAS=2;" "-DLMGS_EMIT_PERSIST_CTAS=3;" > $out/variants.txt 2>&1
cat $out/variants.txt
