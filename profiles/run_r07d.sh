#!/bin/bash
# onesweep ranking variants (m0 current, m1 MATCH.ANY, m2gR pipelined R items)
out=gpurun_out/r07d; mkdir -p $out
B=bench_tools/sweep_bin
{
for v in m0 m1 m2g2 m2g4 m0n3; do
  for rep in 1 2; do
  echo -n "$v: "; timeout 60 $B/tsb_$v 20700000 8160
  echo -n "$v: "; timeout 60 $B/tsb_$v 20700000 32400
  echo -n "$v: "; timeout 60 $B/sb_$v 6000000 4 3 1
  echo -n "$v: "; timeout 60 $B/sb_$v 20700000 8 2
  done
done
} > $out/rank_variants.txt 2>&1
