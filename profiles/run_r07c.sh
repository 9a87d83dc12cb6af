#!/bin/bash
# tile-sort variants: timings + per-pass ncu launch lists
out=gpurun_out/r07c; mkdir -p $out
B=bench_tools/sweep_bin
{
for v in pk4 pk3 nopk; do
  for args in "20700000 8160" "20700000 32400" "1000 8160" "4097 257"; do
    echo -n "$v: "; timeout 60 $B/tsb_$v $args
  done
done
} > $out/tile_sort.txt 2>&1
for v in pk4 pk3 nopk; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $out/launches_$v.csv $B/tsb_$v 20700000 8160 > /dev/null 2>&1
python profiles/launch_table.py $out/launches_$v.csv > $out/launch_table_$v.txt 2>&1
done
