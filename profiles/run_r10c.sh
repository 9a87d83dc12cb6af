#!/bin/bash
# fused emission + tile sort, second cut: A/B tests, bench stage times, launch list, ncu of the passes
out=gpurun_out/r10c; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_pipeline.py -q -x -p no:cacheprovider > $out/pytest_fused.log 2>&1
tail -3 $out/pytest_fused.log
timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-c5 > $out/bench.log 2>&1
tail -1 $out/bench.log | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['value'],1), d['e2e']['value'], {k: round(v,4) for k,v in d['roofline']['stage_ms_per_frame'].items()})"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $out/launches.csv python profiles/view_probe.py 1 > /dev/null 2>&1
python profiles/launch_table.py $out/launches.csv > $out/launch_table.txt 2>&1
cat $out/launch_table.txt | grep -v "at::"
for ks in "unsigned long, 2" "unsigned int, 1, 0" "k_rank_scan" "k_tile_plan"; do
  nm=$(echo "$ks" | tr -c 'a-z0-9\n' '_')
  timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$ks" -s 1 -c 1 -o $out/$nm -f \
      python profiles/view_probe.py 2 > $out/ncu_$nm.log 2>&1
  python profiles/ncu_summary.py $out/$nm.ncu-rep > $out/${nm}_summary.txt 2>&1
  head -30 $out/${nm}_summary.txt
done
