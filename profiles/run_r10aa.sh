#!/bin/bash
# warp instructions and time per kernel of one serial c3 view (issue-slot budget of the batch)
out=gpurun_out/r10aa; mkdir -p $out
timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
    --log-file $out/inst.csv python profiles/view_probe.py 2 1920 1080 2 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/r10aa/inst.csv")))
h = None; agg = collections.OrderedDict()
for r in rows:
    if len(r) > 10 and r[0] == "ID": h = r; continue
    if not h or len(r) != len(h): continue
    d = dict(zip(h, r))
    k = d["Kernel Name"][:60]; m = d["Metric Name"]; v = float(d["Metric Value"].replace(",", ""))
    agg.setdefault(k, collections.defaultdict(list))[m].append(v)
tot = 0
for k, m in agg.items():
    inst = m["smsp__inst_executed.sum"]; t = m["gpu__time_duration.sum"]
    n = len(inst); s = sum(inst) / 1e6
    tot += s
    print(f"{k:60s} n={n:3d} Minst/launch={s/n:8.1f} us/launch={sum(t)/n/1e3 if max(t) > 1e4 else sum(t)/n:8.1f} issue%={sum(m['smsp__issue_active.avg.pct_of_peak_sustained_active'])/n:5.1f}")
print("total Minst", round(tot, 1))
PY
