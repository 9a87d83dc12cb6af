"""Per-kernel duration table from an ncu --csv gpu__time_duration launch list.
usage: python launch_table.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
mi = h.index("Metric Name") if "Metric Name" in h else None
dram = collections.defaultdict(float)
seq = []
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    if mi is not None and r[mi] != "gpu__time_duration.sum":
        if r[mi].startswith("dram__bytes"):
            dram[r[ki].split("(")[0].replace("lmgs::<unnamed>::", "")[:48]] += float(
                r[vi].replace(",", ""))
        continue
    v = float(r[vi].replace(",", ""))
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
          "ms": 1e3}.get(r[ui], 1.0)
    seq.append((r[ki].split("(")[0].replace("lmgs::<unnamed>::", "")[:48], v))
agg = collections.OrderedDict()
for n, v in seq:
    agg.setdefault(n, []).append(v)
print(f"{'kernel':50s} {'n':>4s} {'mean_us':>9s} {'min_us':>9s} {'max_us':>9s} {'MB/launch':>10s}")
for k, v in agg.items():
    mb = dram.get(k, 0.0) / len(v) / 1e6
    print(f"{k:50s} {len(v):4d} {sum(v)/len(v):9.1f} {min(v):9.1f} {max(v):9.1f} {mb:10.1f}")
if len(sys.argv) > 2:
    for n, v in seq:
        print(f"  {n:50s} {v:9.1f}")
