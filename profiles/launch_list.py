"""Print an ncu launch-list CSV (time + DRAM bytes per launch).
usage: python launch_list.py launches.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
by = {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        e = by.setdefault(int(d["ID"]), {"name": d["Kernel Name"]})
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
print(f"{'id':>3} {'kernel':58s} {'us':>9} {'rd MB':>8} {'wr MB':>8} {'GB/s':>7}")
for i, e in sorted(by.items()):
    t = e.get("gpu__time_duration.sum", 0) / 1e3
    rd = e.get("dram__bytes_read.sum", 0) / 1e6
    wr = e.get("dram__bytes_write.sum", 0) / 1e6
    name = e["name"].replace("lmgs::<unnamed>::", "").replace("(anonymous namespace)::", "")
    print(f"{i:3d} {name[:58]:58s} {t:9.1f} {rd:8.1f} {wr:8.1f} {(rd + wr) / t * 1e3 if t else 0:7.0f}")
