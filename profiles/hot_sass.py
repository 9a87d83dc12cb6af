"""Summarise an `ncu --page source --csv --print-source sass` dump: top SASS
lines by stall samples (usage: python hot_sass.py dump.csv [N])."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
si = h.index("Warp Stall Sampling (All Samples)")
src = h.index("Source")
addr = h.index("Address")
data = []
for r in rows[2:]:
    if len(r) <= si:
        continue
    try:
        v = int(r[si] or 0)
    except ValueError:
        continue
    data.append((v, r[addr], r[src]))
tot = sum(d[0] for d in data) or 1
for v, a, s in sorted(data, reverse=True)[:n]:
    print(f"{100 * v / tot:5.1f}%  {a}  {s[:110]}")
