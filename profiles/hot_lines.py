"""Top CUDA source lines of an ncu report by warp-stall samples.
usage: python hot_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
data = []
fname = ""
h = None
for r in rows:
    if len(r) == 2 and r[0] == "File Name":
        fname = r[1].rsplit("/", 1)[-1]
        h = None
        continue
    if r and r[0] == "Line No" or (r and r[0] == "#"):
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        try:
            v = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        if v:
            data.append((v, f"{fname}:{d.get('Line No', d.get('#'))}", d.get("Source", "").strip()))
tot = sum(x[0] for x in data) or 1
for v, loc, s in sorted(data, reverse=True)[:n]:
    print(f"{100 * v / tot:5.1f}%  {loc:18s} {s[:100]}")
