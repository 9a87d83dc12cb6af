"""Stall samples per CUDA source line from an ncu report (needs -lineinfo).
usage: python line_stalls.py report.ncu-rep [N] [file-substring]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
want = sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass,cuda"],
                     capture_output=True, text=True).stdout
agg, src, stalls = {}, {}, {}
fname, hdr, cur = "", None, None
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 5:
        continue
    if r[0] and r[0] != "-":
        try:
            cur = (fname, int(r[0]))
        except ValueError:
            continue
        src[cur] = r[1]
        continue
    if cur is None or r[2] in ("...", "-"):
        continue
    try:
        v = int(r[4] or 0)
    except ValueError:
        continue
    agg[cur] = agg.get(cur, 0) + v
    st = stalls.setdefault(cur, {})
    for i, name in enumerate(hdr):
        if name.startswith("stall_") and "Not Issued" not in name and i < len(r):
            try:
                st[name[6:]] = st.get(name[6:], 0) + int(r[i] or 0)
            except ValueError:
                pass
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:n]:
    if want and want not in k[0]:
        continue
    top = sorted(stalls.get(k, {}).items(), key=lambda x: -x[1])[:2]
    tops = " ".join(f"{a}:{100 * b / v:.0f}%" for a, b in top if v)
    print(f"{100 * v / tot:5.1f}% {k[0]}:{k[1]:<4d} [{tops:28s}] {src[k].strip()[:80]}")
