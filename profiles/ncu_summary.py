"""One-screen summary of an ncu report: duration, throughputs, occupancy,
DRAM bytes, top stall reasons.  usage: python ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
for row in rows[2:]:
    d = dict(zip(h, row))
    name = d.get("Kernel Name", "")[:70]
    print(f"== {name}  grid={d.get('Grid Size')} block={d.get('Block Size')}")

    def g(k):
        return d.get(k, "")

    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__occupancy_limit_registers",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "lts__t_bytes.sum", "l1tex__t_bytes.sum"]
    for k in keys:
        if k in d:
            print(f"  {k:60s} {g(k)}")
    st = []
    for k in h:
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st.append((float(d[k].replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    print("  stalls: " + ", ".join(f"{n} {100*v/tot:.0f}%" for v, n in sorted(st, reverse=True)[:7]))
