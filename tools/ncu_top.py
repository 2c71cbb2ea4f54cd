"""Summarise an ncu report: headline metrics + top source lines by
instructions executed and by stall samples.  Usage: ncu_top.py REP [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
want = ("Duration", "Executed Ipc Active", "Issued Instructions", "Achieved Active Warps Per SM",
        "Theoretical Active Warps per SM", "No Eligible", "Avg. Active Threads Per Warp",
        "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Block Size", "Grid Size", "Compute (SM) Throughput",
        "Warp Cycles Per Issued Instruction", "Branch Efficiency")
rows = list(csv.reader(io.StringIO(det)))
h = rows[0]
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in want:
        print(f"{d.get('Kernel Name','')[:40]:40s} {d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = []
fname = None
for r in csv.reader(io.StringIO(src)):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] in ("Line No", "Function Name") or r[0] == "":
        continue
    try:
        agg.append((fname, int(r[0]), r[1][:80], int(r[4]), int(r[7])))
    except ValueError:
        pass
ts = sum(a[3] for a in agg) or 1
ti = sum(a[4] for a in agg) or 1
print(f"samples {ts} warp-instructions {ti}")
for a in sorted(agg, key=lambda x: -x[4])[:n]:
    print(f"{a[0]}:{a[1]:4d} inst {100*a[4]/ti:5.1f}% samp {100*a[3]/ts:5.1f}%  {a[2]}")
