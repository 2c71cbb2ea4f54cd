"""Summarise a round's ncu artefacts into profiles/<round>/.

    python tools/summarize_profiles.py r1

Reads gpurun_out/launches_<r>.csv (the `--metrics gpu__time_duration.sum`
launch list of one bench run) and gpurun_out/prof_<kernel>_<r>.ncu-rep (one
`--set full` capture per hot kernel), writes:
  profiles/<r>/launches_<r>.csv      the launch list (copied)
  profiles/<r>/kernel_metrics.csv    key metrics per captured kernel
  profiles/<r>/ncu_traffic.json      DRAM bytes per launch (bench.py roofline.traffic)
  profiles/<r>/SUMMARY.md            shares of the step + per-kernel table
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

R = sys.argv[1] if len(sys.argv) > 1 else "r1"
W = sys.argv[2] if len(sys.argv) > 2 else "c5"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out")
DST = os.path.join(ROOT, "profiles", R)
os.makedirs(DST, exist_ok=True)

METRICS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_B",
    "dram__bytes_write.sum": "dram_write_B",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_wavefronts_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    h, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(h, vals))
    u = dict(zip(h, units))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
             "second": 1e9, "s": 1e9}
    res = {"kernel": d.get("Kernel Name", "")}
    for k, name in METRICS.items():
        v = d.get(k)
        if v is not None:
            try:
                res[name] = float(v.replace(",", "")) * scale.get(u.get(k, ""), 1)
            except ValueError:
                res[name] = v
    return res


kernels = []
for f in sorted(os.listdir(SRC)):
    if f.startswith("prof_plz_") and f.endswith(f"_{R}.ncu-rep"):
        m = raw(os.path.join(SRC, f))
        if m:
            m["report"] = f
            kernels.append(m)
            shutil.copy(os.path.join(SRC, f), os.path.join(DST, f))

with open(os.path.join(DST, "kernel_metrics.csv"), "w", newline="") as fh:
    cols = ["kernel", "report"] + list(METRICS.values())
    w = csv.DictWriter(fh, fieldnames=cols, extrasaction="ignore")
    w.writeheader()
    for k in kernels:
        w.writerow(k)

traffic = {}
for k in kernels:
    name = k["kernel"].split("(")[0].split("::")[-1].split("<")[0].strip()
    if "dram_read_B" in k and "dram_write_B" in k:
        traffic[name] = {"dram_bytes_per_launch": k["dram_read_B"] + k["dram_write_B"],
                         "duration_ns_ncu": k.get("duration_ns"), "report": k["report"]}
with open(os.path.join(DST, "ncu_traffic.json"), "w") as fh:
    json.dump(traffic, fh, indent=1)

# launch list shares
shares = {}
launch_csv = os.path.join(SRC, f"launches_{R}.csv")
if os.path.exists(launch_csv):
    shutil.copy(launch_csv, os.path.join(DST, f"launches_{R}.csv"))
    text = open(launch_csv).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].split("::")[-1].split("<")[0].strip()
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        s = shares.setdefault(name, [0, 0.0])
        s[0] += 1
        s[1] += v

lines = [f"# Profiles — round {R}", "",
         "Produced by `tools/profile_round.sh " + R + "` on one B200 (gpurun) and summarised by",
         "`tools/summarize_profiles.py " + R + "`.  ncu times are cold-cache and serialised:",
         "compare SHARES, not absolute times, with bench.py's CUDA-event numbers.", ""]
if shares:
    tot = sum(v[1] for v in shares.values())
    lines += ["## Launch list (all kernels of `bench.py --steps 2 --warmup 1`)", "",
              "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for name, (n, t) in sorted(shares.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {name} | {n} | {t / 1e6:.3f} | {100 * t / tot:.1f} % |")
    lines.append("")
lines += [f"## Per-kernel (one `--set full` capture each, {W} workload)", "",
          "| kernel | dur µs | DRAM MB (r+w) | DRAM % | SM % | ALU pipe % | FMA pipe % | issue % | occ % | warp-instr |",
          "|---|---|---|---|---|---|---|---|---|---|"]
for k in kernels:
    name = k["kernel"].split("(")[0].split("::")[-1].strip()
    dram = (k.get("dram_read_B", 0) + k.get("dram_write_B", 0)) / 1e6
    lines.append(
        f"| {name} | {k.get('duration_ns', 0) / 1e3:.1f} | {dram:.1f} | "
        f"{k.get('dram_throughput_pct', 0):.1f} | {k.get('sm_throughput_pct', 0):.1f} | "
        f"{k.get('alu_pipe_pct', 0):.1f} | {k.get('fma_pipe_pct', 0):.1f} | "
        f"{k.get('issue_active_pct', 0):.1f} | {k.get('achieved_occupancy_pct', 0):.1f} | "
        f"{k.get('warp_instructions', 0):.3g} |")
with open(os.path.join(DST, "SUMMARY.md"), "w") as fh:
    fh.write("\n".join(lines) + "\n")
print("\n".join(lines))
