"""Summarise a round's ncu evidence into profiles/.

    python tools/profile_report.py --tag r01 --launches gpurun_out/launches.csv \
        --full gpurun_out/prof_cfg2.ncu-rep [--bench gpurun_out/bench.log]

Writes profiles/<tag>_launches.csv (per-kernel/grid launch times, shares of
the bench process), profiles/<tag>_ncu_full.txt (key metrics of the top
kernel) and profiles/ncu_summary.json (dram bytes per launch, read by
bench.py for roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--tag", required=True)
ap.add_argument("--launches")
ap.add_argument("--full")
a = ap.parse_args()
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
summary = {"tag": a.tag}

if a.launches:
    rows = [r for r in csv.reader(open(a.launches)) if len(r) > 5]
    hdr = rows[0]
    agg = defaultdict(list)
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3}.get(d["Metric Unit"], 1e-3)
            agg[(d["Kernel Name"].split("(")[0], d["Grid Size"])].append(float(d["Metric Value"].replace(",", "")) * scale)
    total = sum(sum(v) for v in agg.values())
    out = os.path.join(ROOT, "profiles", f"{a.tag}_launches.csv")
    with open(out, "w") as f:
        f.write("kernel,grid,launches,mean_us,total_us,share_of_profiled_time\n")
        for (k, g), v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"\"{k}\",\"{g}\",{len(v)},{sum(v)/len(v):.2f},{sum(v):.1f},{sum(v)/total:.4f}\n")
    print(open(out).read())

if a.full:
    det = subprocess.run(["ncu", "-i", a.full, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", a.full, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    d = dict(zip(rr[0], rr[2] if len(rr) > 2 else rr[1]))
    def num(k):
        try:
            return float(d[k].replace(",", ""))
        except Exception:
            return None
    units = dict(zip(rr[0], rr[1])) if len(rr) > 2 else {}
    def bytes_of(k):
        v = num(k)
        u = units.get(k, "byte")
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        return None if v is None else v * mult
    rd, wr = bytes_of("dram__bytes_read.sum"), bytes_of("dram__bytes_write.sum")
    summary.update({
        "kernel": d.get("Kernel Name"),
        "duration_us": num("gpu__time_duration.sum") / 1e3 if units.get("gpu__time_duration.sum") == "nsecond" else num("gpu__time_duration.sum"),
        "dram_bytes_read": rd, "dram_bytes_write": wr,
        "dram_bytes_per_launch": (rd or 0) + (wr or 0),
        "sm_inst_executed": num("smsp__inst_executed.sum"),
        "ipc": num("sm__inst_executed.avg.per_cycle_active"),
        "issue_active_pct": num("sm__inst_issued.avg.pct_of_peak_sustained_active"),
        "pipe_fma_pct": num("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
        "pipe_alu_pct": num("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
        "pipe_xu_pct": num("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
        "registers": num("launch__registers_per_thread"),
        "occupancy_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "sm_mhz": num("smsp__cycles_elapsed.avg.per_second"),
    })
    keep = {"Duration", "Executed Ipc Active", "Issue Slots Busy", "Executed Instructions", "No Eligible",
            "Eligible Warps Per Scheduler", "Achieved Occupancy", "Registers Per Thread",
            "Dynamic Shared Memory Per Block", "Theoretical Occupancy", "Compute (SM) Throughput",
            "DRAM Throughput", "SM Frequency", "Grid Size", "Block Size", "Memory Throughput"}
    lines = [f"ncu --set full capture: {os.path.basename(a.full)} ({d.get('Kernel Name')})"]
    rdr = csv.reader(io.StringIO(det))
    h = next(rdr)
    for row in rdr:
        e = dict(zip(h, row))
        if e.get("Metric Name") in keep:
            lines.append(f"  {e['Metric Name']:40s} {e['Metric Value']} {e['Metric Unit']}")
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(k) for k in d
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    stalls = {k: v for k, v in stalls.items() if v}
    tot = sum(stalls.values()) or 1
    lines.append("  stall samples: " + ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in
                                                 sorted(stalls.items(), key=lambda kv: -kv[1])[:10]))
    for k in ("pipe_fma_pct", "pipe_alu_pct", "pipe_xu_pct", "dram_bytes_read", "dram_bytes_write"):
        lines.append(f"  {k:40s} {summary[k]}")
    out = os.path.join(ROOT, "profiles", f"{a.tag}_ncu_full.txt")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    with open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
