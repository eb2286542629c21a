"""Summarise ncu captures into profiles/ (run in the build container).

    python tools/ncu_summary.py <launches.csv> <pass.ncu-rep> [<other.ncu-rep> ...] --tag r01
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Registers Per Thread", "Achieved Occupancy", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "No Eligible",
        "Block Size", "Grid Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
       "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct",
       "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    out = [{"kernel": k, "launches": len(v), "total_us": sum(v), "avg_us": sum(v) / len(v),
            "share": sum(v) / tot} for k, v in agg.items()]
    return sorted(out, key=lambda d: -d["total_us"])


def details(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    d = {}
    for r in rows[1:]:
        row = dict(zip(h, r))
        if row.get("Metric Name") in WANT:
            d[row["Metric Name"]] = f'{row["Metric Value"]} {row["Metric Unit"]}'.strip()
            d["kernel"] = row.get("Kernel Name", "")[:120]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) > 2:
        h, units, vals = rr[0], rr[1], rr[2]
        for name in RAW:
            if name in h:
                i = h.index(name)
                d[name] = f"{vals[i]} {units[i]}".strip()
    return d


def to_bytes(s):
    v, u = s.split()[0].replace(",", ""), (s.split() + [""])[1]
    mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return float(v) * mul.get(u, 1.0)


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    tag = sys.argv[sys.argv.index("--tag") + 1] if "--tag" in sys.argv else "r01"
    points = int(sys.argv[sys.argv.index("--points") + 1]) if "--points" in sys.argv else 16000000
    args = [a for a in args if a not in (tag, str(points))]
    summary = {"launches": launches(args[0]), "kernels": {}}
    for rep in args[1:]:
        summary["kernels"][os.path.basename(rep)] = details(rep)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    p = summary["kernels"].get(os.path.basename(args[1]), {})
    if "dram__bytes_read.sum" in p:
        dram = to_bytes(p["dram__bytes_read.sum"]) + to_bytes(p["dram__bytes_write.sum"])
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w") as fh:
            json.dump({"rigid_pass": {"points": points, "dram_bytes": dram,
                                      "source": f"profiles/{tag}_ncu.json"}}, fh, indent=1)
    print(json.dumps(summary, indent=1)[:6000])


if __name__ == "__main__":
    main()
