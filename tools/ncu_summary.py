"""Summarise ncu captures into profiles/ (run in the build container).

    python tools/ncu_summary.py <launches.csv> <capture.ncu-rep> [<other.ncu-rep> ...] --tag r02
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
       "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "launch__grid_size",
       "launch__block_size", "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
       "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
       "l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum",
       "lts__t_sectors_srcunit_tex_op_read.sum", "local_load_bytes", "local_store_bytes"]


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
    """Per captured launch: the WANT rows of the details page and the RAW
    metrics (one dict per launch, in capture order)."""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    per = defaultdict(dict)
    for r in rows[1:]:
        row = dict(zip(h, r))
        key = row.get("ID", "0")
        if row.get("Metric Name") in WANT:
            per[key][row["Metric Name"]] = f'{row["Metric Value"]} {row["Metric Unit"]}'.strip()
            per[key]["kernel"] = row.get("Kernel Name", "")[:120]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    out = []
    if len(rr) > 2:
        h, units = rr[0], rr[1]
        for vals in rr[2:]:
            key = vals[h.index("ID")] if "ID" in h else str(len(out))
            d = dict(per.get(key, {}))
            for name in RAW:
                if name in h:
                    i = h.index(name)
                    d[name] = f"{vals[i]} {units[i]}".strip()
            out.append(d)
    return out


def to_bytes(s):
    v, u = s.split()[0].replace(",", ""), (s.split() + [""])[1]
    mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return float(v) * mul.get(u, 1.0)


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    tag = sys.argv[sys.argv.index("--tag") + 1] if "--tag" in sys.argv else "r02"
    args = [a for a in args if a != tag]
    summary = {"launches": launches(args[0]), "captures": {}}
    for rep in args[1:]:
        summary["captures"][os.path.basename(rep)] = details(rep)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps(summary, indent=1)[:8000])


if __name__ == "__main__":
    main()
