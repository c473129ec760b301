"""Summarise an ncu report: key metrics per kernel + top stall lines.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--source]
"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Issue Slots Busy", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "L1/TEX Hit Rate", "L2 Hit Rate", "DRAM Throughput",
        "Compute (SM) Throughput", "Memory Throughput", "Executed Instructions"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    res = {}
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        res.setdefault((r[0], r[ki]), {})[r[mi]] = (r[vi], r[ui])
    return res


def raw(rep, metrics):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(metrics)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows


if __name__ == "__main__":
    rep = sys.argv[1]
    for (idx, k), m in details(rep).items():
        print(f"== [{idx}] {k[:90]}")
        for key in KEYS:
            if key in m:
                print(f"   {key:40s} {m[key][0]} {m[key][1]}")
    rows = raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                     "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                     "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"])
    for r in rows:
        print("   ", ",".join(x[:40] for x in r[:3] + r[-6:]))
