"""Summarise an ncu report (details page) into a compact text table: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Executed Instructions", "Dynamic Shared Memory Per Block", "Grid Size",
        "Block Size", "One or More Eligible", "No Eligible", "Active Warps Per Scheduler", "Eligible Warps Per Scheduler"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    idi = h.index("ID")
    cur = None
    for r in rows[1:]:
        if r[idi] != cur:
            cur = r[idi]
            print(f"== launch {cur}: {r[ki][:110]}")
        if r[mi] in KEYS:
            print(f"   {r[mi]:40s} {r[vi]:>16s} {r[ui]}")


if __name__ == "__main__":
    main(sys.argv[1])
