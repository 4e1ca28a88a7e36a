"""Key metrics and stall breakdown from an ncu --page raw --csv export: python tools/ncu_raw_summary.py f.csv"""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "sm__inst_executed.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__maximum_warps_per_active_cycle_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]


def main(path):
    rows = list(csv.reader(open(path)))
    h, units, vals = rows[0], rows[1], rows[2]
    print(vals[h.index("Kernel Name")][:90] if "Kernel Name" in h else path)
    for i, k in enumerate(h):
        if k in KEYS:
            print(f"  {k:70s} {units[i]:10s} {vals[i]}")
    st = []
    for i, k in enumerate(h):
        if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
            try:
                st.append((float(vals[i].replace(",", "")), k.split("stalled_")[-1]))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    print("  stalls: " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(st, reverse=True)[:8]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
