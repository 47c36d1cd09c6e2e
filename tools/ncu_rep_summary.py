"""Key metrics + top source lines of one kernel in an ncu --set full report."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            print(f"{k} {units[i]} {vals[i]}")
    stalls = [(h, v) for h, v in zip(hdr, vals) if h.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not h.endswith("_not_issued")]
    tot = sum(float(v or 0) for _, v in stalls) or 1
    print("## warp stall samples (share)")
    for h, v in sorted(stalls, key=lambda x: -float(x[1] or 0))[:10]:
        print(f"  {h.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * float(v or 0) / tot:.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
