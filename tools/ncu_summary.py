"""Key metrics + top stall reasons from an ncu report (run here, no GPU needed)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "lts__t_bytes.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print(r[hdr.index("Kernel Name")][:60])
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"   {k:70s} {r[i]} {units[i]}")
        stalls = [(hdr[i], r[i]) for i in range(len(hdr))
                  if hdr[i].startswith("smsp__average_warp_latency_issue_stalled") and hdr[i].endswith(".ratio")]
        stalls = sorted(((float(v.replace(",", "")), k) for k, v in stalls if v), reverse=True)[:6]
        for v, k in stalls:
            print(f"   stall {k.replace('smsp__average_warp_latency_issue_stalled_', ''):50s} {v:.2f}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
