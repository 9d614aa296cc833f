"""Summarise an ncu report (run locally): key throughput, memory and stall metrics."""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
    "lts__t_bytes.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sass__inst_executed_local_loads",
    "sass__inst_executed_local_stores", "smsp__inst_executed.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]


def main(path, kernel_filter=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")]
        if kernel_filter and kernel_filter not in name:
            continue
        print(f"== {name[:100]}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:70s} {vals[i]:>18s} {units[i]}")
        stalls = [(hdr[i], vals[i]) for i in range(len(hdr))
                  if hdr[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not hdr[i].endswith("not_issued")]
        tot = sum(float(v or 0) for _, v in stalls) or 1.0
        for h, v in sorted(stalls, key=lambda x: -float(x[1] or 0))[:8]:
            print(f"  stall {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):40s} {100 * float(v or 0) / tot:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
