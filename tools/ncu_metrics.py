"""Print the headline counters of an `ncu --page raw --csv` export (one
column per launch): duration, DRAM throughput / bytes, occupancy, warp
stall mix, tensor-pipe activity.

Usage: python tools/ncu_metrics.py gpurun_out/full_<tag>.csv.gz [more metric substrings]"""

import csv
import gzip
import io
import sys

KEYS = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__registers_per_thread", "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed"]


def main():
    path = sys.argv[1]
    extra = sys.argv[2:]
    raw = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
    rows = list(csv.reader(io.StringIO(raw.read())))
    head, units, data = rows[0], rows[1], rows[2:]
    for k in KEYS + [h for h in head if any(e in h for e in extra)]:
        if k not in head:
            continue
        i = head.index(k)
        vals = [r[i] for r in data]
        name = k if len(k) < 70 else k[:67] + "..."
        print(f"{name:72s} {units[i]:>10s}  " + " | ".join(v[:40] for v in vals))


if __name__ == "__main__":
    main()
