"""Compact markdown summary of ncu --set full reports (one row per profiled
launch): duration, grid, registers, occupancy, issue-slot use, tensor-pipe
activity, DRAM throughput / bytes and the top warp-stall reasons.

Usage: python tools/ncu_summary.py label=report.ncu-rep [label=report.ncu-rep ...]"""

import csv
import io
import subprocess
import sys

M = {
    "dur_us": "gpu__time_duration.sum",
    "grid": "launch__grid_size",
    "regs": "launch__registers_per_thread",
    "occ_%": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_%": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "tensor_%": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "dram_%": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_rd_MB": "dram__bytes_read.sum",
    "dram_wr_MB": "dram__bytes_write.sum",
}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units = r[0], r[1]
    for row in r[2:]:
        yield dict(zip(h, row)), dict(zip(h, units))


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


def main():
    print("| launch | kernel | " + " | ".join(M) + " | top stalls |")
    print("|" + "---|" * (len(M) + 3))
    for arg in sys.argv[1:]:
        label, rep = arg.split("=", 1)
        for i, (d, u) in enumerate(rows(rep)):
            name = d.get("Kernel Name", "")[:48]
            vals = []
            for k, m in M.items():
                v = num(d.get(m, ""))
                if v is not None and k.endswith("_MB"):
                    unit = u.get(m, "")
                    v *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
                if v is not None and k == "dur_us":
                    v *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(u.get(m, ""), 1.0)
                vals.append("" if v is None else f"{v:.2f}" if v < 10 else f"{v:.1f}" if v < 1e5 else f"{v:.0f}")
            st = {k[33:]: num(v) for k, v in d.items()
                  if k.startswith("smsp__pcsamp_warps_issue_stalled") and
                  not k.endswith("not_issued") and num(v)}
            tot = sum(st.values()) or 1.0
            top = ", ".join(f"{k} {v / tot:.2f}" for k, v in
                            sorted(st.items(), key=lambda x: -x[1])[:3])
            print(f"| {label}#{i} | `{name}` | " + " | ".join(vals) + f" | {top} |")


if __name__ == "__main__":
    main()
