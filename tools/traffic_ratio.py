"""Match an ncu per-launch CSV (gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum; --cache-control none) of tools/profile_traffic.py
against the engine's per-launch log of the same run, launch by launch, and
print per kernel class: launches, algorithmic bytes per launch (SURVEY §8(d)
counts), DRAM bytes per launch, their ratio, ncu time share.

Usage: python tools/traffic_ratio.py gpurun_out/traffic_<tag>.csv gpurun_out/prof_log_<tag>.npz"""

import csv
import json
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
CLASSES = ("embed", "gemm_enc", "attn_enc", "norm", "gemm_dec", "attn_dec", "vocab_argmax",
           "search", "other")


def read_ncu(path):
    rows = defaultdict(dict)
    order = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        key = int(r["ID"])
        if key not in rows:
            order.append(key)
        v = float(r["Metric Value"].replace(",", "")) if r["Metric Value"] else 0.0
        unit = r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
                 "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(unit, 1.0)
        rows[key]["name"] = r["Kernel Name"]
        rows[key][r["Metric Name"]] = v * scale
    return [rows[k] for k in order]


def group_of_name(name):
    n = name.split("(")[0].split("<")[0].split("::")[-1].strip()
    for pre, g in (("attn_dec", "attn_dec"), ("dec_layer", "attn_dec"), ("attn_varlen", "attn_enc"), ("add_norm", "norm"),
                   ("embed", "embed"), ("greedy_update", "search"), ("beam_row_reduce", "search"),
                   ("beam_select", "search"), ("gemm_", "gemm")):
        if n.startswith(pre):
            return g
    return None


def group_of_cls(c):
    return "gemm" if c in ("gemm_enc", "gemm_dec", "vocab_argmax") else \
        (None if c == "other" else c)


def main():
    launches = read_ncu(sys.argv[1])
    log = np.load(sys.argv[2])
    cls = [CLASSES[int(c)] for c in log["cls"]]
    # match launch by launch within each kernel group (unprofiled helper
    # kernels and the "other" class are skipped on both sides)
    by_ncu, by_log = defaultdict(list), defaultdict(list)
    for r in launches:
        g = group_of_name(r["name"])
        if g:
            by_ncu[g].append(r)
    for i, c in enumerate(cls):
        g = group_of_cls(c)
        if g:
            by_log[g].append(i)
    agg = defaultdict(lambda: {"n": 0, "alg": 0.0, "dram": 0.0, "t": 0.0, "flops": 0.0})
    for g in by_log:
        if len(by_ncu[g]) != len(by_log[g]):
            print(f"warning: group {g}: ncu {len(by_ncu[g])} launches, log {len(by_log[g])}",
                  file=sys.stderr)
        for r, i in zip(by_ncu[g], by_log[g]):
            a = agg[cls[i]]
            a["n"] += 1
            a["alg"] += float(log["bytes"][i])
            a["flops"] += float(log["flops"][i])
            a["dram"] += r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0)
            a["t"] += r.get("gpu__time_duration.sum", 0)
    tt = sum(a["t"] for a in agg.values()) or 1.0
    res = {}
    for c, a in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
        res[c] = {"launches": a["n"], "alg_bytes_per_launch": a["alg"] / a["n"],
                  "dram_bytes_per_launch": a["dram"] / a["n"],
                  "dram_over_alg": a["dram"] / a["alg"] if a["alg"] else None,
                  "ncu_ms": a["t"] * 1e3, "ncu_share": a["t"] / tt,
                  "ncu_gbs": a["alg"] / a["t"] / 1e9 if a["t"] else None,
                  "ncu_tflops": a["flops"] / a["t"] / 1e12 if a["t"] and a["flops"] else None}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
