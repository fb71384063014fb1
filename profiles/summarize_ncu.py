#!/usr/bin/env python
"""Summarise an ncu launch list (profiles/run_ncu.sh step 1) per kernel class.

Classes follow the engine's profile classes (bench.py kernel_profile):
the launch order of one lane is phase-ordered — ``gather_batch_kernel``
starts a batch (encoder phase: embed, GEMMs, varlen attention, add+norm,
then the cross-K/V GEMMs), ``init_decode_kernel`` starts the decode loop
(decoder GEMMs; the GEMM right before ``greedy_update_kernel`` / a beam
kernel is the vocab projection).

Writes ``profiles/ncu_traffic.json`` (class -> DRAM bytes per launch, read by
bench.py for ``roofline.traffic``) and prints a markdown table.

Usage: python profiles/summarize_ncu.py gpurun_out/launches_r1b.csv.gz [out.md]
"""

from __future__ import annotations

import csv
import gzip
import io
import json
import sys
from collections import defaultdict
from pathlib import Path


def rows_of(path: Path):
    raw = gzip.open(path, "rt") if path.suffix == ".gz" else open(path)
    text = raw.read()
    start = text.find('"ID"')
    rd = csv.DictReader(io.StringIO(text[start:]))
    launches = {}
    for r in rd:
        i = int(r["ID"])
        L = launches.setdefault(i, {"name": r["Kernel Name"], "m": {}})
        val = r["Metric Value"].replace(",", "")
        unit = r.get("Metric Unit", "")
        try:
            v = float(val)
        except ValueError:
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
                 "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
        L["m"][r["Metric Name"]] = v * scale
    return [launches[k] for k in sorted(launches)]


def classify(launches):
    phase = "enc"
    out = []
    for i, L in enumerate(launches):
        n = L["name"]
        if "gather_batch" in n:
            phase = "enc"
        elif "init_decode" in n or "beam_init" in n:
            phase = "dec"
        if "gemm_tc" in n or "gemm_simt" in n:
            nxt = launches[i + 1]["name"] if i + 1 < len(launches) else ""
            if phase == "dec" and ("greedy_update" in nxt or "beam_row" in nxt or "topk" in nxt):
                c = "vocab_argmax"
            else:
                c = "gemm_dec" if phase == "dec" else "gemm_enc"
        elif "attn_varlen" in n:
            c = "attn_enc"
        elif "attn_decode" in n:
            c = "attn_dec"
        elif "add_norm" in n:
            c = "norm"
        elif "embed" in n:
            c = "embed"
        elif "greedy_update" in n or "beam_" in n or "keys_to_index" in n:
            c = "search"
        elif "q_minmax" in n or "q_quant" in n:
            c = "quant"
        else:
            c = "other"
        out.append((c, L))
    return out


def main():
    src = Path(sys.argv[1])
    cl = classify(rows_of(src))
    agg = defaultdict(lambda: {"n": 0, "ms": 0.0, "rd": 0.0, "wr": 0.0})
    for c, L in cl:
        a = agg[c]
        a["n"] += 1
        a["ms"] += L["m"].get("gpu__time_duration.sum", 0.0)
        a["rd"] += L["m"].get("dram__bytes_read.sum", 0.0)
        a["wr"] += L["m"].get("dram__bytes_write.sum", 0.0)
    tot = sum(a["ms"] for a in agg.values()) or 1.0
    lines = ["| class | launches | total ms | share | avg us | DRAM MB / launch |",
             "|---|---|---|---|---|---|"]
    traffic = {}
    for c, a in sorted(agg.items(), key=lambda kv: -kv[1]["ms"]):
        per = (a["rd"] + a["wr"]) / max(a["n"], 1)
        traffic[c] = round(per)
        lines.append(f"| {c} | {a['n']} | {a['ms']:.3f} | {a['ms'] / tot:.3f} | "
                     f"{1e3 * a['ms'] / max(a['n'], 1):.2f} | {per / 1e6:.2f} |")
    lines.append(f"| **total** | {sum(a['n'] for a in agg.values())} | {tot:.3f} | 1.000 | | |")
    text = "\n".join(lines)
    print(text)
    (Path(__file__).resolve().parent / "ncu_traffic.json").write_text(
        json.dumps({"source": str(src.name), "unit": "DRAM bytes (read+write) per launch, "
                    "ncu serialised / cold L2", **traffic}, indent=1))
    if len(sys.argv) > 2:
        Path(sys.argv[2]).write_text(text + "\n")


if __name__ == "__main__":
    main()
