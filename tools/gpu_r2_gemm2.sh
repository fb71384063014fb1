mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.max,sm__cycles_active.avg,launch__grid_size --csv --log-file gpurun_out/gemm_cold.csv python tools/perf_gemm.py dec > /dev/null 2>&1
timeout 600 ncu --cache-control none --metrics gpu__time_duration.sum,sm__cycles_active.max,sm__cycles_active.avg,launch__grid_size --csv --log-file gpurun_out/gemm_warm.csv python tools/perf_gemm.py dec > /dev/null 2>&1
python - <<'PY'
import csv, collections
for f in ("gpurun_out/gemm_cold.csv", "gpurun_out/gemm_warm.csv"):
    rows = list(csv.reader(open(f)))
    i = next(k for k, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[i]; L = collections.OrderedDict()
    for r in rows[i + 1:]:
        d = L.setdefault(r[h.index("ID")], {})
        d[r[h.index("Metric Name")]] = r[h.index("Metric Value")]
    print(f)
    v = list(L.values())
    for j in range(0, len(v), 20):   # one line per shape (first launch of each graph replay group)
        d = v[j + 5] if j + 5 < len(v) else v[j]
        print("  ", {k: d[k] for k in d})
PY
