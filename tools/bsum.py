"""One-line summary of a bench JSON line (value, e2e, parity, clocks, kernel classes)."""
import json
import sys

for p in sys.argv[1:]:
    d = json.loads(open(p).read().strip().splitlines()[-1])
    par = d.get("parity") or {}
    print(p, "value %.0f e2e %.0f ms/step %.1f" % (d["value"], d["e2e"]["value"], d["ms_per_step"]),
          "parity %s/%s near-ties %s" % (par.get("identical"), par.get("sentences"), par.get("all_near_ties")),
          "sm_mhz", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    print("   roofline", {k: d["roofline"].get(k) for k in ("kernel", "achieved", "frac", "path_tflops")})
    for k, v in d.get("kernel_profile", {}).items():
        print("   %-13s %8.3f ms %5d launches  %.2f us/launch" % (k, v["ms"], v["launches"], 1e3 * v["ms"] / max(1, v["launches"])))
