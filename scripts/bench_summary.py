"""Dev tool: one-screen summary of a bench.py JSON line (file argument)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value", d["value"], "dense", d.get("dense_us_per_step"), "speedup", d.get("speedup_vs_dense"))
print("e2e", d["e2e"]["value"], "clocks", d["clocks"])
r = d["roofline"]
print("roofline frac", r["frac"], "achieved", r["achieved"], "phases", r.get("phases"))
for c in d.get("other_configs", []):
    print(" ", c["config"][:34], "routed", c["routed_us"], "dense", c["dense_us"], "x", c["speedup_vs_dense"])
for s in d.get("sweep", []):
    print(" ", s["context"], [p["us"] for p in s["points"]], "dense", s["dense_us"])
for k, v in d.get("next_rows", {}).items():
    print(" ", k, {a: b for a, b in v.items() if a != "note"})
print("cpu_baseline", d.get("cpu_baseline", {}).get("value"))
