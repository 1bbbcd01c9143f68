"""Print the headline and per-stage times of a bench.py JSON line (dev tool)."""
import json, sys
d = json.load(open(sys.argv[1]))
print("steps/s", round(d["value"], 1), "ms", round(d["ms_per_step"], 4), "clocks", d.get("clocks"))
for k, v in d["stages"].items():
    if "gbs" in v:
        print(f"  {k:16s} {1e3 * v['ms']:8.1f} us  {v['gbs']:7.0f} GB/s")
