"""Print the headline figures of a bench.py JSON line: python tools/bench_brief.py FILE..."""
import json
import sys

for f in sys.argv[1:]:
    d = json.load(open(f))
    w = d["config"].get("window") or {}
    ks = {k: round(v["ms"] / max(v["launches"], 1), 4) for k, v in d["roofline"].get("kernels", {}).items()}
    print(f, round(d["value"], 3), d["unit"], "window", round(w.get("steps_per_s", 0), 3), "e2e",
          (d.get("e2e") or {}).get("value"), ks)
