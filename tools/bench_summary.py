"""Print the compact fields of the last bench.py JSON line in a log file."""
import json
import sys

line = [l for l in open(sys.argv[1]).read().strip().splitlines() if l.startswith("{")][-1]
d = json.loads(line)
out = {k: d.get(k) for k in ("value", "ms_per_step", "kernels_ms_per_step", "residual_rel", "gpu_launches")}
out["roofline"] = {k: d["roofline"].get(k) for k in ("kernel", "bound", "achieved", "frac")} if d.get("roofline") else None
out["e2e"] = d["e2e"]["value"] if d.get("e2e") else None
print(json.dumps(out))
