"""Print value + the top per-kernel CUDA-event times of a bench JSON line."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
pk = d["roofline"]["per_kernel"]
print(round(d["value"]), "passes/s;", round(d["ms_per_step"]), "ms/step; e2e", round(d["e2e"]["value"]))
print({k: round(v["ms"]) for k, v in sorted(pk.items(), key=lambda kv: -kv[1]["ms"])[:14]})
