#!/bin/bash
# A/B sweep of engine options (CQG_OPTS) on the default bench step, one short
# bench run per variant (no CPU leg, no ACDC). Usage (from the repo root,
# under gpurun): tools/ab_sweep.sh "" "fix_g=2" "fix_cpi=4" ...
# Prints value and the top per-kernel times per variant -> gpurun_out/ab_*.json
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
i=0
for v in "$@"; do
  CQG_OPTS="$v" timeout 600 python bench.py --no-cpu --no-acdc --steps 2 --warmup 3 ${BENCH_ARGS} \
    > "gpurun_out/ab_$i.json" 2> "gpurun_out/ab_$i.err"
  python - "$i" "$v" <<'PY'
import json, sys
i, v = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/ab_{i}.json").read().strip().splitlines()[-1])
except Exception as ex:
    print(i, repr(v), "FAILED", ex); sys.exit()
pk = d["roofline"]["per_kernel"]
top = {k: round(x["ms"]) for k, x in sorted(pk.items(), key=lambda kv: -kv[1]["ms"])[:9]}
print(i, repr(v), round(d["value"]), round(d["ms_per_step"]), top, flush=True)
PY
  i=$((i+1))
done
