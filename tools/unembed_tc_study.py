"""Dev study (GPU): the tensor-core unembed on the bench workload. Scores one
full ACDC iteration-1 step (every edge, GPT-2-small IOI B=64) three ways:
exact logits; tensor-core logits with no fallback (tol huge); the certified
default. Writes gpurun_out/unembed_tc_study.json (per-edge relative
deviations vs the exact path, exact-row shares, device times)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2510_23264_b200 import engine as eng  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "gpt2s"
cfg, w, ds = bench.make_inputs(name)
e = eng.Engine(w)
e.set_dataset(ds, eng.KL)
mask = np.ones(e.n_edges, bool)
edges = eng.sweep_order(cfg, mask)
pol = eng.PrecisionPolicy.head_quantized()
out = {}
res = {}
for tag, opts in (("exact", {"unembed_tc": 0}), ("tc_nofallback", {"unembed_tc": 1, "unembed_tol_e9": 10**18}),
                  ("tc_certified", {"unembed_tc": 1, "unembed_tol_e9": 100000})):
    for k, v in opts.items():
        e.set_option(k, v)
    e.score_edges(mask, edges, pol, True, eng.LOSS)  # warm
    s = e.score_edges(mask, edges, pol, True, eng.LOSS)
    st = e.stats()
    res[tag] = s
    out[tag] = {"ms_device": st["ms_device"], "rows": st["unembed_rows"], "exact_rows": st["unembed_exact_rows"]}
    print(tag, out[tag], flush=True)
for tag in ("tc_nofallback", "tc_certified"):
    r = np.abs(res[tag] - res["exact"]) / np.maximum(np.abs(res["exact"]), 1e-300)
    out[tag]["rel_vs_exact"] = {q: float(np.quantile(r, q)) for q in (0.5, 0.9, 0.99, 0.999, 1.0)}
    out[tag]["n_over_1e-4"] = int((r > 1e-4).sum())
    out[tag]["n_over_1e-6"] = int((r > 1e-6).sum())
    print(tag, out[tag], flush=True)
out["score_quantiles"] = {q: float(np.quantile(res["exact"], q)) for q in (0.0, 0.01, 0.5, 0.99, 1.0)}
print(out["score_quantiles"])
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"unembed_tc_study_{name}.json"), "w"), indent=1)
