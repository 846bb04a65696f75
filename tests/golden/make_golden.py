"""Regenerates the golden fixtures under tests/golden/ from the REFERENCE.

Run in the build container (needs /root/reference and oracle/_ref):
    python tests/golden/make_golden.py

* planted_<preset>_s<seed>/  — save_task output of the reference's planted
  task generator (proj/src/eval.cpp:1087-1117). Its weights draw from
  std::normal_distribution, so they must be consumed, not regenerated
  (SURVEY.md §4 caveat).
* golden.json — reference outputs: known-answer AUCs, run_acdc records for
  the toy config, per-edge scores for the tiny config, frozen values.
Doubles are stored as float.hex strings (bit-exact).
"""
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle.oracle import Policy, Ref  # noqa: E402
from helpers import TINY, TOY, make, write  # noqa: E402

PRESETS = {"standard": 0, "underflow": 1, "interference": 2, "two_hop": 3, "carrier": 4}


def hx(a):
    return [float(x).hex() for x in np.asarray(a, np.float64).ravel()]


def main():
    ref = Ref()
    out = {}
    # --- planted tasks + known-answer AUCs (proj/tests/test_eval.cpp:174-295)
    taus = ref.threshold_grid(0.001, 3.16, 21)
    out["threshold_grid"] = hx(taus)
    out["planted"] = {}
    for name, pid in PRESETS.items():
        d = os.path.join(HERE, f"planted_{name}_s1")
        ref.gen_planted(pid, 1, d)
        rec = {}
        for mname, mid in (("acdc", 0), ("rtn8", 1), ("pahq", 2)):
            auc, tpr, fpr, kept = ref.roc_sweep(d, mid, taus)
            rec[mname] = {"auc": float(auc).hex(), "tpr": hx(tpr), "fpr": hx(fpr),
                          "kept": [int(k) for k in kept]}
        out["planted"][name] = rec
    # --- toy config (BASELINE config 1): full PAHQ-ACDC, KL, tau 0.01
    with tempfile.TemporaryDirectory() as t:
        w, ds = make(TOY, wseed=1, items=16, dseed=2)
        wp, dp = write(t, w, ds)
        m = ref.open(wp, dp, 0)
        pr = ref.method_config(2, 8)
        pr.tau, pr.max_steps = 0.01, 10
        r = m.run_acdc(pr)
        out["toy_pahq"] = {"steps": r.steps, "final_mask": r.final_mask.astype(int).tolist(),
                           "records": [[s, e, float(sc).hex(), k] for s, e, sc, k in r.records]}
        m.close()
    # --- tiny config: every edge, several policies / metrics / masks
    with tempfile.TemporaryDirectory() as t:
        w, ds = make(TINY, wseed=101, items=3, dseed=7)
        wp, dp = write(t, w, ds)
        out["tiny"] = {}
        for metric in (0, 1):
            m = ref.open(wp, dp, metric)
            E = m.n_edges
            for mask_seed in (None, 5):
                mask = None if mask_seed is None else (np.random.RandomState(mask_seed).rand(E) < 0.6)
                edges = np.arange(E) if mask is None else np.nonzero(mask)[0]
                for pname, pol, per in (("fp32", Policy.all_fp32(), False),
                                        ("hq", Policy.head_quantized(), False),
                                        ("pahq", Policy.head_quantized(), True),
                                        ("low", Policy.all_low(), False)):
                    for mode in (0, 1):
                        key = f"m{metric}_mask{mask_seed}_{pname}_mode{mode}"
                        sc = m.score_edges(edges, pol, per_edge=per, mode=mode,
                                           mask=None if mask is None else mask.astype(np.uint8))
                        out["tiny"][key] = {"edges": edges.tolist(), "scores": hx(sc)}
            m.close()
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=0)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
