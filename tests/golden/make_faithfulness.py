"""Golden faithfulness / task_accuracy (eval.cpp:1240-1254) of the planted
tasks under the ground-truth mask and a random mask, computed by the
REFERENCE library compiled in place (oracle/_ref/libcqref.so):

    python tests/golden/make_faithfulness.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT]

import numpy as np  # noqa: E402

from oracle.oracle import Ref  # noqa: E402
from paper_2510_23264_b200 import formats  # noqa: E402
from paper_2510_23264_b200.engine import graph_edges  # noqa: E402


def main():
    ref = Ref()
    out = {}
    for preset in ("standard", "underflow", "interference", "two_hop", "carrier"):
        d = os.path.join(HERE, f"planted_{preset}_s1")
        w = formats.load_weights(os.path.join(d, "weights.bin"))
        n_edges = len(graph_edges(w.cfg)[1])
        gt = json.load(open(os.path.join(d, "task.json")))["ground_truth"]
        masks = {"ground_truth": np.isin(np.arange(n_edges), gt),
                 "random": np.random.RandomState(5).rand(n_edges) < 0.5}
        for name, m in masks.items():
            f, a = ref.faithfulness(d, m)
            out[f"{preset}/{name}"] = {"mask": m.astype(int).tolist(), "faithfulness": float(f).hex(),
                                       "task_accuracy": float(a).hex()}
            print(preset, name, f, a)
    json.dump(out, open(os.path.join(HERE, "faithfulness.json"), "w"))


if __name__ == "__main__":
    main()
