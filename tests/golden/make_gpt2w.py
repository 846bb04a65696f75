"""Golden scores for the GPT-2-width slice test (tests/test_gpu_parity.py::
test_gpt2_width_slice_matches_reference), computed by the REFERENCE library
compiled in place (oracle/_ref/libcqref.so, reference delta_l in its OpenMP
loop). Run here where /root/reference exists:

    python tests/golden/make_gpt2w.py
"""
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.dirname(HERE)]

import numpy as np  # noqa: E402

from helpers import make  # noqa: E402
from oracle.oracle import KL, Policy, Ref  # noqa: E402
from paper_2510_23264_b200 import formats  # noqa: E402

CFG = formats.ModelConfig(2, 12, 768, 64, 1024, 16, 1, 1)
WSEED, ITEMS, DSEED = 1, 4, 3


def edges_of(n_edges):
    return np.unique(np.r_[np.arange(0, n_edges, 23), n_edges - 1]).astype(np.int32)


def main():
    w, ds = make(CFG, WSEED, ITEMS, DSEED)
    ref = Ref()
    ref.set_threads(ref.max_threads())
    with tempfile.TemporaryDirectory() as t:
        wp, dp = os.path.join(t, "w.bin"), os.path.join(t, "d.jsonl")
        formats.save_weights(w, wp)
        formats.save_dataset_jsonl(ds, dp)
        m = ref.open(wp, dp, KL)
        from paper_2510_23264_b200.engine import graph_edges
        n_edges = len(graph_edges(CFG)[1])
        edges = edges_of(n_edges)
        s = m.score_edges(edges, Policy.head_quantized(), True)
        m.close()
    out = {"config": [int(v) for v in vars(CFG).values()], "wseed": WSEED, "items": ITEMS, "dseed": DSEED,
           "edges": edges.tolist(), "scores": [float(x).hex() for x in s]}
    json.dump(out, open(os.path.join(HERE, "gpt2w_slice.json"), "w"), indent=1)
    print(len(edges), "edges:", s[:4])


if __name__ == "__main__":
    main()
