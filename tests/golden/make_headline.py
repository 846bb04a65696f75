"""Golden per-edge scores at the bench's model shapes, computed by the
REFERENCE library compiled in place (oracle/_ref/libcqref.so: the reference's
own ImageBank, DeltaLEngine::refresh_baselines per policy and delta_l in its
OpenMP loop, proj/src/patching.cpp:191-239, via oracle/ref_shim.cpp
cqref_score_edges). Run here, where /root/reference exists:

    python tests/golden/make_headline.py [gpt2s_ioi|gpt2m_slice|pythia_slice ...]

Each case writes tests/golden/<case>.json: the model config, the generator
seeds (weights and prompts regenerate byte-identically from
paper_2510_23264_b200.synth, pinned against the reference in
tests/test_formats.py), the edge ids and the reference's scores (hex floats).

Edge sample: a fixed list of source nodes covering every node kind and depth
(embed, early/middle/final-layer heads, MLPs); for each source its out-edges
at positions 0, 1/3, 2/3 and last (the last one is always src -> unembed), so
destinations span the next stage, the middle of the graph, and the unembed.
Per-edge PAHQ policies (policy_for_edge, pahq.cpp:198-209) over the
head_quantized base: every source runs its own baseline refresh.
"""
import json
import os
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.dirname(HERE)]

import numpy as np  # noqa: E402

from oracle.oracle import KL, Policy, Ref  # noqa: E402
from paper_2510_23264_b200 import formats, synth  # noqa: E402

CASES = {
    # BASELINE config 2 (the bench's headline workload): full GPT-2-small
    # shape, V=50257, IOI-shaped prompts
    "gpt2s_ioi": dict(cfg=(12, 12, 768, 64, 50257, 16, 1, 1), data="ioi", items=4, dseed=1,
                      srcs=lambda L, H: [0, (0, 0), (0, 7), ("m", 0), (3, 4), ("m", 5), (8, 2),
                                         ("m", 9), (10, 11), (11, 3), (11, 11), ("m", 11)]),
    # BASELINE config 4 widths (GPT-2-medium: D=1024, H=16), 2 layers, full vocabulary
    "gpt2m_slice": dict(cfg=(2, 16, 1024, 64, 50257, 16, 1, 1), data="ioi", items=2, dseed=2,
                        srcs=lambda L, H: [0, (0, 0), (0, 15), ("m", 0), (1, 9), ("m", 1)]),
    # BASELINE config 5 widths (Pythia-1.4B: D=2048, d_k=128, S=32, V=50304), 2 layers
    "pythia_slice": dict(cfg=(2, 16, 2048, 128, 50304, 32, 1, 1), data="docstring", items=2,
                         dseed=3, srcs=lambda L, H: [0, (0, 3), ("m", 0), (1, 12), ("m", 1)]),
}
WSEED = 1


def node_id(s, H):
    if s == 0:
        return 0
    if s[0] == "m":
        return 1 + s[1] * (H + 1) + H
    return 1 + s[0] * (H + 1) + s[1]


def dataset(cfg, kind, items, seed):
    gen = {"ioi": synth.ioi_dataset, "docstring": synth.docstring_dataset,
           "greater_than": synth.greater_than_dataset}[kind]
    return gen(cfg, items, seed)


def pick_edges(ref, cfg8, srcs):
    _, _, _, src, _ = ref.graph(cfg8)
    out = []
    for s in srcs:
        oe = np.nonzero(src == s)[0]
        for k in sorted({0, len(oe) // 3, (2 * len(oe)) // 3, len(oe) - 1}):
            out.append(int(oe[k]))
    return np.array(sorted(set(out)), np.int32)


def make_case(name):
    c = CASES[name]
    cfg = formats.ModelConfig(*c["cfg"])
    w = synth.random_weights(cfg, WSEED)
    ds = dataset(cfg, c["data"], c["items"], c["dseed"])
    ref = Ref()
    ref.set_threads(ref.max_threads())
    srcs = [node_id(s, cfg.n_heads) for s in c["srcs"](cfg.n_layers, cfg.n_heads)]
    edges = pick_edges(ref, cfg.fields8(), srcs)
    t0 = time.time()
    with tempfile.TemporaryDirectory() as t:
        wp, dp = os.path.join(t, "w.bin"), os.path.join(t, "d.jsonl")
        formats.save_weights(w, wp)
        formats.save_dataset_jsonl(ds, dp)
        m = ref.open(wp, dp, KL)
        s = m.score_edges(edges, Policy.head_quantized(), True)
        m.close()
    out = {"case": name, "config": list(c["cfg"]), "wseed": WSEED, "data": c["data"],
           "items": c["items"], "dseed": c["dseed"], "policy": "head_quantized E4M3, per-edge",
           "metric": "kl", "edges": edges.tolist(), "scores": [float(x).hex() for x in s],
           "ref_seconds": round(time.time() - t0, 1)}
    json.dump(out, open(os.path.join(HERE, f"{name}.json"), "w"), indent=1)
    print(name, len(edges), "edges in", out["ref_seconds"], "s; scores", s[:4], flush=True)


if __name__ == "__main__":
    os.environ.setdefault("CQREF_NO_RTN4", "1")
    for n in sys.argv[1:] or list(CASES):
        make_case(n)
