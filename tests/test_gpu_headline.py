"""GPU parity at the bench's own model shapes, against scores of the
REFERENCE library (tests/golden/make_headline.py ran proj/src's
DeltaLEngine::refresh_baselines + delta_l, patching.cpp:191-239, on the same
synthetic weights and prompts):

* gpt2s_ioi   — BASELINE config 2, the headline workload: full GPT-2-small
  shape (12 layers, V = 50257), IOI-shaped prompts, per-edge PAHQ policies,
  edges from 12 sources spanning every node kind and depth, incl. src->unembed;
  also with the memory budget forced down so every source group is split into
  one-edge launch batches (the multi-batch path configs 4-5 need);
* gpt2m_slice — GPT-2-medium widths (D = 1024, H = 16), 2 layers, V = 50257;
* pythia_slice — Pythia-1.4B widths (D = 2048, d_k = 128, S = 32, V = 50304),
  2 layers, docstring-shaped prompts.

Tolerance: |gpu - ref| <= 1e-9 |ref| + 2^-44 (see test_gpu_parity.py).

Also: per-edge policies over a base policy that carries its own target
(policy_for_edge resets it, pahq.cpp:198-209) against the oracle.
"""
import json
import os

import numpy as np
import pytest

from oracle.oracle import KL, Policy, Port
from paper_2510_23264_b200 import engine as eng
from paper_2510_23264_b200 import formats, synth
from helpers import GOLDEN, SMALL, make
from test_gpu_parity import close, gpol

pytestmark = pytest.mark.gpu


def load_case(name):
    g = json.load(open(os.path.join(GOLDEN, f"{name}.json")))
    cfg = formats.ModelConfig(*g["config"])
    w = synth.random_weights(cfg, g["wseed"])
    gen = {"ioi": synth.ioi_dataset, "docstring": synth.docstring_dataset,
           "greater_than": synth.greater_than_dataset}[g["data"]]
    ds = gen(cfg, g["items"], g["dseed"])
    edges = np.array(g["edges"], np.int32)
    want = np.array([float.fromhex(x) for x in g["scores"]])
    return cfg, w, ds, edges, want


@pytest.mark.parametrize("case,opts", [("gpt2s_ioi", {}), ("gpt2s_ioi", {"mem_budget": 1}),
                                       ("gpt2s_ioi", {"env:CQG_LN_LANE_MIN": 1}),
                                       ("gpt2m_slice", {}), ("gpt2m_slice", {"env:CQG_LN_LANE_MIN": 1}),
                                       ("pythia_slice", {})])
def test_model_shapes_match_reference(case, opts, monkeypatch):
    """(env:CQG_LN_LANE_MIN=1 runs every layer norm through ln_lane_kernel,
    the big-launch LN kernel, which the bench step uses but these small
    golden cases would not reach.)"""
    cfg, w, ds, edges, want = load_case(case)
    e = eng.Engine(w)
    for k, v in opts.items():
        if k.startswith("env:"):
            monkeypatch.setenv(k[4:], str(v))
        else:
            e.set_option(k, v)
    e.set_dataset(ds, eng.KL)
    mask = np.ones(e.n_edges, bool)
    got = e.score_edges(mask, edges, eng.PrecisionPolicy.head_quantized(), True, eng.LOSS)
    rel = np.abs(got - want) / (np.abs(want) + 1e-300)
    assert close(got, want), (case, opts, float(rel.max()), int(np.argmax(rel)))
    assert e.stats()["kernel_launches"] > 0
    e.close()


def test_per_edge_policies_over_a_targeted_base():
    """A base policy with its own target head / MLP under per-edge policies:
    every scored pass runs policy_for_edge(edge, base), which drops the base's
    targets; the shared baseline prefix must therefore be target-free too."""
    w, ds = make(SMALL, 5, 3, 9)
    p = Port(SMALL, w.mats)
    e = eng.Engine(w)
    e.set_dataset(ds, KL)
    mask = np.ones(p.n_edges, bool)
    mask[np.random.RandomState(3).rand(p.n_edges) < 0.3] = False
    edges = np.nonzero(mask)[0].astype(np.int32)
    for base in (Policy.make(th=(0, 1)), Policy.make(tm=2), Policy.make(th=(2, 3), tm=0)):
        want = p.score_edges(ds, edges, base, per_edge=True, metric=KL, mask=mask)
        got = e.score_edges(mask, edges, gpol(base), True, eng.LOSS)
        assert close(got, want), (base.target_head_layer, base.target_mlp)
        # and the base policy itself (no per-edge policies) keeps its targets
        want = p.score_edges(ds, edges, base, per_edge=False, metric=KL, mask=mask)
        got = e.score_edges(mask, edges, gpol(base), False, eng.LOSS)
        assert close(got, want)
    e.close()
