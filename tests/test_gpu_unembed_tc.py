"""The optional tensor-core unembed of the patched passes (engine option
unembed_tc=1; the default is the exact SIMT unembed): the FP32 logits on the
tcgen05 tensor cores (6-term BF16 split, gemm_tc.cu split_rows/split_cols)
with the KL-level certificate (kernels.cu KlCert): every (edge, item) row
whose estimated KL deviation exceeds tol * KL is recomputed on the exact
reference-order path (gemm_exact_rows + kl_rows).

Bars:
* tol -> 0 (unembed_tol_e9 = 0): every row is sent to the exact path, so the
  scores equal the exact-logit engine's bit for bit (the fallback machinery);
* default tol (1e-4, BASELINE north_star "per-edge KL within 1e-4
  relative"): every per-edge score within 1e-4 relative of the exact-logit
  engine and of the reference library (GPT-2-small IOI golden); the measured
  maximum deviation and the exact-row share are recorded in
  gpurun_out/unembed_tc.json. (At GPT-2 width the certificate sends nearly
  every row to the exact path: that is the measured reason the option is off
  by default.)
"""
import json
import os

import numpy as np
import pytest

from oracle.oracle import KL, Policy
from paper_2510_23264_b200 import engine as eng
from paper_2510_23264_b200 import formats, synth
from helpers import SMALL, make
from test_gpu_headline import load_case

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NORTH_STAR_RTOL = 1e-4
RESULTS = {}
# GPT-2-width slice: D = 768, V = 50257 (the bench's unembed shape), 2 layers
GPT2W = formats.ModelConfig(2, 12, 768, 64, 50257, 16, 1, 1)


def record(name, **kv):
    RESULTS[name] = kv
    p = os.path.join(ROOT, "gpurun_out", "unembed_tc.json")
    os.makedirs(os.path.dirname(p), exist_ok=True)
    json.dump(RESULTS, open(p, "w"), indent=1)


def scores(w, ds, mask, edges, per_edge, **opts):
    e = eng.Engine(w, options=opts)
    e.set_dataset(ds, KL)
    s = e.score_edges(mask, edges, eng.PrecisionPolicy.head_quantized(), per_edge, eng.LOSS)
    st = e.stats()
    e.close()
    return s, st


def rel(a, b):
    return np.abs(a - b) / np.maximum(np.abs(b), 1e-300)


@pytest.mark.parametrize("cfg,items", [(SMALL, 5), (GPT2W, 4)])
def test_all_rows_flagged_equals_exact(cfg, items):
    w, ds = make(cfg, 3, items, 4)
    mask = np.ones(len(eng.graph_edges(cfg)[1]), bool)
    edges = np.nonzero(mask)[0].astype(np.int32)
    if len(edges) > 120:
        edges = edges[np.linspace(0, len(edges) - 1, 120).astype(int)]
    # (the exact logits' KL through the same stored-logit KL kernel: the fused
    # unembed + KL epilogue evaluates the same KL with another rounding)
    want, _ = scores(w, ds, mask, edges, True, unembed_tc=0, kl_fused=0)
    got, st = scores(w, ds, mask, edges, True, unembed_tc=1, unembed_tol_e9=0)
    assert st["unembed_rows"] > 0 and st["unembed_exact_rows"] == st["unembed_rows"]
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("cfg,items,per_edge", [(SMALL, 5, True), (SMALL, 5, False), (GPT2W, 4, True)])
def test_certified_scores_within_north_star(cfg, items, per_edge):
    w, ds = make(cfg, 5, items, 6)
    n_e = len(eng.graph_edges(cfg)[1])
    mask = np.random.RandomState(1).rand(n_e) < 0.8
    edges = np.nonzero(mask)[0].astype(np.int32)
    want, _ = scores(w, ds, mask, edges, per_edge, unembed_tc=0)
    got, st = scores(w, ds, mask, edges, per_edge, unembed_tc=1)  # certified, default tol
    r = rel(got, want)
    record(f"engine_{cfg.d_model}_{per_edge}", max_rel=float(r.max()), median_rel=float(np.median(r)),
           rows=int(st["unembed_rows"]), exact_rows=int(st["unembed_exact_rows"]))
    assert st["unembed_rows"] > 0
    assert r.max() <= NORTH_STAR_RTOL, float(r.max())


def test_headline_golden_within_north_star():
    """GPT-2-small, IOI prompts, per-edge PAHQ policies: the reference
    library's delta_l scores (tests/golden/gpt2s_ioi.json)."""
    cfg, w, ds, edges, want = load_case("gpt2s_ioi")
    e = eng.Engine(w, options={"unembed_tc": 1})
    e.set_dataset(ds, eng.KL)
    got = e.score_edges(np.ones(e.n_edges, bool), edges, eng.PrecisionPolicy.head_quantized(), True,
                        eng.LOSS)
    st = e.stats()
    e.close()
    r = rel(got, want)
    record("gpt2s_ioi_golden", max_rel=float(r.max()), median_rel=float(np.median(r)),
           rows=int(st["unembed_rows"]), exact_rows=int(st["unembed_exact_rows"]))
    assert r.max() <= NORTH_STAR_RTOL, float(r.max())
