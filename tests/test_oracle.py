"""The CPU oracle (oracle/cq_oracle.c) pinned to the reference.

* against the reference's own frozen values (proj/tests/test_numerics.cpp,
  test_patching.cpp, test_acdc.cpp, test_eval.cpp) via tests/golden/;
* bit-for-bit against the reference library compiled in place (oracle/_ref)
  when it is present (build container and GPU box).
"""
import json
import math
import os

import numpy as np
import pytest

from oracle.oracle import KL, LOGITDIFF, Policy, Port, Prune
from paper_2510_23264_b200 import formats, synth
from paper_2510_23264_b200.engine import PrecisionPolicy, method_prune_config, threshold_grid
from helpers import GOLDEN, SMALL, TINY, TOY, bits, make, random_mask, write

G = json.load(open(os.path.join(GOLDEN, "golden.json")))


def port_for(cfg, wseed, items, dseed):
    w, ds = make(cfg, wseed, items, dseed)
    return Port(cfg, w.mats), w, ds


# --- numerics (proj/tests/test_numerics.cpp) -------------------------------
def test_e4m3_landmarks():
    p, _, _ = port_for(TINY, 1, 1, 1)
    lib = p.lib
    enc = lambda x: lib.cqo_encode_f8(x)  # noqa: E731
    assert enc(448.0) == 0x7E and enc(1000.0) == 0x7E and enc(-1000.0) == 0xFE
    assert enc(0.015625) == 0x08
    assert enc(0.3) == enc(0.3125)
    assert enc(0.0) == 0x00
    assert enc(float("nan")) == 0x7F
    assert enc(2.0 ** -11) == 0 and enc(2.0 ** -10) == 0
    assert enc(1.5 * 2.0 ** -10) == 0x01


def test_e4m3_decode_table_all_patterns():
    p, _, _ = port_for(TINY, 1, 1, 1)
    import ctypes as C
    p.lib.cqo_decode_f8.restype = C.c_double
    p.lib.cqo_decode_f8.argtypes = [C.c_uint8]
    vals = [p.lib.cqo_decode_f8(b) for b in range(256)]
    nans = [b for b, v in enumerate(vals) if math.isnan(v)]
    assert nans == [0x7F, 0xFF]
    pos = {v for b, v in enumerate(vals) if not (b & 0x80) and not math.isnan(v)}
    assert len(pos) == 127 and max(pos) == 448.0
    for b in range(256):  # encode(decode(p)) round trip
        if b in nans:
            continue
        assert p.lib.cqo_encode_f8(vals[b]) == b or (b == 0x80)  # -0 encodes to 0x80


def test_rtn_frozen_examples():
    # test_numerics.cpp:221-244
    from oracle.oracle import Ref, ref_available
    x = np.array([1.0, -2.0, 0.3], np.float32)
    import ctypes as C
    p, _, _ = port_for(TINY, 1, 1, 1)
    d = C.c_double()
    y = x.copy()
    p.lib.cqo_quantize_rtn(y.ctypes.data_as(C.c_void_p), C.c_int64(3), 8, C.byref(d))
    assert d.value == 2.0 / 128.0 and y[0] == 1.0 and y[1] == -2.0 and y[2] == np.float32(0.296875)


def test_kl_frozen_value():
    # test_patching.cpp:53-73, acceptance_tests.cpp:553-558
    import ctypes as C
    p, _, _ = port_for(TINY, 1, 1, 1)
    f = np.array([0.0, 0.0], np.float32)
    t = np.array([0.0, 1.0], np.float32)
    kl = p.lib.cqo_metric_kl(f.ctypes.data_as(C.c_void_p), t.ctypes.data_as(C.c_void_p), 2)
    assert abs(kl - 0.12011450695827752) <= 1e-12 * 0.12011450695827752
    assert p.lib.cqo_metric_kl(f.ctypes.data_as(C.c_void_p), f.ctypes.data_as(C.c_void_p), 2) == 0.0
    l3 = np.array([0.0, np.float32(math.log(3.0))], np.float32)
    kl3 = p.lib.cqo_metric_kl(f.ctypes.data_as(C.c_void_p), l3.ctypes.data_as(C.c_void_p), 2)
    assert abs(kl3 - 0.5 * math.log(4.0 / 3.0)) <= 1e-6


def test_threshold_grid_frozen():
    # test_acdc.cpp:277-294
    g = threshold_grid(0.001, 3.16, 21)
    assert g[0] == 0.001 and g[-1] == 3.16
    assert abs(g[1] - 0.0014961817537620622) <= 1e-12 * g[1]
    assert abs(g[2] - 0.002238559840290518) <= 1e-12 * g[2]
    assert abs(g[19] - 2.112042866486218) <= 1e-12 * g[19]
    assert [float(x).hex() for x in g] == G["threshold_grid"]


# --- graph (model.cpp:166-246) ---------------------------------------------
@pytest.mark.parametrize("cfg,n_nodes,n_edges", [(TOY, 10, 33), (TINY, 8, 26)])
def test_graph_counts(cfg, n_nodes, n_edges):
    p = Port(cfg, synth.random_weights(cfg, 1).mats)
    assert (p.n_nodes, p.n_edges) == (n_nodes, n_edges)


def test_gpt2_graph_edge_count():
    # SURVEY.md §0.7 (measured with the reference's ComputationalGraph)
    from paper_2510_23264_b200.engine import graph_edges
    from helpers import GPT2S
    n, src, dst = graph_edges(GPT2S)
    assert n == 158 and len(src) == 11611
    med = formats.ModelConfig(24, 16, 1024, 64, 50257, 16, 1, 1)
    assert len(graph_edges(med)[1]) == 80965


# --- scores / ACDC against the reference's recorded outputs -----------------
def test_tiny_scores_match_golden():
    p, w, ds = port_for(TINY, 101, 3, 7)
    pols = {"fp32": (Policy.all_fp32(), False), "hq": (Policy.head_quantized(), False),
            "pahq": (Policy.head_quantized(), True), "low": (Policy.all_low(), False)}
    for key, rec in G["tiny"].items():
        metric = int(key[1])
        mask_seed = key.split("_")[1][4:]
        mask = None if mask_seed == "None" else (
            np.random.RandomState(int(mask_seed)).rand(p.n_edges) < 0.6)
        pname = key.split("_")[2]
        mode = int(key[-1])
        pol, per = pols[pname]
        got = p.score_edges(ds, rec["edges"], pol, per_edge=per, metric=metric, mode=mode,
                            mask=mask)
        assert [float(x).hex() for x in got] == rec["scores"], key


def test_toy_pahq_acdc_matches_golden():
    p, w, ds = port_for(TOY, 1, 16, 2)
    pr = Prune()
    pr.tau, pr.max_steps, pr.min_change_rate, pr.mode, pr.act_floor = 0.01, 10, 0.0, 0, 0.0
    pr.per_edge_policy, pr.heads_only = 1, 0
    pr.base = Policy.head_quantized()
    r = p.run_acdc(ds, pr, KL)
    g = G["toy_pahq"]
    assert r.steps == g["steps"]
    assert r.final_mask.astype(int).tolist() == g["final_mask"]
    assert [[s, e, float(sc).hex(), k] for s, e, sc, k in r.records] == g["records"]


@pytest.mark.parametrize("preset", ["standard", "underflow", "two_hop"])
def test_planted_auc_known_answers(preset):
    """roc_sweep (eval.cpp:1193-1226) restated over the oracle reproduces the
    reference's exact AUCs (test_eval.cpp:174-294)."""
    d = os.path.join(GOLDEN, f"planted_{preset}_s1")
    w = formats.load_weights(os.path.join(d, "weights.bin"))
    ds = formats.load_dataset_jsonl(os.path.join(d, "dataset.jsonl"))
    gt = set(json.load(open(os.path.join(d, "task.json")))["ground_truth"])
    p = Port(w.cfg, w.mats)
    taus = threshold_grid(0.001, 3.16, 21)
    for mname, mid in (("acdc", 0), ("rtn8", 1), ("pahq", 2)):
        cfg = method_prune_config(mid)
        pts = []
        for tau in taus:
            pr = Prune()
            pr.tau, pr.max_steps, pr.min_change_rate, pr.mode = tau, cfg.max_steps, 0.0, 0
            pr.act_floor, pr.per_edge_policy, pr.heads_only = 0.0, int(cfg.per_edge_policy), 0
            b = cfg.base_policy
            pr.base = Policy.make(b.attention_default, b.mlp_default, b.embed_precision,
                                  b.unembed_precision, b.low_mode)
            r = p.run_acdc(ds, pr, LOGITDIFF)
            kept = np.nonzero(r.final_mask)[0]
            tp = sum(1 for e in kept if e in gt)
            pts.append((tp / len(gt), (len(kept) - tp) / (p.n_edges - len(gt))))
        auc = auc_from_points(pts)
        assert float(auc).hex() == G["planted"][preset][mname]["auc"], (preset, mname, auc)


def auc_from_points(pts):
    """eval.cpp:1149-1166"""
    ps = sorted(pts, key=lambda p: (p[1], p[0]))
    x = y = area = 0.0
    for tpr, fpr in ps:
        if tpr <= y:
            continue
        if fpr > x:
            area += (fpr - x) * y
            x = fpr
        y = tpr
    return area + (1.0 - x) * y


# --- bit-for-bit against the compiled reference ------------------------------
@pytest.mark.parametrize("cfg", [TINY, SMALL, TOY])
def test_port_forward_equals_reference(ref, cfg, tmp_path):
    w, ds = make(cfg, 3, 2, 4)
    wp, dp = write(str(tmp_path), w, ds)
    rm = ref.open(wp, dp, 0)
    p = Port(cfg, w.mats)
    L, H = cfg.n_layers, cfg.n_heads
    pols = [Policy.all_fp32(), Policy.head_quantized(), Policy.all_low(),
            Policy.make(th=(L - 1, H - 1)), Policy.head_quantized(mode=1),
            Policy.make(att=1), Policy.make(mode=1, th=(0, 0)), Policy.all_low(1),
            Policy.make(att=0, mlp=0, mode=1, tm=0 if cfg.has_mlp else None)]
    if cfg.has_mlp:
        pols.append(Policy.make(tm=0))
    for i, pol in enumerate(pols):
        mask = random_mask(p.n_edges, i, 0.7) if i % 2 else None
        a = rm.forward(ds.clean[0], pol, mask=mask)
        b = p.forward(ds.clean[0], pol, mask=mask)
        assert np.array_equal(bits(a), bits(b)), i
    rm.close()


def test_port_run_acdc_equals_reference_small(ref, tmp_path):
    w, ds = make(SMALL, 5, 3, 6)
    wp, dp = write(str(tmp_path), w, ds)
    rm = ref.open(wp, dp, 0)
    p = Port(SMALL, w.mats)
    pr = ref.method_config(2, 8)
    pr.tau, pr.max_steps = 0.002, 3
    a = rm.run_acdc(pr)
    b = p.run_acdc(ds, pr, KL)
    assert a.steps == b.steps and np.array_equal(a.final_mask, b.final_mask)
    assert a.records == b.records
    rm.close()


def test_port_targeted_base_per_edge_equals_reference(ref, tmp_path):
    """Per-edge policies over a base that carries its own target head / MLP
    (policy_for_edge resets it, pahq.cpp:198-209): the restatement equals the
    reference library bit for bit (the GPU test compares against the port)."""
    from helpers import write
    w, ds = make(SMALL, 5, 3, 9)
    p = Port(SMALL, w.mats)
    mask = np.ones(p.n_edges, bool)
    mask[np.random.RandomState(3).rand(p.n_edges) < 0.3] = False
    edges = np.nonzero(mask)[0].astype(np.int32)
    wp, dp = write(str(tmp_path), w, ds)
    m = ref.open(wp, dp, KL)
    for base in (Policy.make(th=(0, 1)), Policy.make(tm=2), Policy.make(th=(2, 3), tm=0)):
        for pe in (True, False):
            a = p.score_edges(ds, edges, base, per_edge=pe, metric=KL, mask=mask)
            b = m.score_edges(edges, base, pe, 0, mask)
            assert np.array_equal(a, b), (pe, base.target_head_layer, base.target_mlp)
    m.close()


# --- INT8 per-channel RTN (extension, BASELINE config 2; parity unpinned) ------
def _int8_col(col):
    """quantize_rtn conventions (numerics.cpp:105-120) with N = 8 on one
    group, plus the INT8 clamp q <= 127 (restated independently here)."""
    col = np.asarray(col, np.float32)
    mx = float(np.max(np.abs(col.astype(np.float64)))) if col.size else 0.0
    if mx == 0.0:
        return col.copy()
    d = mx / 128.0
    # numpy rounds half to even; int64 as round_half_even's return type (a
    # zero quotient gives +0, numerics.cpp:21-28)
    q = np.minimum(np.round(col.astype(np.float64) / d).astype(np.int64), 127)
    return (d * q).astype(np.float32)


def test_int8_rtn_conventions():
    """Frozen values: quantize_rtn's N = 8 example (test_numerics.cpp:221-229:
    {1, -2, 0.3} -> delta 2/128, 0.3 -> 0.296875, -2 -> -128 delta kept), the
    +128 endpoint (a positive group maximum saturates to 127 delta) and an
    all-zero group (unchanged), through the oracle's W_Q image columns."""
    from oracle.oracle import INT8, P8
    cfg = formats.ModelConfig(1, 1, 3, 3, 5, 2, 1, 0)
    w = synth.random_weights(cfg, 1)
    wq = np.zeros((3, 3), np.float32)
    wq[:, 0] = [1.0, -2.0, 0.3]
    wq[:, 1] = [2.0, -1.0, 0.3]
    w.mats[4] = wq.ravel().copy()
    p = Port(cfg, w.mats)
    img = p.image(4, P8, INT8).reshape(3, 3)
    assert img[:, 0].tolist() == [1.0, -2.0, 0.296875]
    assert img[:, 1].tolist() == [np.float32(127 / 64), -1.0, 0.296875]
    assert img[:, 2].tolist() == [0.0, 0.0, 0.0]


@pytest.mark.parametrize("cfg", [SMALL, TOY])
def test_int8_images_per_channel(cfg):
    """Every INT8 image equals the independent restatement: W_Q/K/V/W_in/
    W_out/W_u/W_e/W_pos per output column, W_O per (head, column) block of
    d_k rows, LN vectors as one group."""
    from oracle.oracle import INT8, P8
    w, _ = make(cfg, 2, 1, 1)
    p = Port(cfg, w.mats)
    D, dk, H, V = cfg.d_model, cfg.d_k, cfg.n_heads, cfg.vocab
    for idx, (name, shape) in enumerate(cfg.matrix_specs()):
        m = np.asarray(w.mats[idx], np.float32).reshape(shape)
        got = p.image(idx, P8, INT8).reshape(shape)
        if len(shape) == 1:
            want = _int8_col(m)
        elif name.endswith("w_o"):
            want = np.empty_like(m)
            for h in range(H):
                for c in range(D):
                    want[h * dk:(h + 1) * dk, c] = _int8_col(m[h * dk:(h + 1) * dk, c])
        else:
            want = np.stack([_int8_col(m[:, c]) for c in range(shape[1])], axis=1)
        assert np.array_equal(bits(got), bits(want)), name


def test_int8_forward_per_token_grids():
    """Under an INT8 policy every low-precision head output row (one token,
    D values) is an INT8 grid: at most 256 distinct values, all multiples of
    one step (per-token dynamic activation scales)."""
    from oracle.oracle import INT8
    w, ds = make(SMALL, 3, 2, 4)
    p = Port(SMALL, w.mats)
    out = p.forward(ds.clean[0], Policy.make(mode=INT8))
    S, D = SMALL.seq_len, SMALL.d_model
    for n in range(1, 1 + SMALL.n_heads):  # layer-0 heads (nodes 1..H)
        rows = out[n * S * D:(n + 1) * S * D].reshape(S, D).astype(np.float64)
        for r in rows:
            mx = np.max(np.abs(r))
            q = r / (mx / 127.0) if np.any(r == mx) and mx > 0 else r / (mx / 128.0)
            assert len(np.unique(r)) <= 256
            assert np.allclose(q, np.round(q), atol=1e-4), (n, q[:4])


# --- Q/K/V-split edges (extension, BASELINE config 3; parity unpinned) ---------
def test_qkv_split_edge_counts():
    """Each head has q / k / v input receivers: 32,491 edges at GPT-2-small
    (config 3's "~32k"); 49 + 481 l per layer plus 157 into the unembed."""
    from helpers import GPT2S
    w = synth.random_weights(GPT2S, 1)
    p = Port(GPT2S, w.mats, qkv_split=True)
    assert p.n_edges == 32491
    L, H = 3, 2
    cfg = formats.ModelConfig(L, H, 8, 4, 11, 3, 1, 1)
    p = Port(cfg, synth.random_weights(cfg, 1).mats, qkv_split=True)
    # receivers: per layer 3H head inputs (1 + (H+1) l senders) + MLP (1 + (H+1) l + H)
    want = sum(3 * H * (1 + (H + 1) * l) + 1 + (H + 1) * l + H for l in range(L)) + 1 + (H + 1) * L
    assert p.n_edges == want


def test_qkv_split_numbering_and_sweep_order():
    """Edges are numbered receiver-major (node asc, component q < k < v), then
    source ascending (model.cpp:192-201 with the receiver in place of the
    node); the sweep order is receiver descending, source descending
    (model.cpp:238-246)."""
    p = Port(SMALL, make(SMALL)[0].mats, qkv_split=True)
    k, l, h, src, dst = p.graph()
    comp = p.edge_comp()
    key = [(int(d), int(c), int(s)) for s, d, c in zip(src, dst, comp)]
    assert key == sorted(key)
    assert all(c == 0 for d, c in zip(dst, comp) if k[d] != 1)
    assert list(p.sweep_order()) == list(range(p.n_edges))[::-1]


@pytest.mark.parametrize("cfg", [TINY, SMALL, TOY])
def test_qkv_split_pins_against_the_reference_graph(cfg):
    """Where the split graph has a reference counterpart it equals it bit for
    bit: the full graph (every receiver of a head sums the same sources), and
    any mask that drops (u -> h.q, u -> h.k, u -> h.v) together (= dropping
    u -> h in the reference's graph), under several policies. The unsplit
    oracle is itself pinned to the reference library (test_port_forward_equals_reference)."""
    w, ds = make(cfg, 4, 2, 5)
    a, b = Port(cfg, w.mats), Port(cfg, w.mats, qkv_split=True)
    _, _, _, sa, da = a.graph()
    _, _, _, sb, db = b.graph()
    idx = {(int(s), int(d)): i for i, (s, d) in enumerate(zip(sa, da))}
    rng = np.random.RandomState(7)
    L = cfg.n_layers
    for pol in (Policy.head_quantized(), Policy.all_fp32(), Policy.make(th=(L - 1, 0))):
        fa = a.forward(ds.clean[0], pol)
        fb = b.forward(ds.clean[0], pol)
        assert np.array_equal(bits(fa), bits(fb))
        ma = rng.rand(a.n_edges) < 0.7
        mb = np.array([ma[idx[(int(s), int(d))]] for s, d in zip(sb, db)])
        fa = a.forward(ds.clean[1], pol, mask=ma)
        fb = b.forward(ds.clean[1], pol, mask=mb)
        assert np.array_equal(bits(fa), bits(fb))


def test_qkv_split_patch_moves_one_component():
    """A patch on u -> h.q changes h's queries only: patching with the clean
    value is a no-op (test_model.cpp:381-396), and a patch on one component
    gives a different output from the same patch on another."""
    w, ds = make(SMALL, 4, 2, 5)
    p = Port(SMALL, w.mats, qkv_split=True)
    k, l, h, src, dst = p.graph()
    comp = p.edge_comp()
    S, D = SMALL.seq_len, SMALL.d_model
    base = p.forward(ds.clean[0], Policy.head_quantized())
    eq = [e for e in range(p.n_edges) if k[dst[e]] == 1 and l[dst[e]] == 1 and comp[e] == 0][0]
    ek = eq + sum(1 for e in range(p.n_edges) if dst[e] == dst[eq] and comp[e] == 0)  # same source, k input
    assert src[ek] == src[eq] and comp[ek] == 1
    s = int(src[eq])
    same = p.forward(ds.clean[0], Policy.head_quantized(), patch_edge=eq,
                     patch_value=base[s * S * D:(s + 1) * S * D])
    assert np.array_equal(bits(same), bits(base))
    pv = np.random.RandomState(1).randn(S * D).astype(np.float32)
    fq = p.forward(ds.clean[0], Policy.head_quantized(), patch_edge=eq, patch_value=pv)
    fk = p.forward(ds.clean[0], Policy.head_quantized(), patch_edge=ek, patch_value=pv)
    n = int(dst[eq])
    assert not np.array_equal(fq[n * S * D:(n + 1) * S * D], fk[n * S * D:(n + 1) * S * D])
    # nodes before the destination's stage are untouched
    assert np.array_equal(bits(fq[:n * S * D - (h[n]) * S * D]), bits(base[:n * S * D - (h[n]) * S * D]))
