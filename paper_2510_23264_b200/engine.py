"""Python mirror of the reference's scoring/driver interface over libcqg.so.

Names and argument meaning follow proj/include/circuitquant/{precision_policy,
patching,acdc,eval}.hpp so parity tests read like the reference's own tests.
All compute happens in libcqg.so (sm_100a CUDA); there is no CPU fallback —
constructing an Engine without the built library or without a GPU raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from .formats import Dataset, ModelConfig, WeightSet, validate_dataset

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcqg.so")

# Precision (numerics.hpp:19), LowMode (numerics.hpp:25), Metric, ScoreMode, Method
P8, P16, P32 = 0, 1, 2
E4M3, RTN4, INT8 = 0, 1, 2  # INT8: extension (per-channel weights, per-token activations)
KL, LOGITDIFF = 0, 1
LOSS, ACT = 0, 1
ACDC, RTN8, PAHQ = 0, 1, 2


class CqgPolicy(C.Structure):
    _fields_ = [("attention_default", C.c_int8), ("mlp_default", C.c_int8),
                ("embed_precision", C.c_int8), ("unembed_precision", C.c_int8),
                ("low_mode", C.c_int8), ("target_head_layer", C.c_int32),
                ("target_head_head", C.c_int32), ("target_mlp", C.c_int32)]


class CqgPrune(C.Structure):
    _fields_ = [("tau", C.c_double), ("max_steps", C.c_int32), ("min_change_rate", C.c_double),
                ("mode", C.c_int32), ("act_floor", C.c_double), ("per_edge_policy", C.c_int32),
                ("heads_only", C.c_int32), ("base", CqgPolicy)]


class CqgConfig(C.Structure):
    _fields_ = [("n_layers", C.c_uint32), ("n_heads", C.c_uint32), ("d_model", C.c_uint32),
                ("d_k", C.c_uint32), ("vocab", C.c_uint32), ("seq_len", C.c_uint32),
                ("has_mlp", C.c_uint32), ("qkv_split", C.c_uint32)]


class CqgStats(C.Structure):
    _fields_ = [("ms_total", C.c_double), ("ms_device", C.c_double), ("ms_baseline", C.c_double),
                ("ms_passes", C.c_double), ("passes", C.c_int64), ("kernel_launches", C.c_int64),
                ("fallback_elems", C.c_int64), ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
                ("unembed_rows", C.c_int64), ("unembed_exact_rows", C.c_int64)]


@dataclass
class PrecisionPolicy:
    """PrecisionPolicy (precision_policy.hpp:36-58)."""

    attention_default: int = P8
    mlp_default: int = P16
    embed_precision: int = P32
    unembed_precision: int = P32
    low_mode: int = E4M3
    target_head: Optional[tuple] = None  # (layer, head)
    target_mlp: Optional[int] = None

    @staticmethod
    def all_fp32():
        return PrecisionPolicy(P32, P32, P32, P32, E4M3)

    @staticmethod
    def all_low(mode=E4M3):
        return PrecisionPolicy(P8, P8, P8, P8, mode)

    @staticmethod
    def head_quantized(attention_default=P8, mode=E4M3):
        return PrecisionPolicy(attention_default, P16, P32, P32, mode)

    def c(self) -> CqgPolicy:
        th = self.target_head or (-1, -1)
        return CqgPolicy(self.attention_default, self.mlp_default, self.embed_precision,
                         self.unembed_precision, self.low_mode, th[0], th[1],
                         -1 if self.target_mlp is None else self.target_mlp)


@dataclass
class PruneConfig:
    """PruneConfig (acdc.hpp:19-36)."""

    tau: float = 0.01
    max_steps: int = 10
    min_change_rate: float = 0.0
    mode: int = LOSS
    act_floor: float = 0.0
    per_edge_policy: bool = False
    base_policy: PrecisionPolicy = field(default_factory=PrecisionPolicy)
    heads_only: bool = False

    def c(self) -> CqgPrune:
        return CqgPrune(self.tau, self.max_steps, self.min_change_rate, self.mode, self.act_floor,
                        int(self.per_edge_policy), int(self.heads_only), self.base_policy.c())


def ablation_policy(bits: int) -> PrecisionPolicy:
    """eval.cpp:1043-1050"""
    if bits == 4:
        return PrecisionPolicy.head_quantized(P8, RTN4)
    if bits == 8:
        return PrecisionPolicy.head_quantized(P8, E4M3)
    if bits == 16:
        return PrecisionPolicy.head_quantized(P16, E4M3)
    raise ValueError("ablation_policy: bits must be 4, 8, or 16")


def method_prune_config(method: int, bits: int = 8) -> PruneConfig:
    """eval.cpp:1052-1076"""
    if bits not in (4, 8, 16):
        raise ValueError("method_prune_config: bits must be 4, 8, or 16")
    if method != PAHQ and bits != 8:
        raise ValueError("method_prune_config: only pahq varies the bit width")
    if method == ACDC:
        return PruneConfig(per_edge_policy=False, base_policy=PrecisionPolicy.all_fp32())
    if method == RTN8:
        return PruneConfig(per_edge_policy=False, base_policy=PrecisionPolicy.all_low(E4M3))
    return PruneConfig(per_edge_policy=True, base_policy=ablation_policy(bits))


def threshold_grid(lo: float, hi: float, n: int) -> List[float]:
    """acdc.cpp:90-102"""
    import math
    if not (lo > 0.0) or not (hi > lo):
        raise ValueError("threshold_grid: need 0 < lo < hi")
    if n < 2:
        raise ValueError("threshold_grid: need n >= 2")
    llo, lhi = math.log(lo), math.log(hi)
    g = [math.exp(llo + (lhi - llo) * i / (n - 1)) for i in range(n)]
    g[0], g[-1] = lo, hi
    return g


@dataclass
class EdgeScore:
    edge: int
    score: float
    kept: bool


@dataclass
class IterationRecord:
    step: int
    present_before: int
    present_after: int
    scores: List[EdgeScore]


@dataclass
class CircuitResult:
    iterations: List[IterationRecord]
    final_mask: np.ndarray
    last_score: np.ndarray
    steps: int


@dataclass
class RocPoint:
    """RocPoint (eval.hpp): threshold, TPR, FPR, kept edges (+ iterations)."""
    tau: float
    tpr: float
    fpr: float
    kept: int
    steps: int = 0


@dataclass
class RocCurve:
    points: List[RocPoint]
    auc: float


def auc_from_points(points) -> float:
    """eval.cpp:1149-1166 (points: RocPoint or (tpr, fpr) pairs)."""
    pts = [(p.tpr, p.fpr) if isinstance(p, RocPoint) else tuple(p) for p in points]
    if not pts:
        raise ValueError("auc_from_points: no points")
    x = y = area = 0.0
    for tpr, fpr in sorted(pts, key=lambda p: (p[1], p[0])):
        if tpr <= y:
            continue
        if fpr > x:
            area += (fpr - x) * y
            x = fpr
        y = tpr
    return area + (1.0 - x) * y


_lib = None


def load_library():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with "
                           "`python -m paper_2510_23264_b200.build` (no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    lib.cqg_last_error.restype = C.c_char_p
    lib.cqg_fnv1a64.restype = C.c_uint64
    lib.cqg_fnv1a64.argtypes = [C.c_void_p, C.c_size_t]
    vp = C.c_void_p
    lib.cqg_create.argtypes = [C.POINTER(CqgConfig), vp, C.c_int, C.POINTER(vp)]
    lib.cqg_destroy.argtypes = [vp]
    lib.cqg_set_dataset.argtypes = [vp, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int]
    lib.cqg_get_unique_id.argtypes = [vp]
    lib.cqg_init_comm.argtypes = [vp, vp, C.c_int, C.c_int]
    lib.cqg_score_edges.argtypes = [vp, vp, vp, C.c_int, C.POINTER(CqgPolicy), C.c_int, C.c_int, vp]
    lib.cqg_run_acdc.argtypes = [vp, C.POINTER(CqgPrune), C.POINTER(C.c_int), vp, vp,
                                 C.POINTER(C.c_int), vp, vp, vp, vp, C.c_int]
    lib.cqg_quantize_matrix.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp]
    lib.cqg_roc_sweep.argtypes = [vp, C.POINTER(CqgPrune), vp, C.c_int, vp, C.c_int, vp, vp, vp, vp,
                                  C.POINTER(C.c_double)]
    lib.cqg_forward.argtypes = [vp, vp, vp, C.POINTER(CqgPolicy), C.c_int, vp, vp]
    lib.cqg_circuit_stats.argtypes = [vp, vp, vp, vp, vp]
    lib.cqg_graph_info.argtypes = [C.POINTER(CqgConfig), C.POINTER(C.c_int), C.POINTER(C.c_int)]
    lib.cqg_graph_edges.argtypes = [C.POINTER(CqgConfig), vp, vp]
    lib.cqg_last_stats.argtypes = [vp, C.POINTER(CqgStats)]
    lib.cqg_set_option.argtypes = [vp, C.c_char_p, C.c_int64]
    lib.cqg_profile_count.argtypes = [vp]
    lib.cqg_profile_entry.argtypes = [vp, C.c_int, C.c_char_p, vp, vp, vp, vp]
    lib.cqg_diag_e4m3_range.argtypes = [C.c_uint32, C.c_uint64, vp]
    lib.cqg_diag_bf16_range.argtypes = [C.c_uint32, C.c_uint64, vp]
    lib.cqg_diag_libm_range.argtypes = [C.c_int, C.c_uint32, C.c_uint64, vp]
    _lib = lib
    return lib


class CqgError(RuntimeError):
    pass


def _check(rc: int):
    if rc == 0:
        return
    msg = load_library().cqg_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 3:
        raise MemoryError(msg)
    raise CqgError(msg)


def _vp(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def fnv1a64(data: bytes) -> int:
    lib = load_library()
    buf = (C.c_char * len(data)).from_buffer_copy(data)
    return int(lib.cqg_fnv1a64(C.cast(buf, C.c_void_p), len(data)))


def config_struct(cfg: ModelConfig, qkv_split: bool = False) -> CqgConfig:
    return CqgConfig(cfg.n_layers, cfg.n_heads, cfg.d_model, cfg.d_k, cfg.vocab, cfg.seq_len,
                     cfg.has_mlp, int(bool(qkv_split)))


def graph_edges(cfg: ModelConfig, qkv_split: bool = False):
    """Edge list in the reference numbering (model.cpp:192-201); qkv_split:
    the Q/K/V-split graph (extension, include/cqg.h)."""
    lib = load_library()
    c = config_struct(cfg, qkv_split)
    nn, ne = C.c_int(), C.c_int()
    _check(lib.cqg_graph_info(C.byref(c), C.byref(nn), C.byref(ne)))
    src = np.empty(ne.value, np.int32)
    dst = np.empty(ne.value, np.int32)
    _check(lib.cqg_graph_edges(C.byref(c), _vp(src), _vp(dst)))
    return nn.value, src, dst


def graph_edge_comp(cfg: ModelConfig, qkv_split: bool = False) -> np.ndarray:
    """Receiver component of each edge: 0/1/2 = q/k/v input of a split head."""
    lib = load_library()
    c = config_struct(cfg, qkv_split)
    nn, ne = C.c_int(), C.c_int()
    _check(lib.cqg_graph_info(C.byref(c), C.byref(nn), C.byref(ne)))
    comp = np.empty(ne.value, np.int32)
    _check(lib.cqg_graph_edge_comp(C.byref(c), _vp(comp)))
    return comp


def sweep_order(cfg: ModelConfig, mask: np.ndarray, qkv_split: bool = False) -> np.ndarray:
    """model.cpp:238-246 (dst descending, src descending within a dst; split
    graph: receiver descending)."""
    idx = np.nonzero(np.asarray(mask, bool))[0]
    # edges are numbered receiver-major ascending, src ascending -> reverse order
    return idx[::-1].astype(np.int32)


class Engine:
    """One GPU context (cqg_ctx): HBM-resident weights + dataset shard."""

    def __init__(self, weights: WeightSet, device: int = 0, options: Optional[dict] = None,
                 qkv_split: bool = False):
        """options: cqg_set_option knobs applied at creation (after any given
        in the CQG_OPTS environment variable, "key=value,key=value").
        qkv_split: the Q/K/V-split edge graph (extension, include/cqg.h)."""
        self.lib = load_library()
        self.cfg = weights.cfg
        self.cfg.validate()
        self._mats = [np.ascontiguousarray(m, np.float32) for m in weights.mats]
        ptrs = (C.c_void_p * len(self._mats))(*[m.ctypes.data for m in self._mats])
        self.qkv_split = bool(qkv_split)
        c = config_struct(self.cfg, self.qkv_split)
        h = C.c_void_p()
        _check(self.lib.cqg_create(C.byref(c), C.cast(ptrs, C.c_void_p), device, C.byref(h)))
        self.h = h
        self._mats = None  # copied into HBM
        self.n_nodes, self.edge_src, self.edge_dst = graph_edges(self.cfg, self.qkv_split)
        self.n_edges = len(self.edge_src)
        self.n_items = 0
        opts = {}
        for kv in filter(None, os.environ.get("CQG_OPTS", "").split(",")):
            k, v = kv.split("=")
            opts[k.strip()] = int(v)
        opts.update(options or {})
        for k, v in opts.items():
            self.set_option(k, v)

    def close(self):
        if getattr(self, "h", None):
            self.lib.cqg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_dataset(self, ds: Dataset, metric: int = KL, item_offset: int = 0,
                    item_total: Optional[int] = None):
        validate_dataset(ds, self.cfg)
        cl = np.ascontiguousarray(ds.clean, np.int32)
        co = np.ascontiguousarray(ds.corrupt, np.int32)
        an = np.ascontiguousarray(ds.answer, np.int32)
        di = np.ascontiguousarray(ds.distractor, np.int32)
        _check(self.lib.cqg_set_dataset(self.h, _vp(cl), _vp(co), _vp(an), _vp(di), len(ds),
                                        item_offset, item_total or len(ds), metric))
        self.n_items = len(ds)

    def init_comm(self, unique_id: bytes, rank: int, world: int):
        buf = (C.c_char * 128).from_buffer_copy(unique_id)
        _check(self.lib.cqg_init_comm(self.h, C.cast(buf, C.c_void_p), rank, world))

    @staticmethod
    def unique_id() -> bytes:
        lib = load_library()
        buf = (C.c_char * 128)()
        _check(lib.cqg_get_unique_id(C.cast(buf, C.c_void_p)))
        return bytes(buf)

    def score_edges(self, mask, edges, base: PrecisionPolicy, per_edge_policy: bool = True,
                    mode: int = LOSS) -> np.ndarray:
        m = np.ascontiguousarray(np.asarray(mask, bool), np.uint8)
        e = np.ascontiguousarray(edges, np.int32)
        out = np.empty(e.size, np.float64)
        p = base.c()
        _check(self.lib.cqg_score_edges(self.h, _vp(m), _vp(e), e.size, C.byref(p),
                                        int(per_edge_policy), mode, _vp(out)))
        return out

    def run_acdc(self, prune: PruneConfig) -> CircuitResult:
        E = self.n_edges
        cap = E * max(1, prune.max_steps)
        steps, nrec = C.c_int(), C.c_int()
        fm = np.empty(E, np.uint8)
        ls = np.empty(E, np.float64)
        rs, re_ = np.empty(cap, np.int32), np.empty(cap, np.int32)
        rsc, rk = np.empty(cap, np.float64), np.empty(cap, np.uint8)
        pc = prune.c()
        _check(self.lib.cqg_run_acdc(self.h, C.byref(pc), C.byref(steps), _vp(fm), _vp(ls),
                                     C.byref(nrec), _vp(rs), _vp(re_), _vp(rsc), _vp(rk), cap))
        n = min(nrec.value, cap)
        its: List[IterationRecord] = []
        present = E
        for i in range(n):
            if not its or its[-1].step != rs[i]:
                its.append(IterationRecord(int(rs[i]), present, present, []))
            its[-1].scores.append(EdgeScore(int(re_[i]), float(rsc[i]), bool(rk[i])))
            if not rk[i]:
                present -= 1
            its[-1].present_after = present
        return CircuitResult(its, fm.astype(bool), ls, steps.value)

    def roc_sweep(self, prune: PruneConfig, taus: Sequence[float], ground_truth) -> "RocCurve":
        """roc_sweep (eval.cpp:1193-1226) through cqg_roc_sweep: iteration 1 is
        scored once and shared across the thresholds."""
        t = np.ascontiguousarray(taus, np.float64)
        gt = np.ascontiguousarray(sorted(set(int(x) for x in ground_truth)), np.int32)
        n = t.size
        tpr, fpr = np.empty(n), np.empty(n)
        kept, steps = np.empty(n, np.int32), np.empty(n, np.int32)
        auc = C.c_double()
        pc = prune.c()
        _check(self.lib.cqg_roc_sweep(self.h, C.byref(pc), _vp(t), n, _vp(gt), gt.size, _vp(tpr),
                                      _vp(fpr), _vp(kept), _vp(steps), C.byref(auc)))
        pts = [RocPoint(float(t[i]), float(tpr[i]), float(fpr[i]), int(kept[i]), int(steps[i]))
               for i in range(n)]
        return RocCurve(pts, auc.value)

    def quantize_matrix(self, idx: int, precision: int, low_mode: int = E4M3) -> np.ndarray:
        shape = self.cfg.matrix_specs()[idx][1]
        out = np.empty(int(np.prod(shape)), np.float32)
        _check(self.lib.cqg_quantize_matrix(self.h, idx, precision, low_mode, _vp(out)))
        return out.reshape(shape)

    def forward(self, tokens, policy: PrecisionPolicy, mask=None, patch_edge: int = -1,
                patch_value=None) -> np.ndarray:
        c = self.cfg
        SD = c.seq_len * c.d_model
        outs = np.empty((self.n_nodes - 1) * SD + c.seq_len * c.vocab, np.float32)
        tok = np.ascontiguousarray(tokens, np.int32)
        m = None if mask is None else np.ascontiguousarray(np.asarray(mask, bool), np.uint8)
        pv = None if patch_value is None else np.ascontiguousarray(patch_value, np.float32)
        p = policy.c()
        _check(self.lib.cqg_forward(self.h, _vp(tok), None if m is None else _vp(m), C.byref(p),
                                    patch_edge, None if pv is None else _vp(pv), _vp(outs)))
        return outs

    def stats(self) -> dict:
        s = CqgStats()
        _check(self.lib.cqg_last_stats(self.h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in CqgStats._fields_}

    def profile(self) -> dict:
        """Per-kernel-class totals of the last score call (cqg_profile_entry)."""
        out = {}
        n = self.lib.cqg_profile_count(self.h)
        for i in range(n):
            name = C.create_string_buffer(64)
            ms, fl, by = C.c_double(), C.c_double(), C.c_double()
            la = C.c_int64()
            _check(self.lib.cqg_profile_entry(self.h, i, name, C.byref(ms), C.byref(fl),
                                              C.byref(by), C.byref(la)))
            out[name.value.decode()] = {"ms": ms.value, "flops": fl.value, "bytes": by.value,
                                        "launches": la.value}
        return out

    def set_option(self, key: str, value: int):
        _check(self.lib.cqg_set_option(self.h, key.encode(), int(value)))


class DeltaLEngine:
    """Facade with the reference's DeltaLEngine surface (patching.hpp:69-121).

    Baselines are refreshed inside every device call, so refresh_baselines /
    prepare_policy only record the mask, mirroring the reference's contract
    (scoring throws if the mask changed since the last refresh)."""

    def __init__(self, engine: Engine, dataset: Dataset, metric: int = KL):
        self.engine = engine
        self.metric = metric
        engine.set_dataset(dataset, metric)
        self._mask = np.ones(engine.n_edges, bool)
        self._refreshed = None

    def set_mask(self, mask):
        self._mask = np.asarray(mask, bool).copy()

    def prepare_policy(self, policy: PrecisionPolicy):
        pass

    def refresh_baselines(self, policy: PrecisionPolicy):
        self._refreshed = self._mask.copy()

    def _check_fresh(self):
        if self._refreshed is None or not np.array_equal(self._refreshed, self._mask):
            raise RuntimeError("DeltaLEngine: baselines stale for mask; call refresh_baselines")

    def delta_l(self, edge: int, policy: PrecisionPolicy) -> float:
        self._check_fresh()
        return float(self.engine.score_edges(self._mask, [edge], policy, False, LOSS)[0])

    def act_diff(self, edge: int, policy: PrecisionPolicy) -> float:
        self._check_fresh()
        return float(self.engine.score_edges(self._mask, [edge], policy, False, ACT)[0])

    def score(self, edge: int, policy: PrecisionPolicy, mode: int) -> float:
        return self.delta_l(edge, policy) if mode == LOSS else self.act_diff(edge, policy)

    def epsilon_precision(self, edge: int, low: PrecisionPolicy) -> float:
        """|delta_l(e, all_fp32) - delta_l(e, low)| (patching.cpp:266-268)."""
        return abs(self.delta_l(edge, PrecisionPolicy.all_fp32()) - self.delta_l(edge, low))


@dataclass
class CircuitStats:
    clean_ld: np.ndarray
    corrupt_ld: np.ndarray
    circuit_ld: np.ndarray


def _mean(xs) -> float:
    s = 0.0
    for x in xs:  # sequential, as eval.cpp's mean()
        s += float(x)
    return s / len(xs)


def circuit_stats(engine: "Engine", mask) -> CircuitStats:
    """eval.cpp:960-985 on the GPU: clean / corrupt / circuit last-row logit
    differences at FP32 for the engine's dataset (absent edges read the
    corrupt run)."""
    m = np.ascontiguousarray(np.asarray(mask, bool), np.uint8)
    if m.size != engine.n_edges:
        raise ValueError("circuit_stats: mask size mismatch")
    n = engine.n_items
    cl, co, ci = np.empty(n), np.empty(n), np.empty(n)
    _check(engine.lib.cqg_circuit_stats(engine.h, _vp(m), _vp(cl), _vp(co), _vp(ci)))
    return CircuitStats(cl, co, ci)


def faithfulness(engine: "Engine", mask) -> float:
    """eval.cpp:1240-1247"""
    st = circuit_stats(engine, mask)
    denom = _mean(st.clean_ld) - _mean(st.corrupt_ld)
    if abs(denom) < 1e-9:
        raise RuntimeError("faithfulness: degenerate clean-corrupt gap")
    return (_mean(st.circuit_ld) - _mean(st.corrupt_ld)) / denom


def task_accuracy(engine: "Engine", mask) -> float:
    """eval.cpp:1249-1254"""
    st = circuit_stats(engine, mask)
    return float(sum(1 for ld in st.circuit_ld if ld > 0.0)) / len(st.circuit_ld)


@dataclass
class EpsilonReport:
    eps: np.ndarray   # per present edge, sweep order
    edges: np.ndarray
    eps_mean: float
    eps_max: float


def epsilon_report(engine: Engine, mask, prune: PruneConfig) -> EpsilonReport:
    """The run-acdc epsilon post-pass (proj/tools/circuitquant_main.cpp:280-299):
    over the edges that survived, the score error the method's precision
    introduces, |delta_l(e, all_fp32) - delta_l(e, policy(e))|, as two batched
    device calls (FP32 and the method's per-edge policies) instead of two
    delta_l per edge."""
    mask = np.asarray(mask, bool)
    edges = sweep_order(engine.cfg, mask)
    if edges.size == 0:
        return EpsilonReport(np.zeros(0), edges, 0.0, 0.0)
    full = engine.score_edges(mask, edges, PrecisionPolicy.all_fp32(), False, LOSS)
    low = engine.score_edges(mask, edges, prune.base_policy, prune.per_edge_policy, LOSS)
    eps = np.abs(full - low)
    total = 0.0
    for x in eps:  # sequential, as the reference accumulates
        total += float(x)
    return EpsilonReport(eps, edges, total / eps.size, float(eps.max()))


def run_acdc(engine: Engine, prune: PruneConfig) -> CircuitResult:
    """run_acdc (acdc.cpp:23-88): greedy loop in C++ inside libcqg.so."""
    return engine.run_acdc(prune)


def diag_e4m3(lo: int, count: int) -> np.ndarray:
    out = np.empty(count, np.uint8)
    _check(load_library().cqg_diag_e4m3_range(lo, count, _vp(out)))
    return out


def diag_bf16(lo: int, count: int) -> np.ndarray:
    out = np.empty(count, np.uint16)
    _check(load_library().cqg_diag_bf16_range(lo, count, _vp(out)))
    return out


def diag_libm(which: int, lo: int, count: int) -> np.ndarray:
    out = np.empty(count, np.float32)
    _check(load_library().cqg_diag_libm_range(which, lo, count, _vp(out)))
    return out
