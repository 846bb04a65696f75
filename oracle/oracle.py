"""ctypes bindings for the CHECKERS (test infrastructure only).

* ``Ref``  — the unmodified reference library compiled in place
  (oracle/_ref/libcqref.so, see oracle/Makefile + ref_shim.cpp).
* ``Port`` — our plain-C restatement (oracle/libcqoracle.so, cq_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libcqref.so")
PORT_SO = os.path.join(HERE, "libcqoracle.so")

P8, P16, P32 = 0, 1, 2
E4M3, RTN4, INT8 = 0, 1, 2  # INT8: extension (per-channel weights, per-token activations)
KL, LOGITDIFF = 0, 1


class Policy(C.Structure):
    _fields_ = [("attention_default", C.c_int8), ("mlp_default", C.c_int8),
                ("embed_precision", C.c_int8), ("unembed_precision", C.c_int8),
                ("low_mode", C.c_int8), ("target_head_layer", C.c_int32),
                ("target_head_head", C.c_int32), ("target_mlp", C.c_int32)]

    @staticmethod
    def make(att=P8, mlp=P16, emb=P32, unemb=P32, mode=E4M3, th=None, tm=None):
        p = Policy(att, mlp, emb, unemb, mode, -1, -1, -1)
        if th is not None:
            p.target_head_layer, p.target_head_head = th
        if tm is not None:
            p.target_mlp = tm
        return p

    # precision_policy.hpp:85-109
    @staticmethod
    def head_quantized(att=P8, mode=E4M3):
        return Policy.make(att, P16, P32, P32, mode)

    @staticmethod
    def all_fp32():
        return Policy.make(P32, P32, P32, P32, E4M3)

    @staticmethod
    def all_low(mode=E4M3):
        return Policy.make(P8, P8, P8, P8, mode)


class Prune(C.Structure):
    _fields_ = [("tau", C.c_double), ("max_steps", C.c_int32), ("min_change_rate", C.c_double),
                ("mode", C.c_int32), ("act_floor", C.c_double), ("per_edge_policy", C.c_int32),
                ("heads_only", C.c_int32), ("base", Policy)]


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class AcdcResult:
    def __init__(self, steps, final_mask, last_score, records):
        self.steps = steps
        self.final_mask = final_mask
        self.last_score = last_score
        self.records = records  # list of (step, edge, score, kept)


class Ref:
    """The reference library (proj/src/*.cpp) behind ref_shim.cpp."""

    _lib = None

    def __init__(self):
        if Ref._lib is None:
            if not os.path.exists(REF_SO):
                raise RuntimeError(f"{REF_SO} missing: run `make -C oracle ref` where "
                                   "/root/reference exists")
            lib = C.CDLL(REF_SO)
            lib.cqref_last_error.restype = C.c_char_p
            lib.cqref_decode_f8.restype = C.c_double
            lib.cqref_encode_f8.restype = C.c_uint8
            lib.cqref_encode_f8.argtypes = [C.c_double]
            lib.cqref_encode_bf16.restype = C.c_uint16
            lib.cqref_encode_bf16.argtypes = [C.c_float]
            lib.cqref_metric_kl.restype = C.c_double
            lib.cqref_encode_f8_range.argtypes = [C.c_uint32, C.c_uint64, C.c_void_p]
            lib.cqref_encode_bf16_range.argtypes = [C.c_uint32, C.c_uint64, C.c_void_p]
            lib.cqref_gen_random.argtypes = [C.c_void_p, C.c_uint32, C.c_float, C.c_int,
                                             C.c_uint32, C.c_char_p, C.c_char_p]
            lib.cqref_gen_planted.argtypes = [C.c_int, C.c_uint32, C.c_int, C.c_double, C.c_char_p]
            lib.cqref_open.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
            lib.cqref_close.argtypes = [C.c_void_p]
            lib.cqref_threshold_grid.argtypes = [C.c_double, C.c_double, C.c_int, C.c_void_p]
            Ref._lib = lib
        self.lib = Ref._lib

    def check(self, rc):
        if rc != 0:
            msg = self.lib.cqref_last_error().decode()
            raise (ValueError if rc == 1 else RuntimeError)(msg)

    def set_threads(self, n):
        self.lib.cqref_set_threads(n)

    def max_threads(self):
        return self.lib.cqref_max_threads()

    # numerics
    def encode_f8(self, x: float) -> int:
        return self.lib.cqref_encode_f8(float(x))

    def encode_f8_range(self, lo: int, count: int) -> np.ndarray:
        out = np.empty(count, np.uint8)
        self.lib.cqref_encode_f8_range(lo, count, out.ctypes.data_as(C.c_void_p))
        return out

    def encode_bf16_range(self, lo: int, count: int) -> np.ndarray:
        out = np.empty(count, np.uint16)
        self.lib.cqref_encode_bf16_range(lo, count, out.ctypes.data_as(C.c_void_p))
        return out

    def quantize_rtn(self, x: np.ndarray, bits: int):
        x = np.ascontiguousarray(x, np.float32).copy()
        d = C.c_double()
        self.check(self.lib.cqref_quantize_rtn_f32(_p(x, C.c_float), C.c_int64(x.size), bits,
                                                   C.byref(d)))
        return x, d.value

    def quantize_rtn_f64(self, x, bits):
        x = np.ascontiguousarray(x, np.float64).copy()
        d = C.c_double()
        self.check(self.lib.cqref_quantize_rtn_f64(_p(x, C.c_double), C.c_int64(x.size), bits,
                                                   C.byref(d)))
        return x, d.value

    def metric_kl(self, c, p):
        c = np.ascontiguousarray(c, np.float32)
        p = np.ascontiguousarray(p, np.float32)
        return self.lib.cqref_metric_kl(_p(c, C.c_float), _p(p, C.c_float), C.c_int64(c.size))

    def threshold_grid(self, lo, hi, n):
        out = np.empty(n, np.float64)
        self.lib.cqref_threshold_grid(lo, hi, n, out.ctypes.data_as(C.c_void_p))
        return out

    # generators
    def gen_random(self, cfg8, wseed, items, dseed, wpath, dpath, wscale=0.0):
        c = np.asarray(cfg8, np.uint32)
        self.check(self.lib.cqref_gen_random(c.ctypes.data_as(C.c_void_p), wseed, wscale, items, dseed,
                                             (wpath or "").encode(), (dpath or "").encode()))

    def gen_planted(self, preset, seed, outdir, items=6, signal_scale=1.0):
        self.check(self.lib.cqref_gen_planted(preset, seed, items, signal_scale, outdir.encode()))

    def roc_sweep(self, taskdir, method, taus, metric=LOGITDIFF, bits=8):
        taus = np.ascontiguousarray(taus, np.float64)
        n = taus.size
        tpr, fpr = np.empty(n), np.empty(n)
        kept = np.empty(n, np.int32)
        auc = C.c_double()
        self.check(self.lib.cqref_roc_sweep(taskdir.encode(), method, bits, metric,
                                            _p(taus, C.c_double), n, _p(tpr, C.c_double),
                                            _p(fpr, C.c_double), _p(kept, C.c_int),
                                            C.byref(auc)))
        return auc.value, tpr, fpr, kept

    def faithfulness(self, taskdir, mask):
        """(faithfulness, task_accuracy) of the reference (eval.cpp:1240-1254)."""
        m = np.ascontiguousarray(mask, np.uint8)
        f, a = C.c_double(), C.c_double()
        self.check(self.lib.cqref_faithfulness(taskdir.encode(), m.ctypes.data_as(C.c_void_p), m.size,
                                               C.byref(f), C.byref(a)))
        return f.value, a.value

    def method_config(self, method, bits=8) -> Prune:
        p = Prune()
        self.check(self.lib.cqref_method_config(method, bits, C.byref(p)))
        return p

    def graph(self, cfg8):
        c = np.asarray(cfg8, np.uint32)
        nn, ne = C.c_int(), C.c_int()
        self.check(self.lib.cqref_graph(c.ctypes.data_as(C.c_void_p), C.byref(nn), C.byref(ne), None, None, None,
                                        None, None))
        kind = np.empty(nn.value, np.int32)
        layer, head = np.empty_like(kind), np.empty_like(kind)
        src = np.empty(ne.value, np.int32)
        dst = np.empty_like(src)
        self.check(self.lib.cqref_graph(c.ctypes.data_as(C.c_void_p), C.byref(nn), C.byref(ne), kind.ctypes.data_as(C.c_void_p),
                                        layer.ctypes.data_as(C.c_void_p), head.ctypes.data_as(C.c_void_p), src.ctypes.data_as(C.c_void_p),
                                        dst.ctypes.data_as(C.c_void_p)))
        return kind, layer, head, src, dst

    def sweep_order(self, cfg8, mask=None):
        c = np.asarray(cfg8, np.uint32)
        _, _, _, src, _ = self.graph(cfg8)
        out = np.empty(src.size, np.int32)
        n = C.c_int()
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        self.check(self.lib.cqref_sweep_order(c.ctypes.data_as(C.c_void_p), None if m is None else m.ctypes.data_as(C.c_void_p),
                                              out.ctypes.data_as(C.c_void_p), C.byref(n)))
        return out[:n.value]

    def open(self, wpath, dpath, metric=KL) -> "RefModel":
        h = C.c_void_p()
        self.check(self.lib.cqref_open(wpath.encode(), dpath.encode(), metric, C.byref(h)))
        return RefModel(self, h)


class RefModel:
    def __init__(self, ref: Ref, h):
        self.ref, self.lib, self.h = ref, ref.lib, h
        cfg = np.empty(8, np.uint32)
        items = C.c_int()
        ref.check(self.lib.cqref_config(h, cfg.ctypes.data_as(C.c_void_p), C.byref(items)))
        self.cfg8 = [int(x) for x in cfg]
        self.items = items.value
        L, H, D, dk, V, S, _, mlp = self.cfg8
        self.n_nodes = 2 + L * (H + mlp)
        self.n_edges = len(ref.graph(self.cfg8)[3])
        self.S, self.D, self.V = S, D, V

    def close(self):
        if self.h:
            self.lib.cqref_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def image(self, idx, precision, mode, size):
        out = np.empty(size, np.float32)
        self.ref.check(self.lib.cqref_image(self.h, idx, precision, mode, out.ctypes.data_as(C.c_void_p)))
        return out

    def forward(self, tokens, policy: Policy, mask=None, patch_edge=-1, patch_value=None,
                with_inputs=False):
        tok = np.ascontiguousarray(tokens, np.int32)
        SD = self.S * self.D
        outs = np.empty((self.n_nodes - 1) * SD + self.S * self.V, np.float32)
        ins = np.empty(self.n_nodes * SD, np.float32) if with_inputs else None
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        pv = None if patch_value is None else np.ascontiguousarray(patch_value, np.float32)
        self.ref.check(self.lib.cqref_forward(
            self.h, tok.ctypes.data_as(C.c_void_p), None if m is None else m.ctypes.data_as(C.c_void_p), C.byref(policy),
            patch_edge, None if pv is None else pv.ctypes.data_as(C.c_void_p), outs.ctypes.data_as(C.c_void_p),
            None if ins is None else ins.ctypes.data_as(C.c_void_p)))
        return (outs, ins) if with_inputs else outs

    def score_edges(self, edges, policy: Policy, per_edge=True, mode=0, mask=None):
        e = np.ascontiguousarray(edges, np.int32)
        out = np.empty(e.size, np.float64)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        self.ref.check(self.lib.cqref_score_edges(self.h, None if m is None else m.ctypes.data_as(C.c_void_p),
                                                  e.ctypes.data_as(C.c_void_p), e.size, C.byref(policy),
                                                  int(per_edge), mode, out.ctypes.data_as(C.c_void_p)))
        return out

    def time_delta_l(self, edges, policy: Policy, per_edge=True):
        """(scores, ms_refresh, ms_score): delta_l over edges in an OpenMP
        parallel-for (acdc.cpp:55-60), baseline refresh timed separately."""
        e = np.ascontiguousarray(edges, np.int32)
        out = np.empty(e.size, np.float64)
        mr, ms = C.c_double(), C.c_double()
        self.ref.check(self.lib.cqref_time_delta_l(self.h, e.ctypes.data_as(C.c_void_p), e.size,
                                                   C.byref(policy), int(per_edge),
                                                   out.ctypes.data_as(C.c_void_p), C.byref(mr),
                                                   C.byref(ms)))
        return out, mr.value, ms.value

    def run_acdc(self, prune: Prune) -> AcdcResult:
        E = self.n_edges
        cap = E * max(1, prune.max_steps)
        steps = C.c_int()
        fm = np.empty(E, np.uint8)
        ls = np.empty(E, np.float64)
        nrec = C.c_int()
        rs, re_ = np.empty(cap, np.int32), np.empty(cap, np.int32)
        rsc, rk = np.empty(cap, np.float64), np.empty(cap, np.uint8)
        self.ref.check(self.lib.cqref_run_acdc(self.h, C.byref(prune), C.byref(steps),
                                               fm.ctypes.data_as(C.c_void_p), ls.ctypes.data_as(C.c_void_p), C.byref(nrec),
                                               rs.ctypes.data_as(C.c_void_p), re_.ctypes.data_as(C.c_void_p), rsc.ctypes.data_as(C.c_void_p),
                                               rk.ctypes.data_as(C.c_void_p), cap))
        n = min(nrec.value, cap)
        recs = list(zip(rs[:n].tolist(), re_[:n].tolist(), rsc[:n].tolist(), rk[:n].tolist()))
        return AcdcResult(steps.value, fm.astype(bool), ls, recs)


class Port:
    """Our plain-C restatement (cq_oracle.c)."""

    _lib = None

    def __init__(self, cfg, mats, qkv_split=False):
        if Port._lib is None:
            if not os.path.exists(PORT_SO):
                raise RuntimeError(f"{PORT_SO} missing: run `make -C oracle port`")
            lib = C.CDLL(PORT_SO)
            lib.cqo_last_error.restype = C.c_char_p
            lib.cqo_model_new.restype = C.c_void_p
            lib.cqo_model_new_split.restype = C.c_void_p
            lib.cqo_model_free.argtypes = [C.c_void_p]
            lib.cqo_encode_f8.restype = C.c_uint8
            lib.cqo_encode_f8.argtypes = [C.c_double]
            lib.cqo_encode_bf16.restype = C.c_uint16
            lib.cqo_encode_bf16.argtypes = [C.c_float]
            lib.cqo_metric_kl.restype = C.c_double
            lib.cqo_metric_kl.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
            for fn in ("cqo_n_nodes", "cqo_n_edges", "cqo_graph", "cqo_sweep_order", "cqo_image",
                       "cqo_forward", "cqo_score_edges", "cqo_run_acdc"):
                getattr(lib, fn).argtypes = None
            Port._lib = lib
        self.lib = Port._lib
        self.cfg = cfg
        self._mats = [np.ascontiguousarray(m, np.float32) for m in mats]
        ptrs = (C.c_void_p * len(self._mats))(*[m.ctypes.data_as(C.c_void_p) for m in self._mats])
        c7 = np.asarray([cfg.n_layers, cfg.n_heads, cfg.d_model, cfg.d_k, cfg.vocab, cfg.seq_len,
                         cfg.has_mlp], np.uint32)
        self.qkv_split = bool(qkv_split)
        self.h = self.lib.cqo_model_new_split(c7.ctypes.data_as(C.c_void_p), ptrs, int(self.qkv_split))
        if not self.h:
            raise ValueError(self.lib.cqo_last_error().decode())
        self.h = C.c_void_p(self.h)
        self.n_nodes = self.lib.cqo_n_nodes(self.h)
        self.n_edges = self.lib.cqo_n_edges(self.h)

    def __del__(self):
        try:
            if self.h:
                self.lib.cqo_model_free(self.h)
        except Exception:
            pass

    def check(self, rc):
        if rc != 0:
            msg = self.lib.cqo_last_error().decode()
            raise (ValueError if rc == 1 else RuntimeError)(msg)

    def graph(self):
        k = np.empty(self.n_nodes, np.int32)
        l, h = np.empty_like(k), np.empty_like(k)
        s = np.empty(self.n_edges, np.int32)
        d = np.empty_like(s)
        self.lib.cqo_graph(self.h, k.ctypes.data_as(C.c_void_p), l.ctypes.data_as(C.c_void_p),
                           h.ctypes.data_as(C.c_void_p), s.ctypes.data_as(C.c_void_p),
                           d.ctypes.data_as(C.c_void_p))
        return k, l, h, s, d

    def edge_comp(self):
        """Receiver component per edge: 0/1/2 = q/k/v input of a head (split
        graph), 0 otherwise."""
        c = np.empty(self.n_edges, np.int32)
        self.lib.cqo_graph_comp(self.h, c.ctypes.data_as(C.c_void_p))
        return c

    def sweep_order(self, mask=None):
        out = np.empty(self.n_edges, np.int32)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        n = self.lib.cqo_sweep_order(self.h, None if m is None else m.ctypes.data_as(C.c_void_p),
                                     out.ctypes.data_as(C.c_void_p))
        return out[:n]

    def image(self, idx, precision, mode):
        out = np.empty(self._mats[idx].size, np.float32)
        self.check(self.lib.cqo_image(self.h, C.c_int(idx), C.c_int(precision), C.c_int(mode),
                                      out.ctypes.data_as(C.c_void_p)))
        return out

    def forward(self, tokens, policy: Policy, mask=None, patch_edge=-1, patch_value=None):
        c = self.cfg
        SD = c.seq_len * c.d_model
        outs = np.empty((self.n_nodes - 1) * SD + c.seq_len * c.vocab, np.float32)
        tok = np.ascontiguousarray(tokens, np.int32)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        pv = None if patch_value is None else np.ascontiguousarray(patch_value, np.float32)
        self.check(self.lib.cqo_forward(self.h, tok.ctypes.data_as(C.c_void_p),
                                        None if m is None else m.ctypes.data_as(C.c_void_p),
                                        C.byref(policy), C.c_int(patch_edge),
                                        None if pv is None else pv.ctypes.data_as(C.c_void_p),
                                        outs.ctypes.data_as(C.c_void_p)))
        return outs

    def _ds(self, ds):
        return [np.ascontiguousarray(a, np.int32) for a in (ds.clean, ds.corrupt, ds.answer,
                                                            ds.distractor)]

    def score_edges(self, ds, edges, policy: Policy, per_edge=True, metric=KL, mode=0, mask=None):
        cl, co, an, di = self._ds(ds)
        e = np.ascontiguousarray(edges, np.int32)
        out = np.empty(e.size, np.float64)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        v = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        self.check(self.lib.cqo_score_edges(self.h, v(cl), v(co), v(an), v(di), C.c_int(len(ds)),
                                            None if m is None else v(m), v(e), C.c_int(e.size),
                                            C.byref(policy), C.c_int(int(per_edge)),
                                            C.c_int(metric), C.c_int(mode), v(out)))
        return out

    def run_acdc(self, ds, prune: Prune, metric=KL) -> AcdcResult:
        cl, co, an, di = self._ds(ds)
        E = self.n_edges
        cap = E * max(1, prune.max_steps)
        steps, nrec = C.c_int(), C.c_int()
        fm = np.empty(E, np.uint8)
        ls = np.empty(E, np.float64)
        rs, re_ = np.empty(cap, np.int32), np.empty(cap, np.int32)
        rsc, rk = np.empty(cap, np.float64), np.empty(cap, np.uint8)
        v = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        self.check(self.lib.cqo_run_acdc(self.h, v(cl), v(co), v(an), v(di), C.c_int(len(ds)),
                                         C.c_int(metric), C.byref(prune), C.byref(steps), v(fm),
                                         v(ls), C.byref(nrec), v(rs), v(re_), v(rsc), v(rk),
                                         C.c_int(cap)))
        n = min(nrec.value, cap)
        recs = list(zip(rs[:n].tolist(), re_[:n].tolist(), rsc[:n].tolist(), rk[:n].tolist()))
        return AcdcResult(steps.value, fm.astype(bool), ls, recs)


def ref_available() -> bool:
    return os.path.exists(REF_SO)
