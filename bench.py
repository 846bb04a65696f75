#!/usr/bin/env python
"""Benchmark of the PAHQ-ACDC patched-forward hot path (BASELINE.json metric:
"patched forward passes/sec and ACDC end-to-end s").

One STEP = scoring every present edge of ACDC iteration 1 (full mask; the
run_acdc scoring block, proj/src/acdc.cpp:42-60) over the whole prompt batch,
i.e. n_edges x items patched passes, through the C-ABI cqg_score_edges.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config gpt2s]
    python bench.py --impl reference ...    # reference CPU path on host cores

Multi-GPU (torchrun, one rank per GPU): the prompt batch is sharded over
ranks, per-edge partial KL sums are NCCL-allreduced inside libcqg.so; value
is whole-job passes/s over the max-over-ranks device time ("strong" scaling:
the total batch is fixed).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2510_23264_b200 import formats, synth  # noqa: E402
from paper_2510_23264_b200 import shard as shard_mod  # noqa: E402

CONFIGS = {
    # BASELINE.json configs[1]: GPT-2-small shape, IOI-shaped prompts, batch 64
    "gpt2s": dict(cfg=formats.ModelConfig(12, 12, 768, 64, 50257, 16, 1, 1), items=64,
                  data="ioi"),
    # configs[0]: toy attention-only transformer, batch 16
    "toy": dict(cfg=formats.ModelConfig(2, 4, 128, 32, 512, 16, 1, 0), items=16, data="random"),
    # configs[2]: GPT-2-small shape, Greater-Than-shaped prompts (S = 12), E4M3 heads
    "gpt2s_gt": dict(cfg=formats.ModelConfig(12, 12, 768, 64, 50257, 12, 1, 1), items=64,
                     data="greater_than"),
    # configs[3]: GPT-2-medium shape, batch 256
    "gpt2m": dict(cfg=formats.ModelConfig(24, 16, 1024, 64, 50257, 16, 1, 1), items=256,
                  data="ioi"),
    # configs[4]: Pythia-1.4B shape (d_k = 128, V = 50304), docstring-shaped prompts
    # (S = 32); batch 512 over 8 GPUs, i.e. 64 items per GPU
    "pythia": dict(cfg=formats.ModelConfig(24, 16, 2048, 128, 50304, 32, 1, 1), items=512,
                   data="docstring"),
}
METRIC = "patched forward passes/sec and ACDC end-to-end s (1/2/4/8 B200 vs host CPU)"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        # tensor kernels run inside a long step: the sustained bf16 figure
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops_sustained", d.get("bf16_tflops", 1590.0)), \
            "measured (MEASURED_PEAKS.json)"
    return 6650.0, 1590.0, "fallback"


def make_inputs(name, weight_scale=0.0):
    c = CONFIGS[name]
    cfg = c["cfg"]
    w = synth.random_weights(cfg, 1, weight_scale)
    if c["data"] == "ioi":
        ds = synth.ioi_dataset(cfg, c["items"], 1)
    elif c["data"] == "greater_than":
        ds = synth.greater_than_dataset(cfg, c["items"], 1)
    elif c["data"] == "docstring":
        ds = synth.docstring_dataset(cfg, c["items"], 1)
    else:
        ds = synth.random_dataset(cfg, c["items"], 2)
    return cfg, w, ds


class ClockSampler:
    """nvidia-smi clocks/throttle reasons during the timed region."""

    def __init__(self, index=0):
        self.index, self.proc, self.lines = index, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# ------------------------------------------------------------------------------
# reference CPU arm
# ------------------------------------------------------------------------------
def cpu_sample(cfg, w, ds, steps, warmup, threads=None):
    """delta_l of the reference library (oracle/_ref) over a bounded sample:
    the out-edges of head a0.0 (one policy) x 1 prompt, one pass per host
    thread, in the reference's own OpenMP parallel-for (acdc.cpp:55-60)."""
    os.environ.setdefault("CQREF_NO_RTN4", "1")
    from oracle.oracle import Policy, Ref, ref_available
    kind = "reference"
    ref = Ref()
    nthreads = threads or ref.max_threads()
    ref.set_threads(nthreads)
    with tempfile.TemporaryDirectory() as t:
        wp, dp = os.path.join(t, "w.bin"), os.path.join(t, "d.jsonl")
        write_ref_inputs(ref, cfg, ds.subset([0]), wp, dp)
        m = ref.open(wp, dp, 0)
        # edges from the reference's own ComputationalGraph (model.cpp:182-203):
        # this arm never loads libcqg.so
        _, _, _, src, _ = ref.graph(cfg.fields8())
        cand = np.nonzero(src == 1)[0]  # node 1 = head a0.0
        n = int(min(len(cand), max(8, nthreads)))
        edges = cand[:n]
        times = []
        for i in range(warmup + steps):
            _, ms_refresh, ms_score = m.time_delta_l(edges, Policy.head_quantized(), True)
            if i >= warmup:
                times.append(ms_score / 1e3)
        m.close()
    passes = n * 1
    value = passes * len(times) / sum(times)
    return {"value": value, "unit": "passes/s", "cores": nthreads, "kind": kind,
            "cpu_model": cpu_model(),
            "sample": f"delta_l of {n} out-edges of a0.0 x 1 IOI prompt per step "
                      f"(reference library compiled in place, OpenMP {nthreads} threads; "
                      f"refresh_baselines excluded), {len(times)} steps",
            "s_per_step": float(np.mean(times))}


def self_launch(n, argv):
    """`python bench.py --gpus N` without torchrun: start N ranks (one per
    GPU) with torch.distributed.run on 127.0.0.1 and pass rank 0's line through."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + list(argv)
    return subprocess.call(cmd)


def toy_acdc_pair(eng):
    """BASELINE config 1 end to end on both sides: full PAHQ-ACDC (tau=0.01,
    acdc.cpp:23-88) through cqg_run_acdc on the GPU and the reference library's
    own run_acdc on all host threads, wall seconds each, and whether the two
    pruned edge sets are identical."""
    from oracle.oracle import Ref
    cfg, w, ds = make_inputs("toy")
    ref = Ref()
    nthreads = ref.max_threads()
    ref.set_threads(nthreads)
    with tempfile.TemporaryDirectory() as t:
        wp, dp = os.path.join(t, "w.bin"), os.path.join(t, "d.jsonl")
        write_ref_inputs(ref, cfg, ds, wp, dp)
        m = ref.open(wp, dp, 0)
        pc = ref.method_config(2, 8)
        t0 = time.perf_counter()
        rr = m.run_acdc(pc)
        cpu_s = time.perf_counter() - t0
        m.close()
    e = eng.Engine(w, device=int(os.environ.get("LOCAL_RANK", 0)))
    e.set_dataset(ds, eng.KL)
    c = eng.method_prune_config(eng.PAHQ)
    e.run_acdc(c)  # warm-up (weight images, packed operands, buffers)
    t0 = time.perf_counter()
    r = e.run_acdc(c)
    gpu_s = time.perf_counter() - t0
    e.close()
    return {"workload": "toy L2 H4 d128 V512 S16, random prompts batch 16, PAHQ tau=0.01",
            "gpu_s": gpu_s, "cpu_s": cpu_s, "cpu_threads": nthreads, "steps": r.steps,
            "kept_edges": int(r.final_mask.sum()),
            "same_circuit": bool(np.array_equal(r.final_mask, rr.final_mask)),
            "same_steps": r.steps == rr.steps}


def timed_roc_sweep(eng, e, scores, edges, barrier, max_over_ranks, iter1_s):
    """BASELINE config 5's 'full ACDC threshold sweep' (roc_sweep,
    eval.cpp:1193-1226) over threshold_grid(0.001, 3.16, 21) (acdc.cpp:90-102)
    through cqg_roc_sweep, which scores iteration 1 once and shares it across
    the 21 thresholds. Ground truth: the 16 top-scored iteration-1 edges (a
    synthetic model has no planted circuit; the AUC is not the point here,
    the time is). 21 independent run_acdc calls would each score iteration 1
    again: at least 21 x the iteration-1 time."""
    taus = eng.threshold_grid(0.001, 3.16, 21)
    gt = [int(x) for x in np.asarray(edges)[np.argsort(-np.asarray(scores))[:16]]]
    c = eng.method_prune_config(eng.PAHQ)
    barrier()
    t0 = time.perf_counter()
    curve = e.roc_sweep(c, taus, gt)
    barrier()
    sweep_s = max_over_ranks(time.perf_counter() - t0)
    return {"seconds": sweep_s, "thresholds": len(taus), "grid": "threshold_grid(0.001, 3.16, 21)",
            "iteration1_s": iter1_s, "independent_runs_lower_bound_s": 21 * iter1_s,
            "kept": [p.kept for p in curve.points], "auc_vs_synthetic_gt": curve.auc}


def toy_roc_pair(eng):
    """Config 1: the 21-threshold sweep with iteration 1 shared vs 21
    independent run_acdc calls, wall seconds each, same kept counts."""
    cfg, w, ds = make_inputs("toy")
    e = eng.Engine(w, device=int(os.environ.get("LOCAL_RANK", 0)))
    e.set_dataset(ds, eng.KL)
    c = eng.method_prune_config(eng.PAHQ)
    taus = eng.threshold_grid(0.001, 3.16, 21)
    gt = list(range(8))
    e.roc_sweep(c, taus, gt)  # warm-up
    t0 = time.perf_counter()
    curve = e.roc_sweep(c, taus, gt)
    shared_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    kept = []
    for t in taus:
        c.tau = float(t)
        kept.append(int(e.run_acdc(c).final_mask.sum()))
    indep_s = time.perf_counter() - t0
    e.close()
    return {"shared_s": shared_s, "independent_s": indep_s,
            "same_kept": kept == [p.kept for p in curve.points]}


def write_ref_inputs(ref, cfg, ds, wp, dp):
    """weights.bin by the reference's own generator and writer (support.hpp
    random_weights(seed 1) -> save_weights, byte-identical to synth.random_weights,
    tests/test_formats.py), then this workload's prompts as dataset.jsonl: the
    reference arm needs nothing from the product library."""
    ref.gen_random(cfg.fields8(), 1, 1, 1, wp, dp)
    formats.save_dataset_jsonl(ds, dp)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg, w, ds = make_inputs(args.config, getattr(args, "weight_scale", 0.0))
    try:
        cb = cpu_sample(cfg, w, ds, args.steps, args.warmup)
    except Exception as e:  # the oracle library always exists in-tree
        print(json.dumps({"impl": "reference", "unavailable": f"{type(e).__name__}: {e}"}))
        return
    out = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "passes/s",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": cb["s_per_step"] * 1e3, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "fp32-emulated e4m3/bf16", "data": "synthetic",
           "config": config_block(args), "cpu_baseline": cb,
           "e2e": {"value": cb["value"], "unit": "passes/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def config_block(args, n_edges_all=None, n_scored=None):
    c = CONFIGS[args.config]
    cfg = c["cfg"]
    items = min(args.items, c["items"]) if getattr(args, "items", 0) else c["items"]
    sampled = n_scored is not None and n_edges_all is not None and n_scored < n_edges_all
    out = {"workload": f"{args.config}: L{cfg.n_layers} H{cfg.n_heads} d{cfg.d_model} "
                       f"V{cfg.vocab} S{cfg.seq_len}, {c['data']}-shaped prompts batch "
                       f"{items}, PAHQ (E4M3 heads, BF16 MLP, FP32 source/unembed), "
                       f"KL, ACDC iteration-1 scoring of "
                       + (f"a strided sample of {n_scored} of the {n_edges_all} edges" if sampled
                          else "every edge"),
           "items": items, "parallelism": f"items sharded over {args.gpus} GPU(s)",
           "edges": "Q/K/V-split graph (extension, include/cqg.h)" if getattr(args, "qkv_split", False)
                    else "the reference's graph (model.cpp:192-201)",
            "low_precision": ("int8 per-channel RTN (extension, exact SIMT path)"
                              if getattr(args, "low", "e4m3") == "int8"
                              else "e4m3 (reference-pinned; INT8 per-channel: --low int8)"),
           "l2": "inputs >> L2 (activations per step ~GBs)"}
    if sampled:
        out["edges_sampled"] = {"scored": n_scored, "of": n_edges_all}
    if items != c["items"]:
        out["items_note"] = f"{items} of the config's {c['items']} items (one GPU's shard)"
    return out


# ------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------
def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="gpt2s", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--acdc", action="store_true", default=True,
                    help="also time a full PAHQ-ACDC run (default; the metric's 'ACDC end-to-end s')")
    ap.add_argument("--no-acdc", dest="acdc", action="store_false")
    ap.add_argument("--ncu", action="store_true",
                    help="profiling mode: one untimed scoring step, no JSON line (for ncu "
                         "launch lists; no number from it is a bench value)")
    ap.add_argument("--items", type=int, default=0,
                    help="prompt batch (default: the config's; e.g. the per-GPU shard of an "
                         "8-GPU config on one GPU)")
    ap.add_argument("--low", default="e4m3", choices=["e4m3", "int8"],
                    help="low precision of the heads: e4m3 (reference-pinned, tensor cores) or "
                         "int8 (per-channel RTN extension, exact path)")
    ap.add_argument("--qkv-split", action="store_true",
                    help="the Q/K/V-split edge graph (extension; config 3's ~32k edges)")
    ap.add_argument("--max-edges", type=int, default=0,
                    help="score an evenly strided sample of at most this many iteration-1 edges "
                         "(configs 4-5 on one GPU; reported in config.edges_sampled)")
    ap.add_argument("--weight-scale", type=float, default=0.0,
                    help="uniform half-width of the attention / MLP weight matrices (default: "
                         "support.hpp's 0.8/sqrt(d)); larger values model trained-weight "
                         "magnitudes: E4M3 weights leave the subnormal range and the "
                         "certificate flags more elements")
    ap.add_argument("--acdc-quantile", type=float, default=0.99,
                    help="ACDC end-to-end threshold = this quantile of the iteration-1 scores "
                         "(a non-trivial circuit survives); tau=0.01 is timed as well")
    args = ap.parse_args(argv)
    rank, world, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args.gpus, argv if argv is not None else sys.argv[1:])
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return run_reference(args)

    from paper_2510_23264_b200 import engine as eng
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    cfg, w, ds = make_inputs(args.config, getattr(args, "weight_scale", 0.0))
    if args.items:
        ds = ds.subset(list(range(min(args.items, len(ds)))))
    items = len(ds)
    lo, hi = shard_mod.item_block(rank, world, items)
    shard = ds.subset(list(range(lo, hi)))
    e = eng.Engine(w, device=local, qkv_split=args.qkv_split)
    for kv in filter(None, os.environ.get("CQG_OPTS", "").split(",")):  # e.g. exact_x2=0
        k, v = kv.split("=")
        e.set_option(k, int(v))
    e.set_dataset(shard, eng.KL, lo, items)
    if world > 1:
        import torch
        obj = [eng.Engine.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        e.init_comm(obj[0], rank, world)
    mask = np.ones(e.n_edges, bool)
    edges = eng.sweep_order(cfg, mask)
    n_edges_all = len(edges)
    if args.max_edges and len(edges) > args.max_edges:  # strided: every source depth is sampled
        edges = edges[::-(-len(edges) // args.max_edges)]
    pol = eng.PrecisionPolicy.head_quantized(eng.P8, eng.INT8 if args.low == "int8" else eng.E4M3)
    passes_per_step = len(edges) * items

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(x):
        if not dist:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    if args.ncu:
        e.score_edges(mask, edges, pol, True, eng.LOSS)
        print(f"ncu step: {passes_per_step} passes, {e.stats()['kernel_launches']} launches")
        return
    for _ in range(args.warmup):
        e.score_edges(mask, edges, pol, True, eng.LOSS)
    barrier()
    dev_ms = 0.0
    launches = 0
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            scores = e.score_edges(mask, edges, pol, True, eng.LOSS)
            st = e.stats()
            dev_ms += st["ms_device"]
            launches += st["kernel_launches"]
        wall = time.perf_counter() - t0
    barrier()
    dev_s = max_over_ranks(dev_ms / 1e3)
    wall = max_over_ranks(wall)
    value = passes_per_step * args.steps / dev_s

    # end to end through the C-ABI with host buffers: dataset tokens H2D
    # (cqg_set_dataset) + mask/edge list H2D + per-edge scores D2H each step
    barrier()
    t0 = time.perf_counter()
    e2e_parts = []
    for _ in range(args.steps):
        t1 = time.perf_counter()
        e.set_dataset(shard, eng.KL, lo, items)
        t2 = time.perf_counter()
        e.score_edges(mask, edges, pol, True, eng.LOSS)
        st = e.stats()
        e2e_parts.append({"set_dataset_s": t2 - t1, "score_wall_s": time.perf_counter() - t2,
                          "score_device_s": st["ms_device"] / 1e3,
                          "baseline_s": st.get("ms_baseline", 0) / 1e3})
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    h2d = shard.clean.nbytes + shard.corrupt.nbytes + shard.answer.nbytes + \
        shard.distractor.nbytes + mask.size + edges.size * 4
    d2h = edges.size * 8

    # one profiled step for the roofline of the dominant kernel
    e.set_option("profile", 1)
    e.score_edges(mask, edges, pol, True, eng.LOSS)
    prof = e.profile()
    flagged = int(e.stats()["fallback_elems"])
    e.set_option("profile", 0)
    # tensor-core output elements of the step (flops / 2K per GEMM class) and
    # the share the certificate sent to the exact fixup
    kdim = {"qkv": cfg.d_model, "wo": cfg.d_k, "mlp_in": cfg.d_model, "mlp_out": 4 * cfg.d_model}
    tc_el = sum(v["flops"] / (2 * kdim[k.split("gemm_tc_")[1].split("_", 1)[1]])
                for k, v in prof.items() if "gemm_tc_" in k)
    certificate = {"flagged_elems_per_step": flagged, "tc_elems_per_step": int(tc_el),
                   "flagged_share": flagged / tc_el if tc_el else None,
                   "weight_scale": getattr(args, "weight_scale", 0.0) or "support.hpp default 0.8/sqrt(d)"}
    hbm, bf16, src = load_peaks()
    name, p = max(prof.items(), key=lambda kv: kv[1]["ms"])
    # FP32 CUDA-core rate for separately rounded mul + add (the reference's
    # dot_col semantics forbid FMA): 148 SMs x 128 lanes x 1 instr/clk, 2 instr
    # per multiply-add, counted as 2 flops
    simt_peak = 148 * 128 * 1.965e9 / 1e12
    traffic, traffic_note = None, None
    for tp in (os.path.join(ROOT, "profiles", "r2_ncu_traffic.json"),
               os.path.join(ROOT, "profiles", "r1_ncu_traffic.json")):
        if traffic is None and os.path.exists(tp):  # committed ncu --set full capture of this class
            t = json.load(open(tp)).get(name.split(":")[-1])
            if t:
                traffic = t["traffic_bytes"]
                traffic_note = (f"dram bytes of one captured launch ({t['launch']}); algorithmic "
                                f"{t['algorithmic_bytes']} B for that launch ({os.path.basename(tp)})")
    cls = name.split(":")[-1]  # "base:" = per-source baseline runs
    if p["flops"] > 0:
        ach = p["flops"] / (p["ms"] / 1e3) / 1e12
        if cls.startswith("gemm_tc_fp8"):
            peak, unit, bound, psrc = 2 * bf16, "TFLOP/s", "tensor", f"2x {src} sustained bf16 (fp8 rate)"
        elif cls.startswith("gemm_tc"):
            peak, unit, bound, psrc = bf16, "TFLOP/s", "tensor", f"{src} sustained bf16"
        else:
            peak, unit, bound, psrc = simt_peak, "TFLOP/s", "fp32-simt", \
                "FP32 CUDA-core issue rate, no FMA (148 SM x 128 lanes x 1.965 GHz)"
    else:
        ach = p["bytes"] / (p["ms"] / 1e3) / 1e9
        peak, unit, bound, psrc = hbm, "GB/s", "hbm", src
    kernel_note = None
    if cls == "gemm_unembed" and os.environ.get("CQG_OPTS", "").find("kl_fused=0") < 0:
        kernel_note = ("gemm_unembed_kl_kernel: the exact FP32 unembed with the log-softmax + KL "
                       "reduction fused into its epilogue (FP64 expm1 / dot partials per tile, no "
                       "logits stored); achieved counts only the GEMM's 2 D V flops per row. The "
                       "GEMM alone (kl_fused=0) runs at ~32.4 TFLOP/s = 0.87 of this peak, plus a "
                       "separate 0.21 s KL kernel (profiles/r2_klfused_ab_*.json)")
    roofline = {"bound": bound, "kernel": name, "achieved": ach, "peak": peak, "unit": unit,
                "frac": ach / peak, "traffic": traffic, "traffic_note": traffic_note,
                "kernel_note": kernel_note, "peak_source": psrc,
                "kernel_share_of_step": p["ms"] / max(1e-9, sum(v["ms"] for v in prof.values())),
                "per_kernel": {k: {"ms": v["ms"], "launches": v["launches"],
                                   "tflops": v["flops"] / max(v["ms"], 1e-9) / 1e9,
                                   "gbs": v["bytes"] / max(v["ms"], 1e-9) / 1e6}
                               for k, v in prof.items()},
                "per_kernel_note": "gbs = algorithmic bytes (every operand read counted, incl. re-reads "
                                   "served by L2) / CUDA-event time; measured DRAM throughput: hbm_kernels_ncu"}
    dp = os.path.join(ROOT, "profiles", "r2_dram_per_kernel.json")
    if os.path.exists(dp):  # committed per-launch ncu DRAM bytes of one whole step
        dk = json.load(open(dp))
        roofline["hbm_kernels_ncu"] = {
            "source": "profiles/r2_dram_per_kernel.json (" + dk["source"] + ")",
            "kernels": {k: dk["kernels"][k] for k in dk["kernels"]
                        if any(x in k for x in ("fold", "ln_small_kernel<4>", "kl_reduce", "attention"))}}

    acdc = None
    if args.acdc:  # every rank runs the loop on its item block; scores are all-reduced per iteration
        def timed_acdc(tau):
            c = eng.method_prune_config(eng.PAHQ)
            c.tau = float(tau)
            barrier()
            t0 = time.perf_counter()
            r = e.run_acdc(c)
            barrier()
            return {"seconds": max_over_ranks(time.perf_counter() - t0), "steps": r.steps,
                    "kept_edges": int(r.final_mask.sum()), "tau": c.tau,
                    "kept_per_iteration": [it.present_after for it in r.iterations],
                    "passes": int(sum(len(it.scores) for it in r.iterations)) * items}
        # tau at a high quantile of this workload's iteration-1 scores, so a
        # non-trivial circuit survives and several iterations run
        tau_q = float(np.quantile(scores, args.acdc_quantile))
        sweep = timed_roc_sweep(eng, e, scores, edges, barrier, max_over_ranks, dev_s / args.steps)
        # headline: the largest grid threshold whose final circuit keeps at
        # least 16 edges (the sweep's kept counts are identical on every rank:
        # scores are all-reduced), so the timed run prunes to a non-empty circuit
        grid = eng.threshold_grid(0.001, 3.16, 21)
        nt = [t for t, k in zip(grid, sweep["kept"]) if k >= 16]
        tau_nt = float(max(nt)) if nt else float(grid[0])
        acdc = timed_acdc(tau_nt)
        acdc["tau_rule"] = ("largest threshold_grid(0.001, 3.16, 21) value whose final circuit "
                            "keeps >= 16 edges (from the roc_sweep below)")
        acdc[f"tau_quantile_{args.acdc_quantile}"] = timed_acdc(tau_q)
        acdc["tau_0.01"] = timed_acdc(0.01)
        acdc["roc_sweep"] = sweep

    if rank == 0:
        cb = None
        toy = None
        if not args.no_cpu:
            try:
                cb = cpu_sample(cfg, w, ds, steps=1, warmup=0)
            except Exception as ex:
                cb = {"unavailable": f"{type(ex).__name__}: {ex}"}
            if world == 1 and args.acdc:
                try:
                    toy = toy_acdc_pair(eng)
                    toy["roc_sweep"] = toy_roc_pair(eng)
                except Exception as ex:
                    toy = {"unavailable": f"{type(ex).__name__}: {ex}"}
        out = {"metric": METRIC, "value": value, "unit": "passes/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": dev_s / args.steps * 1e3, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "e4m3/bf16/fp32 (exact)",
               "data": f"synthetic (random-init weights per support.hpp, "
                       f"{CONFIGS[args.config]['data']}-shaped prompts)",
               "config": config_block(args, n_edges_all, len(edges)), "clocks": clk.summary(),
               "e2e": {"value": passes_per_step * args.steps / e2e_s, "unit": "passes/s",
                       "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                       "parts": e2e_parts},
               "gpu_launches": int(launches), "wall_s": wall, "roofline": roofline,
               "cpu_baseline": cb, "passes_per_step": passes_per_step, "certificate": certificate,
               "acdc_end_to_end": acdc, "acdc_toy_gpu_vs_cpu": toy}
        print(json.dumps(out))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
