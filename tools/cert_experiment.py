"""Dev experiment (GPU): how the raw tcgen05 BF16 accumulation error and the
reference's sequential FP32 error scale on structured data. Writes
gpurun_out/cert_experiment.json. Not a test."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from test_gpu_parity import _bf16_grid, _tc_gemm  # noqa: E402

U = 2.0 ** -24


def data(kind, M, N, K, rng):
    A = rng.randn(M, K)
    Bt = rng.randn(N, K) * 0.03
    if kind.startswith("cancel"):
        nb = int(kind[6:])
        A = np.abs(A)
        Bt = np.abs(Bt)
        L = K // nb
        for b in range(1, nb, 2):
            A[:, b * L:(b + 1) * L] *= -1
    elif kind == "ramp":  # slow drift: products biased positive then negative
        A = A + np.linspace(2, -2, K)[None, :]
        Bt = np.abs(Bt)
    return _bf16_grid(A.astype(np.float32)), _bf16_grid(Bt.astype(np.float32))


def seq(A, Bt):
    s = np.zeros((A.shape[0], Bt.shape[0]), np.float32)
    path_abs = np.zeros(s.shape)
    path_sq = np.zeros(s.shape)
    tsum = np.zeros(s.shape)
    ex = np.zeros(s.shape)
    for k in range(A.shape[1]):
        p = (A[:, k:k + 1] * Bt[:, k][None, :]).astype(np.float64)
        s = (s + p.astype(np.float32)).astype(np.float32)
        ex += p
        path_abs += np.abs(ex)
        path_sq += ex ** 2
        if (k + 1) % 16 == 0:
            tsum += ex
    return s, ex, path_abs, path_sq, tsum


out = {}
M = N = 128
for K in (768, 3072):
    for kind in ("iid", "cancel2", "cancel4", "cancel8", "cancel16", "ramp"):
        rng = np.random.RandomState(K)
        A, Bt = data(kind, M, N, K, rng)
        raw, _, _ = _tc_gemm(1, 2, 0, A, Bt)
        s, ex, pa, ps, ts = seq(A, Bt)
        na = np.sqrt((A.astype(np.float64) ** 2).sum(1))
        nb = np.sqrt((Bt.astype(np.float64) ** 2).sum(1))
        nn = np.outer(na, nb)
        e_tc = raw.astype(np.float64) - ex
        e_ref = s.astype(np.float64) - ex
        r = {
            "tc_over_u_T16": float(np.max(np.abs(e_tc) / (U * np.abs(ts) + U * nn))),
            "tc_signed_fit": float(np.sum(e_tc * ts) / np.sum(ts * ts) / U),
            "tc_over_u_pathabs16": float(np.max(np.abs(e_tc) / (U * pa / 16))),
            "ref_over_u_rms_path": float(np.max(np.abs(e_ref) / (U * np.sqrt(ps)))),
            "ref_over_u_pathabs": float(np.max(np.abs(e_ref) / (U * pa))),
            "tc_over_u_nn": float(np.max(np.abs(e_tc) / (U * nn))),
            "ref_over_u_nn": float(np.max(np.abs(e_ref) / (U * nn))),
            "diff_over_u_nn": float(np.max(np.abs(raw.astype(np.float64) - s) / (U * nn))),
        }
        out[f"K{K}_{kind}"] = r
        print(K, kind, r, flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "cert_experiment.json"), "w"), indent=1)
