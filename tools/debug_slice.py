"""Localise a headline-slice score mismatch: per-edge score error vs the
reference golden, then node-by-node forward comparison (engine vs the C
oracle) for the clean, corrupt and patched runs of one edge.
usage: python tools/debug_slice.py pythia_slice [edge]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from oracle.oracle import Policy, Port  # noqa: E402
from paper_2510_23264_b200 import engine as eng  # noqa: E402
from helpers import bits  # noqa: E402
from test_gpu_headline import load_case  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "pythia_slice"
cfg, w, ds, edges, want = load_case(case)
e = eng.Engine(w)
e.set_dataset(ds, eng.KL)
mask = np.ones(e.n_edges, bool)
got = e.score_edges(mask, edges, eng.PrecisionPolicy.head_quantized(), True, eng.LOSS)
rel = np.abs(got - want) / (np.abs(want) + 1e-300)
for i, ed in enumerate(edges):
    print(f"edge {ed}: got {got[i]:.17g} want {want[i]:.17g} rel {rel[i]:.3e}")
bad = int(sys.argv[2]) if len(sys.argv) > 2 else int(edges[int(np.argmax(rel))])
p = Port(cfg, w.mats)
_, es, ed_ = eng.graph_edges(cfg)
src, dst = int(es[bad]), int(ed_[bad])
print("edge", bad, "src", src, "dst", dst)
SD = cfg.seq_len * cfg.d_model
nn = int(eng.graph_edges(cfg)[0])
pol = Policy.head_quantized()
gp = eng.PrecisionPolicy.head_quantized()


def cmp(a, b, what):
    n_bad = 0
    for n in range(nn):
        sz = SD if n < nn - 1 else cfg.seq_len * cfg.vocab
        x, y = a[n * SD:n * SD + sz], b[n * SD:n * SD + sz]
        if not np.array_equal(bits(x), bits(y)):
            d = np.nonzero(bits(x) != bits(y))[0]
            print(f"  {what} node {n}: {d.size} elems differ, first {d[:6]}, "
                  f"ref {x[d[:3]]} gpu {y[d[:3]]}")
            n_bad += 1
    print(f"{what}: {n_bad} nodes differ")


for it in range(len(ds)):
    a = p.forward(ds.clean[it], pol)
    b = e.forward(ds.clean[it], gp)
    cmp(a, b, f"clean item {it}")
    c = p.forward(ds.corrupt[it], pol)
    d = e.forward(ds.corrupt[it], gp)
    cmp(c, d, f"corrupt item {it}")
    pv = c[src * SD:(src + 1) * SD]
    a = p.forward(ds.clean[it], pol, patch_edge=bad, patch_value=pv)
    b = e.forward(ds.clean[it], gp, patch_edge=bad, patch_value=pv)
    cmp(a, b, f"patched item {it}")
