import sys, os, faulthandler
faulthandler.enable()
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, 'tests'))
import numpy as np
from oracle.oracle import Policy, Port
from paper_2510_23264_b200 import engine as eng
from helpers import TOY, make, bits, random_mask
from test_gpu_parity import gpol
cfg = TOY
w, ds = make(cfg, 3, 2, 4)
p = Port(cfg, w.mats); e = eng.Engine(w)
L, H = cfg.n_layers, cfg.n_heads
pols = [Policy.all_fp32(), Policy.head_quantized(), Policy.all_low(), Policy.make(th=(L - 1, H - 1)), Policy.make(att=1), Policy.make(th=(0, 1))]
SD = cfg.seq_len * cfg.d_model
rng = np.random.RandomState(0)
for i, pol in enumerate(pols):
    mask = random_mask(p.n_edges, i, 0.7) if i % 2 else None
    pe, pv = -1, None
    if i >= 2:
        cand = np.nonzero(mask)[0] if mask is not None else np.arange(p.n_edges)
        pe = int(cand[rng.randint(len(cand))]); pv = rng.randn(SD).astype(np.float32)
    print(i, 'port', flush=True)
    a = p.forward(ds.clean[1], pol, mask=mask, patch_edge=pe, patch_value=pv)
    print(i, 'gpu', flush=True)
    b = e.forward(ds.clean[1], gpol(pol), mask=mask, patch_edge=pe, patch_value=pv)
    print(i, np.array_equal(bits(a), bits(b)), flush=True)
