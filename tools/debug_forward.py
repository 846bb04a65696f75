import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), 'tests'))
import numpy as np
from oracle.oracle import Policy, Port
from paper_2510_23264_b200 import engine as eng
from helpers import TINY, SMALL, TOY, make, bits
cfg = {'tiny': TINY, 'small': SMALL, 'toy': TOY}[sys.argv[1] if len(sys.argv) > 1 else 'tiny']
w, ds = make(cfg, 3, 2, 4)
p = Port(cfg, w.mats); e = eng.Engine(w)
SD = cfg.seq_len * cfg.d_model
for pol in [Policy.all_fp32(), Policy.head_quantized()]:
    a = p.forward(ds.clean[1], pol); b = e.forward(ds.clean[1], eng.PrecisionPolicy(pol.attention_default, pol.mlp_default, pol.embed_precision, pol.unembed_precision, pol.low_mode))
    for n in range(p.n_nodes):
        sz = SD if n < p.n_nodes - 1 else cfg.seq_len * cfg.vocab
        x, y = a[n*SD:n*SD+sz], b[n*SD:n*SD+sz]
        ok = np.array_equal(bits(x), bits(y))
        print(n, ok, '' if ok else (np.max(np.abs(x-y)), x[:4], y[:4]))
