import sys, os
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, 'tests'))
import numpy as np
from oracle.oracle import Policy, Port
from paper_2510_23264_b200 import engine as eng, formats, synth
cfg = formats.ModelConfig(2, 2, 32, 16, 41, 6, 1, 1)
w = synth.random_weights(cfg, 7); ds = synth.random_dataset(cfg, 4, 8)
e = eng.Engine(w); e.set_dataset(ds, eng.KL)
p = Port(cfg, w.mats)
mask = np.ones(e.n_edges, bool); edges = np.arange(e.n_edges, dtype=np.int32)
for per in (False, True):
    want = p.score_edges(ds, edges, Policy.head_quantized(), per_edge=per)
    got = e.score_edges(mask, edges, eng.PrecisionPolicy.head_quantized(), per, eng.LOSS)
    one = np.array([e.score_edges(mask, [x], eng.PrecisionPolicy.head_quantized(), per, eng.LOSS)[0] for x in edges])
    print("per_edge", per)
    for i in edges:
        r = abs(got[i]-want[i])/(abs(want[i])+1e-15); r1 = abs(one[i]-want[i])/(abs(want[i])+1e-15)
        print(f"{i:3d} {e.edge_src[i]:2d}->{e.edge_dst[i]:2d} want {want[i]:.6e} got {got[i]:.6e} rel {r:.1e} single {r1:.1e}")
