import sys, os, time
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, R)
import numpy as np
from paper_2510_23264_b200 import engine as eng, formats, synth
cfg = formats.ModelConfig(*[int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "12,12,768,64,50257,16,1,1").split(",")])
items = int(sys.argv[2]) if len(sys.argv) > 2 else 64
nsrc = int(sys.argv[3]) if len(sys.argv) > 3 else 0
t = time.time(); w = synth.random_weights(cfg, 1); ds = synth.ioi_dataset(cfg, items, 1); print("gen", time.time()-t, flush=True)
t = time.time(); e = eng.Engine(w); e.set_dataset(ds, eng.KL); print("create", time.time()-t, flush=True)
mask = np.ones(e.n_edges, bool)
edges = eng.sweep_order(cfg, mask)
if nsrc: # restrict to edges from a few sources spread over depth
    srcs = sorted(set(e.edge_src.tolist()))
    pick = set(srcs[:: max(1, len(srcs)//nsrc)][:nsrc])
    edges = np.array([x for x in edges if e.edge_src[x] in pick], np.int32)
print("edges", len(edges), flush=True)
e.set_option("profile", 1)
for it in range(2):
    t = time.time(); s = e.score_edges(mask, edges, eng.PrecisionPolicy.head_quantized(), True, eng.LOSS); dt = time.time()-t
    st = e.stats()
    print(f"step {it}: wall {dt:.2f}s device {st['ms_device']/1e3:.2f}s passes {st['passes']} -> {st['passes']/dt:.0f} passes/s launches {st['kernel_launches']}", flush=True)
prof = e.profile()
for k, v in sorted(prof.items(), key=lambda kv: -kv[1]['ms']):
    print(f"  {k:12s} {v['ms']:10.1f} ms  launches {v['launches']:6d}  TFLOP/s {v['flops']/max(v['ms'],1e-9)/1e9:8.2f}  GB/s {v['bytes']/max(v['ms'],1e-9)/1e6:8.1f}")
print("fallback elems", e.stats()["fallback_elems"], "passes", e.stats()["passes"])
