import sys, os, ctypes as C
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, R)
import numpy as np
from paper_2510_23264_b200 import engine as eng
lib = eng.load_library()
lib.cqg_diag_gemm_tc.argtypes = [C.c_int]*6 + [C.c_void_p]*5
def run(elem, prec, epi, M, N, K, A, Bt):
    o1 = np.empty((M, N), np.float32); o2 = np.empty((M, N), np.float32); nf = np.zeros(1, np.uint32)
    rc = lib.cqg_diag_gemm_tc(elem, prec, epi, M, N, K, A.ctypes.data, Bt.ctypes.data, o1.ctypes.data, o2.ctypes.data, nf.ctypes.data)
    return rc, o1, o2, int(nf[0])
def grid(x, elem):
    import torch
    t = torch.from_numpy(x)
    return (t.to(torch.float8_e4m3fn) if elem == 0 else t.to(torch.bfloat16)).float().numpy()
rng = np.random.RandomState(0)
for elem in (0, 1):
    for (M, N, K) in [(128, 128, 128), (256, 384, 768), (1000, 300, 768), (256, 256, 64 if elem == 0 else 64), (512, 768, 3072)]:
        if elem == 0 and K == 3072: continue
        A = grid((rng.randn(M, K)).astype(np.float32), elem)
        Bt = grid((rng.rand(N, K).astype(np.float32) - 0.5) * 0.0288, elem)
        rc, raw, _, _ = run(elem, 2, 0, M, N, K, A, Bt)
        exact = A.astype(np.float64) @ Bt.astype(np.float64).T
        seq = np.zeros((M, N), np.float32)
        for k in range(K): seq = (seq + (A[:, k:k+1] * Bt[:, k][None, :]).astype(np.float32)).astype(np.float32)
        print(f"elem {elem} M{M} N{N} K{K} rc {rc}: raw-exact max {np.max(np.abs(raw-exact)):.3e} (rel {np.max(np.abs(raw-exact)/(np.abs(exact)+1e-30)):.2e}) raw==seq {np.mean(raw==seq):.4f} seq-exact {np.max(np.abs(seq-exact)):.3e}")
        for prec, epi in ((elem, 0), (elem, 1)) if elem == 1 else ((0, 0),):
            rc, tc, ex, nf = run(elem, prec, epi, M, N, K, A, Bt)
            print(f"   prec {prec} epi {epi}: bitexact {np.array_equal(tc.view(np.uint32), ex.view(np.uint32))} mismatches {int(np.sum(tc.view(np.uint32) != ex.view(np.uint32)))} fixed {nf} ({nf/(M*N):.4%})")
