import sys, os, ctypes as C
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, R)
import numpy as np
from paper_2510_23264_b200 import engine as eng
lib = eng.load_library()
lib.cqg_diag_gemm_tc.argtypes = [C.c_int]*6 + [C.c_void_p]*5
def bf16(x):
    u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)
rng = np.random.RandomState(1)
u = 2.0**-24
for (M, N, K) in [(8192, 3072, 768), (8192, 768, 3072)]:
    if K == 768:
        A = bf16(rng.randn(M, K).astype(np.float32) * (1 + 0.2*(rng.rand(K)-0.5)).astype(np.float32))
    else:  # gelu outputs: mostly positive, heavy at 0
        x = rng.randn(M, K).astype(np.float32) * 0.2
        A = bf16(0.5 * x * (1 + np.tanh(0.79788456 * (x + 0.044715 * x**3))))
    Bt = bf16((rng.rand(N, K).astype(np.float32) - 0.5) * np.float32(0.8/np.sqrt(768)))
    o1 = np.empty((M, N), np.float32); o2 = np.empty((M, N), np.float32); nf = np.zeros(1, np.uint32)
    rc = lib.cqg_diag_gemm_tc(1, 2, 0, M, N, K, A.ctypes.data, Bt.ctypes.data, o1.ctypes.data, o2.ctypes.data, nf.ctypes.data)
    na = np.sqrt((A.astype(np.float64)**2).sum(1)); nb = np.sqrt((Bt.astype(np.float64)**2).sum(1))
    floor = u * na[:, None] * nb[None, :]
    d = np.abs(o1.astype(np.float64) - o2.astype(np.float64))
    r1 = d / floor
    r2 = d / (u * np.sqrt(K) * np.maximum(np.abs(o2), na[:, None]*nb[None, :]/np.sqrt(K)))
    print(f"M{M} N{N} K{K} rc{rc}: |tc-seq|/(u na nb): mean {r1.mean():.3f} p99.99 {np.quantile(r1, 0.9999):.3f} max {r1.max():.3f};  in margin units (kappa=1): max {r2.max():.3f} p99.999 {np.quantile(r2, 0.99999):.3f}")
    # flagged fraction as function of kappa
    for kappa in (2, 3, 4, 6, 8):
        m = kappa * u * np.sqrt(K) * np.maximum(np.abs(o1), na[:, None]*nb[None, :]/np.sqrt(K))
        def rb(x):
            uu = x.astype(np.float32).view(np.uint32).astype(np.uint64); lsb = (uu >> 16) & 1
            return ((uu + 0x7FFF + lsb) & 0xFFFF0000).astype(np.uint32)
        amb = rb((o1 - m).astype(np.float32)) != rb((o1 + m).astype(np.float32))
        print(f"   kappa {kappa}: flagged {amb.mean():.4%}")
