/* cqg_diag.h — diagnostic entry points of libcqg.so used by the parity tests
 * to check the device numerics exhaustively (no reference interface is
 * replaced by these; they expose the scalar device functions of
 * csrc/numerics.cuh over ranges of FP32 bit patterns). */
#ifndef CQG_DIAG_H
#define CQG_DIAG_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
/* E4M3 codes of the floats with bit patterns lo .. lo+count-1
 * (== cq::encode_f8, proj/src/numerics.cpp:41-64). */
int cqg_diag_e4m3_range(uint32_t lo, uint64_t count, uint8_t* out_host);
/* BF16 codes (== cq::encode_bf16, numerics.cpp:84-94). */
int cqg_diag_bf16_range(uint32_t lo, uint64_t count, uint16_t* out_host);
/* which: 0 glibc-exact expf, 1 glibc-exact erff, 2 reference gelu
 * (kernels.cpp:226). */
int cqg_diag_libm_range(int which, uint32_t lo, uint64_t count, float* out_host);
/* The W_in epilogue's GELU of every BF16 code: out_lut = the full
 * device-built table (round_bf16(gelu(x)), kernels.cpp:221-234, glibc-exact
 * erff), out_code = gelu_code (shared-memory slice + closed forms),
 * out_fast = the fast path's slice lookup for codes inside the slice
 * (|x| in [2^-24, 8)), 0 elsewhere. */
int cqg_diag_gelu_codes(uint16_t* out_lut, uint16_t* out_code, uint16_t* out_fast);
/* One tensor-core GEMM C = round(A . B^T) (A: M x K, Bt: N x K, values on
 * the elem grid: 0 E4M3, 1 BF16) through the production tcgen05 kernel +
 * exactness fixup, and the same product through the exact sequential SIMT
 * kernel. prec: output rounding (0 E4M3, 1 BF16, 2 none = raw accumulators);
 * epi 1 = round-gelu-round. *n_fix = elements recomputed exactly. */
int cqg_diag_gemm_tc(int elem, int prec, int epi, int M, int N, int K, const float* A,
                     const float* Bt, float* out_tc, float* out_exact, uint32_t* n_fix);
#ifdef __cplusplus
}
#endif
#endif
