// kernels.h — job descriptors and launchers for the sm_100a kernels.
//
// Activation layout in HBM: a "segment" is one evaluation context (the
// baseline, or one patched edge) over the local item batch: [B][S][D] FP32,
// contiguous. Kernels take flat job lists so one launch covers every segment
// of a step (no per-edge launches).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cqg {

// ---- K2a: receiver-input fold (sum_inputs, model.cpp:537-552) -------------
// dst = (a ? a : 0.0f) + b elementwise, ops of a program run in order per
// element (so a later op may read an earlier op's dst). a == kRegPrev reuses
// the previous op's result held in a register; dst == nullptr keeps it there.
// Node-output storage types: node outputs that the reference rounds to E4M3 or
// BF16 (low-precision heads, the BF16 MLP) are stored as their 1- or 2-byte
// codes (bit-exact: the codes decode to the rounded FP32 values).
enum OutType { kOutF32 = 0, kOutE4M3 = 1, kOutBF16 = 2 };

struct FoldOp {
  const float* a;
  const float* b;  // element type btype (OutType)
  float* dst;
  int btype;
};
struct FoldProg {
  int op_begin, op_end;
};
#define CQG_REG_PREV (reinterpret_cast<const float*>(uintptr_t(1)))
void launch_fold(const FoldOp* d_ops, const FoldProg* d_progs, int n_progs, int64_t n_elems,
                 cudaStream_t st);

// ---- K2b: layer norm + precision rounding (kernels.cpp:127-163) -----------
// Exact reference order: sequential FP32 sums per row.
struct LnJob {
  const float* in;  // rows selected as in + r*in_stride
  float* xln;       // [rows][D] (may be null)
  float* xq;        // [rows][D] rounded at prec (may be null)
  int rows;
  int in_stride;
  void* xqp;        // packed copy of xq for the tensor cores (may be null)
  int pack;         // 1: E4M3 bytes, 2: BF16
  float* xnorm;     // [rows] ||xq row|| * 1.0001 (sign: BF16 row not FMA-safe) (may be null)
};
void launch_layernorm(const LnJob* d_jobs, int n_jobs, int max_rows, const float* gamma,
                      const float* beta, int D, int prec, cudaStream_t st);

// ---- exact SIMT GEMM (dot_col, kernels.cpp:44-52) --------------------------
// C[M][N] = round_prec(sum_k A[m][k]*B[k][n]) with k ascending, every product
// rounded then added (no FMA), as the reference. epi=1: C = round(gelu(round(acc))).
struct GemmJob {
  const float* A;
  const float* B;
  float* C;
  int M, N, K, lda, ldb, ldc;
  int prec, epi;
};
void launch_gemm_exact(const GemmJob* d_jobs, const int* d_tile_start, int n_jobs, int total_tiles,
                       cudaStream_t st);
int gemm_exact_tiles(int M, int N);
// 128 x 128-tile variant for large jobs (same numerics)
void launch_gemm_exact_big(const GemmJob* d_jobs, const int* d_tile_start, int n_jobs,
                           int total_tiles, cudaStream_t st);
int gemm_exact_big_tiles(int M, int N);
// 64 x 256-tile paired-FP32 variant for jobs with at most 64 rows (same numerics)
void launch_gemm_exact_wide(const GemmJob* d_jobs, const int* d_tile_start, int n_jobs,
                            int total_tiles, cudaStream_t st);
int gemm_exact_wide_tiles(int M, int N);
extern int g_exact_x2;  // 1: FFMA2/FADD2 variant of the big exact GEMM

// ---- K5: causal attention (kernels.cpp:167-219) + z rounding ---------------
struct AttnJob {
  const float* q;
  const float* k;
  const float* v;
  float* z;
  int ld;    // row stride of q/k/v (elements)
  int prec;  // rounding of z (model.cpp:688-689)
  int ldz;   // row stride of z / z8
  uint8_t* z8;  // packed E4M3 copy of z for the tensor-core W_O (may be null)
  int q0;       // first query row computed (S-1: last position only); z rows
                // are compact: item * (S - q0) + (i - q0)
  float* znorm;  // [z rows] ||z8 row|| * 1.0001 for W_O's certificate (may be null)
  const uint8_t* q8;  // E4M3 codes of q/k/v instead of q/k/v (row stride ld bytes), or null
  const uint8_t* k8;
  const uint8_t* v8;
};
void launch_attention(const AttnJob* d_jobs, int n_jobs, int B, int S, int dk, cudaStream_t st);

// ---- embed (model.cpp:608-620) ---------------------------------------------
void launch_embed(const int* tokens, const float* we, const float* wpos, float* out, int B, int S,
                  int D, int prec, cudaStream_t st);

// ---- K8: KL / logit-diff against the baseline (patching.cpp:108-161) -------
// logits: [rows][V] (patched last rows), row r belongs to item item_of[r];
// base: [B][V] baseline last-row logits; base_lse[B]. out[r] (double).
// base_p (optional): [B][V] exp(base - lse) from launch_lse's p_out
void launch_kl(const float* logits, const float* base, const double* base_lse, const int* item_of,
               int rows, int V, double* out, int* nan_flag, cudaStream_t st,
               const double* base_p = nullptr);
// KL with the tensor-core unembed's certificate (kernels.cu, KlCert): rows
// whose estimated deviation from the reference's exact-logit KL exceeds tol *
// KL are appended to list (count[0]; count[1] += the same, a running total).
void launch_kl_cert(const float* logits, const float* base, const double* base_lse, const int* item_of,
                    int rows, int V, double* out, int* nan_flag, const double* base_p, const float* anorm,
                    const float* wnorm, int K, double tol, int* list, int* count, cudaStream_t st);
// the KL of the listed rows (rows[0 .. *count)), persistent grid
void launch_kl_rows(const float* logits, const float* base, const double* base_lse, const int* item_of,
                    int V, double* out, int* nan_flag, const double* base_p, const int* rows,
                    const int* count, cudaStream_t st);
// the exact GEMM of jb over the listed rows of A / C (jb.M ignored)
void launch_gemm_exact_rows(const GemmJob& jb, const int* rows, const int* count, cudaStream_t st);
void launch_lse(const float* base, int rows, int V, double* lse, int* nan_flag, cudaStream_t st,
                double* p_out = nullptr, double* p_sum = nullptr);
// Fused unembed + KL (kernels.cu, gemm_unembed_kl_kernel): per 128-column
// tile partials (T, S) of the patched rows against the baseline item
// (row % nb): xb [nb][ld] baseline logits (as doubles), eb [nb][ld] exp(lp),
// both zero-padded to ld = V rounded up to 128 (launch_pad_baselines).
struct KlFuse {
  const double* xb;
  const double* eb;
  double2* part;  // [rows][n_ct]
  int nb, n_ct, ld;
};
void launch_gemm_unembed_kl(const GemmJob& jb, const KlFuse& kf, cudaStream_t st);
int unembed_kl_col_tiles(int V);
void launch_pad_baselines(const float* logits, const double* prob, int nb, int V, int ld, double* xbd,
                          double* ebd, cudaStream_t st);
// L2 prefetch (cp.async.bulk.prefetch.L2) of up to three column slices
// (rows x cols floats at pitch ld floats; null: none) and two whole matrices;
// addresses 16-byte aligned, sizes multiples of 16. Passed by value: no
// device-side list, nothing for the host to wait on.
struct PfJob {
  const float* col[3];
  int rows, ld, cols;
  const void* blk[2];
  uint64_t blk_bytes[2];
};
void launch_prefetch_l2(const PfJob& j, cudaStream_t st);
// KL per row = E log1p((E - 1) + T) - S from the row's partials (NaN -> flag)
void launch_kl_reduce(const double2* part, int rows, int n_ct, const double* esum, int nb, double* out,
                      int* nan_flag, cudaStream_t st);
void launch_logitdiff(const float* logits, const float* base, const int* item_of,
                      const int* answer, const int* distractor, int rows, int V, double* out,
                      int* nan_flag, cudaStream_t st);

// ---- act_diff RMS (patching.cpp:241-259) -----------------------------------
// out[j] = sqrt(sum((a-b)^2)/n) per job over n contiguous floats.
struct RmsJob {
  const float* a;
  const float* b;
  int64_t n;
  double* out;
  int atype, btype;  // OutType of a / b
};
void launch_rms(const RmsJob* d_jobs, int n_jobs, cudaStream_t st);

// ---- K1: weight images (ImageBank, model.cpp:473-491) ----------------------
void launch_quantize(const float* in, float* out, int64_t n, int prec, cudaStream_t st);
void launch_pack_e4m3(const float* in, uint8_t* out, int64_t n, cudaStream_t st);
void launch_pack_bf16(const float* in, uint16_t* out, int64_t n, cudaStream_t st);
// Rtn4 per group: groups are `n_groups` blocks of rows x cols taken with a
// row stride `ld` starting at base + g*group_off (model.cpp:445-469).
void launch_rtn_groups(const float* in, float* out, int n_groups, int64_t group_off, int rows,
                       int cols, int ld, int bits, cudaStream_t st, int qmax = 0);

// ---- Rtn4 activations (quantize_span P8/Rtn4, kernels.cpp:236-251) ---------
// In place: each of n_groups groups (one per item) is a rows x cols block
// with row stride ld, groups group_off apart; the whole group shares one
// delta = max|x| / 2^(bits-1) (quantize_rtn, numerics.cpp:105-120).
// gelu = 1 applies gelu_ref first (the MLP's round -> GELU -> round chain).
struct RtnJob {
  float* p;
  int64_t group_off;
  int rows, cols, ld, gelu;
};
// qmax: INT8 extension clamp (127), 0 = none
void launch_rtn_act(const RtnJob* d_jobs, int n_jobs, int n_groups, int bits, cudaStream_t st, int qmax = 0);
// rows = 1 groups (per-token scales): one warp per group
void launch_rtn_rows(const RtnJob* d_jobs, int n_jobs, int n_groups, int bits, cudaStream_t st, int qmax = 0);

// ---- tests: exhaustive scalar checks on the device --------------------------
void launch_e4m3_all(uint8_t* out, uint32_t lo, uint64_t count, cudaStream_t st);
void launch_bf16_all(uint16_t* out, uint32_t lo, uint64_t count, cudaStream_t st);
void launch_libm_all(float* out, uint32_t lo, uint64_t count, int which, cudaStream_t st);

}  // namespace cqg
