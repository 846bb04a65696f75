// gemm_tc.h — tcgen05 tensor-core GEMMs for the low-precision projections
// (E4M3 head Q/K/V and W_O, BF16 MLP) with an exactness-certified epilogue.
//
// C[m][n] = round_prec( sum_k A[m][k] * B[n][k] )      (A, B K-major)
//
// The reference accumulates each dot product sequentially in FP32
// (kernels.cpp:44-52) and then rounds to E4M3/BF16. Products of two E4M3 or
// two BF16 values are exact in FP32, so the tensor-core sum r_tc and the
// reference's sequential sum r_ref differ only by accumulation rounding. The
// epilogue rounds r_tc and flags every element whose rounding is not
// certified: round(r_tc - m) != round(r_tc + m) for the error margin
//   m = kappa * 2^-24 * sqrt(K) * max(|r_tc|, ||a_m|| ||b_n|| / sqrt(K)),
// (a ~kappa-sigma bound on |r_tc - r_ref| for FP32 accumulation of K terms).
// Flagged elements are recomputed by the exact sequential kernel
// (fixup), so the stored result equals the reference's bit for bit.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace cqg {

enum TcElem : int { kTcE4M3 = 0, kTcBF16 = 1 };

struct TcJob {
  int a_row0;        // first A row (global row index in the A tensor)
  int b_row0;        // first B row (= output column 0) in the B tensor
  int b_k0;          // K offset inside B rows (W_O head slices)
  int M, N, K;       // K in elements, multiple of 32 bytes
  float* out_f32;    // [M][ldo] FP32 values (may be null)
  void* out_pack;    // [M][ldo] packed E4M3/BF16 of the output (may be null)
  int ldo;
  int tile0;         // first tile index of this job
  const float* b_norm;  // [N] ||B row n|| over [b_k0, b_k0+K)
  int prec;          // output rounding: 0 E4M3, 1 BF16, 2 none
  int epi;           // 1: round -> gelu -> round (MLP in, kernels.cpp:226)
};

struct TcLaunch {
  CUtensorMap tmA, tmB;
  const uint8_t* A;  // global base of A, row pitch lda bytes
  const uint8_t* B;
  int64_t lda, ldb;  // bytes
  const float* a_norm;  // [rows of A] ||A row|| (sign bit: row not FMA-safe), or null with a_ss
  const float* a_ss;     // alternative: [rows of A] sum of squares and
  const uint32_t* a_bad; //   nonzero where the row is not FMA-safe (written by a producer epilogue)
  float* out_ss;         // producer side: accumulate the output rows' sums of squares (atomics)
  uint32_t* out_bad;     //   and their not-FMA-safe flags (both zeroed before the launch)
  int elem;          // TcElem
  int prec, epi;     // launch-uniform output rounding / GELU epilogue (== every job's)
  int n_jobs, total_tiles;
  uint32_t* fix_mask;   // [total_tiles][kFixWords] flagged bits, row r at r*4 (words = 32 cols);
                        // valid for the 32 x 32 parts whose bit is set in tile_mark
  uint32_t* fix_tiles;  // [total_tiles] tiles with flagged elements
  uint32_t* tile_mark;  // [total_tiles] flagged-part bits (row quarter q + 4 * column chunk); zero between launches
  int fix_g;            // tile-fixup unit: 2 (2 x 2-tile super-tiles, fix_st) or 1 (listed tiles)
  const int4* fix_st;   // [n_fix_st] the launch's 2 x 2-tile super-tiles {job, row tile, col tile, 0}
  int n_fix_st;
  uint64_t* fix_items;  // [units][fix_item_cap(fix_g)] item lists (fix_plan_kernel)
  uint32_t* fix_n;      // [units] items | columns-per-item << 24 of each unit
  uint32_t* fix_count;  // [0] tiles listed by this launch, [1] fixup CTAs finished (both
                        //   zeroed by the fixup's last CTA),
                        // [2..3] u64 running total of flagged elements,
                        // [4] block-fixup chunk queue (reset by its last CTA)
  float kappa;
  int fix_cpi;  // fixup columns per work item: 0 adaptive, else 1 / 2 / 4
  int fix_dry;  // timing experiment only: the tile fixup streams and stages but runs no chains
  const int* tile_job;  // [total_tiles] job index of each tile (may be null: binary search)
  const uint16_t* gelu_lut;  // bf16 -> round_bf16(gelu(x)) for all 2^16 inputs
  // block fixup (BF16): SW32 maps of A / B (32-byte K slices x 256 rows) and
  // the launch's chunk list {job, first row tile, first column tile,
  // row tiles | column tiles << 8} (<= 4 x 6 tiles), taken in order through
  // the queue counter fix_count[4]
  CUtensorMap fxA, fxB;
  const int4* fix_blocks;
  int n_fix_blocks;
};

// Builds 2D K-major tensor maps (SW128, box = 128 B x box_rows) for A/B.
bool tc_make_map(CUtensorMap* map, const void* base, int elem, uint64_t rows, uint64_t cols_elems,
                 uint64_t pitch_bytes, uint32_t box_rows);

void launch_gemm_tc(const TcLaunch& L, const TcJob* d_jobs, cudaStream_t st);
void launch_gemm_fixup(const TcLaunch& L, const TcJob* d_jobs, cudaStream_t st);
// BF16 only: persistent CTAs over chunks of up to 4 x 6 tiles (gemm_tc.cu)
void launch_gemm_fixup_blk(const TcLaunch& L, const TcJob* d_jobs, cudaStream_t st);
// the chunk list of a launch's jobs: 4-row-tile chunks first, then 2, then 1
// (persistent CTAs take them in order: a balanced tail)
std::vector<int4> fixup_chunks(const TcJob* jobs, int n_jobs, int ctas);
// the tile fixup's 2 x 2-tile super-tiles of a launch's jobs (gemm_tc.cu)
std::vector<int4> fixup_super_tiles(const TcJob* jobs, int n_jobs);
bool tc_make_map_sw32(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols_elems,
                      uint64_t pitch_bytes);
// lut[b] = enc_bf16(round_bf16(gelu_ref(dec_bf16(b)))) (glibc-exact erff)
void launch_gelu_lut(uint16_t* lut, cudaStream_t st);
void launch_gelu_codes(const uint16_t* lut, uint16_t* out, uint16_t* out_fast, cudaStream_t st);
// ||row|| of a packed [rows][K] operand (elements starting at col k0)
void launch_rownorm(const uint8_t* A, int64_t lda, int elem, int rows, int k0, int K, float* out,
                    cudaStream_t st);
// transpose + pack: out[n][k] = enc(in[k][n]) for a row-major K x N FP32 image
void launch_pack_t(const float* in, int K, int N, int ld_in, void* out, int64_t ld_out, int elem,
                   cudaStream_t st);

// The FP32 unembed on the tensor cores (6-term BF16 split, gemm_tc.cu):
// A6 [rows][6D] (+ ||a|| per row) from the FP32 LN output rows (pitch ldx),
// and B6 [V][6D] (+ ||w_j|| per column) from the [D][V] FP32 image.
void launch_split_rows(const float* x, int rows, int D, int ldx, uint16_t* out, float* anorm,
                       cudaStream_t st);
void launch_split_cols(const float* w, int D, int V, uint16_t* out, float* wnorm, cudaStream_t st);

constexpr int kTcBM = 128;
constexpr int kTcBN = 128;
constexpr int kFixWords = kTcBM * kTcBN / 32;
// item capacity of one tile-fixup unit of g x g tiles (= fix_cap in gemm_tc.cu)
constexpr int fix_item_cap(int g) { return g * kTcBM * g * kTcBN / 4 + g * kTcBM; }

}  // namespace cqg
