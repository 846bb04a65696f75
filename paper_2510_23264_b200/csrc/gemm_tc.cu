// gemm_tc.cu — tcgen05 / TMA / TMEM GEMM for sm_100a (see gemm_tc.h).
//
// One CTA computes one 128 x 128 output tile:
//   warp 0      TMA producer  (cp.async.bulk.tensor.2d, SWIZZLE_128B, mbarrier tx)
//   warp 1      MMA issuer    (tcgen05.mma.cta_group::1, kind::f8f6f4 | kind::f16,
//                              FP32 accumulator in TMEM; TMEM alloc/dealloc)
//   warps 2..5  epilogue      (tcgen05.ld 32x32b -> round -> certify -> store)
// A 4-stage smem ring (32 KB/stage) keeps the tensor pipe fed.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>

#include "gemm_tc.h"
#include "numerics.cuh"

namespace cqg {

namespace {

constexpr int kStages = 4;
constexpr int kBKBytes = 128;  // one SW128 atom row
constexpr int kAStage = kTcBM * kBKBytes;  // 16 KB
constexpr int kBStage = kTcBN * kBKBytes;  // 16 KB
constexpr int kEpiWarps = 16;  // 4 per TMEM lane quarter, one 32-column chunk each
constexpr int kEpiWarp0 = 3;  // warps: 0 TMA, 1 MMA, 2 tile metadata, 3.. epilogue
constexpr int kThreads = 32 * kEpiWarp0 + 32 * kEpiWarps;
constexpr size_t kStageFloats = 32 * 36;  // per epilogue warp store staging

// Per-tile metadata staged in shared memory by the metadata warp one TMEM
// buffer ahead of the epilogue (job lookup, row / column norms), so the
// epilogue warps never wait on dependent global loads.
struct TileMeta {
  TcJob jb;
  int mt, nt;
  alignas(16) float na[kTcBM];  // ||A row|| bound per tile row (0 outside the job)
  alignas(16) float nb[kTcBN];  // ||B row|| per tile column (0 outside the job)
  float nbmax[kTcBN / 32];       // max of nb over each 32-column chunk
};
constexpr size_t kMetaBytes = (sizeof(TileMeta) + 15) & ~size_t(15);
// TMEM accumulator buffers (128 columns each; 4 = all 512 columns): the MMA
// and the metadata warp run up to kAccBufs - 1 tiles ahead of the epilogue,
// which hides the per-tile TMA -> MMA -> commit latency of short-K GEMMs (W_O).
constexpr int kAccBufs = 4;
// Certified BF16 outputs accumulate K in two halves into two TMEM
// accumulators (the buffer count halves to 2): the epilogue adds them and
// also knows the partial sum at K/2, so a sign-ordered (cancelling) row, whose
// partial sums run far above the result, gets a margin on that scale.
__host__ __device__ constexpr int split_of(int elem, int prec) { return elem == kTcBF16 && prec == 1 ? 2 : 1; }
__device__ __forceinline__ int split_kh(int nk) { return (nk + 1) >> 1; }
constexpr size_t kSmemBytes = 1024 + (size_t)kStages * (kAStage + kBStage) + 256 +
                              kEpiWarps * kStageFloats * sizeof(float) + kAccBufs * kMetaBytes +
                              2 * 2 * 27 * 128;  // GELU LUT slice (kGeluSm uint16)
static_assert(kSmemBytes <= 227 * 1024, "tcgen05 GEMM shared memory");

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// K-major SWIZZLE_128B smem matrix descriptor (cute::UMMA::SmemDescriptor):
// start>>4 [0,14), LBO>>4 [16,30) (=1, unused for swizzled K-major),
// SBO>>4 [32,46) (=1024 B: 8 rows x 128 B), version 1 [46,48), layout 2 [61,64).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor (cute::UMMA::InstrDescriptor): c_format F32 [4,6),
// a/b format [7,10)/[10,13) (E4M3=0 for f8f6f4, BF16=1 for f16), K-major A/B,
// N>>3 [17,23), M>>4 [24,29).
template <int ELEM>
__device__ __forceinline__ uint32_t instr_desc() {
  uint32_t d = 0;
  d |= 1u << 4;
  const uint32_t f = ELEM == kTcBF16 ? 1u : 0u;
  d |= f << 7;
  d |= f << 10;
  d |= (uint32_t)(kTcBN >> 3) << 17;
  d |= (uint32_t)(kTcBM >> 4) << 24;
  return d;
}

template <int ELEM>
__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                    uint32_t accum) {
  if (ELEM == kTcBF16) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accum));
  } else {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accum));
  }
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ||A row|| bound and FMA safety of A row r (rownorm_kernel's encoding, or
// the sum of squares accumulated by the producing GEMM's epilogue)
__device__ __forceinline__ float a_norm_of(const TcLaunch& L, int r) {
  return L.a_ss ? sqrtf(L.a_ss[r]) * 1.0001f : fabsf(L.a_norm[r]);
}
__device__ __forceinline__ bool a_fma_safe(const TcLaunch& L, int r) {
  return L.a_ss ? L.a_bad[r] == 0u : (__float_as_uint(L.a_norm[r]) >> 31) == 0;
}

__device__ __forceinline__ float round_out(float x, int prec) {
  return prec == 2 ? x : round_p(x, prec);
}

__device__ __forceinline__ int find_job(const TcJob* jobs, int n, int t) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].tile0 <= t) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// job owning a tile: one load from the host-built tile -> job map (the
// binary search over the job list is a chain of dependent loads, a visible
// per-tile latency for the single-thread producer / MMA and the metadata warp
// on short-K launches with thousands of jobs)
__device__ __forceinline__ int job_of(const TcLaunch& L, const TcJob* jobs, int t) {
  return L.tile_job ? __ldg(L.tile_job + t) : find_job(jobs, L.n_jobs, t);
}

__device__ __forceinline__ void store_out(const TcJob& jb, int row, int col, float v) {
  const int64_t o = (int64_t)row * jb.ldo + col;
  if (jb.out_f32) jb.out_f32[o] = v;
  if (jb.out_pack) {
    if (jb.prec == 1) reinterpret_cast<uint16_t*>(jb.out_pack)[o] = enc_bf16(v);
    else reinterpret_cast<uint8_t*>(jb.out_pack)[o] = enc_e4m3(v);
  }
}

// E4M3 round trip of two values with the paired hardware conversions
// (F2FP.SATFINITE.E4M3 / F2FP.F16.E4M3 unpack); NaN -> 0x7F as enc_e4m3.
__device__ __forceinline__ float2 round_e4m3x2(float a, float b) {
  const __nv_fp8x2_storage_t p = __nv_cvt_float2_to_fp8x2(make_float2(a, b), __NV_SATFINITE, __NV_E4M3);
  float2 f = __half22float2(__half2(__nv_cvt_fp8x2_to_halfraw2(p, __NV_E4M3)));
  const float qnan = dec_e4m3(0x7F);
  if (a != a) f.x = qnan;
  if (b != b) f.y = qnan;
  return f;
}

template <int PREC>
__device__ __forceinline__ void round_pair(float& a, float& b) {
  if (PREC == 0) {
    const float2 f = round_e4m3x2(a, b);
    a = f.x, b = f.y;
  } else if (PREC == 1) {
    a = round_bf16(a), b = round_bf16(b);
  }
}

// Paired E4M3 codes of (a, b) (cvt.rn.satfinite.e4m3x2; reference NaN code 0x7F)
__device__ __forceinline__ uint32_t e4m3x2_code(float a, float b) {
  uint32_t c = (uint32_t)__nv_cvt_float2_to_fp8x2(make_float2(a, b), __NV_SATFINITE, __NV_E4M3);
  if (a != a) c = (c & 0xFF00u) | 0x7Fu;
  if (b != b) c = (c & 0x00FFu) | 0x7F00u;
  return c;
}
__device__ __forceinline__ float2 e4m3x2_value(uint32_t c) {
  return __half22float2(__half2(__nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)c, __NV_E4M3)));
}

// BF16 certificate in integer form: the reference's value lies in
// [acc - m, acc + m]; its RNE rounding to BF16 can differ from acc's only if
// that interval reaches the rounding midpoint nearest to acc, i.e. if the
// distance from acc's discarded 16 bits to 0x8000 (in units of acc's FP32
// ulp, 2^(E-150)) is at most m / ulp. Binade edges cannot matter because m is
// far below a BF16 ulp. Non-finite, tiny (|acc| < 2^-95) or NaN-margin
// elements are always flagged.
__device__ __forceinline__ bool bf16_ambiguous(float acc, float m) {
  // branch-free: |acc| minus its BF16 truncation is exact in FP32; its
  // distance to half a BF16 ulp (2^(e-8)) is the distance to the midpoint
  const uint32_t ab = __float_as_uint(acc) & 0x7FFFFFFFu;
  const float dl = __uint_as_float(ab) - __uint_as_float(ab & 0xFFFF0000u);
  const float h = __uint_as_float((ab & 0x7F800000u) - (8u << 23));  // 2^(e-8)
  const bool odd = ab >= 0x7F800000u || ab < (32u << 23);
  return odd | !(fabsf(dl - h) > m);  // m carries the 1.001 guard for its own FP32 rounding
}

// RNE of an FP32 value to its BF16 grid (integer form). No NaN special case:
// a NaN accumulator is always flagged (bf16_ambiguous: odd) and its element
// recomputed and stored by the exact fixup.
__device__ __forceinline__ float rne_bf16_bits(float x) {
  const uint32_t u = __float_as_uint(x);
  return __uint_as_float((u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u);
}

// round_bf16 of a GELU input's code through the shared-memory slice of the
// LUT (|x| in [2^-24, 8), both signs) and the closed forms outside it
// (checked against the full table for all 2^16 codes): x >= 8 -> x,
// x <= -8 -> -0, |x| < 2^-10 -> round_bf16(0.5 x); Inf / NaN via the table.
constexpr int kGeluE0 = 103, kGeluNE = 27;
constexpr int kGeluSm = 2 * kGeluNE * 128;
static_assert(2 * kGeluSm == 2 * 2 * 27 * 128, "kSmemBytes holds the GELU slice");
__device__ __forceinline__ uint32_t gelu_code(uint32_t c, const uint16_t* lut_s, const uint16_t* lut_g) {
  const uint32_t E = (c >> 7) & 0xFFu;
  const uint32_t t = E - kGeluE0;
  const bool in = t < (uint32_t)kGeluNE;
  const uint32_t g = lut_s[in ? (c >> 15) * (kGeluNE * 128) + (c & 0x7FFFu) - kGeluE0 * 128 : 0];
  // |x| < 2^-10: round_bf16(0.5 x) (x is a BF16 value, 0.5 x is exact in FP32)
  const uint32_t hb = __float_as_uint(0.5f * __uint_as_float(c << 16));
  const uint32_t half = (hb + 0x7FFFu + ((hb >> 16) & 1u)) >> 16;
  const uint32_t big = (c & 0x8000u) ? 0x8000u : c;  // x >= 8 -> x, x <= -8 -> -0
  uint32_t r = in ? g : (E > kGeluE0 ? big : half);
  if (E == 255u) r = __ldg(lut_g + c);  // Inf / NaN (rare)
  return r;
}

// The rare half-chunks with a code outside the slice: out of line, so the
// closed forms' registers do not weigh on the fast path's allocation
struct F16 {
  float x[16];
};
__device__ __noinline__ F16 gelu16_slow(F16 v, const uint16_t* gelu_s, const uint16_t* lut) {
#pragma unroll
  for (int j = 0; j < 16; ++j) v.x[j] = __uint_as_float(gelu_code(__float_as_uint(v.x[j]) >> 16, gelu_s, lut) << 16);
  return v;
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
      "[%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Per-lane state of one epilogue chunk (32 rows x 32 columns of a tile).
struct EpiRow {
  float oss;      // sum of squares of the stored outputs (out_ss)
  bool obad;      // a stored output is not FMA-safe
};

// 16 columns [c0, c0 + 16) of the warp's chunk: TMEM -> rounding ->
// certificate flags (returned, bit j = column c0 + j) -> GELU -> out_ss;
// FP32 values to the staging row (stage, when the job stores FP32) and the
// packed codes to pk (BF16: 8 words, E4M3: 4 words).
template <int ELEM, int PREC, int EPI>
__device__ __forceinline__ uint32_t epilogue16(const TcLaunch& L, const TileMeta& md, uint32_t tacc, int q,
                                               int c0, int ncol, bool rvalid, float na, float sk, float ku,
                                               bool two, float* srow, uint32_t* pk, EpiRow& st,
                                               const uint16_t* gelu_s) {
  const TcJob& jb = md.jb;
  constexpr int kSplitE = split_of(ELEM, PREC);
  uint32_t r[16];
  tmem_ld16(tacc + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, r);
  // split accumulation: r = first-half sum, r2 = second half; acc = r + r2,
  // and |first half| joins the margin's scale (h1)
  float h1[kSplitE == 2 ? 16 : 1];
  if (kSplitE == 2) {
    if (two) {
      uint32_t r2[16];
      tmem_ld16(tacc + kTcBN + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, r2);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        h1[j] = fabsf(__uint_as_float(r[j]));
        r[j] = __float_as_uint(__uint_as_float(r[j]) + __uint_as_float(r2[j]));
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) h1[j] = 0.f;
    }
  }
  uint32_t fl = 0;
  float v[16];
  bool have_codes = false;
  // E4M3 x E4M3 products are multiples of 2^-18; if every partial sum is
  // below 2^6 (|s_k| <= ||a|| ||b||) all of them are exact in FP32, so the
  // reference's sequential sum is the exact sum and so is the tensor-core
  // sum: the rounding is certified without a fixup. Checked for the whole
  // warp chunk at once (uniform branch) with the chunk's largest column norm.
  const bool cert_all = ELEM == kTcE4M3 && PREC == 0 &&
                        __all_sync(0xffffffffu, na * md.nbmax[c0 >> 5] < 63.99f);
  if (PREC == 0 && cert_all) {
#pragma unroll
    for (int j = 0; j < 16; j += 4)
      pk[j >> 2] = e4m3x2_code(__uint_as_float(r[j]), __uint_as_float(r[j + 1])) |
                   (e4m3x2_code(__uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])) << 16);
    have_codes = true;
    if (jb.out_f32 || EPI == 1 || L.out_ss) {
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        const float2 x = e4m3x2_value(pk[j >> 2] & 0xFFFFu), y = e4m3x2_value(pk[j >> 2] >> 16);
        v[j] = x.x, v[j + 1] = x.y, v[j + 2] = y.x, v[j + 3] = y.y;
      }
    }
  } else if (PREC == 1 && ncol > 0) {
    // BF16: RNE by integer add, certificate in integer form
    const float nas = na / sk;
    const float ku1 = ku * 1.001f;  // (the guard for the FP32 rounding of the margin)
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      const float4 t4 = *reinterpret_cast<const float4*>(md.nb + c0 + j);
      const float nb4[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float acc = __uint_as_float(r[j + t]);
        v[j + t] = rne_bf16_bits(acc);
        float sc = fabsf(acc);
        if (kSplitE == 2) sc = fmaxf(sc, h1[(j + t) & (kSplitE == 2 ? 15 : 0)]);
        const float m = ku1 * fmaxf(sc, nas * nb4[t]);
        if (bf16_ambiguous(acc, m)) fl |= 1u << (j + t);
      }
    }
    if (!rvalid) fl = 0;
    if (ncol < 16) fl &= (1u << max(ncol, 0)) - 1u;
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
#pragma unroll
    for (int j = 0; j < 16; j += 2) round_pair<PREC>(v[j], v[j + 1]);
    if (PREC != 2 && ncol > 0) {
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        float lo[2], hi[2];
        bool chk[2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const float nb = md.nb[c0 + j + t];  // (uniform: broadcast shared loads)
          const float acc = __uint_as_float(r[j + t]);
          chk[t] = !(ELEM == kTcE4M3 && na * nb < 63.99f);
          const float m = ku * fmaxf(fabsf(acc), na * nb / sk);
          lo[t] = acc - m, hi[t] = acc + m;
          if (!(acc == acc)) fl |= 1u << (j + t);
        }
        if (chk[0] || chk[1]) {
          round_pair<PREC>(lo[0], lo[1]);
          round_pair<PREC>(hi[0], hi[1]);
#pragma unroll
          for (int t = 0; t < 2; ++t)
            if (chk[t] && !(lo[t] == hi[t])) fl |= 1u << (j + t);
        }
      }
      if (!rvalid) fl = 0;
      if (ncol < 16) fl &= (1u << max(ncol, 0)) - 1u;
    }
  }
  if (EPI == 1 && ncol > 0) {
    if (PREC == 1) {
      // fast path: every code of the 16 inside the shared-memory slice
      // (|x| in [2^-24, 8): all but ~1e-7 of the pre-activations) -> one
      // lookup each; otherwise gelu_code's closed forms
      uint32_t u[16];
      bool all_in = true;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        u[j] = (__float_as_uint(v[j]) >> 16 & 0x7FFFu) - (uint32_t)(kGeluE0 * 128);
        all_in = all_in && u[j] < (uint32_t)(kGeluNE * 128);
      }
      if (all_in) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          v[j] = __uint_as_float(
              (uint32_t)gelu_s[u[j] + (__float_as_uint(v[j]) >> 31) * (uint32_t)(kGeluNE * 128)] << 16);
      } else {
        F16 t;
#pragma unroll
        for (int j = 0; j < 16; ++j) t.x[j] = v[j];
        t = gelu16_slow(t, gelu_s, L.gelu_lut);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = t.x[j];
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = round_out(gelu_ref(v[j]), PREC);
      have_codes = false;
    }
  }
  if (L.out_ss && ncol > 0 && rvalid) {
    // (columns >= ncol hold zero-padded accumulators: they add nothing)
    uint32_t ebad = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      // a flagged element is recomputed later: bound |final| by the
      // neighbouring rounding candidates (GELU is 1.13-Lipschitz)
      const float vb = (fl >> j) & 1u ? fabsf(v[j]) + 0.02f * fabsf(__uint_as_float(r[j])) : v[j];
      st.oss = fmaf(vb, vb, st.oss);
      // not FMA-safe: nonzero |v| outside [2^-67, 2^64)
      const uint32_t ab = __float_as_uint(v[j]) & 0x7FFFFFFFu;
      ebad |= (uint32_t)(ab - (60u << 23) >= (131u << 23)) & (uint32_t)(ab != 0u);
    }
    st.obad = st.obad || ebad != 0;
  }
  if (jb.out_f32) {
#pragma unroll
    for (int j = 0; j < 16; j += 4) *reinterpret_cast<float4*>(srow + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
  }
  if (jb.out_pack) {
    if (PREC == 1) {
#pragma unroll
      for (int w = 0; w < 8; ++w)
        pk[w] = (__float_as_uint(v[2 * w]) >> 16) | (__float_as_uint(v[2 * w + 1]) & 0xFFFF0000u);
    } else if (!have_codes) {
#pragma unroll
      for (int w = 0; w < 4; ++w)
        pk[w] = enc_e4m3(v[4 * w]) | ((uint32_t)enc_e4m3(v[4 * w + 1]) << 8) |
                ((uint32_t)enc_e4m3(v[4 * w + 2]) << 16) | ((uint32_t)enc_e4m3(v[4 * w + 3]) << 24);
    }
  }
  return fl;
}

// Epilogue of one tile for one warp: 32 TMEM lanes (rows) x 32 columns
// (column chunk cq of the tile), in two 16-column halves (registers: 16
// epilogue warps share the SM's register file).
template <int ELEM, int PREC, int EPI>
__device__ __forceinline__ void epilogue_tile(const TcLaunch& L, const TileMeta& md, int tile,
                                              uint32_t tacc, int q, int cq, int lane, float* stage,
                                              const uint16_t* gelu_s) {
  const TcJob& jb = md.jb;
  const int mt = md.mt, nt = md.nt;
  const int row = mt * kTcBM + q * 32 + lane;
  const bool rvalid = row < jb.M;
  const float sk = sqrtf((float)jb.K);
  const float na = md.na[q * 32 + lane];
  const float ku = L.kappa * 5.9604644775390625e-08f * sk;
  const int row0 = mt * kTcBM + q * 32;
  const int nrow = min(32, jb.M - row0);
  constexpr int kSplitE = split_of(ELEM, PREC);
  // the second accumulator exists when K spans at least two k-blocks
  const bool two = kSplitE == 2 && (jb.K * (ELEM == kTcBF16 ? 2 : 1) + kBKBytes - 1) / kBKBytes >= 2;
  const int c0 = cq * 32;
  const int colb = nt * kTcBN + c0;
  const int ncol = min(32, jb.N - colb);
  EpiRow st{0.f, false};
  uint32_t pk[16];  // packed output codes of the 32 columns (BF16: 16 words, E4M3: 8)
  constexpr int hw = PREC == 1 ? 8 : 4;  // packed words per 16 columns
  uint32_t fl = epilogue16<ELEM, PREC, EPI>(L, md, tacc, q, c0, ncol, rvalid, na, sk, ku, two,
                                            stage + lane * 36, pk, st, gelu_s);
  fl |= epilogue16<ELEM, PREC, EPI>(L, md, tacc, q, c0 + 16, ncol - 16, rvalid, na, sk, ku, two,
                                    stage + lane * 36 + 16, pk + hw, st, gelu_s) << 16;
  // Stores: the 32 x 32 block is transposed through a warp-private smem
  // tile with 16-byte accesses (row pitch padded by 4 words: conflict-free),
  // then written as whole row segments with 16-byte global stores.
  if (ncol > 0) {
    uint32_t* sw = reinterpret_cast<uint32_t*>(stage);
    if (jb.out_f32) {
      __syncwarp();
      const bool vec = ncol == 32 && ((reinterpret_cast<uintptr_t>(jb.out_f32) & 15) == 0) && (jb.ldo & 3) == 0;
      if (vec) {
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int rr = it * 4 + (lane >> 3), cw = (lane & 7) * 4;
          if (rr < nrow)
            *reinterpret_cast<float4*>(jb.out_f32 + (int64_t)(row0 + rr) * jb.ldo + colb + cw) =
                *reinterpret_cast<const float4*>(stage + rr * 36 + cw);
        }
      } else {
        float* dst = jb.out_f32 + (int64_t)row0 * jb.ldo + colb + lane;
        for (int rr = 0; rr < nrow; ++rr)
          if (lane < ncol) dst[(int64_t)rr * jb.ldo] = stage[rr * 36 + lane];
      }
      __syncwarp();
    }
    if (jb.out_pack) {
      constexpr int esz = PREC == 1 ? 2 : 1;
      constexpr int words = 32 * esz / 4;  // per row: 16 (bf16) or 8 (e4m3)
      constexpr int pitch = words + 4;
      uint8_t* base = reinterpret_cast<uint8_t*>(jb.out_pack);
      const bool vec = ncol == 32 && ((reinterpret_cast<uintptr_t>(base) & 15) == 0) &&
                       ((int64_t)jb.ldo * esz) % 16 == 0 && (colb * esz) % 16 == 0;
      if (vec) {
#pragma unroll
        for (int w = 0; w < words; w += 4)
          *reinterpret_cast<uint4*>(sw + lane * pitch + w) = make_uint4(pk[w], pk[w + 1], pk[w + 2], pk[w + 3]);
        __syncwarp();
        constexpr int lanes_per_row = words / 4;  // 4 (bf16) or 2 (e4m3)
        constexpr int rows_per_it = 32 / lanes_per_row;
#pragma unroll
        for (int it = 0; it < 32 / rows_per_it; ++it) {
          const int rr = it * rows_per_it + lane / lanes_per_row, cw = (lane % lanes_per_row) * 4;
          if (rr < nrow)
            *reinterpret_cast<uint4*>(base + ((int64_t)(row0 + rr) * jb.ldo + colb) * esz + cw * 4) =
                *reinterpret_cast<const uint4*>(sw + rr * pitch + cw);
        }
        __syncwarp();
      } else {
#pragma unroll
        for (int w = 0; w < words; ++w) sw[lane * (words + 1) + w] = pk[w];
        __syncwarp();
        for (int rr = 0; rr < nrow; ++rr) {
          if (lane < ncol) {
            const uint32_t wv = sw[rr * (words + 1) + lane * esz / 4];
            const int64_t o = (int64_t)(row0 + rr) * jb.ldo + colb + lane;
            if (PREC == 1) reinterpret_cast<uint16_t*>(base)[o] = (uint16_t)(wv >> (16 * (lane & 1)));
            else base[o] = (uint8_t)(wv >> (8 * (lane & 3)));
          }
        }
        __syncwarp();
      }
    }
  }
  if (L.out_ss && rvalid) {
    atomicAdd(L.out_ss + jb.a_row0 + row, st.oss);
    if (st.obad) atomicOr(L.out_bad + jb.a_row0 + row, 1u);
  }
  // Record the flagged bits of this warp's 32 x 32 part (word cq of each row;
  // part bit q + 4 cq); the first part of a tile to flag anything lists the
  // tile for the fixup kernel.
  if (!__any_sync(0xffffffffu, fl != 0)) return;
  L.fix_mask[(size_t)tile * kFixWords + (q * 32 + lane) * 4 + cq] = fl;
  int total = __popc(fl);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
  if (lane == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(L.fix_count + 2), (unsigned long long)total);
    if (atomicOr(L.tile_mark + tile, 1u << (q + 4 * cq)) == 0u)
      L.fix_tiles[atomicAdd(L.fix_count, 1u)] = (uint32_t)tile;
  }
}

// Persistent warp-specialised kernel: the TMEM accumulator is double
// buffered, so the epilogue of tile i overlaps the MMAs of tile i+1.
template <int ELEM, int PREC, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ TcLaunch L, const TcJob* __restrict__ jobs) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment by pointer arithmetic on the shared array itself, so
  // the compiler keeps every derived access in the shared address space
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kAStage;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * kBStage);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;   // [kAccBufs]
  uint64_t* tempty = tfull + kAccBufs;  // [kAccBufs]
  uint64_t* mfull = tempty + kAccBufs;  // [kAccBufs] metadata ready (32 arrivals)
  uint64_t* mempty = mfull + kAccBufs;  // [kAccBufs] metadata consumed (kEpiWarps arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mempty + kAccBufs);
  float* stage_all = reinterpret_cast<float*>(smem + kStages * (kAStage + kBStage) + 256);
  TileMeta* meta = reinterpret_cast<TileMeta*>(stage_all + (size_t)kEpiWarps * kStageFloats);
  uint16_t* gelu_s = reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(meta) + kAccBufs * kMetaBytes);
  if (EPI == 1 && PREC == 1)  // the GELU LUT slice |x| in [2^-24, 8) (made visible by the barrier below)
    for (int i = threadIdx.x; i < kGeluSm; i += blockDim.x) {
      const int sg = i / (kGeluNE * 128), rem = i % (kGeluNE * 128);
      gelu_s[i] = L.gelu_lut[(sg << 15) | ((kGeluE0 + rem / 128) << 7) | (rem % 128)];
    }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int esz = ELEM == kTcBF16 ? 2 : 1;
  constexpr int bke = kBKBytes / esz;  // elements per stage along K
  constexpr int kSplit = split_of(ELEM, PREC);
  constexpr int kBufs = kAccBufs / kSplit;  // TMEM accumulator buffers in flight

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < kBufs; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps);
      mbar_init(&mfull[b], 32);
      mbar_init(&mempty[b], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kAccBufs * kTcBN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      uint32_t it = 0;
      for (int tile = blockIdx.x; tile < L.total_tiles; tile += gridDim.x) {
        const TcJob& jb = jobs[job_of(L, jobs, tile)];
        const int tiles_n = (jb.N + kTcBN - 1) / kTcBN;
        const int mt = (tile - jb.tile0) / tiles_n, nt = (tile - jb.tile0) % tiles_n;
        const int nk = (jb.K * esz + kBKBytes - 1) / kBKBytes;
        const int arow = jb.a_row0 + mt * kTcBM, brow = jb.b_row0 + nt * kTcBN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % kStages;
          mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
          mbar_expect_tx(&full[s], kAStage + kBStage);
          tma_load_2d(sA + s * kAStage, &L.tmA, &full[s], kb * bke, arow);
          tma_load_2d(sB + s * kBStage, &L.tmB, &full[s], jb.b_k0 + kb * bke, brow);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      const uint32_t idesc = instr_desc<ELEM>();
      uint32_t it = 0, ti = 0;
      for (int tile = blockIdx.x; tile < L.total_tiles; tile += gridDim.x, ++ti) {
        const TcJob& jb = jobs[job_of(L, jobs, tile)];
        const int kbytes = jb.K * esz;
        const int nk = (kbytes + kBKBytes - 1) / kBKBytes;
        const uint32_t b = ti % kBufs, bph = (ti / kBufs) & 1;
        mbar_wait(&tempty[b], bph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t tacc = tmem + b * kSplit * kTcBN;
        // split accumulation (kSplit == 2): k-blocks [0, kh) into the first
        // accumulator, [kh, nk) into the second (the epilogue sees the
        // partial sum at K/2: the trend term of the certificate)
        const int kh = kSplit == 2 ? split_kh(nk) : nk;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % kStages;
          mbar_wait(&full[s], (it / kStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const int nmma = min(4, (kbytes - kb * kBKBytes) / 32);
          const uint32_t a0 = smem_u32(sA + s * kAStage), b0 = smem_u32(sB + s * kBStage);
          const uint32_t tdst = kb < kh ? tacc : tacc + kTcBN;
          const int kb0 = kb < kh ? 0 : kh;
          for (int k = 0; k < nmma; ++k)
            mma<ELEM>(tdst, sw128_desc(a0 + k * 32), sw128_desc(b0 + k * 32), idesc,
                      (kb != kb0 || k != 0) ? 1u : 0u);
          mma_commit(&empty[s]);
        }
        mma_commit(&tfull[b]);
      }
    }
  } else if (warp == 2) {  // tile metadata, one TMEM buffer ahead of the epilogue
    uint32_t ti = 0;
    for (int tile = blockIdx.x; tile < L.total_tiles; tile += gridDim.x, ++ti) {
      const uint32_t b = ti % kBufs, bph = (ti / kBufs) & 1;
      mbar_wait(&mempty[b], bph ^ 1);
      TileMeta& md = meta[b];
      const int ji = job_of(L, jobs, tile);
      const TcJob& jg = jobs[ji];
      const int M = jg.M, N = jg.N, a_row0 = jg.a_row0;
      const float* bn = jg.b_norm;
      const int tiles_n = (N + kTcBN - 1) / kTcBN;
      const int mt = (tile - jg.tile0) / tiles_n, nt = (tile - jg.tile0) % tiles_n;
      if (lane == 0) md.jb = jg, md.mt = mt, md.nt = nt;
      const bool need = PREC != 2 && (L.a_norm || L.a_ss);
#pragma unroll
      for (int k = 0; k < kTcBM / 32; ++k) {
        const int r = mt * kTcBM + k * 32 + lane;
        md.na[k * 32 + lane] = need && r < M ? a_norm_of(L, a_row0 + r) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < kTcBN / 32; ++k) {
        const int c = nt * kTcBN + k * 32 + lane;
        float x = PREC != 2 && bn && c < N ? fabsf(__ldg(bn + c)) : 0.f;
        md.nb[k * 32 + lane] = x;
        // NaN-propagating max (a NaN norm must defeat the certificate shortcut)
        for (int o = 16; o > 0; o >>= 1) {
          const float y = __shfl_xor_sync(0xffffffffu, x, o);
          x = (x != x || y != y) ? __int_as_float(0x7FC00000) : fmaxf(x, y);
        }
        if (lane == 0) md.nbmax[k] = x;
      }
      mbar_arrive(&mfull[b]);  // count 32: every lane's stores are released
    }
  } else {  // epilogue warps: lanes quarter (warp % 4), 32-column chunk
    const int q = warp & 3, half = (warp - kEpiWarp0) >> 2;  // (half: the chunk index cq)
    uint32_t ti = 0;
    for (int tile = blockIdx.x; tile < L.total_tiles; tile += gridDim.x, ++ti) {
      const uint32_t b = ti % kBufs, bph = (ti / kBufs) & 1;
      mbar_wait(&mfull[b], bph);
      mbar_wait(&tfull[b], bph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      epilogue_tile<ELEM, PREC, EPI>(L, meta[b], tile, tmem + b * kSplit * kTcBN, q, half, lane,
                                     stage_all + (size_t)(warp - kEpiWarp0) * kStageFloats, gelu_s);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&tempty[b]);
        mbar_arrive(&mempty[b]);
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kAccBufs * kTcBN));
  }
}

template <int ELEM>
__device__ __forceinline__ void dec16(const uint4 v, float* out) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  if (ELEM == kTcBF16) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      out[2 * t] = __uint_as_float(w[t] << 16);
      out[2 * t + 1] = __uint_as_float(w[t] & 0xFFFF0000u);
    }
  } else {
#pragma unroll
    for (int t = 0; t < 16; ++t) out[t] = dec_e4m3((uint8_t)(w[t / 4] >> (8 * (t & 3))));
  }
}

constexpr int kFixThreads = 512;
constexpr int kFixCols = 4;   // flagged columns of one row per work item
constexpr int kFixPer = 2;    // work items per thread per round
// The fixup works on 2 x 2-tile super-tiles (256 x 256 outputs): the chains
// of ~4x as many flagged elements are in flight per SM (the chains are
// latency-bound: one dependent FHFMA chain per flagged element), and each
// K slice of the 256 A rows and 256 B rows is streamed once for 4 tiles.
constexpr int kFixStages = 6;  // ring slots (max) of g = 1 units (3 for g = 2)
#ifndef L_FIX_SLOTS1
#define L_FIX_SLOTS1 4
#endif
constexpr int kFixRows = 2 * kTcBM;                        // super-tile rows (= columns)
constexpr int kFixStageBytes = kFixRows * kBKBytes;        // 32 KB per operand per stage
constexpr int kFixMaxSplit = 4;  // CTAs sharing one super-tile when they are few
constexpr int kFixMaxItems = kFixRows * kFixRows / kFixCols + kFixRows;
// units of the tile fixup: 2 x 2-tile super-tiles (fix_g 2, the host table
// fix_st; BF16 K < 2048, where the chains are short and many flagged tiles
// share rows) or the GEMM's listed flagged tiles (fix_g 1, fix_tiles, count
// on the device; long chains and the near-empty E4M3 launches)
__host__ __device__ constexpr int fix_cap(int g) { return g * kTcBM * g * kTcBN / kFixCols + g * kTcBM; }
__device__ __forceinline__ int fix_n_units(const TcLaunch& L) {
  return L.fix_g == 2 ? L.n_fix_st : (int)*L.fix_count;
}
template <int G>
__device__ __forceinline__ int4 fix_unit_g(const TcLaunch& L, const TcJob* jobs, int i) {
  if (G == 2) return L.fix_st[i];
  const int tile = (int)L.fix_tiles[i];
  const int j = job_of(L, jobs, tile);
  const int tiles_n = (jobs[j].N + kTcBN - 1) / kTcBN;
  return make_int4(j, (tile - jobs[j].tile0) / tiles_n, (tile - jobs[j].tile0) % tiles_n, 0);
}
__device__ __forceinline__ int4 fix_unit(const TcLaunch& L, const TcJob* jobs, int i) {
  if (L.fix_g == 2) return L.fix_st[i];
  const int tile = (int)L.fix_tiles[i];
  const int j = job_of(L, jobs, tile);
  const int tiles_n = (jobs[j].N + kTcBN - 1) / kTcBN;
  return make_int4(j, (tile - jobs[j].tile0) / tiles_n, (tile - jobs[j].tile0) % tiles_n, 0);
}
constexpr size_t kFixSmem = 1024 + (size_t)3 * 2 * kFixStageBytes + 256 + 1024;
// ring slots and slot size per operand of a unit of g x g tiles (same bytes)
template <int G> constexpr int kFixSlots = G == 2 ? 3 : L_FIX_SLOTS1;

// A row's norm carries a sign bit when the row holds a value whose products
// might not be exact in FP32 (rownorm_kernel); otherwise fl(s + fl(a*b)) ==
// fma(a, b, s) bit for bit, because the product is exact.
__device__ __forceinline__ bool fma_safe(float norm) { return (__float_as_uint(norm) >> 31) == 0; }

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}

// k then k+1 (low half first) of two packed BF16 pairs: fma.rn.f32.bf16 is
// one rounding of the exact a*b + s (FHFMA.BF16 on sm_100a, no unpacking)
__device__ __forceinline__ float fma_bf16x2(uint32_t a, uint32_t b, float s) {
  asm("{\n.reg .b16 al, ah, bl, bh;\nmov.b32 {al, ah}, %1;\nmov.b32 {bl, bh}, %2;\n"
      "fma.rn.f32.bf16 %0, al, bl, %0;\nfma.rn.f32.bf16 %0, ah, bh, %0;\n}"
      : "+f"(s)
      : "r"(a), "r"(b));
  return s;
}

// Chains of one work item over 16-byte K units [u0, u0 + NU) of one chunk
// (SW128 layout: unit u of row r lives at (u ^ (r & 7)) << 4 within the row).
// All shared loads of the group are issued first (they are volatile, so the
// compiler keeps their order), then the CPI chains consume them.
template <int ELEM, bool FMA, int CPI, int NU>
__device__ __forceinline__ void fix_units(uint32_t a_row, uint32_t ra16, const uint32_t (&b_row)[kFixCols],
                                          const uint32_t (&rb16)[kFixCols], int u0,
                                          float (&acc)[kFixCols]) {
  uint4 av[NU], bv[CPI][NU];
#pragma unroll
  for (int u = 0; u < NU; ++u) av[u] = lds128(a_row | (((uint32_t)(u0 + u) << 4) ^ ra16));
#pragma unroll
  for (int c = 0; c < CPI; ++c)
#pragma unroll
    for (int u = 0; u < NU; ++u) bv[c][u] = lds128(b_row[c] | (((uint32_t)(u0 + u) << 4) ^ rb16[c]));
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    if (ELEM == kTcBF16 && FMA) {
#pragma unroll
      for (int c = 0; c < CPI; ++c) {
        float s = acc[c];
        s = fma_bf16x2(av[u].x, bv[c][u].x, s);
        s = fma_bf16x2(av[u].y, bv[c][u].y, s);
        s = fma_bf16x2(av[u].z, bv[c][u].z, s);
        s = fma_bf16x2(av[u].w, bv[c][u].w, s);
        acc[c] = s;
      }
    } else {
      constexpr int vel = ELEM == kTcBF16 ? 8 : 16;
      float x[vel];
      dec16<ELEM>(av[u], x);
#pragma unroll
      for (int c = 0; c < CPI; ++c) {
        float y[vel];
        dec16<ELEM>(bv[c][u], y);
        float s = acc[c];
#pragma unroll
        for (int t = 0; t < vel; ++t) s = FMA ? __fmaf_rn(x[t], y[t], s) : __fadd_rn(s, __fmul_rn(x[t], y[t]));
        acc[c] = s;
      }
    }
  }
}

template <int ELEM, bool FMA, int CPI>
__device__ __forceinline__ void fix_chunk(uint32_t a_row, uint32_t ra16, uint32_t b_stage,
                                          const int (&col)[kFixCols], int nu, float (&acc)[kFixCols]) {
  uint32_t b_row[kFixCols], rb16[kFixCols];
#pragma unroll
  for (int c = 0; c < CPI; ++c) b_row[c] = b_stage + col[c] * kBKBytes, rb16[c] = (col[c] & 7) << 4;
  if (nu == 8) {
    fix_units<ELEM, FMA, CPI, 4>(a_row, ra16, b_row, rb16, 0, acc);
    fix_units<ELEM, FMA, CPI, 4>(a_row, ra16, b_row, rb16, 4, acc);
  } else {
    for (int u = 0; u < nu; ++u) fix_units<ELEM, FMA, CPI, 1>(a_row, ra16, b_row, rb16, u, acc);
  }
}

struct FixItem {
  int row;  // -1: none
  int nc;
  bool fma;
  int col[kFixCols];
  float acc[kFixCols];
};

// A TMA stream of the tile fixup: one round of one super-tile's K extent.
struct FixStream {
  int valid, arow, brow, bk0, nk, g;  // g: 128-row boxes per operand
};

template <int ELEM, int G>
__device__ __forceinline__ void fix_issue(const TcLaunch& L, uint8_t* sA, uint8_t* sB, uint64_t* full,
                                          uint64_t* empty, uint32_t& ld, const FixStream& f, int kb) {
  constexpr int bke = kBKBytes / (ELEM == kTcBF16 ? 2 : 1);
  constexpr int ns = kFixSlots<G>, sb = G * kTcBM * kBKBytes;
  const int s = ld % ns;
  mbar_wait(&empty[s], ((ld / ns) & 1) ^ 1);
  mbar_expect_tx(&full[s], 2 * sb);
  uint8_t* a = sA + s * sb;
  uint8_t* b = sB + s * sb;
  // G 128-row boxes per operand: row r of the unit sits at r * 128 B (past a
  // job's or tensor's last row: unused rows / TMA zero fill)
#pragma unroll
  for (int h = 0; h < G; ++h) {
    tma_load_2d(a + h * kTcBM * kBKBytes, &L.tmA, &full[s], kb * bke, f.arow + h * kTcBM);
    tma_load_2d(b + h * kTcBN * kBKBytes, &L.tmB, &full[s], f.bk0 + kb * bke, f.brow + h * kTcBN);
  }
  ++ld;
}

// One round of the TMA ring over the tile's K extent for this thread's items.
// The producer (thread 0) keeps the ring full across rounds: once the current
// stream's stages are all issued it issues the next round's (nxt), so the
// next tile's first stages arrive while this round's chains finish.
template <int ELEM, int G, int CPI>
__device__ __forceinline__ void fix_round(const TcLaunch& L, FixItem (&w)[kFixPer], uint8_t* sA,
                                          uint8_t* sB, uint64_t* full, uint64_t* empty,
                                          const FixStream& cur, const FixStream& nxt, int& nxt_issued,
                                          int kbytes, uint32_t& ld, uint32_t& it) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int nk = cur.nk;
  constexpr int ns = kFixSlots<G>, sb = G * kTcBM * kBKBytes;
  for (int kb = 0; kb < nk; ++kb, ++it) {
    const int s = it % ns;
    if (L.fix_dry != 2) mbar_wait(&full[s], (it / ns) & 1);
    const uint32_t a0 = smem_u32(sA + s * sb), b0 = smem_u32(sB + s * sb);
    const int nu = min(8, (kbytes - kb * kBKBytes) / 16);
#pragma unroll
    for (int j = 0; j < kFixPer; ++j) {
      // (timing experiments, wrong results: fix_dry 1 streams without chains,
      // 2 runs the chains on whatever shared memory holds, without streaming)
      if (w[j].row < 0 || L.fix_dry == 1) continue;
      const uint32_t ar = a0 + w[j].row * kBKBytes, ra16 = (w[j].row & 7) << 4;
      if (w[j].fma) fix_chunk<ELEM, true, CPI>(ar, ra16, b0, w[j].col, nu, w[j].acc);
      else fix_chunk<ELEM, false, CPI>(ar, ra16, b0, w[j].col, nu, w[j].acc);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (tid == 0 && L.fix_dry != 2) {
      if (kb + ns < nk) fix_issue<ELEM, G>(L, sA, sB, full, empty, ld, cur, kb + ns);
      else if (nxt.valid && kb + ns - nk < nxt.nk && nxt_issued == kb + ns - nk) {
        fix_issue<ELEM, G>(L, sA, sB, full, empty, ld, nxt, nxt_issued);
        ++nxt_issued;
      }
    }
  }
}

// Item lists of the launch's super-tiles (fix_plan_kernel): per super-tile,
// up to kFixMaxItems 64-bit items  row | ncol << 8 | col_c << (16 + 12 c)
// (rows / columns 0..255 of the super-tile), the FMA-safety of the item in
// bit 27 (col_0's spare bit 11), and the count n | cpi << 24 in fix_n. Built
// once per launch by a separate kernel, so the fixup's per-super-tile setup
// is one load of n and one load of each thread's items.
constexpr uint64_t kFixItemFma = 1ull << 27;

template <int ELEM>
__global__ void __launch_bounds__(kFixRows) fix_plan_kernel(const __grid_constant__ TcLaunch L,
                                                            const TcJob* __restrict__ jobs) {
  __shared__ int wsum[kFixRows / 32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = L.fix_g, n_units = fix_n_units(L), cap = fix_cap(g);
  for (int si = blockIdx.x; si < n_units; si += gridDim.x) {
    const int4 sd = fix_unit(L, jobs, si);  // job, first row tile, first column tile
    const TcJob& jb = jobs[sd.x];
    const int tiles_m = (jb.M + kTcBM - 1) / kTcBM, tiles_n = (jb.N + kTcBN - 1) / kTcBN;
    const int mt = sd.y + tid / kTcBM, rr = tid % kTcBM, q = rr >> 5;
    uint32_t wm[8];
#pragma unroll
    for (int ct = 0; ct < 2; ++ct) {
      uint4 m = make_uint4(0u, 0u, 0u, 0u);
      uint32_t parts = 0u;
      if (tid < g * kTcBM && ct < g && mt < tiles_m && sd.z + ct < tiles_n) {
        const int tile = jb.tile0 + mt * tiles_n + sd.z + ct;
        parts = L.tile_mark[tile];
        if (parts) m = *reinterpret_cast<const uint4*>(L.fix_mask + (size_t)tile * kFixWords + rr * 4);
      }
      // (word k of a row is valid where its 32 x 32 part, bit q + 4 k, flagged)
      wm[4 * ct + 0] = (parts >> q) & 1u ? m.x : 0u;
      wm[4 * ct + 1] = (parts >> (q + 4)) & 1u ? m.y : 0u;
      wm[4 * ct + 2] = (parts >> (q + 8)) & 1u ? m.z : 0u;
      wm[4 * ct + 3] = (parts >> (q + 12)) & 1u ? m.w : 0u;
    }
    int pc = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) pc += __popc(wm[k]);
    if (!__syncthreads_or(pc)) {  // nothing flagged in this unit (most E4M3 tiles)
      if (tid == 0) L.fix_n[si] = 0u;
      continue;
    }
    int tot = pc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    __syncthreads();  // (wsum reuse)
    if (lane == 0) wsum[warp] = tot;
    __syncthreads();
    int n_el = 0;
#pragma unroll
    for (int w = 0; w < kFixRows / 32; ++w) n_el += wsum[w];
    // columns per item: one while the fixup CTA has idle threads, up to
    // kFixCols when there is work to spare or the list would overflow
    const int need = (n_el + kFixThreads * kFixPer - 1) / (kFixThreads * kFixPer);
    const int cap_cpi = n_el + g * kTcBM <= cap ? 1 : (n_el / 2 + g * kTcBM <= cap ? 2 : kFixCols);
    const int cpi = L.fix_cpi ? max(L.fix_cpi, cap_cpi) : max(cap_cpi, need <= 1 ? 1 : (need == 2 ? 2 : kFixCols));
    const int cnt = (pc + cpi - 1) / cpi;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    __syncthreads();
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int pos = incl - cnt, n = 0;
    for (int w = 0; w < kFixRows / 32; ++w) {
      if (w < warp) pos += wsum[w];
      n += wsum[w];
    }
    const int grow = sd.y * kTcBM + tid;  // row within the job
    // (rows past the job have no flagged elements: their norms are not read)
    const bool row_ok = ELEM == kTcE4M3 || grow >= jb.M || a_fma_safe(L, jb.a_row0 + grow);
    uint64_t* out = L.fix_items + (size_t)si * cap;
    uint64_t item = 0;
    int nc = 0;
    bool ok = row_ok;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t mm = wm[k];
      while (mm) {
        const int bit = __ffs(mm) - 1;
        mm &= mm - 1;
        const int col = k * 32 + bit;
        item |= (uint64_t)col << (16 + 12 * nc);
        if (ELEM == kTcBF16) ok = ok && fma_safe(jb.b_norm[sd.z * kTcBN + col]);
        if (++nc == cpi) {
          out[pos++] = item | (uint64_t)tid | ((uint64_t)nc << 8) | (ok ? kFixItemFma : 0ull);
          item = 0, nc = 0, ok = row_ok;
        }
      }
    }
    if (nc) out[pos++] = item | (uint64_t)tid | ((uint64_t)nc << 8) | (ok ? kFixItemFma : 0ull);
    if (tid == 0) L.fix_n[si] = (uint32_t)n | ((uint32_t)cpi << 24);
  }
}

// The stream (geometry) of super-tile si
template <int ELEM, int G>
__device__ __forceinline__ FixStream fix_stream_of(const TcLaunch& L, const TcJob* jobs, uint32_t si) {
  const int4 sd = fix_unit_g<G>(L, jobs, (int)si);
  const TcJob& jb = jobs[sd.x];
  FixStream f;
  f.valid = 1, f.arow = jb.a_row0 + sd.y * kTcBM, f.brow = jb.b_row0 + sd.z * kTcBN, f.bk0 = jb.b_k0;
  f.nk = (jb.K * (ELEM == kTcBF16 ? 2 : 1) + kBKBytes - 1) / kBKBytes;
  f.g = G;
  return f;
}

// Exact sequential recomputation of the flagged elements (dot_col order,
// kernels.cpp:44-52: every product rounded, then added, k ascending). One
// CTA per listed tile: the tile's A rows and B rows stream through a TMA ring
// (the GEMM's own SW128 tensor maps) once per round, and every thread runs
// the FP32 chains of its work items out of shared memory. A work item is up
// to kFixCols flagged columns of one row (the A unit is loaded once for all).
// Where every product is exact in FP32 the chain uses FMA (identical
// result), for BF16 straight from the packed pairs (FHFMA.BF16).
template <int ELEM, int G>
__global__ void __launch_bounds__(kFixThreads, 1)
    gemm_fixup_kernel(const __grid_constant__ TcLaunch L, const TcJob* __restrict__ jobs) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment by pointer arithmetic on the shared array itself, so
  // the compiler keeps every derived access in the shared address space
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  constexpr int ring = kFixSlots<G> * G * kTcBM * kBKBytes;  // bytes per operand
  uint8_t* sB = smem + ring;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + ring);
  uint64_t* empty = full + kFixStages;
  constexpr int esz = ELEM == kTcBF16 ? 2 : 1;
  constexpr int kWarps = kFixThreads / 32;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kFixSlots<G>; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t n_tiles = *L.fix_count;  // (listed GEMM tiles: their marks are reset at the end)
  uint32_t ld = 0, it = 0;  // TMA loads issued / chunks consumed (ring phases)
  // Few super-tiles (small launches): split each one's work items over up to
  // kFixMaxSplit CTAs (each streams the operands; L2 absorbs the repeats) so
  // every SM has work.
  const uint32_t n_st = G == 2 ? (uint32_t)L.n_fix_st : *L.fix_count;
  const uint32_t split = n_st ? min((uint32_t)kFixMaxSplit, max(1u, gridDim.x / n_st)) : 1u;
  const uint32_t n_vt = n_st * split;
  constexpr int cap = fix_cap(G);
  auto range = [&](uint32_t vt, int& lo, int& hi) {  // item range of virtual tile vt
    const uint32_t n = L.fix_n[vt / split] & 0xFFFFFFu, part = vt % split;
    lo = (int)((uint64_t)n * part / split), hi = (int)((uint64_t)n * (part + 1) / split);
  };
  // thread 0's lookahead: the next round's stream and how many of its stages are issued
  FixStream nxt{0, 0, 0, 0, 0, 1};
  int nxt_issued = 0;
  for (uint32_t vt = blockIdx.x; vt < n_vt; vt += gridDim.x) {
    int e_lo, e_hi;
    range(vt, e_lo, e_hi);
    if (e_lo >= e_hi) continue;
    const uint32_t ti = vt / split;  // super-tile
    const int cpi = (int)(L.fix_n[ti] >> 24);
    const int4 sd = fix_unit_g<G>(L, jobs, (int)ti);
    const TcJob jb = jobs[sd.x];
    const int mt = sd.y, nt = sd.z;  // first row / column tile
    const FixStream cur = fix_stream_of<ELEM, G>(L, jobs, ti);
    const int kbytes = jb.K * esz;
    const uint64_t* items = L.fix_items + (size_t)ti * cap;
    for (int e0 = e_lo; e0 < e_hi; e0 += kFixThreads * kFixPer) {
      if (tid == 0 && L.fix_dry != 2) {
        // prologue: the stages of this round the previous round did not issue
        for (int kb = nxt_issued; kb < min(kFixSlots<G>, cur.nk); ++kb)
          fix_issue<ELEM, G>(L, sA, sB, full, empty, ld, cur, kb);
        nxt_issued = 0;
        // the round after this one: this unit again, or the next non-empty virtual unit
        nxt.valid = 0;
        if (e0 + kFixThreads * kFixPer < e_hi) {
          nxt = cur;
        } else {
          for (uint32_t v2 = vt + gridDim.x; v2 < n_vt; v2 += gridDim.x) {
            int l2, h2;
            range(v2, l2, h2);
            if (l2 < h2) {
              nxt = fix_stream_of<ELEM, G>(L, jobs, v2 / split);
              break;
            }
          }
        }
      }
      FixItem w[kFixPer];
#pragma unroll
      for (int j = 0; j < kFixPer; ++j) {
        const int e = e0 + j * kFixThreads + tid;
        const uint64_t item = e < e_hi ? __ldg(items + e) : 0ull;
        w[j].row = e < e_hi ? (int)(item & 0xFF) : -1;  // (0..255: the super-tile row)
        w[j].nc = (int)((item >> 8) & 0xFF);
        w[j].fma = (item & kFixItemFma) != 0;
#pragma unroll
        for (int c = 0; c < kFixCols; ++c) {
          // missing columns of a short item repeat its first (results unused)
          w[j].col[c] = c < w[j].nc ? (int)((item >> (16 + 12 * c)) & 0x7FF) : (int)((item >> 16) & 0x7FF);
          w[j].acc[c] = 0.f;
        }
      }
      if (cpi == 1) fix_round<ELEM, G, 1>(L, w, sA, sB, full, empty, cur, nxt, nxt_issued, kbytes, ld, it);
      else if (cpi == 2) fix_round<ELEM, G, 2>(L, w, sA, sB, full, empty, cur, nxt, nxt_issued, kbytes, ld, it);
      else fix_round<ELEM, G, kFixCols>(L, w, sA, sB, full, empty, cur, nxt, nxt_issued, kbytes, ld, it);
#pragma unroll
      for (int j = 0; j < kFixPer; ++j) {
        if (w[j].row < 0 || L.fix_dry) continue;  // (timing experiments store nothing)
#pragma unroll
        for (int c = 0; c < kFixCols; ++c) {
          if (c >= w[j].nc) continue;
          float v = round_out(w[j].acc[c], jb.prec);
          if (jb.epi == 1) {
            if (jb.prec == 1 && L.gelu_lut) v = dec_bf16(L.gelu_lut[enc_bf16(v)]);
            else v = round_out(gelu_ref(v), jb.prec);
          }
          store_out(jb, mt * kTcBM + w[j].row, nt * kTcBN + w[j].col[c], v);
        }
      }
    }
  }
  // The last CTA to finish clears the listed tiles' marks and the count for
  // the next launch (fix_count[1] counts finished CTAs).
  __shared__ int last_cta;
  if (tid == 0) {
    __threadfence();
    last_cta = atomicAdd(L.fix_count + 1, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last_cta) {
    __threadfence();
    for (uint32_t i = tid; i < n_tiles; i += blockDim.x) L.tile_mark[L.fix_tiles[i]] = 0u;
    __syncthreads();
    if (tid == 0) {
      L.fix_count[0] = 0u;
      L.fix_count[1] = 0u;
    }
  }
}

// ---- block fixup (BF16) ---------------------------------------------------------
// The tile fixup above streams a whole 128 x 128 tile's operands (A 128 x K
// and B 128 x K) through shared memory to recompute the 2.5-4.5% of its
// elements the certificate flags: as many operand bytes as the GEMM itself, so
// it runs at L2 -> SM streaming speed. Here a CTA owns a chunk of up to 4 x 6
// GEMM tiles (512 rows x 768 columns): each 32-byte K slice of the chunk's A
// rows and B rows is loaded once (TMA, SWIZZLE_32B) and serves every flagged
// element of the chunk. The chains stay exact and sequential (dot_col,
// kernels.cpp:44-52).
//
// Lanes: a warp runs "packs" of up to 32 flagged elements drawn from one group
// of 8 consecutive chunk rows, 4 elements per column class (col mod 8). In the
// SW32 layout row r's 16-byte unit u sits in bank group
// 2 (r & 3) + (u ^ ((r >> 2) & 1)), distinct for the 8 rows of a group, and a
// column's likewise per column class. A 128-bit shared load is served per
// quarter-warp, and every quarter holds one lane per column class: both
// operands of a pack are conflict-free (4 wavefronts each; empty lanes read
// their own class's column and the group's first row). Each lane keeps one FP32 chain per pack it
// holds (kFbSlots accumulators), run kFbChunk at a time without branches.
//
// Scheduling: persistent CTAs take chunks from a host-built list through an
// atomic counter; the list starts with 4-row-tile chunks and ends with
// 1-row-tile ones, so the tail is balanced.
constexpr int kFbStages = 4;
constexpr int kFbThreads = 512, kFbWarps = kFbThreads / 32;
constexpr int kFbSlots = 16;   // packs per lane per round (register accumulators)
constexpr int kFbChunk = 8;    // chains run together (independent FHFMA chains, loads in flight)
constexpr int kFbGroup = 8;    // rows per pack group
constexpr int kFbMaxCT = 6;    // column tiles per chunk (768 columns)
constexpr uint32_t kFbBox = 256 * 32;  // one TMA box: 256 rows x 32 B
constexpr uint32_t kFbStageA = 2 * kFbBox, kFbStageB = 3 * kFbBox;  // 512 / 768 rows
constexpr size_t kFbSmem = 1024 + (size_t)kFbStages * (kFbStageA + kFbStageB) + 512 +
                           (size_t)kFbWarps * kFbSlots * 32 * 4;
constexpr uint32_t kFbEmpty = 0x80000000u, kFbUnsafe = 0x40000000u;

// byte offset of row r's unit 0 in a stage (256-row SW32 boxes)
__device__ __forceinline__ uint32_t fb_off(uint32_t r) {
  return (r >> 8) * kFbBox + (r & 255u) * 32u + (((r >> 2) & 1u) << 4);
}

__device__ __forceinline__ void fb_issue(const TcLaunch& L, uint8_t* sA, uint8_t* sB, uint64_t* full,
                                         uint64_t* empty, uint32_t& ld, int sg, int arow, int brow,
                                         int nba, int nbb) {
  const int s = ld % kFbStages;
  mbar_wait(&empty[s], ((ld / kFbStages) & 1) ^ 1);
  mbar_expect_tx(&full[s], (uint32_t)(nba + nbb) * kFbBox);
  uint8_t* a = sA + s * kFbStageA;
  uint8_t* b = sB + s * kFbStageB;
  for (int h = 0; h < nba; ++h) tma_load_2d(a + h * kFbBox, &L.fxA, &full[s], sg * 16, arow + 256 * h);
  for (int h = 0; h < nbb; ++h) tma_load_2d(b + h * kFbBox, &L.fxB, &full[s], sg * 16, brow + 256 * h);
  ++ld;
}

// 8 products of one 16-byte unit, k ascending, not FMA-safe (fmul + fadd)
__device__ __forceinline__ float fb_slow(uint4 a, uint4 b, float s) {
  float x[8], y[8];
  dec16<kTcBF16>(a, x);
  dec16<kTcBF16>(b, y);
#pragma unroll
  for (int t = 0; t < 8; ++t) s = __fadd_rn(s, __fmul_rn(x[t], y[t]));
  return s;
}

// One ring stage (two 16-byte K units) of the lane's packs, kFbChunk chains
// at a time (their 2 x kFbChunk shared loads are issued together).
// FMA: FHFMA.BF16 (every product exact in FP32); otherwise fmul + fadd.
template <bool FMA>
__device__ __forceinline__ void fb_stage(const uint8_t* as, const uint8_t* bs, const uint32_t (&ra)[kFbSlots],
                                         const uint32_t (&cb)[kFbSlots], float (&acc)[kFbSlots], int nch) {
#pragma unroll
  for (int u = 0; u < 2; ++u) {
#pragma unroll
    for (int jc = 0; jc < kFbSlots / kFbChunk; ++jc) {
      if (jc < nch) {
        uint4 av[kFbChunk], bv[kFbChunk];
#pragma unroll
        for (int t = 0; t < kFbChunk; ++t) {
          av[t] = *reinterpret_cast<const uint4*>(as + (ra[kFbChunk * jc + t] ^ (u << 4)));
          bv[t] = *reinterpret_cast<const uint4*>(bs + (cb[kFbChunk * jc + t] ^ (u << 4)));
        }
        float* a = acc + kFbChunk * jc;
        if (FMA) {
#pragma unroll
          for (int t = 0; t < kFbChunk; ++t) a[t] = fma_bf16x2(av[t].x, bv[t].x, a[t]);
#pragma unroll
          for (int t = 0; t < kFbChunk; ++t) a[t] = fma_bf16x2(av[t].y, bv[t].y, a[t]);
#pragma unroll
          for (int t = 0; t < kFbChunk; ++t) a[t] = fma_bf16x2(av[t].z, bv[t].z, a[t]);
#pragma unroll
          for (int t = 0; t < kFbChunk; ++t) a[t] = fma_bf16x2(av[t].w, bv[t].w, a[t]);
        } else {
#pragma unroll
          for (int t = 0; t < kFbChunk; ++t) a[t] = fb_slow(av[t], bv[t], a[t]);
        }
      }
    }
  }
}

__global__ void __launch_bounds__(kFbThreads, 1)
    gemm_fixup_blk_kernel(const __grid_constant__ TcLaunch L, const TcJob* __restrict__ jobs) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + kFbStages * kFbStageA;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kFbStages * kFbStageB);
  uint64_t* empty = full + kFbStages;
  uint32_t* rbad = reinterpret_cast<uint32_t*>(empty + kFbStages);  // [16] rows not FMA-safe
  uint32_t* cbad = rbad + 16;                                      // [24] columns not FMA-safe
  int* s_chunk = reinterpret_cast<int*>(cbad + 24);
  uint32_t* packs = reinterpret_cast<uint32_t*>(smem + kFbStages * (kFbStageA + kFbStageB) + 512);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t* wp = packs + warp * kFbSlots * 32;
  if (tid == 0) {
    for (int s = 0; s < kFbStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kFbWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t ld = 0, it = 0;  // stages loaded / consumed (ring phases)
  // column class (col mod 8) and index within the class: a 128-bit shared
  // load is served per quarter-warp (8 lanes), so each quarter holds the 8
  // classes once (B conflict-free) and rows of one group (A conflict-free)
  const int lb = lane & 7, lt = lane >> 3;
  const uint32_t cmask = 0x01010101u << lb;
  for (;;) {
    __syncthreads();  // (previous chunk's shared state is dead)
    if (tid == 0) *s_chunk = (int)atomicAdd(L.fix_count + 4, 1u);
    __syncthreads();
    const int ci = *s_chunk;
    if (ci >= L.n_fix_blocks) break;
    const int4 cd = L.fix_blocks[ci];  // job, first row tile, first column tile, nrt | nct << 8
    const TcJob jb = jobs[cd.x];
    const int tiles_n = (jb.N + kTcBN - 1) / kTcBN;
    const int mt0 = cd.y, nt0 = cd.z, nrt = cd.w & 255, nct = cd.w >> 8;
    const int n_stages = jb.K / 16;  // K is a multiple of 16 (tc_dims_ok)
    const int arow = jb.a_row0 + mt0 * kTcBM, brow = jb.b_row0 + nt0 * kTcBN;
    const int nba = (nrt * kTcBM + 255) / 256, nbb = (nct * kTcBN + 255) / 256;
    const int W = nct * 4;  // flag words per chunk row
    // FMA safety of the chunk's rows and columns (one bit each)
    {
      const bool rb = tid < nrt * kTcBM && !a_fma_safe(L, arow + tid);
      const uint32_t br = __ballot_sync(0xffffffffu, rb);
      if (lane == 0) rbad[warp] = br;
      for (int c = tid; c < 768; c += kFbThreads) {
        const bool bc = c < nct * kTcBN && !fma_safe(jb.b_norm[nt0 * kTcBN + c]);
        const uint32_t bb = __ballot_sync(0xffffffffu, bc);
        if (lane == 0) cbad[c >> 5] = bb;
      }
    }
    __syncthreads();
    const int n_groups = nrt * (kTcBM / kFbGroup);
    int g = warp;  // this warp's current group ...
    int p0 = 0;    // ... and its first pack not yet run
    for (;;) {     // rounds: up to kFbSlots packs per warp, one pass over K each
      int ns = 0;
      while (g < n_groups && ns < kFbSlots) {
        const int r0 = g * kFbGroup, rt = r0 >> 7;
        // flag words of the group's 8 rows x W words: lane holds word lane + 32 q
        uint32_t wv[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) {
          const int k = lane + 32 * q, i = k / W, w = k - i * W, ct = w >> 2;
          wv[q] = 0u;
          if (i < kFbGroup) {
            const int tile = jb.tile0 + (mt0 + rt) * tiles_n + nt0 + ct;
            const int rr = (r0 + i) & 127;
            const uint32_t parts = L.tile_mark[tile];
            if ((parts >> ((rr >> 5) + 4 * (w & 3))) & 1u)
              wv[q] = L.fix_mask[(size_t)tile * kFixWords + rr * 4 + (w & 3)];
          }
        }
        const int room = kFbSlots - ns;
        int n = 0;  // elements of this lane's column class seen so far
#pragma unroll
        for (int q = 0; q < 6; ++q) {
          if (32 * q >= kFbGroup * W) break;
#pragma unroll 1
          for (int s = 0; s < 32; ++s) {
            uint32_t m = __shfl_sync(0xffffffffu, wv[q], s) & cmask;
            while (m) {
              const int bit = __ffs(m) - 1;
              m &= m - 1;
              const int pk = n >> 2;
              if ((n & 3) == lt && pk >= p0 && pk < p0 + room) {
                const int k = s + 32 * q, i = k / W, rb = r0 + i, col = (k - i * W) * 32 + bit;
                const bool bad = ((rbad[rb >> 5] >> (rb & 31)) | (cbad[col >> 5] >> (col & 31))) & 1u;
                wp[(ns + pk - p0) * 32 + lane] = ((uint32_t)rb << 16) | (uint32_t)col | (bad ? kFbUnsafe : 0u);
              }
              ++n;
            }
          }
        }
        const int pg = (__reduce_max_sync(0xffffffffu, (uint32_t)n) + 3) >> 2;  // packs of the group
        const int take = min(pg - p0, room);
        for (int s = 0; s < take; ++s)  // this lane's empty slots of those packs
          if (4 * (p0 + s) + lt >= n) wp[(ns + s) * 32 + lane] = kFbEmpty | ((uint32_t)r0 << 16) | (uint32_t)lb;
        ns += take;
        if (p0 + take >= pg) g += kFbWarps, p0 = 0;
        else p0 += take;
      }
      const int nch = (ns + kFbChunk - 1) / kFbChunk;
      for (int s = ns; s < kFbChunk * nch; ++s) wp[s * 32 + lane] = kFbEmpty | (uint32_t)lb;
      __syncwarp();
      if (!__syncthreads_or(ns > 0)) break;
      uint32_t ra[kFbSlots], cb[kFbSlots];
      float acc[kFbSlots];
      bool unsafe = false;
#pragma unroll
      for (int j = 0; j < kFbSlots; ++j) {
        const uint32_t d = j < kFbChunk * nch ? wp[j * 32 + lane] : kFbEmpty;
        ra[j] = fb_off((d >> 16) & 511u);
        cb[j] = fb_off(d & 1023u);
        acc[j] = 0.f;
        unsafe = unsafe || (d & kFbUnsafe) != 0u;
      }
      unsafe = __any_sync(0xffffffffu, unsafe);
      if (tid == 0)
        for (int sg = 0; sg < min(kFbStages, n_stages); ++sg)
          fb_issue(L, sA, sB, full, empty, ld, sg, arow, brow, nba, nbb);
      for (int sg = 0; sg < n_stages; ++sg, ++it) {
        const int s = it % kFbStages;
        mbar_wait(&full[s], (it / kFbStages) & 1);
        const uint8_t* as = sA + s * kFbStageA;
        const uint8_t* bs = sB + s * kFbStageB;
        if (!unsafe) fb_stage<true>(as, bs, ra, cb, acc, nch);
        else fb_stage<false>(as, bs, ra, cb, acc, nch);  // (rare: some product not exact in FP32)
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (tid == 0 && sg + kFbStages < n_stages)
          fb_issue(L, sA, sB, full, empty, ld, sg + kFbStages, arow, brow, nba, nbb);
      }
#pragma unroll
      for (int j = 0; j < kFbSlots; ++j) {
        const uint32_t d = j < kFbChunk * nch ? wp[j * 32 + lane] : kFbEmpty;  // (the list is still in place)
        if (!(d & kFbEmpty)) {
          float v = round_out(acc[j], jb.prec);
          if (jb.epi == 1) {
            if (jb.prec == 1 && L.gelu_lut) v = dec_bf16(L.gelu_lut[enc_bf16(v)]);
            else v = round_out(gelu_ref(v), jb.prec);
          }
          store_out(jb, mt0 * kTcBM + (int)((d >> 16) & 511u), nt0 * kTcBN + (int)(d & 1023u), v);
        }
      }
      __syncwarp();  // (the pack list is rebuilt by the next round)
    }
  }
  // The last CTA to finish clears the listed tiles' marks and the counters
  // for the next launch (fix_count[1] counts finished CTAs, [4] the chunk queue).
  __shared__ int last_cta;
  if (tid == 0) {
    __threadfence();
    last_cta = atomicAdd(L.fix_count + 1, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last_cta) {
    __threadfence();
    const uint32_t n_tiles = *reinterpret_cast<volatile uint32_t*>(L.fix_count);
    for (uint32_t i = tid; i < n_tiles; i += blockDim.x) L.tile_mark[L.fix_tiles[i]] = 0u;
    __syncthreads();
    if (tid == 0) {
      L.fix_count[0] = 0u;
      L.fix_count[1] = 0u;
      L.fix_count[4] = 0u;
    }
  }
}

// ---- the FP32 unembed on the tensor cores: 6-term BF16 split ------------------
// x = x0 + x1 + x2 + O(2^-27 |x|) with x0 = bf16(x), x1 = bf16(x - x0),
// x2 = bf16(x - x0 - x1) (each difference exact in FP32). The six products
// x2 w0, x1 w1, x0 w2, x1 w0, x0 w1, x0 w0 are exact in FP32 and carry the
// full FP32 dot product (the dropped x1 w2, x2 w1, x2 w2 are ~2^-24 relative).
// Operands are concatenated along K (6 blocks of D), small terms first so the
// accumulator is still small while they are added: A rows [x2|x1|x0|x1|x0|x0],
// B rows (vocabulary columns) [w0|w1|w2|w0|w1|w0].
__device__ __forceinline__ void split3(float x, uint16_t& h0, uint16_t& h1, uint16_t& h2) {
  h0 = enc_bf16(x);
  const float r1 = x - dec_bf16(h0);
  h1 = enc_bf16(r1);
  h2 = enc_bf16(r1 - dec_bf16(h1));
}

// one warp per row: A6 row + the row's L2 norm (the certificate's ||a||)
__global__ void split_rows_kernel(const float* __restrict__ x, int rows, int D, int ldx,
                                  uint16_t* __restrict__ out, float* __restrict__ anorm) {
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* xr = x + (int64_t)r * ldx;
  uint16_t* o = out + (int64_t)r * 6 * D;
  float ss = 0.f;
  for (int k = lane; k < D; k += 32) {
    const float v = xr[k];
    ss = fmaf(v, v, ss);
    uint16_t h0, h1, h2;
    split3(v, h0, h1, h2);
    o[k] = h2, o[D + k] = h1, o[2 * D + k] = h0, o[3 * D + k] = h1, o[4 * D + k] = h0, o[5 * D + k] = h0;
  }
  for (int s = 16; s > 0; s >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, s);
  if (lane == 0) anorm[r] = sqrtf(ss);
}

// W [D][V] row-major (the FP32 unembed image) -> B6 [V][6D] + column norms
__global__ void split_cols_kernel(const float* __restrict__ w, int D, int V, uint16_t* __restrict__ out) {
  __shared__ float t[32][33];
  const int k0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int k = k0 + i, n = n0 + threadIdx.x;
    t[i][threadIdx.x] = (k < D && n < V) ? w[(int64_t)k * V + n] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int n = n0 + i, k = k0 + threadIdx.x;
    if (n < V && k < D) {
      uint16_t h0, h1, h2;
      split3(t[threadIdx.x][i], h0, h1, h2);
      uint16_t* o = out + (int64_t)n * 6 * D;
      o[k] = h0, o[D + k] = h1, o[2 * D + k] = h2, o[3 * D + k] = h0, o[4 * D + k] = h1, o[5 * D + k] = h0;
    }
  }
}

__global__ void colnorm_kernel(const float* __restrict__ w, int D, int V, float* __restrict__ out) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= V) return;
  float ss = 0.f;
  for (int k = 0; k < D; ++k) {
    const float v = w[(int64_t)k * V + n];
    ss = fmaf(v, v, ss);
  }
  out[n] = sqrtf(ss);
}

__global__ void gelu_lut_kernel(uint16_t* lut) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < 65536u) lut[i] = enc_bf16(round_bf16(gelu_ref(dec_bf16((uint16_t)i))));
}

__global__ void rownorm_kernel(const uint8_t* A, int64_t lda, int elem, int rows, int k0, int K,
                               float* out) {
  const int warps = blockDim.x >> 5;
  const int r = blockIdx.x * warps + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int lane = threadIdx.x & 31;
  float s = 0.f;
  bool bad = false;  // a value whose products with the other operand may be inexact in FP32
  const uint8_t* p = A + (int64_t)r * lda;
  for (int k = lane; k < K; k += 32) {
    const float x = elem == kTcBF16 ? dec_bf16(reinterpret_cast<const uint16_t*>(p)[k0 + k])
                                    : dec_e4m3(p[k0 + k]);
    s = fmaf(x, x, s);
    // BF16 x BF16: 16 significant bits; exact iff |a|,|b| in [2^-67, 2^64) (or 0)
    const float ax = fabsf(x);
    bad = bad || !(ax == 0.f || (ax >= 6.7762635780344027e-21f && ax < 1.8446744073709552e19f));
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  bad = __any_sync(0xffffffffu, bad);
  // tiny guard for the FP32 sum itself; the sign bit marks "not FMA-safe"
  if (lane == 0) out[r] = (bad && elem == kTcBF16) ? -(sqrtf(s) * 1.0001f) : sqrtf(s) * 1.0001f;
}

__global__ void pack_t_kernel(const float* __restrict__ in, int K, int N, int ld_in, void* out,
                              int64_t ld_out, int elem) {
  __shared__ float t[32][33];
  const int k0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int k = k0 + i, n = n0 + threadIdx.x;
    t[i][threadIdx.x] = (k < K && n < N) ? in[(int64_t)k * ld_in + n] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int n = n0 + i, k = k0 + threadIdx.x;
    if (n < N && k < K) {
      const float v = t[threadIdx.x][i];
      if (elem == kTcBF16) reinterpret_cast<uint16_t*>(out)[(int64_t)n * ld_out + k] = enc_bf16(v);
      else reinterpret_cast<uint8_t*>(out)[(int64_t)n * ld_out + k] = enc_e4m3(v);
    }
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

}  // namespace

bool tc_make_map(CUtensorMap* map, const void* base, int elem, uint64_t rows, uint64_t cols_elems,
                 uint64_t pitch_bytes, uint32_t box_rows) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  const int esz = elem == kTcBF16 ? 2 : 1;
  cuuint64_t dims[2] = {cols_elems, rows};
  cuuint64_t strides[1] = {pitch_bytes};
  cuuint32_t box[2] = {(cuuint32_t)(kBKBytes / esz), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, elem == kTcBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8,
                  2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool tc_make_map_sw32(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols_elems,
                      uint64_t pitch_bytes) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols_elems, rows};
  cuuint64_t strides[1] = {pitch_bytes};
  cuuint32_t box[2] = {16, 256};  // 32 bytes of K x 256 rows (BF16)
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

void launch_gemm_tc(const TcLaunch& L, const TcJob* d_jobs, cudaStream_t st) {
  if (L.total_tiles <= 0) return;
  const int grid = std::min(L.total_tiles, 148);
  // (element, output precision, GELU epilogue) specialisations keep each
  // epilogue's code small (the generic one thrashed the instruction cache)
  auto go = [&](auto kern) {
    static bool attr = false;  // one static per instantiation of the lambda body
    (void)attr;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    kern<<<grid, kThreads, kSmemBytes, st>>>(L, d_jobs);
  };
  if (L.elem == kTcBF16) {
    if (L.prec == 1 && L.epi == 1) go(gemm_tc_kernel<kTcBF16, 1, 1>);
    else if (L.prec == 1) go(gemm_tc_kernel<kTcBF16, 1, 0>);
    else go(gemm_tc_kernel<kTcBF16, 2, 0>);
  } else {
    if (L.prec == 0 && L.epi == 1) go(gemm_tc_kernel<kTcE4M3, 0, 1>);
    else if (L.prec == 0) go(gemm_tc_kernel<kTcE4M3, 0, 0>);
    else go(gemm_tc_kernel<kTcE4M3, 2, 0>);
  }
}

void launch_gemm_fixup(const TcLaunch& L, const TcJob* d_jobs, cudaStream_t st) {
  if (L.total_tiles <= 0) return;
  const int units = L.fix_g == 2 ? L.n_fix_st : L.total_tiles;  // (g 1: an upper bound)
  if (units <= 0) return;
  // item lists of the launch's units
  if (L.elem == kTcBF16) fix_plan_kernel<kTcBF16><<<std::min(units, 4 * 148), kFixRows, 0, st>>>(L, d_jobs);
  else fix_plan_kernel<kTcE4M3><<<std::min(units, 4 * 148), kFixRows, 0, st>>>(L, d_jobs);
  const int grid = std::min(units * kFixMaxSplit, 148);
  // shared memory of the unit size's ring (a smaller carve-out leaves L1 to the item loads)
  const int slots = L.fix_g == 2 ? 3 : L_FIX_SLOTS1;
  const size_t smem = 1024 + (size_t)2 * slots * L.fix_g * kTcBM * kBKBytes + 256 + 1024;
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFixSmem);
    kern<<<grid, kFixThreads, smem, st>>>(L, d_jobs);
  };
  if (L.elem == kTcBF16) {
    if (L.fix_g == 2) go(gemm_fixup_kernel<kTcBF16, 2>);
    else go(gemm_fixup_kernel<kTcBF16, 1>);
  } else {
    if (L.fix_g == 2) go(gemm_fixup_kernel<kTcE4M3, 2>);
    else go(gemm_fixup_kernel<kTcE4M3, 1>);
  }
}

std::vector<int4> fixup_super_tiles(const TcJob* jobs, int n_jobs) {
  std::vector<int4> st;
  for (int j = 0; j < n_jobs; ++j) {
    const int tm = (jobs[j].M + kTcBM - 1) / kTcBM, tn = (jobs[j].N + kTcBN - 1) / kTcBN;
    for (int m = 0; m < tm; m += 2)
      for (int n = 0; n < tn; n += 2) st.push_back(make_int4(j, m, n, 0));
  }
  return st;
}

std::vector<int4> fixup_chunks(const TcJob* jobs, int n_jobs, int ctas) {
  // rows per chunk: what one round of kFbSlots packs per warp covers at the
  // measured flag rates (~4.5% at K = 3072, ~2.5% at K = 768)
  const long max_rt = n_jobs > 0 && jobs[0].K >= 2048 ? 1 : 2;
  struct Seg { int job, nt0, nct, tm; };
  std::vector<Seg> segs;
  long remaining = 0;  // row-tile units not yet emitted
  for (int j = 0; j < n_jobs; ++j) {
    const int tm = (jobs[j].M + kTcBM - 1) / kTcBM, tn = (jobs[j].N + kTcBN - 1) / kTcBN;
    const int ncb = (tn + kFbMaxCT - 1) / kFbMaxCT;
    for (int c = 0; c < ncb; ++c) {
      const int a = tn * c / ncb, b = tn * (c + 1) / ncb;  // balanced column blocks
      segs.push_back({j, a, b - a, tm});
      remaining += tm;
    }
  }
  std::vector<int4> out;
  for (const Seg& sg : segs)
    for (int mt = 0; mt < sg.tm;) {
      const int want = (int)std::max(1L, std::min(max_rt, remaining / (2L * ctas)));
      const int n = std::min(want, sg.tm - mt);
      out.push_back(make_int4(sg.job, mt, sg.nt0, n | sg.nct << 8));
      mt += n;
      remaining -= n;
    }
  return out;
}

void launch_gemm_fixup_blk(const TcLaunch& L, const TcJob* d_jobs, cudaStream_t st) {
  if (L.n_fix_blocks <= 0) return;
  const int grid = std::min(L.n_fix_blocks, 148);
  cudaFuncSetAttribute(gemm_fixup_blk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFbSmem);
  gemm_fixup_blk_kernel<<<grid, kFbThreads, kFbSmem, st>>>(L, d_jobs);
}

void launch_gelu_lut(uint16_t* lut, cudaStream_t st) { gelu_lut_kernel<<<256, 256, 0, st>>>(lut); }

// (diagnostics) the epilogue's GELU of all 2^16 BF16 codes: the shared-memory
// slice built as in gemm_tc_kernel, out[c] = gelu_code(c) (closed forms +
// slice), out_fast[c] = the fast path's lookup for codes inside the slice
// (0 elsewhere); both must equal the full table lut[c].
__global__ void gelu_codes_kernel(const uint16_t* lut, uint16_t* out, uint16_t* out_fast) {
  __shared__ uint16_t gs[kGeluSm];
  for (int i = threadIdx.x; i < kGeluSm; i += blockDim.x) {
    const int sg = i / (kGeluNE * 128), rem = i % (kGeluNE * 128);
    gs[i] = lut[(sg << 15) | ((kGeluE0 + rem / 128) << 7) | (rem % 128)];
  }
  __syncthreads();
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < 65536; c += gridDim.x * blockDim.x) {
    out[c] = (uint16_t)gelu_code((uint32_t)c, gs, lut);
    const uint32_t u = ((uint32_t)c & 0x7FFFu) - (uint32_t)(kGeluE0 * 128);
    out_fast[c] = u < (uint32_t)(kGeluNE * 128) ? gs[u + ((uint32_t)c >> 15) * (uint32_t)(kGeluNE * 128)] : 0;
  }
}

void launch_gelu_codes(const uint16_t* lut, uint16_t* out, uint16_t* out_fast, cudaStream_t st) {
  gelu_codes_kernel<<<64, 256, 0, st>>>(lut, out, out_fast);
}

void launch_split_rows(const float* x, int rows, int D, int ldx, uint16_t* out, float* anorm,
                       cudaStream_t st) {
  if (rows > 0) split_rows_kernel<<<(rows + 7) / 8, 256, 0, st>>>(x, rows, D, ldx, out, anorm);
}

void launch_split_cols(const float* w, int D, int V, uint16_t* out, float* wnorm, cudaStream_t st) {
  dim3 grid((V + 31) / 32, (D + 31) / 32), block(32, 8);
  split_cols_kernel<<<grid, block, 0, st>>>(w, D, V, out);
  colnorm_kernel<<<(V + 255) / 256, 256, 0, st>>>(w, D, V, wnorm);
}


void launch_rownorm(const uint8_t* A, int64_t lda, int elem, int rows, int k0, int K, float* out,
                    cudaStream_t st) {
  if (rows <= 0) return;
  rownorm_kernel<<<(rows + 7) / 8, 256, 0, st>>>(A, lda, elem, rows, k0, K, out);
}

void launch_pack_t(const float* in, int K, int N, int ld_in, void* out, int64_t ld_out, int elem,
                   cudaStream_t st) {
  dim3 grid((N + 31) / 32, (K + 31) / 32), block(32, 8);
  pack_t_kernel<<<grid, block, 0, st>>>(in, K, N, ld_in, out, ld_out, elem);
}

}  // namespace cqg
