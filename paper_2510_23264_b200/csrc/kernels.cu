// kernels.cu — exact-semantics sm_100a kernels of the patched forward.
//
// Every kernel reproduces the reference's FP32 operation order (no FMA
// contraction: explicit _rn intrinsics) so that its outputs are bit-equal to
// proj/src/kernels.cpp + model.cpp on the same inputs. These are the building
// blocks of the exact path and the fallback of the tensor-core GEMMs
// (gemm_tc.cu).
#include <float.h>
#include <math.h>
#include <stdlib.h>

#include "kernels.h"
#include "numerics.cuh"

namespace cqg {

int g_exact_x2 = 1;  // paired-FP32 big exact GEMM (option "exact_x2")

// ---------------------------------------------------------------------------
// K2a: fold (sum_inputs, model.cpp:537-552). HBM-bound, float4-vectorised.
// ---------------------------------------------------------------------------
// element i (float4 group i for VEC) of a node output of storage type t
__device__ __forceinline__ float4 load_out4(const void* b, int t, int64_t i) {
  if (t == kOutF32) return __ldg(reinterpret_cast<const float4*>(b) + i);
  if (t == kOutE4M3) {
    const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(b) + i);
    const float2 lo = __half22float2(__half2(__nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(w & 0xFFFFu), __NV_E4M3)));
    const float2 hi = __half22float2(__half2(__nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(w >> 16), __NV_E4M3)));
    return make_float4(lo.x, lo.y, hi.x, hi.y);
  }
  const uint2 w = __ldg(reinterpret_cast<const uint2*>(b) + i);
  return make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xFFFF0000u),
                     __uint_as_float(w.y << 16), __uint_as_float(w.y & 0xFFFF0000u));
}
__device__ __forceinline__ float load_out(const void* b, int t, int64_t i) {
  if (t == kOutF32) return reinterpret_cast<const float*>(b)[i];
  if (t == kOutE4M3) return dec_e4m3(reinterpret_cast<const uint8_t*>(b)[i]);
  return dec_bf16(reinterpret_cast<const uint16_t*>(b)[i]);
}

template <bool VEC>
__global__ void __launch_bounds__(256) fold_kernel(const FoldOp* __restrict__ ops,
                                                   const FoldProg* __restrict__ progs,
                                                   int64_t n_elems) {
  const FoldProg p = progs[blockIdx.y];
  if (VEC) {
    const int64_t n4 = n_elems >> 2;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
         i += (int64_t)gridDim.x * blockDim.x) {
      float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int o = p.op_begin; o < p.op_end; ++o) {
        const float* a = ops[o].a;
        float* d = ops[o].dst;
        float4 av;
        if (a == CQG_REG_PREV) av = r;
        else if (a == nullptr) av = make_float4(0.f, 0.f, 0.f, 0.f);
        else av = reinterpret_cast<const float4*>(a)[i];
        const float4 bv = load_out4(ops[o].b, ops[o].btype, i);
        r.x = __fadd_rn(av.x, bv.x);
        r.y = __fadd_rn(av.y, bv.y);
        r.z = __fadd_rn(av.z, bv.z);
        r.w = __fadd_rn(av.w, bv.w);
        if (d) reinterpret_cast<float4*>(d)[i] = r;
      }
    }
  } else {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_elems;
         i += (int64_t)gridDim.x * blockDim.x) {
      float r = 0.f;
      for (int o = p.op_begin; o < p.op_end; ++o) {
        const float* a = ops[o].a;
        float av = (a == CQG_REG_PREV) ? r : (a == nullptr ? 0.f : a[i]);
        r = __fadd_rn(av, load_out(ops[o].b, ops[o].btype, i));
        if (ops[o].dst) ops[o].dst[i] = r;
      }
    }
  }
}

// 16 elements per thread: a packed (E4M3) node output is then one 16-byte
// load per op, enough bytes in flight per thread to keep HBM busy (4-byte
// loads per op left the fold latency-bound at ~3 TB/s).
__device__ __forceinline__ void load_out16(const void* b, int t, int64_t i, float (&v)[16]) {
  if (t == kOutF32) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(b) + 4 * i + q);
      v[4 * q] = x.x, v[4 * q + 1] = x.y, v[4 * q + 2] = x.z, v[4 * q + 3] = x.w;
    }
  } else if (t == kOutE4M3) {
    const uint4 w = __ldg(reinterpret_cast<const uint4*>(b) + i);
    const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 lo = __half22float2(__half2(__nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(ww[q] & 0xFFFFu), __NV_E4M3)));
      const float2 hi = __half22float2(__half2(__nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(ww[q] >> 16), __NV_E4M3)));
      v[4 * q] = lo.x, v[4 * q + 1] = lo.y, v[4 * q + 2] = hi.x, v[4 * q + 3] = hi.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(b) + 2 * i + q);
      const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        v[8 * q + 2 * h] = __uint_as_float(ww[h] << 16);
        v[8 * q + 2 * h + 1] = __uint_as_float(ww[h] & 0xFFFF0000u);
      }
    }
  }
}

// Raw bytes of one op's 16 node-output elements (F32: 4 x 16 B, BF16: 2, E4M3: 1).
struct Raw16 { uint4 q[4]; };

__device__ __forceinline__ void load_raw16(const void* b, int t, int64_t i, Raw16& r) {
  const uint4* p = reinterpret_cast<const uint4*>(b);
  if (t == kOutF32) {
#pragma unroll
    for (int q = 0; q < 4; ++q) r.q[q] = __ldg(p + 4 * i + q);
  } else if (t == kOutE4M3) {
    r.q[0] = __ldg(p + i);
  } else {
#pragma unroll
    for (int q = 0; q < 2; ++q) r.q[q] = __ldg(p + 2 * i + q);
  }
}

__device__ __forceinline__ void decode_raw16(const Raw16& r, int t, float (&v)[16]) {
  if (t == kOutF32) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      v[4 * q] = __uint_as_float(r.q[q].x), v[4 * q + 1] = __uint_as_float(r.q[q].y);
      v[4 * q + 2] = __uint_as_float(r.q[q].z), v[4 * q + 3] = __uint_as_float(r.q[q].w);
    }
  } else if (t == kOutE4M3) {
    const uint32_t ww[4] = {r.q[0].x, r.q[0].y, r.q[0].z, r.q[0].w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 lo = __half22float2(__half2(__nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(ww[q] & 0xFFFFu), __NV_E4M3)));
      const float2 hi = __half22float2(__half2(__nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(ww[q] >> 16), __NV_E4M3)));
      v[4 * q] = lo.x, v[4 * q + 1] = lo.y, v[4 * q + 2] = hi.x, v[4 * q + 3] = hi.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const uint32_t ww[4] = {r.q[q].x, r.q[q].y, r.q[q].z, r.q[q].w};
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        v[8 * q + 2 * h] = __uint_as_float(ww[h] << 16);
        v[8 * q + 2 * h + 1] = __uint_as_float(ww[h] & 0xFFFF0000u);
      }
    }
  }
}

// kPipe: the next op's node-output bytes are loaded before this op's prefix
// store, so one op's HBM/L2 latency overlaps the previous op's add + store
// (the compiler cannot hoist them itself: the dst store may alias as far as it
// knows). Node outputs are read-only during a fold (they were already read
// with ld.global.nc), so the reordering does not change any value.
template <bool kPipe>
__device__ __forceinline__ void fold16_body(const FoldOp* __restrict__ ops,
                                            const FoldProg* __restrict__ progs,
                                            int64_t n_elems) {
  const FoldProg p = progs[blockIdx.y];
  const int64_t n16 = n_elems >> 4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
       i += (int64_t)gridDim.x * blockDim.x) {
    float r[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) r[k] = 0.f;
    Raw16 nxt;
    int tn = 0;
    if (kPipe && p.op_begin < p.op_end) {
      tn = ops[p.op_begin].btype;
      load_raw16(ops[p.op_begin].b, tn, i, nxt);
    }
    for (int o = p.op_begin; o < p.op_end; ++o) {
      const float* a = ops[o].a;
      float* d = ops[o].dst;
      float bv[16];
      if (kPipe) {
        const Raw16 cur = nxt;
        const int tc = tn;
        if (o + 1 < p.op_end) {
          tn = ops[o + 1].btype;
          load_raw16(ops[o + 1].b, tn, i, nxt);
        }
        decode_raw16(cur, tc, bv);
      } else {
        load_out16(ops[o].b, ops[o].btype, i, bv);
      }
      if (a != CQG_REG_PREV) {
        if (a == nullptr) {
#pragma unroll
          for (int k = 0; k < 16; ++k) r[k] = 0.f;
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 x = reinterpret_cast<const float4*>(a)[4 * i + q];
            r[4 * q] = x.x, r[4 * q + 1] = x.y, r[4 * q + 2] = x.z, r[4 * q + 3] = x.w;
          }
        }
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) r[k] = __fadd_rn(r[k], bv[k]);
      if (d)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          reinterpret_cast<float4*>(d)[4 * i + q] = make_float4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
    }
  }
}

__global__ void __launch_bounds__(256) fold16_kernel(const FoldOp* __restrict__ ops,
                                                     const FoldProg* __restrict__ progs,
                                                     int64_t n_elems) {
  fold16_body<false>(ops, progs, n_elems);
}

// Registers capped for four CTAs per SM.
__global__ void __launch_bounds__(256, 4) fold16_pipe_kernel(const FoldOp* __restrict__ ops,
                                                             const FoldProg* __restrict__ progs,
                                                             int64_t n_elems) {
  fold16_body<true>(ops, progs, n_elems);
}

// CQG_FOLD_PIPE=1 selects the pipelined fold. Measured slower: uncapped it
// takes 70 registers (3 CTAs per SM), fold 352 -> 475 ms per step
// (profiles/r2_fold_pipe_ab_*.json); capped at 64 for 4 CTAs per SM it is
// still 457 ms (profiles/r2_fold_pipe4_ab_*.json). The one-op lookahead does
// not pay for the warps it costs. Off by default.
static bool fold_pipe() {
  const char* e = getenv("CQG_FOLD_PIPE");
  return e && e[0] == '1';
}

void launch_fold(const FoldOp* d_ops, const FoldProg* d_progs, int n_progs, int64_t n_elems,
                 cudaStream_t st) {
  if (n_progs <= 0) return;
  if (n_elems % 16 == 0) {
    int gx = (int)std::min<int64_t>((n_elems / 16 + 255) / 256, 4096);
    for (int y0 = 0; y0 < n_progs; y0 += 65535) {
      dim3 grid(gx, (unsigned)std::min(65535, n_progs - y0));
      if (fold_pipe()) fold16_pipe_kernel<<<grid, 256, 0, st>>>(d_ops, d_progs + y0, n_elems);
      else fold16_kernel<<<grid, 256, 0, st>>>(d_ops, d_progs + y0, n_elems);
    }
    return;
  }
  const bool vec = (n_elems % 4) == 0;
  int64_t work = vec ? n_elems / 4 : n_elems;
  int gx = (int)((work + 255) / 256);
  if (gx > 4096) gx = 4096;
  for (int y0 = 0; y0 < n_progs; y0 += 65535) {
    dim3 grid(gx, (unsigned)std::min(65535, n_progs - y0));
    if (vec) fold_kernel<true><<<grid, 256, 0, st>>>(d_ops, d_progs + y0, n_elems);
    else fold_kernel<false><<<grid, 256, 0, st>>>(d_ops, d_progs + y0, n_elems);
  }
}

// ---------------------------------------------------------------------------
// K2b: layer norm (kernels.cpp:127-142): one thread per row, sequential FP32
// sums over the row, staged through padded shared-memory tiles so global
// loads stay coalesced.
// ---------------------------------------------------------------------------
constexpr int kLnRows = 128, kLnCh = 32;

__global__ void __launch_bounds__(kLnRows) ln_kernel(const LnJob* __restrict__ jobs,
                                                     const float* __restrict__ gamma,
                                                     const float* __restrict__ beta, int D,
                                                     int prec) {
  const LnJob j = jobs[blockIdx.y];
  const int r0 = blockIdx.x * kLnRows;
  if (r0 >= j.rows) return;
  __shared__ float tile[kLnRows][kLnCh + 1];
  __shared__ float s_mean[kLnRows], s_inv[kLnRows];
  const int tid = threadIdx.x;
  const int nr = min(kLnRows, j.rows - r0);
  float acc = 0.f;
  for (int pass = 0; pass < 2; ++pass) {
    const float mean = acc;
    acc = 0.f;
    for (int c0 = 0; c0 < D; c0 += kLnCh) {
      __syncthreads();
      for (int idx = tid; idx < kLnRows * kLnCh; idx += kLnRows) {
        const int rr = idx / kLnCh, cc = idx % kLnCh;
        tile[rr][cc] = (rr < nr && c0 + cc < D)
                           ? j.in[(int64_t)(r0 + rr) * j.in_stride + c0 + cc]
                           : 0.f;
      }
      __syncthreads();
      const int lim = min(kLnCh, D - c0);
      if (pass == 0) {
        for (int cc = 0; cc < lim; ++cc) acc = __fadd_rn(acc, tile[tid][cc]);
      } else {
        for (int cc = 0; cc < lim; ++cc) {
          const float c = __fsub_rn(tile[tid][cc], mean);
          acc = __fadd_rn(acc, __fmul_rn(c, c));
        }
      }
    }
    acc = __fdiv_rn(acc, (float)D);  // mean /= d  |  var /= d
    if (pass == 0) s_mean[tid] = acc;
  }
  s_inv[tid] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(acc, 1e-5f)));
  __syncthreads();
  for (int idx = tid; idx < nr * D; idx += kLnRows) {
    const int rr = idx / D, col = idx % D;
    const int64_t row = r0 + rr;
    const float x = j.in[row * j.in_stride + col];
    const float y = __fadd_rn(__fmul_rn(gamma[col], __fmul_rn(__fsub_rn(x, s_mean[rr]), s_inv[rr])),
                              beta[col]);
    if (j.xln) j.xln[row * D + col] = y;
    const float q = round_p(y, prec);
    if (j.xq) j.xq[row * D + col] = q;
    if (j.xqp) {
      if (j.pack == 2) reinterpret_cast<uint16_t*>(j.xqp)[row * D + col] = enc_bf16(q);
      else reinterpret_cast<uint8_t*>(j.xqp)[row * D + col] = enc_e4m3(q);
    }
  }
}

// Warp-per-32-rows variant: each warp owns a private padded 32 x 32 tile, so
// warps progress independently (no block barriers); each lane runs its row's
// sequential FP32 chain while the next 32-column chunk is already loading.
__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// One warp per 32 rows, lane = row for the two sequential reductions
// (mean = sum/D, var = sum((x-mean)^2)/D in column order, kernels.cpp:127-163).
// The row block streams through a cp.async ring of 32 x 32 chunks, so many
// chunks are in flight per warp; pass 3 normalises a chunk per lane-row and
// writes it back row by row (coalesced).
constexpr int kLnStages = 4;
constexpr int kLnWarps = 4;
constexpr int kLnTile = 32 * 33;

// Row norm bookkeeping of a packed tensor-core operand row (as rownorm_kernel
// in gemm_tc.cu): ||q|| * 1.0001 with the sign bit set when a BF16 value's
// products may be inexact in FP32 (|q| outside [2^-67, 2^64) and nonzero).
__device__ __forceinline__ bool bf16_fma_bad(float x) {
  const float ax = fabsf(x);
  return !(ax == 0.f || (ax >= 6.7762635780344027e-21f && ax < 1.8446744073709552e19f));
}

__global__ void __launch_bounds__(32 * kLnWarps) ln_warp_kernel(const LnJob* __restrict__ jobs,
                                                              const float* __restrict__ gamma,
                                                              const float* __restrict__ beta,
                                                              int D, int prec) {
  extern __shared__ float ln_sm[];
  const LnJob j = jobs[blockIdx.y];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = (blockIdx.x * kLnWarps + warp) * 32;
  if (r0 >= j.rows) return;
  float* ring = ln_sm + (size_t)warp * kLnStages * kLnTile;
  const int nr = min(32, j.rows - r0);
  const int nc = (D + 31) / 32;
  // source of element (row r, col c0 + lane), clamped into the valid block
  const int cl = lane;
  auto issue = [&](int ch) {
    float* t = ring + (ch % kLnStages) * kLnTile;
    const int c = min(ch * 32 + cl, D - 1);
#pragma unroll 8
    for (int r = 0; r < 32; ++r) {
      const int rr = min(r, nr - 1);
      cp_async4(t + r * 33 + cl, j.in + (int64_t)(r0 + rr) * j.in_stride + c);
    }
  };
  // vectorised normalisation pass: D and the row pitch in float4 units
  const bool vec = (D & 3) == 0 && (j.in_stride & 3) == 0 &&
                   ((reinterpret_cast<uintptr_t>(j.in) & 15) == 0);
  float mean = 0.f, acc = 0.f, inv = 0.f;
  const int npass = vec ? 2 : 3;
  for (int pass = 0; pass < npass; ++pass) {
    acc = 0.f;
#pragma unroll
    for (int p = 0; p < kLnStages - 1; ++p) {
      if (p < nc) issue(p);
      cp_async_commit();
    }
    float g_l = 0.f, b_l = 0.f;
    for (int ch = 0; ch < nc; ++ch) {
      if (ch + kLnStages - 1 < nc) issue(ch + kLnStages - 1);
      cp_async_commit();
      cp_async_wait<kLnStages - 1>();
      __syncwarp();
      float* t = ring + (ch % kLnStages) * kLnTile;
      const int c0 = ch * 32;
      const int lim = min(32, D - c0);
      if (pass == 0) {
        for (int cc = 0; cc < lim; ++cc) acc = __fadd_rn(acc, t[lane * 33 + cc]);
      } else if (pass == 1) {
        for (int cc = 0; cc < lim; ++cc) {
          const float c = __fsub_rn(t[lane * 33 + cc], mean);
          acc = __fadd_rn(acc, __fmul_rn(c, c));
        }
      } else {
        if (c0 + lane < D) g_l = gamma[c0 + lane], b_l = beta[c0 + lane];
        // y in place (row = lane), then row-wise coalesced stores
        for (int cc = 0; cc < 32; ++cc) {
          const float gc = __shfl_sync(0xffffffffu, g_l, cc), bc = __shfl_sync(0xffffffffu, b_l, cc);
          const float x = t[lane * 33 + cc];
          t[lane * 33 + cc] = __fadd_rn(__fmul_rn(gc, __fmul_rn(__fsub_rn(x, mean), inv)), bc);
        }
        __syncwarp();
        if (lane < lim) {
          for (int r = 0; r < nr; ++r) {
            const int64_t o = (int64_t)(r0 + r) * D + c0 + lane;
            const float y = t[r * 33 + lane];
            if (j.xln) j.xln[o] = y;
            const float q = round_p(y, prec);
            if (j.xq) j.xq[o] = q;
            if (j.xqp) {
              if (j.pack == 2) reinterpret_cast<uint16_t*>(j.xqp)[o] = enc_bf16(q);
              else reinterpret_cast<uint8_t*>(j.xqp)[o] = enc_e4m3(q);
            }
          }
        }
      }
      __syncwarp();  // the stage is refilled by the next iteration's issue
    }
    cp_async_wait<0>();
    if (pass < 2) {
      acc = __fdiv_rn(acc, (float)D);  // mean /= d  |  var /= d
      if (pass == 0) mean = acc;
      else inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(acc, 1e-5f)));
    }
  }
  if (!vec) {
    if (j.xnorm) {  // scalar path: norms from the written outputs (rare shapes)
      for (int r = 0; r < nr; ++r) {
        float ss = 0.f;
        bool bad = false;
        for (int c = lane; c < D; c += 32) {
          const int64_t o = (int64_t)(r0 + r) * D + c;
          const float q = j.xq ? j.xq[o]
                               : (j.pack == 2 ? dec_bf16(reinterpret_cast<const uint16_t*>(j.xqp)[o])
                                              : dec_e4m3(reinterpret_cast<const uint8_t*>(j.xqp)[o]));
          ss = fmaf(q, q, ss);
          bad = bad || bf16_fma_bad(q);
        }
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        bad = __any_sync(0xffffffffu, bad) && j.pack == 2;
        if (lane == 0) j.xnorm[r0 + r] = bad ? -(sqrtf(ss) * 1.0001f) : sqrtf(ss) * 1.0001f;
      }
    }
    return;
  }
  // pass 3, row-major: the warp walks its rows; lane owns float4 column groups
  // lane, lane + 32, ... Same per-element arithmetic (kernels.cpp:155-160),
  // 16-byte loads / stores, and the row norm of the rounded output for the
  // tensor-core exactness certificate.
  const int D4 = D >> 2;
  for (int r = 0; r < nr; ++r) {
    const float m_r = __shfl_sync(0xffffffffu, mean, r), i_r = __shfl_sync(0xffffffffu, inv, r);
    const float4* xin = reinterpret_cast<const float4*>(j.in + (int64_t)(r0 + r) * j.in_stride);
    const int64_t ob = (int64_t)(r0 + r) * D;
    float ss = 0.f;
    bool bad = false;
    for (int c4 = lane; c4 < D4; c4 += 32) {
      const float4 x = xin[c4];
      const float4 gm = __ldg(reinterpret_cast<const float4*>(gamma) + c4);
      const float4 bt = __ldg(reinterpret_cast<const float4*>(beta) + c4);
      float y[4] = {x.x, x.y, x.z, x.w};
      const float gg[4] = {gm.x, gm.y, gm.z, gm.w}, bb[4] = {bt.x, bt.y, bt.z, bt.w};
      float qv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        y[k] = __fadd_rn(__fmul_rn(gg[k], __fmul_rn(__fsub_rn(y[k], m_r), i_r)), bb[k]);
        qv[k] = round_p(y[k], prec);
        ss = fmaf(qv[k], qv[k], ss);
        bad = bad || bf16_fma_bad(qv[k]);
      }
      if (j.xln) reinterpret_cast<float4*>(j.xln + ob)[c4] = make_float4(y[0], y[1], y[2], y[3]);
      if (j.xq) reinterpret_cast<float4*>(j.xq + ob)[c4] = make_float4(qv[0], qv[1], qv[2], qv[3]);
      if (j.xqp) {
        if (j.pack == 2)
          reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(j.xqp) + ob)[c4] =
              make_uint2(enc_bf16(qv[0]) | ((uint32_t)enc_bf16(qv[1]) << 16),
                         enc_bf16(qv[2]) | ((uint32_t)enc_bf16(qv[3]) << 16));
        else
          reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(j.xqp) + ob)[c4] =
              enc_e4m3(qv[0]) | ((uint32_t)enc_e4m3(qv[1]) << 8) | ((uint32_t)enc_e4m3(qv[2]) << 16) |
              ((uint32_t)enc_e4m3(qv[3]) << 24);
      }
    }
    if (j.xnorm) {
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      bad = __any_sync(0xffffffffu, bad) && j.pack == 2;
      if (lane == 0) j.xnorm[r0 + r] = bad ? -(sqrtf(ss) * 1.0001f) : sqrtf(ss) * 1.0001f;
    }
  }
}

// Latency-optimised variant for launches with few rows (the per-source
// baseline runs: one segment of B*S rows per launch). Each warp owns RW rows
// and stages them whole in shared memory (all loads in flight at once, odd
// row pitch so the RW chain lanes hit distinct banks); lanes 0..RW-1 then run
// the two sequential reductions at FADD latency and the whole warp normalises
// row-major from shared memory (same arithmetic as ln_warp_kernel).
constexpr int kLsWarps = 4;

// The two sequential reductions of one row (kernels.cpp:127-142: mean, then
// the mean of squared deviations, k ascending, no FMA) at FADD latency, from
// a 16-byte aligned row in shared memory; inv = 1 / sqrt(var + eps).
__device__ __forceinline__ void ln_row_stats(const float* row, int D, float& mean, float& inv) {
  // sequential chains at FADD latency: 16-byte shared loads (rows are
  // 16-byte aligned, P % 4 == 0), the next 16 elements loaded ahead of the
  // dependent adds of the current 16
  constexpr int U = 16;
  float acc = 0.f;
  float4 cur[U / 4], nxt[U / 4];
  const int Dm = D & ~(U - 1);
  if (Dm) {
#pragma unroll
    for (int k = 0; k < U / 4; ++k) cur[k] = reinterpret_cast<const float4*>(row)[k];
  }
  for (int c = 0; c < Dm; c += U) {
    const bool more = c + U < Dm;
#pragma unroll
    for (int k = 0; k < U / 4; ++k)
      nxt[k] = more ? reinterpret_cast<const float4*>(row + c + U)[k] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int k = 0; k < U / 4; ++k) {
      acc = __fadd_rn(acc, cur[k].x);
      acc = __fadd_rn(acc, cur[k].y);
      acc = __fadd_rn(acc, cur[k].z);
      acc = __fadd_rn(acc, cur[k].w);
    }
#pragma unroll
    for (int k = 0; k < U / 4; ++k) cur[k] = nxt[k];
  }
  for (int c = Dm; c < D; ++c) acc = __fadd_rn(acc, row[c]);
  mean = __fdiv_rn(acc, (float)D);
  acc = 0.f;
  if (Dm) {
#pragma unroll
    for (int k = 0; k < U / 4; ++k) cur[k] = reinterpret_cast<const float4*>(row)[k];
  }
  for (int c = 0; c < Dm; c += U) {
    const bool more = c + U < Dm;
#pragma unroll
    for (int k = 0; k < U / 4; ++k)
      nxt[k] = more ? reinterpret_cast<const float4*>(row + c + U)[k] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int k = 0; k < U / 4; ++k) {
      const float xs[4] = {cur[k].x, cur[k].y, cur[k].z, cur[k].w};
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const float d = __fsub_rn(xs[h], mean);
        acc = __fadd_rn(acc, __fmul_rn(d, d));
      }
    }
#pragma unroll
    for (int k = 0; k < U / 4; ++k) cur[k] = nxt[k];
  }
  for (int c = Dm; c < D; ++c) {
    const float d = __fsub_rn(row[c], mean);
    acc = __fadd_rn(acc, __fmul_rn(d, d));
  }
  acc = __fdiv_rn(acc, (float)D);
  inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(acc, 1e-5f)));
}

// Paired E4M3 codes (cvt.rn.satfinite.e4m3x2, the reference's NaN code 0x7F:
// enc_e4m3 element by element) and their values (dec_e4m3)
__device__ __forceinline__ uint32_t ln_e4m3x2(float a, float b) {
  uint32_t c = (uint32_t)__nv_cvt_float2_to_fp8x2(make_float2(a, b), __NV_SATFINITE, __NV_E4M3);
  if (a != a) c = (c & 0xFF00u) | 0x7Fu;
  if (b != b) c = (c & 0x00FFu) | 0x7F00u;
  return c;
}
__device__ __forceinline__ float2 ln_e4m3x2_val(uint32_t c) {
  return __half22float2(__half2(__nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)c, __NV_E4M3)));
}

// Normalisation of row r (job-local index grow) from shared memory by the
// whole warp: y = gamma (x - mean) inv + beta, rounded at PREC, the packed
// tensor-core copy (PACK 1: E4M3 codes, 2: BF16 codes, 0: none) and the row
// norm of the rounded output (fused). PREC / PACK are compile-time so the
// per-element work is the affine map, one paired conversion and the stores
// (the E4M3 codes are converted once and serve both the rounded value and
// the packed copy).
template <int PREC, int PACK>
__device__ __forceinline__ void ln_row_out_t(const LnJob& j, const float* row, int64_t grow, float m_r,
                                             float i_r, const float* __restrict__ gamma,
                                             const float* __restrict__ beta, int D, int lane) {
  const int D4 = D >> 2;
  const int64_t ob = grow * D;
  float ss = 0.f;
  bool bad = false;
  // the sign flag of xnorm (a BF16 row that is not FMA-safe) matters only for BF16 jobs
  const bool chk = PACK == 2 || (PACK == 0 && j.pack == 2);
  for (int c4 = lane; c4 < D4; c4 += 32) {
    const float4 gm = __ldg(reinterpret_cast<const float4*>(gamma) + c4);
    const float4 bt = __ldg(reinterpret_cast<const float4*>(beta) + c4);
    const float4 xv = reinterpret_cast<const float4*>(row)[c4];
    const float gg[4] = {gm.x, gm.y, gm.z, gm.w}, bb[4] = {bt.x, bt.y, bt.z, bt.w};
    const float xx[4] = {xv.x, xv.y, xv.z, xv.w};
    float y[4], qv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) y[k] = __fadd_rn(__fmul_rn(gg[k], __fmul_rn(__fsub_rn(xx[k], m_r), i_r)), bb[k]);
    uint32_t code = 0;
    if (PREC == kP8) {
      const uint32_t c01 = ln_e4m3x2(y[0], y[1]), c23 = ln_e4m3x2(y[2], y[3]);
      const float2 v01 = ln_e4m3x2_val(c01), v23 = ln_e4m3x2_val(c23);
      qv[0] = v01.x, qv[1] = v01.y, qv[2] = v23.x, qv[3] = v23.y;
      code = c01 | (c23 << 16);
    } else if (PREC == kP16) {
#pragma unroll
      for (int k = 0; k < 4; ++k) qv[k] = round_bf16(y[k]);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) qv[k] = y[k];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      ss = fmaf(qv[k], qv[k], ss);
      if (chk) bad = bad || bf16_fma_bad(qv[k]);
    }
    if (j.xln) reinterpret_cast<float4*>(j.xln + ob)[c4] = make_float4(y[0], y[1], y[2], y[3]);
    if (j.xq) reinterpret_cast<float4*>(j.xq + ob)[c4] = make_float4(qv[0], qv[1], qv[2], qv[3]);
    if (PACK == 2)
      reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(j.xqp) + ob)[c4] =
          make_uint2(enc_bf16(qv[0]) | ((uint32_t)enc_bf16(qv[1]) << 16),
                     enc_bf16(qv[2]) | ((uint32_t)enc_bf16(qv[3]) << 16));
    else if (PACK == 1)
      reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(j.xqp) + ob)[c4] =
          PREC == kP8 ? code
                      : enc_e4m3(qv[0]) | ((uint32_t)enc_e4m3(qv[1]) << 8) | ((uint32_t)enc_e4m3(qv[2]) << 16) |
                            ((uint32_t)enc_e4m3(qv[3]) << 24);
  }
  if (j.xnorm) {
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) j.xnorm[grow] = bad ? -(sqrtf(ss) * 1.0001f) : sqrtf(ss) * 1.0001f;
  }
}

__device__ __forceinline__ void ln_row_out(const LnJob& j, const float* row, int64_t grow, float m_r,
                                           float i_r, const float* __restrict__ gamma,
                                           const float* __restrict__ beta, int D, int prec, int lane) {
  const int pack = j.xqp ? (j.pack == 2 ? 2 : 1) : 0;
#define LN_OUT(P, K) ln_row_out_t<P, K>(j, row, grow, m_r, i_r, gamma, beta, D, lane)
  if (prec == kP8) {
    if (pack == 1) LN_OUT(kP8, 1); else if (pack == 2) LN_OUT(kP8, 2); else LN_OUT(kP8, 0);
  } else if (prec == kP16) {
    if (pack == 1) LN_OUT(kP16, 1); else if (pack == 2) LN_OUT(kP16, 2); else LN_OUT(kP16, 0);
  } else {
    if (pack == 1) LN_OUT(kP32, 1); else if (pack == 2) LN_OUT(kP32, 2); else LN_OUT(kP32, 0);
  }
#undef LN_OUT
}

template <int RW>
__global__ void __launch_bounds__(32 * kLsWarps) ln_small_kernel(const LnJob* __restrict__ jobs,
                                                                 const float* __restrict__ gamma,
                                                                 const float* __restrict__ beta,
                                                                 int D, int prec) {
  extern __shared__ float ls_sm[];
  const LnJob j = jobs[blockIdx.y];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = (blockIdx.x * kLsWarps + warp) * RW;
  if (r0 >= j.rows) return;
  // row pitch D + 4 floats: rows stay 16-byte aligned (16-byte cp.async in,
  // float4 reads in the normalisation pass) and the RW chain lanes start 4
  // banks apart (distinct banks for D % 32 == 0)
  const int P = D + 4;
  float* t = ls_sm + (size_t)warp * RW * P;
  const int nr = min(RW, j.rows - r0);
  const bool a16 = (j.in_stride & 3) == 0 && (reinterpret_cast<uintptr_t>(j.in) & 15) == 0;
  for (int r = 0; r < nr; ++r) {
    const float* src = j.in + (int64_t)(r0 + r) * j.in_stride;
    if (a16)
      for (int c = 4 * lane; c < D; c += 128) cp_async16(t + r * P + c, src + c);
    else
      for (int c = lane; c < D; c += 32) cp_async4(t + r * P + c, src + c);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
  float mean = 0.f, inv = 0.f;
  if (lane < nr) ln_row_stats(t + lane * P, D, mean, inv);
  for (int r = 0; r < nr; ++r) {
    const float m_r = __shfl_sync(0xffffffffu, mean, r), i_r = __shfl_sync(0xffffffffu, inv, r);
    ln_row_out(j, t + r * P, r0 + r, m_r, i_r, gamma, beta, D, prec, lane);
  }
}

// Big launches (the patched passes: tens of thousands of rows): ln_small's
// 4 chain lanes per warp left it issue-bound (ncu: 72% issue-active, 15% of
// HBM; the chain loops cost ~1350 warp-instructions per row). Here a CTA of
// kLlWarps warps stages ROWS rows, warp 0 runs all their chains with one row
// per lane (conflict-free 16-byte loads: the row pitch D + 4 puts lanes 0..7
// of a quarter-warp on distinct bank quads), and every warp then normalises
// a share of the rows. The chain phase of one CTA overlaps the loads and
// normalisation of the others. ROWS = 24 (74 KB, three CTAs per SM: 228 ms
// per step) by default, 32 (99 KB, two CTAs: 251 ms) with
// CQG_LN_LANE_ROWS=32; ln_small: 267 ms. Same arithmetic as ln_small_kernel
// (ln_row_stats / ln_row_out): bit-identical outputs.
constexpr int kLlWarps = 4, kLlRows = 32;
constexpr size_t smem_cap_ll() { return sizeof(float) * kLlRows * (1024 + 4); }

template <int kLlRows>
__global__ void __launch_bounds__(32 * kLlWarps) ln_lane_kernel(const LnJob* __restrict__ jobs,
                                                                const float* __restrict__ gamma,
                                                                const float* __restrict__ beta, int D,
                                                                int prec) {
  extern __shared__ float ll_sm[];
  __shared__ float s_mean[kLlRows], s_inv[kLlRows];
  const LnJob j = jobs[blockIdx.y];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = blockIdx.x * kLlRows;
  if (r0 >= j.rows) return;
  const int P = D + 4;
  const int nr = min(kLlRows, j.rows - r0);
  const bool a16 = (j.in_stride & 3) == 0 && (reinterpret_cast<uintptr_t>(j.in) & 15) == 0;
  for (int r = warp; r < nr; r += kLlWarps) {
    const float* src = j.in + (int64_t)(r0 + r) * j.in_stride;
    if (a16)
      for (int c = 4 * lane; c < D; c += 128) cp_async16(ll_sm + r * P + c, src + c);
    else
      for (int c = lane; c < D; c += 32) cp_async4(ll_sm + r * P + c, src + c);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  if (warp == 0 && lane < nr) {
    float mean, inv;
    ln_row_stats(ll_sm + lane * P, D, mean, inv);
    s_mean[lane] = mean, s_inv[lane] = inv;
  }
  __syncthreads();
  for (int r = warp; r < nr; r += kLlWarps)
    ln_row_out(j, ll_sm + r * P, r0 + r, s_mean[r], s_inv[r], gamma, beta, D, prec, lane);
}

void launch_layernorm(const LnJob* d_jobs, int n_jobs, int max_rows, const float* gamma,
                      const float* beta, int D, int prec, cudaStream_t st) {
  if (n_jobs <= 0 || max_rows <= 0) return;
  // few rows: latency-bound, stage whole rows (RW rows per warp) in shared memory
  // Whole rows staged in shared memory: every row is read from HBM once (the
  // ring kernel below re-streams each row three times and thrashes L2 on big
  // launches), and the chains run at FADD latency.
  const int64_t total_rows = (int64_t)max_rows * n_jobs;
  // CQG_LN_LANE_MIN: launches with at least this many rows use ln_lane_kernel
  // (0: never; tests set 1 to run it on every launch)
  const char* e = getenv("CQG_LN_LANE_MIN");
  const int64_t ll_min_rows = e ? atoll(e) : 4 * kLlRows * 148;
  if ((D & 3) == 0 && D <= 1024 && ll_min_rows > 0 && total_rows >= ll_min_rows) {
    // rows per CTA: 24 (three CTAs per SM; measured 228 ms per step) or,
    // CQG_LN_LANE_ROWS=32, 32 (two CTAs per SM; 251 ms)
    const char* er = getenv("CQG_LN_LANE_ROWS");
    const int rows = er && atoi(er) == 32 ? 32 : 24;
    const size_t smem = sizeof(float) * rows * (D + 4);
    static bool attr_l = false;
    if (!attr_l) {
      cudaFuncSetAttribute(ln_lane_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cap_ll());
      cudaFuncSetAttribute(ln_lane_kernel<24>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cap_ll());
      attr_l = true;
    }
    for (int y0 = 0; y0 < n_jobs; y0 += 65535) {
      dim3 grid((max_rows + rows - 1) / rows, (unsigned)std::min(65535, n_jobs - y0));
      if (rows == 24) ln_lane_kernel<24><<<grid, 32 * kLlWarps, smem, st>>>(d_jobs + y0, gamma, beta, D, prec);
      else ln_lane_kernel<32><<<grid, 32 * kLlWarps, smem, st>>>(d_jobs + y0, gamma, beta, D, prec);
    }
    return;
  }
  if ((D & 3) == 0 && D <= 2048) {
    // rows per warp: 8 (4 for D > 1024) on big launches; fewer when the
    // launch would not give every SM several warps (the per-source baseline
    // runs: 1024-row launches), so more chains run side by side
    int rw = D <= 1024 ? 4 : 2;  // measured: 4 rows per warp beats 8 and 2 at D = 768
    if (const char* e_rw = getenv("CQG_LN_RW")) rw = atoi(e_rw) >= 8 ? 8 : (atoi(e_rw) >= 4 ? 4 : 2);  // (A/B)
    const int64_t total = (int64_t)max_rows * n_jobs;
    while (rw > 1 && total / rw < 4 * 148) rw >>= 1;
    const size_t smem = sizeof(float) * kLsWarps * rw * (D + 4);
    static bool attr_s = false;
    if (!attr_s) {
      cudaFuncSetAttribute(ln_small_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(ln_small_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(ln_small_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(ln_small_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr_s = true;
    }
    for (int y0 = 0; y0 < n_jobs; y0 += 65535) {
      dim3 grid((max_rows + rw * kLsWarps - 1) / (rw * kLsWarps), (unsigned)std::min(65535, n_jobs - y0));
      if (rw == 8) ln_small_kernel<8><<<grid, 32 * kLsWarps, smem, st>>>(d_jobs + y0, gamma, beta, D, prec);
      else if (rw == 4) ln_small_kernel<4><<<grid, 32 * kLsWarps, smem, st>>>(d_jobs + y0, gamma, beta, D, prec);
      else if (rw == 2) ln_small_kernel<2><<<grid, 32 * kLsWarps, smem, st>>>(d_jobs + y0, gamma, beta, D, prec);
      else ln_small_kernel<1><<<grid, 32 * kLsWarps, smem, st>>>(d_jobs + y0, gamma, beta, D, prec);
    }
    return;
  }
  const size_t smem = sizeof(float) * kLnWarps * kLnStages * kLnTile;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(ln_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  for (int y0 = 0; y0 < n_jobs; y0 += 65535) {
    dim3 grid((max_rows + 32 * kLnWarps - 1) / (32 * kLnWarps), (unsigned)std::min(65535, n_jobs - y0));
    ln_warp_kernel<<<grid, 32 * kLnWarps, smem, st>>>(d_jobs + y0, gamma, beta, D, prec);
  }
}

// ---------------------------------------------------------------------------
// Exact SIMT GEMM: per output element the k-ascending chain
// acc = fl(acc + fl(a*b)) of dot_col (kernels.cpp:44-52). 64x64 tiles,
// 256 threads, 4x4 micro-tiles, one launch for a whole job list.
// ---------------------------------------------------------------------------
// Paired-FP32 helpers (sm_100a FFMA2 / FADD2), see gemm_exact_x2_kernel.
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2_fma(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f2_t f2_add(f2_t a, f2_t b) {
  f2_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t f2_pack(float lo, float hi) {
  return (f2_t)__float_as_uint(lo) | ((f2_t)__float_as_uint(hi) << 32);
}
// (a, a) through mov.b64: ptxas folds it into FFMA2's scalar-broadcast operand
__device__ __forceinline__ f2_t f2_dup(float a) {
  f2_t r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(a));
  return r;
}
__device__ __forceinline__ float f2_lo(f2_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float f2_hi(f2_t v) { return __uint_as_float((uint32_t)(v >> 32)); }

constexpr int kBM = 64, kBN = 64, kBK = 16;

int gemm_exact_tiles(int M, int N) { return ((M + kBM - 1) / kBM) * ((N + kBN - 1) / kBN); }

__global__ void __launch_bounds__(256) gemm_exact_kernel(const GemmJob* __restrict__ jobs,
                                                         const int* __restrict__ tile_start,
                                                         int n_jobs, float negz) {
  // locate the job owning this tile
  int lo = 0, hi = n_jobs - 1;
  const int t = blockIdx.x;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (tile_start[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  const GemmJob jb = jobs[lo];
  const int local = t - tile_start[lo];
  const int tiles_n = (jb.N + kBN - 1) / kBN;
  const int m0 = (local / tiles_n) * kBM, n0 = (local % tiles_n) * kBN;

  __shared__ __align__(16) float As[kBK][kBM];
  __shared__ __align__(16) float Bs[kBK][kBN];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  // paired FP32 chains: acc[i][p] holds columns tx*4 + 2p, + 2p + 1 of row ty*4 + i
  const f2_t z2 = f2_pack(negz, negz);
  f2_t acc[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0ull;

  for (int k0 = 0; k0 < jb.K; k0 += kBK) {
    // A tile: 64 rows x 16 k -> As[k][m]
    for (int idx = tid; idx < kBM * kBK; idx += 256) {
      const int mm = idx / kBK, kk = idx % kBK;
      const int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < jb.M && gk < jb.K) ? jb.A[(int64_t)gm * jb.lda + gk] : 0.f;
    }
    for (int idx = tid; idx < kBK * kBN; idx += 256) {
      const int kk = idx / kBN, nn = idx % kBN;
      const int gk = k0 + kk, gn = n0 + nn;
      Bs[kk][nn] = (gk < jb.K && gn < jb.N) ? jb.B[(int64_t)gk * jb.ldb + gn] : 0.f;
    }
    __syncthreads();
    const int kl = min(kBK, jb.K - k0);
    for (int kk = 0; kk < kl; ++kk) {
      const float4 a4 = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 b4 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float a[4] = {a4.x, a4.y, a4.z, a4.w};
      const f2_t b[2] = {f2_pack(b4.x, b4.y), f2_pack(b4.z, b4.w)};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int pp = 0; pp < 2; ++pp) acc[i][pp] = f2_add(acc[i][pp], f2_fma(f2_dup(a[i]), b[pp], z2));
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= jb.M) continue;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int gn = n0 + tx * 4 + jj;
      if (gn >= jb.N) continue;
      float v = round_p((jj & 1) ? f2_hi(acc[i][jj >> 1]) : f2_lo(acc[i][jj >> 1]), jb.prec);
      if (jb.epi == 1) v = round_p(gelu_ref(v), jb.prec);
      jb.C[(int64_t)gm * jb.ldc + gn] = v;
    }
  }
}

void launch_gemm_exact(const GemmJob* d_jobs, const int* d_tile_start, int n_jobs, int total_tiles,
                       cudaStream_t st) {
  if (n_jobs <= 0 || total_tiles <= 0) return;
  gemm_exact_kernel<<<total_tiles, 256, 0, st>>>(d_jobs, d_tile_start, n_jobs, -0.0f);
}

// Large-tile variant (128 x 128, 8 x 8 per thread, register-prefetched k
// tiles): same per-element k-ascending fl(acc + fl(a*b)) chain, ~2x the FP32
// issue efficiency of the 64 x 64 kernel. Used for big exact GEMMs (the
// FP32 unembed of every patched pass).
constexpr int kXBM = 128, kXBN = 128, kXBK = 8;

int gemm_exact_big_tiles(int M, int N) { return ((M + kXBM - 1) / kXBM) * ((N + kXBN - 1) / kXBN); }

__global__ void __launch_bounds__(256) gemm_exact_big_kernel(const GemmJob* __restrict__ jobs,
                                                             const int* __restrict__ tile_start,
                                                             int n_jobs) {
  int lo = 0, hi = n_jobs - 1;
  const int t = blockIdx.x;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (tile_start[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  const GemmJob jb = jobs[lo];
  const int local = t - tile_start[lo];
  const int tiles_m = (jb.M + kXBM - 1) / kXBM;
  // column-major tile raster: consecutive CTAs share the B (weight) tile
  const int m0 = (local % tiles_m) * kXBM, n0 = (local / tiles_m) * kXBN;
  __shared__ __align__(16) float As[2][kXBK][kXBM];
  __shared__ __align__(16) float Bs[2][kXBK][kXBN];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  // loaders: A tile 128 x 8 (each thread 4 consecutive k of one row),
  // B tile 8 x 128 (each thread 4 consecutive n of one k row)
  const int a_r = tid >> 1, a_k = (tid & 1) * 4;
  const int b_k = tid >> 5, b_n = (tid & 31) * 4;
  float ra[4], rb[4];
  auto load = [&](int k0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int gm = m0 + a_r, gk = k0 + a_k + i;
      ra[i] = (gm < jb.M && gk < jb.K) ? jb.A[(int64_t)gm * jb.lda + gk] : 0.f;
      const int gk2 = k0 + b_k, gn = n0 + b_n + i;
      rb[i] = (gk2 < jb.K && gn < jb.N) ? jb.B[(int64_t)gk2 * jb.ldb + gn] : 0.f;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 4; ++i) As[buf][a_k + i][a_r] = ra[i];
    *reinterpret_cast<float4*>(&Bs[buf][b_k][b_n]) = make_float4(rb[0], rb[1], rb[2], rb[3]);
  };
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  load(0);
  store(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < jb.K; k0 += kXBK) {
    const bool more = k0 + kXBK < jb.K;
    if (more) load(k0 + kXBK);
    const int kl = min(kXBK, jb.K - k0);
    for (int kk = 0; kk < kl; ++kk) {
      // rows ty*4 + {0..3} and 64 + ty*4 + {0..3}; cols tx*4 + {0..3} and 64 + tx*4 + {0..3}
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(a[i], b[j]));
    }
    if (more) {
      store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int gm = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (gm >= jb.M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int gn = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (gn >= jb.N) continue;
      float v = round_p(acc[i][j], jb.prec);
      if (jb.epi == 1) v = round_p(gelu_ref(v), jb.prec);
      jb.C[(int64_t)gm * jb.ldc + gn] = v;
    }
  }
}

// Paired-FP32 variant of the big-tile kernel (sm_100a FFMA2 / FADD2): each
// instruction advances two output chains. The product is formed as
// fma(a, b, z) with z = -0.0 supplied at run time, which is exactly fl(a*b)
// (x + -0 == x for every x, including +0) and which ptxas cannot contract
// with the following add (it would for mul.rn.f32x2 + add.rn.f32x2); the add
// is add.rn.f32x2. Per output element the chain is therefore still
// acc = fl(acc + fl(a*b)) in k order, bit-identical to dot_col
// (kernels.cpp:44-52). A is staged in shared memory as broadcast pairs
// (a, a) so that each 16-byte load feeds two rows.

// One 128 x 128 tile. MAP: logical row m of A and C is physical row
// rowmap[m] (the exact recomputation of a device-built list of rows).
// expm1 in double for the fused KL epilogue, branch-free for |d| < 8:
//   d = k/128 + r (k = rint(128 d), r exact, |r| <= 2^-8),
//   expm1(d) = m + (1 + m) expm1(r),  m = expm1(k/128) from a 2049-entry
//   table (g_em1_tab, built once per device with libdevice expm1, <= 1 ulp),
//   expm1(r) by its degree-6 Taylor polynomial (truncation r^7/7! < 3e-21).
// Absolute error ~2^-52 |expm1(d)|: the KL's absolute error stays ~1e-16,
// an order below the reference's own rounding of lse (2^-49). The warp no
// longer diverges into libdevice expm1 (~80 instructions) whenever one lane's
// |d| exceeds a polynomial range; |d| >= 8, Inf and NaN still go there.
__device__ double g_em1_tab[2049];

__global__ void em1_tab_kernel() {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < 2049) g_em1_tab[i] = expm1((double)(i - 1024) * 0.0078125);
}

__device__ __forceinline__ double expm1_tab(double d) {
  if (!(fabs(d) < 8.0)) return expm1(d);
  const double kd = rint(d * 128.0);
  const double r = fma(kd, -0.0078125, d);  // exact: k/128 and d are within 2^-8
  double p = fma(r, 1.0 / 720.0, 1.0 / 120.0);
  p = fma(p, r, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p * r, r, r);
  const double m = __ldg(&g_em1_tab[(int)kd + 1024]);
  return fma(1.0 + m, p, m);
}

template <bool MAP, bool FUSE = false>
__device__ __forceinline__ void x2_tile(const GemmJob& jb, int m0, int n0, const int* __restrict__ rowmap,
                                        float negz, const KlFuse* kf = nullptr) {
  __shared__ __align__(16) float As[2][kXBK][kXBM];  // used as the FFMA2 scalar-broadcast operand
  __shared__ __align__(16) float Bs[2][kXBK][kXBN];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int a_r = tid >> 1, a_k = (tid & 1) * 4;
  const int b_k = tid >> 5, b_n = (tid & 31) * 4;
  const f2_t z2 = f2_pack(negz, negz);
  float ra[4], rb[4];
  // 16-byte loads where the rows are 16-byte aligned and the 4 values in range
  const bool va4 = (jb.lda & 3) == 0 && (reinterpret_cast<uintptr_t>(jb.A) & 15) == 0;
  const bool vb4 = (jb.ldb & 3) == 0 && (reinterpret_cast<uintptr_t>(jb.B) & 15) == 0;
  const int arow = m0 + a_r;
  const int64_t apos = arow < jb.M ? (int64_t)(MAP ? rowmap[arow] : arow) * jb.lda : 0;
  auto load = [&](int k0) {
    const int gm = arow, gka = k0 + a_k;
    if (va4 && gm < jb.M && gka + 3 < jb.K) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(jb.A + apos + gka));
      ra[0] = x.x, ra[1] = x.y, ra[2] = x.z, ra[3] = x.w;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        ra[i] = (gm < jb.M && gka + i < jb.K) ? jb.A[apos + gka + i] : 0.f;
    }
    const int gk2 = k0 + b_k, gnb = n0 + b_n;
    if (vb4 && gk2 < jb.K && gnb + 3 < jb.N) {
      const float4 y = __ldg(reinterpret_cast<const float4*>(jb.B + (int64_t)gk2 * jb.ldb + gnb));
      rb[0] = y.x, rb[1] = y.y, rb[2] = y.z, rb[3] = y.w;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        rb[i] = (gk2 < jb.K && gnb + i < jb.N) ? jb.B[(int64_t)gk2 * jb.ldb + gnb + i] : 0.f;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 4; ++i) As[buf][a_k + i][a_r] = ra[i];
    *reinterpret_cast<float4*>(&Bs[buf][b_k][b_n]) = make_float4(rb[0], rb[1], rb[2], rb[3]);
  };
  // acc[i][p]: row i (ty*4 + i, then 64 + ty*4 + i - 4), column pair p
  // (tx*4 + {0,1}, tx*4 + {2,3}, 64 + tx*4 + {0,1}, 64 + tx*4 + {2,3})
  f2_t acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int p = 0; p < 4; ++p) acc[i][p] = 0ull;
  load(0);
  store(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < jb.K; k0 += kXBK) {
    const bool more = k0 + kXBK < jb.K;
    if (more) load(k0 + kXBK);
    const int kl = min(kXBK, jb.K - k0);
    auto step = [&](int kk) {
      f2_t a[8], b[4];
      {
        // (a, a): ptxas folds the pair into FFMA2's scalar-broadcast operand
        const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
        const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
        a[0] = f2_dup(a0.x), a[1] = f2_dup(a0.y), a[2] = f2_dup(a0.z), a[3] = f2_dup(a0.w);
        a[4] = f2_dup(a1.x), a[5] = f2_dup(a1.y), a[6] = f2_dup(a1.z), a[7] = f2_dup(a1.w);
        const ulonglong2 b0 = *reinterpret_cast<const ulonglong2*>(&Bs[buf][kk][tx * 4]);
        const ulonglong2 b1 = *reinterpret_cast<const ulonglong2*>(&Bs[buf][kk][64 + tx * 4]);
        b[0] = b0.x, b[1] = b0.y, b[2] = b1.x, b[3] = b1.y;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int p = 0; p < 4; ++p) acc[i][p] = f2_add(acc[i][p], f2_fma(a[i], b[p], z2));
    };
    if (kl == kXBK) {
#pragma unroll
      for (int kk = 0; kk < kXBK; ++kk) step(kk);
    } else {
      for (int kk = 0; kk < kl; ++kk) step(kk);
    }
    if (more) {
      store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
  if (FUSE) {
    // KL partials of this tile's 128 vocabulary columns per row (see
    // gemm_unembed_kl_kernel): T = sum e_v expm1(d_v), S = sum e_v d_v with
    // d_v = x_v - xb_v (exact in double), e_v = exp(lp_v) of the baseline.
    // A NaN logit makes both NaN (the reduce kernel raises the flag).
    // baselines are zero-padded to a multiple of 128 columns (kf->ld): the
    // padded columns have e = 0 and x = 0 (zero B columns), adding nothing
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int gm = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
      double T = 0.0, S = 0.0;
      if (gm < jb.M) {
        const int it = gm % kf->nb;
        const double* xb = kf->xb + (int64_t)it * kf->ld + n0 + tx * 4;  // (in double already)
        const double* eb = kf->eb + (int64_t)it * kf->ld + n0 + tx * 4;
        const double2 x0 = __ldg(reinterpret_cast<const double2*>(xb));
        const double2 x1 = __ldg(reinterpret_cast<const double2*>(xb + 2));
        const double2 x2 = __ldg(reinterpret_cast<const double2*>(xb + 64));
        const double2 x3 = __ldg(reinterpret_cast<const double2*>(xb + 66));
        const double2 e0 = __ldg(reinterpret_cast<const double2*>(eb));
        const double2 e1 = __ldg(reinterpret_cast<const double2*>(eb + 2));
        const double2 e2 = __ldg(reinterpret_cast<const double2*>(eb + 64));
        const double2 e3 = __ldg(reinterpret_cast<const double2*>(eb + 66));
        const double xbv[8] = {x0.x, x0.y, x1.x, x1.y, x2.x, x2.y, x3.x, x3.y};
        const double ebv[8] = {e0.x, e0.y, e1.x, e1.y, e2.x, e2.y, e3.x, e3.y};
        double t2[2] = {0.0, 0.0}, s2[2] = {0.0, 0.0};  // two independent chains
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const f2_t pr = acc[i][j >> 1];
          const float x = round_p((j & 1) ? f2_hi(pr) : f2_lo(pr), jb.prec);
          const double d = (double)x - xbv[j];
          s2[j & 1] = fma(ebv[j], d, s2[j & 1]);
          t2[j & 1] = fma(ebv[j], expm1_tab(d), t2[j & 1]);
        }
        T = t2[0] + t2[1], S = s2[0] + s2[1];
      }
      // the 16 threads of a row are one half-warp (tid = ty * 16 + tx)
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
        T += __shfl_xor_sync(0xffffffffu, T, o);
        S += __shfl_xor_sync(0xffffffffu, S, o);
      }
      if (tx == 0 && gm < jb.M) kf->part[(int64_t)gm * kf->n_ct + n0 / kXBN] = make_double2(T, S);
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int gm = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (gm >= jb.M) continue;
    const int64_t crow = (int64_t)(MAP ? rowmap[gm] : gm) * jb.ldc;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int gn = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (gn >= jb.N) continue;
      const f2_t pr = acc[i][j >> 1];
      float v = round_p((j & 1) ? f2_hi(pr) : f2_lo(pr), jb.prec);
      if (jb.epi == 1) v = round_p(gelu_ref(v), jb.prec);
      jb.C[crow + gn] = v;
    }
  }
}

__global__ void __launch_bounds__(256, 2) gemm_exact_x2_kernel(const GemmJob* __restrict__ jobs,
                                                            const int* __restrict__ tile_start,
                                                            int n_jobs, float negz) {
  int lo = 0, hi = n_jobs - 1;
  const int t = blockIdx.x;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (tile_start[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  const GemmJob jb = jobs[lo];
  const int local = t - tile_start[lo];
  const int tiles_m = (jb.M + kXBM - 1) / kXBM;
  x2_tile<false>(jb, (local % tiles_m) * kXBM, (local / tiles_m) * kXBN, nullptr, negz);
}

// ---- K7 + K8 fused: the patched rows' exact unembed with the KL in its
// epilogue (logits are never stored). The reference's per-row
//   KL = sum_v e_v (lp_v - lq_v),  lp_v = xb_v - lse_b,  lq_v = x_v - lse_q
// (patching.cpp:127-161) equals, with d_v = x_v - xb_v and E = sum_v e_v,
//   KL = E (lse_q - lse_b) - sum_v e_v d_v,
//   lse_q - lse_b = log sum_v e_v exp(d_v) = log1p((E - 1) + sum_v e_v expm1(d_v)),
// an identity of the same real numbers. Each 128 x 128 tile writes its
// per-row (T, S) partials; kl_reduce_kernel sums a row's partials and forms
// the KL. Every term is O(|d|) and the final subtraction is of two O(|d|)
// numbers, so the result is accurate to ~1e-16 |d| absolute, below the
// reference's own rounding of lse_q (one ulp of ~log V, i.e. ~2^-49).
__global__ void __launch_bounds__(256, 2) gemm_unembed_kl_kernel(GemmJob jb, KlFuse kf, float negz) {
  const int tiles_m = (jb.M + kXBM - 1) / kXBM;
  const int t = blockIdx.x;
  x2_tile<false, true>(jb, (t % tiles_m) * kXBM, (t / tiles_m) * kXBN, nullptr, negz, &kf);
}

void launch_gemm_unembed_kl(const GemmJob& jb, const KlFuse& kf, cudaStream_t st) {
  if (jb.M <= 0) return;
  static bool tab_ready[64] = {};  // g_em1_tab is per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !tab_ready[dev]) {
    em1_tab_kernel<<<(2049 + 255) / 256, 256, 0, st>>>();
    cudaStreamSynchronize(st);  // once per device: engines on other streams see the table
    tab_ready[dev] = true;
  }
  const int tiles = ((jb.M + kXBM - 1) / kXBM) * ((jb.N + kXBN - 1) / kXBN);
  gemm_unembed_kl_kernel<<<tiles, 256, 0, st>>>(jb, kf, -0.0f);
}

int unembed_kl_col_tiles(int V) { return (V + kXBN - 1) / kXBN; }

// the fused KL's baselines: logits (as doubles) and exp(lp) per item, zero
// padded to the 128-column pitch ld (16-byte aligned rows)
__global__ void pad_baselines_kernel(const float* __restrict__ logits, const double* __restrict__ prob, int V,
                                     int ld, double* __restrict__ xbd, double* __restrict__ ebd) {
  const int it = blockIdx.y;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ld; c += gridDim.x * blockDim.x) {
    const bool in = c < V;
    xbd[(int64_t)it * ld + c] = in ? (double)logits[(int64_t)it * V + c] : 0.0;
    ebd[(int64_t)it * ld + c] = in ? prob[(int64_t)it * V + c] : 0.0;
  }
}

void launch_pad_baselines(const float* logits, const double* prob, int nb, int V, int ld, double* xbd,
                          double* ebd, cudaStream_t st) {
  if (nb > 0) pad_baselines_kernel<<<dim3((ld + 255) / 256, nb), 256, 0, st>>>(logits, prob, V, ld, xbd, ebd);
}

// ---- HeadBundle prefetch (pahq.cpp:93-165, 211-238), B200 form --------------
// The FP32 masters are resident in HBM; what the next source group's
// baseline needs (the elevated head's W_Q/W_K/W_V column slices and its
// layer's W_O, or the elevated MLP's W_in/W_out) is pulled into L2 on a side
// stream while the current group runs (cp.async.bulk.prefetch.L2: no
// registers, no shared memory, no completion to wait for).
__global__ void prefetch_l2_kernel(const PfJob j) {
  const int n_rows = j.col[0] ? 3 * j.rows : 0;
  const int64_t n_blk0 = (int64_t)((j.blk_bytes[0] + 65535) >> 16), n_blk1 = (int64_t)((j.blk_bytes[1] + 65535) >> 16);
  const int64_t n = n_rows + n_blk0 + n_blk1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const void* p;
    uint32_t bytes;
    if (i < n_rows) {  // one row of a column slice (d_k floats)
      p = j.col[i / j.rows] + (i % j.rows) * (int64_t)j.ld;
      bytes = (uint32_t)j.cols * 4u;
    } else {  // a 64 KB piece of a whole matrix
      const int64_t k = i - n_rows, b = k < n_blk0 ? 0 : 1, o = (b ? k - n_blk0 : k) << 16;
      p = reinterpret_cast<const uint8_t*>(j.blk[b]) + o;
      bytes = (uint32_t)min((uint64_t)65536, j.blk_bytes[b] - (uint64_t)o);
    }
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
  }
}

void launch_prefetch_l2(const PfJob& j, cudaStream_t st) {
  prefetch_l2_kernel<<<16, 256, 0, st>>>(j);
}

// one warp per row: sum the row's tile partials, then the KL (above)
__global__ void kl_reduce_kernel(const double2* __restrict__ part, int rows, int n_ct,
                                 const double* __restrict__ esum, int nb, double* out, int* nan_flag) {
  const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  double T = 0.0, S = 0.0;
  for (int c = lane; c < n_ct; c += 32) {
    const double2 p = part[(int64_t)r * n_ct + c];
    T += p.x, S += p.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T += __shfl_xor_sync(0xffffffffu, T, o);
    S += __shfl_xor_sync(0xffffffffu, S, o);
  }
  if (lane == 0) {
    if (T != T || S != S) {  // NaN logits: the score is rejected by the host (patching.cpp:120-123)
      atomicOr(nan_flag, 1);
      out[r] = 0.0;
      return;
    }
    // every d_v = 0: the patched logits are the baseline's bit for bit, so
    // lse_q == lse_b and the reference's KL is exactly 0 (test_patching.cpp:115-130)
    const double E = esum[r % nb];
    out[r] = (T == 0.0 && S == 0.0) ? 0.0 : E * log1p((E - 1.0) + T) - S;
  }
}

void launch_kl_reduce(const double2* part, int rows, int n_ct, const double* esum, int nb, double* out,
                      int* nan_flag, cudaStream_t st) {
  if (rows > 0) kl_reduce_kernel<<<(rows + 7) / 8, 256, 0, st>>>(part, rows, n_ct, esum, nb, out, nan_flag);
}

// The exact (reference-order) GEMM over a device-built row list (rows[0 ..
// *count)), persistent: the count is known only on the device (the unembed
// certificate's flagged rows), so the grid loops over however many tiles it
// implies (none: every CTA exits at once).
__global__ void __launch_bounds__(256, 2) gemm_exact_rows_kernel(GemmJob jb, const int* __restrict__ rows,
                                                              const int* __restrict__ count, float negz) {
  const int cnt = *count;
  jb.M = cnt;
  const int tiles_m = (cnt + kXBM - 1) / kXBM, tiles_n = (jb.N + kXBN - 1) / kXBN;
  for (int t = blockIdx.x; t < tiles_m * tiles_n; t += gridDim.x) {
    __syncthreads();  // shared tiles of the previous iteration
    x2_tile<true>(jb, (t % tiles_m) * kXBM, (t / tiles_m) * kXBN, rows, negz);
  }
}

void launch_gemm_exact_rows(const GemmJob& jb, const int* rows, const int* count, cudaStream_t st) {
  gemm_exact_rows_kernel<<<2 * 148, 256, 0, st>>>(jb, rows, count, -0.0f);
}

// Short-and-wide variant (64 x 256 tiles, 4 rows x 16 columns per thread) of
// the paired-FP32 kernel for jobs with at most 64 rows: the unembed of one
// evaluation context (B last rows) would leave half of every 128-row tile
// empty. Same per-element chain.
constexpr int kSBM = 64, kSBN = 256, kSBK = 8;

int gemm_exact_wide_tiles(int M, int N) { return ((M + kSBM - 1) / kSBM) * ((N + kSBN - 1) / kSBN); }

__global__ void __launch_bounds__(256, 2) gemm_exact_wide_kernel(const GemmJob* __restrict__ jobs,
                                                                 const int* __restrict__ tile_start,
                                                                 int n_jobs, float negz) {
  int lo = 0, hi = n_jobs - 1;
  const int t = blockIdx.x;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (tile_start[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  const GemmJob jb = jobs[lo];
  const int local = t - tile_start[lo];
  const int tiles_m = (jb.M + kSBM - 1) / kSBM;
  const int m0 = (local % tiles_m) * kSBM, n0 = (local / tiles_m) * kSBN;
  __shared__ __align__(16) float As[2][kSBK][kSBM];  // FFMA2 scalar-broadcast operand
  __shared__ __align__(16) float Bs[2][kSBK][kSBN];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int a_r = tid >> 2, a_k = (tid & 3) * 2;
  const int b_k = tid >> 5, b_n = (tid & 31) * 8;
  const f2_t z2 = f2_pack(negz, negz);
  float ra[2], rb[8];
  auto load = [&](int k0) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int gm = m0 + a_r, gk = k0 + a_k + i;
      ra[i] = (gm < jb.M && gk < jb.K) ? jb.A[(int64_t)gm * jb.lda + gk] : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int gk2 = k0 + b_k, gn = n0 + b_n + i;
      rb[i] = (gk2 < jb.K && gn < jb.N) ? jb.B[(int64_t)gk2 * jb.ldb + gn] : 0.f;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 2; ++i) As[buf][a_k + i][a_r] = ra[i];
    *reinterpret_cast<float4*>(&Bs[buf][b_k][b_n]) = make_float4(rb[0], rb[1], rb[2], rb[3]);
    *reinterpret_cast<float4*>(&Bs[buf][b_k][b_n + 4]) = make_float4(rb[4], rb[5], rb[6], rb[7]);
  };
  // acc[i][p]: row ty*4 + i, column pair p (q*64 + tx*4 + {0,1} / {2,3}, q = p / 2)
  f2_t acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int p = 0; p < 8; ++p) acc[i][p] = 0ull;
  load(0);
  store(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < jb.K; k0 += kSBK) {
    const bool more = k0 + kSBK < jb.K;
    if (more) load(k0 + kSBK);
    const int kl = min(kSBK, jb.K - k0);
    auto step = [&](int kk) {
      f2_t a[4], b[8];
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      a[0] = f2_dup(a0.x), a[1] = f2_dup(a0.y), a[2] = f2_dup(a0.z), a[3] = f2_dup(a0.w);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const ulonglong2 bq = *reinterpret_cast<const ulonglong2*>(&Bs[buf][kk][q * 64 + tx * 4]);
        b[2 * q] = bq.x, b[2 * q + 1] = bq.y;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int p = 0; p < 8; ++p) acc[i][p] = f2_add(acc[i][p], f2_fma(a[i], b[p], z2));
    };
    if (kl == kSBK) {
#pragma unroll
      for (int kk = 0; kk < kSBK; ++kk) step(kk);
    } else {
      for (int kk = 0; kk < kl; ++kk) step(kk);
    }
    if (more) {
      store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= jb.M) continue;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int gn = n0 + (j >> 2) * 64 + tx * 4 + (j & 3);
      if (gn >= jb.N) continue;
      const f2_t pr = acc[i][j >> 1];
      float v = round_p((j & 1) ? f2_hi(pr) : f2_lo(pr), jb.prec);
      if (jb.epi == 1) v = round_p(gelu_ref(v), jb.prec);
      jb.C[(int64_t)gm * jb.ldc + gn] = v;
    }
  }
}

void launch_gemm_exact_wide(const GemmJob* d_jobs, const int* d_tile_start, int n_jobs,
                            int total_tiles, cudaStream_t st) {
  if (n_jobs <= 0 || total_tiles <= 0) return;
  gemm_exact_wide_kernel<<<total_tiles, 256, 0, st>>>(d_jobs, d_tile_start, n_jobs, -0.0f);
}

void launch_gemm_exact_big(const GemmJob* d_jobs, const int* d_tile_start, int n_jobs,
                           int total_tiles, cudaStream_t st) {
  if (n_jobs <= 0 || total_tiles <= 0) return;
  if (g_exact_x2)
    gemm_exact_x2_kernel<<<total_tiles, 256, 0, st>>>(d_jobs, d_tile_start, n_jobs, -0.0f);
  else
    gemm_exact_big_kernel<<<total_tiles, 256, 0, st>>>(d_jobs, d_tile_start, n_jobs);
}

// ---------------------------------------------------------------------------
// K5: causal attention (kernels.cpp:167-219), one warp per (item, head job).
// Exact reference order: score = (sum_t q_t k_t sequentially) * (1/sqrt(dk));
// max; p = expf(s - max); den = sequential sum; p /= den; z_t = sequential
// sum over j of p_j v_jt; z rounded at prec. Query rows q0..S-1 only (q0 =
// S-1 when only the last position is consumed); z rows are compact:
// item * (S - q0) + (i - q0).
template <int NT>  // dk = 32 * NT
__global__ void __launch_bounds__(128) attention_warp_kernel(const AttnJob* __restrict__ jobs,
                                                             int n_inst, int B, int S) {
  constexpr int dk = 32 * NT, ldk = dk + 1;
  extern __shared__ float sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w = blockIdx.x * (blockDim.x >> 5) + warp;
  if (w >= n_inst) return;
  const int lds = S + 1;
  float* q = sm + (size_t)warp * (3 * S * ldk + S * lds);
  float* k = q + S * ldk;
  float* v = k + S * ldk;
  float* pr = v + S * ldk;
  const AttnJob& jb = jobs[w / B];
  const int item = w % B;
  const int q0 = jb.q0;
  const int64_t base = (int64_t)item * S;
  if (jb.q8) {
    // E4M3 codes: 16-byte loads (16 codes), decoded into the FP32 tiles
    constexpr int vpr = dk / 16;  // 16-code vectors per row
    for (int idx = lane; idx < S * vpr; idx += 32) {
      const int r = idx / vpr, c0 = (idx % vpr) * 16;
      const int64_t g = (base + r) * jb.ld + c0;
      const uint4 kw = __ldg(reinterpret_cast<const uint4*>(jb.k8 + g));
      const uint4 vw = __ldg(reinterpret_cast<const uint4*>(jb.v8 + g));
      const uint4 qw = r >= q0 ? __ldg(reinterpret_cast<const uint4*>(jb.q8 + g)) : make_uint4(0, 0, 0, 0);
      const uint32_t kk[4] = {kw.x, kw.y, kw.z, kw.w}, vv[4] = {vw.x, vw.y, vw.z, vw.w},
                     qq[4] = {qw.x, qw.y, qw.z, qw.w};
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const int wi = h >> 1, sh = (h & 1) * 16;
        const float2 kf = __half22float2(__half2(__nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)((kk[wi] >> sh) & 0xFFFFu), __NV_E4M3)));
        const float2 vf = __half22float2(__half2(__nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)((vv[wi] >> sh) & 0xFFFFu), __NV_E4M3)));
        k[r * ldk + c0 + 2 * h] = kf.x, k[r * ldk + c0 + 2 * h + 1] = kf.y;
        v[r * ldk + c0 + 2 * h] = vf.x, v[r * ldk + c0 + 2 * h + 1] = vf.y;
        if (r >= q0) {
          const float2 qf = __half22float2(__half2(__nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)((qq[wi] >> sh) & 0xFFFFu), __NV_E4M3)));
          q[r * ldk + c0 + 2 * h] = qf.x, q[r * ldk + c0 + 2 * h + 1] = qf.y;
        }
      }
    }
    __syncwarp();
  } else {
    // every load in flight at once (cp.async: no register staging, no
    // generic-pointer aliasing between the global loads and the smem stores)
    for (int r = 0; r < S; ++r) {
      const int64_t g = (base + r) * jb.ld;
#pragma unroll
      for (int c = 0; c < NT; ++c) {
        const int t = lane + 32 * c;
        if (r >= q0) cp_async4(q + r * ldk + t, jb.q + g + t);
        cp_async4(k + r * ldk + t, jb.k + g + t);
        cp_async4(v + r * ldk + t, jb.v + g + t);
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
  }
  const float scale = __fdiv_rn(1.0f, __fsqrt_rn((float)dk));
  // scores for the causal pairs (i, j <= i), i >= q0
  const int p0 = q0 * (q0 + 1) / 2, np = S * (S + 1) / 2 - p0;
  // two pairs per lane at a time (independent chains: twice the ILP of the
  // FADD-latency-bound dot products; each chain keeps dot_col's order)
  auto pair_ij = [&](int pp, int& i, int& j) {
    i = (int)((sqrtf(8.f * pp + 1.f) - 1.f) * 0.5f);
    while (i * (i + 1) / 2 > pp) --i;
    while ((i + 1) * (i + 2) / 2 <= pp) ++i;
    j = pp - i * (i + 1) / 2;
  };
  for (int pa = lane; pa < np; pa += 64) {
    const int pb = pa + 32;
    const bool two = pb < np;
    int ia, ja, ib, jb2;
    pair_ij(p0 + pa, ia, ja);
    pair_ij(p0 + (two ? pb : pa), ib, jb2);
    const float* qa = q + ia * ldk;
    const float* ka = k + ja * ldk;
    const float* qb = q + ib * ldk;
    const float* kb = k + jb2 * ldk;
    float acc_a = 0.f, acc_b = 0.f;
#pragma unroll 16
    for (int t = 0; t < dk; ++t) {
      acc_a = __fadd_rn(acc_a, __fmul_rn(qa[t], ka[t]));
      acc_b = __fadd_rn(acc_b, __fmul_rn(qb[t], kb[t]));
    }
    pr[ia * lds + ja] = __fmul_rn(acc_a, scale);
    if (two) pr[ib * lds + jb2] = __fmul_rn(acc_b, scale);
  }
  __syncwarp();
  // softmax per query row (kernels.cpp:167-219 order: max, exp, sequential
  // den, divide). The max and the den chains run one row per lane; the exps
  // and the divisions are independent per (i, j) and run over the causal
  // pairs, all lanes busy (row i's max / den parked in its spare column S).
  for (int i = q0 + lane; i < S; i += 32) {
    const float* p = pr + i * lds;
    float mx = -INFINITY;
    for (int j = 0; j <= i; ++j) mx = (mx < p[j]) ? p[j] : mx;
    pr[i * lds + S] = mx;
  }
  __syncwarp();
  for (int pi = lane; pi < np; pi += 32) {
    const int pp = p0 + pi;
    int i = (int)((sqrtf(8.f * pp + 1.f) - 1.f) * 0.5f);
    while (i * (i + 1) / 2 > pp) --i;
    while ((i + 1) * (i + 2) / 2 <= pp) ++i;
    const int j = pp - i * (i + 1) / 2;
    pr[i * lds + j] = glibc_expf(__fsub_rn(pr[i * lds + j], pr[i * lds + S]));
  }
  __syncwarp();
  for (int i = q0 + lane; i < S; i += 32) {
    const float* p = pr + i * lds;
    float den = 0.f;
    for (int j = 0; j <= i; ++j) den = __fadd_rn(den, p[j]);
    pr[i * lds + S] = den;
  }
  __syncwarp();
  for (int pi = lane; pi < np; pi += 32) {
    const int pp = p0 + pi;
    int i = (int)((sqrtf(8.f * pp + 1.f) - 1.f) * 0.5f);
    while (i * (i + 1) / 2 > pp) --i;
    while ((i + 1) * (i + 2) / 2 <= pp) ++i;
    const int j = pp - i * (i + 1) / 2;
    pr[i * lds + j] = __fdiv_rn(pr[i * lds + j], pr[i * lds + S]);
  }
  __syncwarp();
  // P.V: two query rows per iteration (rows i and i + 1: independent chains
  // and interleaved row-norm reductions); each chain is j ascending
  for (int i0 = q0; i0 < S; i0 += 2) {
    const bool two = i0 + 1 < S;
    const int i1 = two ? i0 + 1 : i0;
    const float* p0r = pr + i0 * lds;
    const float* p1r = pr + i1 * lds;
    float acc0[NT], acc1[NT];
#pragma unroll
    for (int c = 0; c < NT; ++c) acc0[c] = 0.f, acc1[c] = 0.f;
    for (int j = 0; j <= i0; ++j) {
      const float pj0 = p0r[j], pj1 = p1r[j];
#pragma unroll
      for (int c = 0; c < NT; ++c) {
        const float vj = v[j * ldk + lane + 32 * c];
        acc0[c] = __fadd_rn(acc0[c], __fmul_rn(pj0, vj));
        acc1[c] = __fadd_rn(acc1[c], __fmul_rn(pj1, vj));
      }
    }
    if (two) {  // row i1's last term (j = i1)
      const float pj1 = p1r[i1];
#pragma unroll
      for (int c = 0; c < NT; ++c) acc1[c] = __fadd_rn(acc1[c], __fmul_rn(pj1, v[i1 * ldk + lane + 32 * c]));
    }
    float ss0 = 0.f, ss1 = 0.f;
    const int64_t zr0 = (int64_t)item * (S - q0) + (i0 - q0), zr1 = zr0 + 1;
#pragma unroll
    for (int c = 0; c < NT; ++c) {
      const float z0 = round_p(acc0[c], jb.prec), z1 = round_p(acc1[c], jb.prec);
      if (jb.z) {
        jb.z[zr0 * jb.ldz + lane + 32 * c] = z0;
        if (two) jb.z[zr1 * jb.ldz + lane + 32 * c] = z1;
      }
      if (jb.z8) {
        jb.z8[zr0 * jb.ldz + lane + 32 * c] = enc_e4m3(z0);
        if (two) jb.z8[zr1 * jb.ldz + lane + 32 * c] = enc_e4m3(z1);
      }
      ss0 = fmaf(z0, z0, ss0);
      ss1 = fmaf(z1, z1, ss1);
    }
    if (jb.znorm) {  // the row norm rownorm_kernel would compute (E4M3: no FMA-safety bit)
      for (int o = 16; o > 0; o >>= 1) {
        ss0 += __shfl_xor_sync(0xffffffffu, ss0, o);
        ss1 += __shfl_xor_sync(0xffffffffu, ss1, o);
      }
      if (lane == 0) {
        jb.znorm[zr0] = sqrtf(ss0) * 1.0001f;
        if (two) jb.znorm[zr1] = sqrtf(ss1) * 1.0001f;
      }
    }
  }
}

// generic dk: one CTA per (item, head job), one thread per query row
__global__ void attention_kernel(const AttnJob* __restrict__ jobs, int S, int dk) {
  extern __shared__ float sm[];
  const AttnJob jb = jobs[blockIdx.y];
  const int item = blockIdx.x;
  const int ldk = dk + 1, lds = S + 1;
  float* q = sm;
  float* k = q + S * ldk;
  float* v = k + S * ldk;
  float* pr = v + S * ldk;
  const int64_t base = (int64_t)item * S;
  for (int idx = threadIdx.x; idx < S * dk; idx += blockDim.x) {
    const int r = idx / dk, c = idx % dk;
    const int64_t g = (base + r) * jb.ld + c;
    q[r * ldk + c] = jb.q[g];
    k[r * ldk + c] = jb.k[g];
    v[r * ldk + c] = jb.v[g];
  }
  __syncthreads();
  const float scale = __fdiv_rn(1.0f, __fsqrt_rn((float)dk));
  for (int i = jb.q0 + threadIdx.x; i < S; i += blockDim.x) {
    float* p = pr + i * lds;
    float mx = -INFINITY;
    for (int jj = 0; jj <= i; ++jj) {
      float acc = 0.f;
      for (int t = 0; t < dk; ++t) acc = __fadd_rn(acc, __fmul_rn(q[i * ldk + t], k[jj * ldk + t]));
      p[jj] = __fmul_rn(acc, scale);
      mx = (mx < p[jj]) ? p[jj] : mx;
    }
    float den = 0.f;
    for (int jj = 0; jj <= i; ++jj) {
      p[jj] = glibc_expf(__fsub_rn(p[jj], mx));
      den = __fadd_rn(den, p[jj]);
    }
    for (int jj = 0; jj <= i; ++jj) p[jj] = __fdiv_rn(p[jj], den);
    const int64_t zr = (int64_t)item * (S - jb.q0) + (i - jb.q0);
    float ss = 0.f;
    for (int t = 0; t < dk; ++t) {
      float acc = 0.f;
      for (int jj = 0; jj <= i; ++jj) acc = __fadd_rn(acc, __fmul_rn(p[jj], v[jj * ldk + t]));
      const float zr_v = round_p(acc, jb.prec);
      if (jb.z) jb.z[zr * jb.ldz + t] = zr_v;
      if (jb.z8) jb.z8[zr * jb.ldz + t] = enc_e4m3(zr_v);
      ss = fmaf(zr_v, zr_v, ss);
    }
    if (jb.znorm) jb.znorm[zr] = sqrtf(ss) * 1.0001f;
  }
}

void launch_attention(const AttnJob* d_jobs, int n_jobs, int B, int S, int dk, cudaStream_t st) {
  if (n_jobs <= 0) return;
  const size_t per_warp = sizeof(float) * (size_t)(3 * S * (dk + 1) + S * (S + 1));
  if (dk % 32 == 0 && dk <= 128 && per_warp <= 200 * 1024) {
    const int wpc = (int)std::max<size_t>(1, std::min<size_t>(4, (200 * 1024) / per_warp));
    const int64_t n_inst = (int64_t)n_jobs * B;
    const unsigned grid = (unsigned)((n_inst + wpc - 1) / wpc);
    const size_t smem = per_warp * wpc;
    auto go = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      kern<<<grid, 32 * wpc, smem, st>>>(d_jobs, (int)n_inst, B, S);
    };
    if (dk == 32) go(attention_warp_kernel<1>);
    else if (dk == 64) go(attention_warp_kernel<2>);
    else go(attention_warp_kernel<4>);
    return;
  }
  const size_t smem = per_warp;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  int threads = ((S + 31) / 32) * 32;
  if (threads > 1024) threads = 1024;
  for (int y0 = 0; y0 < n_jobs; y0 += 65535) {
    dim3 grid(B, (unsigned)std::min(65535, n_jobs - y0));
    attention_kernel<<<grid, threads, smem, st>>>(d_jobs + y0, S, dk);
  }
}

// ---------------------------------------------------------------------------
// embed (model.cpp:608-620)
// ---------------------------------------------------------------------------
__global__ void embed_kernel(const int* __restrict__ tok, const float* __restrict__ we,
                             const float* __restrict__ wpos, float* __restrict__ out, int B, int S,
                             int D, int prec) {
  const int64_t n = (int64_t)B * S * D;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(i % D);
    const int64_t row = i / D;
    const int pos = (int)(row % S);
    const int t = tok[row];
    out[i] = round_p(__fadd_rn(we[(int64_t)t * D + j], wpos[(int64_t)pos * D + j]), prec);
  }
}

void launch_embed(const int* tokens, const float* we, const float* wpos, float* out, int B, int S,
                  int D, int prec, cudaStream_t st) {
  const int64_t n = (int64_t)B * S * D;
  int grid = (int)std::min<int64_t>((n + 255) / 256, 8192);
  embed_kernel<<<grid, 256, 0, st>>>(tokens, we, wpos, out, B, S, D, prec);
}

// ---------------------------------------------------------------------------
// K8: KL / logit diff in FP64 (patching.cpp:108-161).
// ---------------------------------------------------------------------------
// Block-wide reduction; `ident` is the identity of op (0 for sums).
template <typename T, typename Op>
__device__ T block_reduce(T v, Op op, T* sh, T ident) {
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  v = (threadIdx.x < nw) ? sh[threadIdx.x] : ident;
  if (w == 0)
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (threadIdx.x == 0) sh[0] = v;
  __syncthreads();
  return sh[0];
}

struct MaxOp {
  __device__ double operator()(double a, double b) const { return a > b ? a : b; }
};
struct SumOp {
  __device__ double operator()(double a, double b) const { return a + b; }
};
struct OrOp {
  __device__ int operator()(int a, int b) const { return a | b; }
};

__device__ double row_lse(const float* x, int V, int* nan_flag, double* sh, int* shi) {
  double mx = -INFINITY;
  int nan = 0;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const float f = x[i];
    if (f != f) nan = 1;
    mx = fmax(mx, (double)f);
  }
  nan = block_reduce(nan, OrOp(), shi, 0);
  if (nan && threadIdx.x == 0) atomicOr(nan_flag, 1);
  mx = block_reduce(mx, MaxOp(), sh, (double)-INFINITY);
  double s = 0.0;
  for (int i = threadIdx.x; i < V; i += blockDim.x) s += exp((double)x[i] - mx);
  s = block_reduce(s, SumOp(), sh, 0.0);
  return mx + log(s);
}

__global__ void lse_kernel(const float* __restrict__ base, int V, double* lse, int* nan_flag,
                           double* p_out, double* p_sum) {
  __shared__ double sh[32];
  __shared__ int shi[32];
  const float* x = base + (int64_t)blockIdx.x * V;
  const double l = row_lse(x, V, nan_flag, sh, shi);
  if (threadIdx.x == 0) lse[blockIdx.x] = l;
  if (p_out) {  // the baseline distribution exp(lp), reused by every patched row
    double e = 0.0;
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
      const double p = exp((double)x[i] - l);
      p_out[(int64_t)blockIdx.x * V + i] = p;
      e += p;
    }
    e = block_reduce(e, SumOp(), sh, 0.0);
    if (p_sum && threadIdx.x == 0) p_sum[blockIdx.x] = e;  // E = sum_v exp(lp_v) (fused KL)
  }
}

void launch_lse(const float* base, int rows, int V, double* lse, int* nan_flag, cudaStream_t st,
                double* p_out, double* p_sum) {
  if (rows > 0) lse_kernel<<<rows, 256, 0, st>>>(base, V, lse, nan_flag, p_out, p_sum);
}

__global__ void kl_kernel(const float* __restrict__ logits, const float* __restrict__ base,
                          const double* __restrict__ base_lse, const int* __restrict__ item_of,
                          int V, double* out, int* nan_flag) {
  __shared__ double sh[32];
  __shared__ int shi[32];
  const int r = blockIdx.x;
  const float* q = logits + (int64_t)r * V;
  const int it = item_of[r];
  const float* c = base + (int64_t)it * V;
  const double lse_c = base_lse[it];
  const double lse_q = row_lse(q, V, nan_flag, sh, shi);
  double kl = 0.0;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const double lp = (double)c[i] - lse_c;
    const double lq = (double)q[i] - lse_q;
    kl += exp(lp) * (lp - lq);
  }
  kl = block_reduce(kl, SumOp(), sh, 0.0);
  if (threadIdx.x == 0) out[r] = kl;
}

// One 512-thread CTA per patched row, two passes over the row (the second
// from L2): an online max / sum-of-exp pass (one exp per element, NaN check),
// then the KL pass. Same per-element arithmetic as the reference
// (patching.cpp:108-135); only the double reduction order differs.
// exp(y) for y <= 0 in double, table-driven: y = (64 k + j) ln2/64 + r with
// |r| <= ln2/128, exp(y) = 2^k * 2^(j/64) * p(r), p the degree-5 Taylor
// polynomial (truncation 3.5e-17 relative); ln2/64 split hi (32 bits) + lo so
// n * hi is exact. ~2-3e-16 relative error, about half the instructions of
// the libdevice exp. The table lives in shared memory (per-lane indices).
__constant__ double kExp2Tab[64] = {
    1.0, 1.0108892860517005, 1.0218971486541166, 1.0330248790212284,
    1.0442737824274138, 1.0556451783605572, 1.0671404006768237, 1.0787607977571199,
    1.0905077326652577, 1.102382583307841, 1.1143867425958924, 1.1265216186082418,
    1.1387886347566916, 1.1511892299529827, 1.1637248587775775, 1.1763969916502812,
    1.189207115002721, 1.202156731452703, 1.215247359980469, 1.22848053610687,
    1.241857812073484, 1.255380757024691, 1.2690509571917332, 1.2828700160787783,
    1.2968395546510096, 1.3109612115247644, 1.3252366431597413, 1.339667524053303,
    1.3542555469368927, 1.3690024229745905, 1.383909881963832, 1.3989796725383112,
    1.4142135623730951, 1.42961333839197, 1.4451808069770467, 1.460917794180647,
    1.4768261459394993, 1.4929077282912648, 1.5091644275934228, 1.5255981507445384,
    1.5422108254079407, 1.559004400237837, 1.5759808451078865, 1.593142151342267,
    1.6104903319492543, 1.6280274218573478, 1.645755478153965, 1.6636765803267364,
    1.681792830507429, 1.7001063537185235, 1.718619298122478, 1.7373338352737062,
    1.7562521603732995, 1.7753764925265212, 1.7947090750031072, 1.8142521755003989,
    1.8340080864093424, 1.8539791250833855, 1.8741676341103, 1.8945759815869656,
    1.9152065613971474, 1.9360617934922943, 1.9571441241754002, 1.978456026387951};

__device__ __forceinline__ double exp_nonpos(double y, const double* tab) {
  if (y < -744.0) return 0.0;
  const double n = rint(y * 92.33248261689366);
  const int ni = (int)n;
  double r = fma(n, -0.01083042469326756, y);
  r = fma(n, -2.9815858269852933e-12, r);
  double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const int kk = ni >> 6;  // floor division (arithmetic shift), kk in [-1074, 0]
  const double t = tab[ni & 63] * p;
  // 2^kk in two factors so that kk down to -1074 never leaves the exponent range
  const int k1 = kk / 2, k2 = kk - k1;
  return t * __longlong_as_double((long long)(k1 + 1023) << 52) *
         __longlong_as_double((long long)(k2 + 1023) << 52);
}

constexpr int kKlThreads = 512;

__device__ __forceinline__ void lse_merge(double& m, double& s, double m2, double s2) {
  if (m2 > m) {
    s = s * exp(m - m2) + s2;
    m = m2;
  } else if (m2 > -INFINITY) {
    s += s2 * exp(m2 - m);
  }
}

// Certificate of the tensor-core unembed (KlCert): the patched logits x~ of
// the row came from the 6-term BF16-split tcgen05 GEMM, not the reference's
// sequential FP32 dot products. Per column j the deviation d_j = x~_j - x_j
// (tensor-core truncation bias + the reference's own rounding) is modelled
// with the partial-sum scale m_j^2 = x_j^2 / 3 + ||a||^2 ||w_j||^2 / (6K)
// (a random walk ending at x_j):
//   |d_j| <~ c u m_j,  c = K/32 + 2 sqrt(K/12)
// and its coherent part (the truncation shrinks every logit, ~ -u (K/64) x_j)
// is bounded by eps_b = u K / 16 per unit of logit. The KL changes to first
// order by sum_j (q_j - p_j) d_j, to second order by <= sum_j q_j d_j^2:
//   E = eps_b |sum_j (q_j - p_j) x_j| + kappa c u sqrt(sum_j (q_j - p_j)^2 m_j^2)
//       + (c u)^2 sum_j q_j m_j^2,  kappa = 8
// A row whose E exceeds tol * KL (or whose KL is not positive and finite) is
// listed for the exact recomputation (gemm_exact_rows + kl over the list).
struct KlCert {
  const float* anorm;  // [rows] ||a|| of the unembed input row (after LN)
  const float* wnorm;  // [V] ||w_j|| of the unembed image columns
  float K;             // D
  double tol;
  int* list;           // flagged rows
  int* count;          // [0] rows listed by this launch, [1] running total (stats)
};

template <bool CERT>
__device__ __forceinline__ void kl_online_row(int r, const float* __restrict__ logits,
                                              const float* __restrict__ base,
                                              const double* __restrict__ base_lse,
                                              const int* __restrict__ item_of, int V, double* out,
                                              int* nan_flag, const double* __restrict__ base_p,
                                              const KlCert& C, double* shm, double* shs, double* sh,
                                              int* shi, const double* tab) {
  const float* q = logits + (int64_t)r * V;
  const int it = item_of[r];
  const float* c = base + (int64_t)it * V;
  int nan = 0;
  double m = -INFINITY, s = 0.0;
  for (int i = threadIdx.x; i < V; i += kKlThreads) {
    const float f = q[i];
    if (f != f) {
      nan = 1;
      continue;
    }
    const double x = (double)f;
    if (x > m) {
      s = s * exp_nonpos(m - x, tab) + 1.0;
      m = x;
    } else {
      s += exp_nonpos(x - m, tab);
    }
  }
  nan = block_reduce(nan, OrOp(), shi, 0);
  if (nan) {  // NaN logits: the score is rejected by the host (patching.cpp:120-123)
    if (threadIdx.x == 0) {
      atomicOr(nan_flag, 1);
      out[r] = 0.0;
      if (CERT) {  // (the exact path decides)
        C.list[atomicAdd(C.count, 1)] = r;
        atomicAdd(C.count + 1, 1);
      }
    }
    return;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    lse_merge(m, s, m2, s2);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) shm[w] = m, shs[w] = s;
  __syncthreads();
  m = shm[0], s = shs[0];
  for (int k = 1; k < kKlThreads / 32; ++k) lse_merge(m, s, shm[k], shs[k]);
  const double lse_q = m + log(s), lse_c = base_lse[it];
  double kl = 0.0, g = 0.0;
  float s2 = 0.f, q2 = 0.f;
  const double* pc = base_p ? base_p + (int64_t)it * V : nullptr;
  const float a2k = CERT ? C.anorm[r] * C.anorm[r] / (6.f * C.K) : 0.f;
  for (int i = threadIdx.x; i < V; i += kKlThreads) {
    const double lp = (double)__ldg(c + i) - lse_c;
    const float xf = q[i];
    const double lq = (double)xf - lse_q;
    const double pp = pc ? __ldg(pc + i) : exp(lp);
    kl += pp * (lp - lq);
    if (CERT) {
      const float qf = __expf((float)lq);
      const float dqp = qf - (float)pp;
      const float wn = __ldg(C.wnorm + i);
      const float m2 = xf * xf * (1.f / 3.f) + a2k * wn * wn;
      g += (double)dqp * (double)xf;
      s2 = fmaf(dqp * dqp, m2, s2);
      q2 = fmaf(qf, m2, q2);
    }
  }
  kl = block_reduce(kl, SumOp(), sh, 0.0);
  if (CERT) {
    g = block_reduce(g, SumOp(), sh, 0.0);
    const double S2 = block_reduce((double)s2, SumOp(), sh, 0.0);
    const double Q2 = block_reduce((double)q2, SumOp(), sh, 0.0);
    if (threadIdx.x == 0) {
      const double u = 5.9604644775390625e-08, K = C.K;
      const double cu = (K / 32.0 + 2.0 * sqrt(K / 12.0)) * u;
      const double E = u * K / 16.0 * fabs(g) + 8.0 * cu * sqrt(S2) + cu * cu * Q2;
      if (!(E <= C.tol * kl)) {
        C.list[atomicAdd(C.count, 1)] = r;
        atomicAdd(C.count + 1, 1);
      }
    }
  }
  if (threadIdx.x == 0) out[r] = kl;
}

__global__ void __launch_bounds__(kKlThreads) kl_online_kernel(const float* __restrict__ logits,
                                                               const float* __restrict__ base,
                                                               const double* __restrict__ base_lse,
                                                               const int* __restrict__ item_of, int V,
                                                               double* out, int* nan_flag,
                                                               const double* __restrict__ base_p,
                                                               KlCert cert, int certify) {
  __shared__ double shm[kKlThreads / 32], shs[kKlThreads / 32];
  __shared__ double sh[32];
  __shared__ int shi[32];
  __shared__ double tab[64];
  if (threadIdx.x < 64) tab[threadIdx.x] = kExp2Tab[threadIdx.x];
  __syncthreads();
  if (certify)
    kl_online_row<true>(blockIdx.x, logits, base, base_lse, item_of, V, out, nan_flag, base_p, cert,
                        shm, shs, sh, shi, tab);
  else
    kl_online_row<false>(blockIdx.x, logits, base, base_lse, item_of, V, out, nan_flag, base_p, cert,
                         shm, shs, sh, shi, tab);
}

// KL of a device-built row list (the certificate's flagged rows after their
// exact recomputation), persistent over the device-side count.
__global__ void __launch_bounds__(kKlThreads) kl_rows_kernel(const float* __restrict__ logits,
                                                             const float* __restrict__ base,
                                                             const double* __restrict__ base_lse,
                                                             const int* __restrict__ item_of, int V,
                                                             double* out, int* nan_flag,
                                                             const double* __restrict__ base_p,
                                                             const int* __restrict__ rows,
                                                             const int* __restrict__ count) {
  __shared__ double shm[kKlThreads / 32], shs[kKlThreads / 32];
  __shared__ double sh[32];
  __shared__ int shi[32];
  __shared__ double tab[64];
  if (threadIdx.x < 64) tab[threadIdx.x] = kExp2Tab[threadIdx.x];
  __syncthreads();
  const int cnt = *count;
  const KlCert none{};
  for (int i = blockIdx.x; i < cnt; i += gridDim.x)
    kl_online_row<false>(rows[i], logits, base, base_lse, item_of, V, out, nan_flag, base_p, none,
                         shm, shs, sh, shi, tab);
}

void launch_kl_rows(const float* logits, const float* base, const double* base_lse, const int* item_of,
                    int V, double* out, int* nan_flag, const double* base_p, const int* rows,
                    const int* count, cudaStream_t st) {
  kl_rows_kernel<<<2 * 148, kKlThreads, 0, st>>>(logits, base, base_lse, item_of, V, out, nan_flag,
                                                 base_p, rows, count);
}

void launch_kl_cert(const float* logits, const float* base, const double* base_lse, const int* item_of,
                    int rows, int V, double* out, int* nan_flag, const double* base_p, const float* anorm,
                    const float* wnorm, int K, double tol, int* list, int* count, cudaStream_t st) {
  if (rows <= 0) return;
  KlCert c{anorm, wnorm, (float)K, tol, list, count};
  kl_online_kernel<<<rows, kKlThreads, 0, st>>>(logits, base, base_lse, item_of, V, out, nan_flag, base_p,
                                                c, 1);
}

void launch_kl(const float* logits, const float* base, const double* base_lse, const int* item_of,
               int rows, int V, double* out, int* nan_flag, cudaStream_t st, const double* base_p) {
  if (rows <= 0) return;
  kl_online_kernel<<<rows, kKlThreads, 0, st>>>(logits, base, base_lse, item_of, V, out, nan_flag,
                                                base_p, KlCert{}, 0);
}

__global__ void logitdiff_kernel(const float* __restrict__ logits, const float* __restrict__ base,
                                 const int* __restrict__ item_of, const int* __restrict__ ans,
                                 const int* __restrict__ dis, int V, double* out, int* nan_flag) {
  __shared__ int shi[32];
  const int r = blockIdx.x;
  const float* q = logits + (int64_t)r * V;
  const int it = item_of[r];
  const float* c = base + (int64_t)it * V;
  int nan = 0;
  for (int i = threadIdx.x; i < V; i += blockDim.x)
    if (q[i] != q[i] || c[i] != c[i]) nan = 1;
  nan = block_reduce(nan, OrOp(), shi, 0);
  if (threadIdx.x == 0) {
    if (nan) atomicOr(nan_flag, 1);
    const int a = ans[it], d = dis[it];
    const double ldp = (double)q[a] - (double)q[d];
    const double ldc = (double)c[a] - (double)c[d];
    out[r] = fabs(ldp - ldc);
  }
}

void launch_logitdiff(const float* logits, const float* base, const int* item_of,
                      const int* answer, const int* distractor, int rows, int V, double* out,
                      int* nan_flag, cudaStream_t st) {
  if (rows > 0)
    logitdiff_kernel<<<rows, 256, 0, st>>>(logits, base, item_of, answer, distractor, V, out,
                                           nan_flag);
}

// ---------------------------------------------------------------------------
// act_diff RMS (patching.cpp:249-256)
// ---------------------------------------------------------------------------
__global__ void rms_kernel(const RmsJob* __restrict__ jobs) {
  __shared__ double sh[32];
  const RmsJob j = jobs[blockIdx.x];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < j.n; i += blockDim.x) {
    const double d = (double)load_out(j.a, j.atype, i) - (double)load_out(j.b, j.btype, i);
    acc += d * d;
  }
  acc = block_reduce(acc, SumOp(), sh, 0.0);
  if (threadIdx.x == 0) *j.out = sqrt(acc / (double)j.n);
}

void launch_rms(const RmsJob* d_jobs, int n_jobs, cudaStream_t st) {
  if (n_jobs > 0) rms_kernel<<<n_jobs, 256, 0, st>>>(d_jobs);
}

// ---------------------------------------------------------------------------
// K1: weight images.
// ---------------------------------------------------------------------------
__global__ void quantize_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t n,
                                int prec) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = round_p(in[i], prec);
}

void launch_quantize(const float* in, float* out, int64_t n, int prec, cudaStream_t st) {
  int grid = (int)std::min<int64_t>((n + 255) / 256, 16384);
  quantize_kernel<<<grid, 256, 0, st>>>(in, out, n, prec);
}

__global__ void pack_e4m3_kernel(const float* __restrict__ in, uint8_t* __restrict__ out,
                                 int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = enc_e4m3(in[i]);
}

void launch_pack_e4m3(const float* in, uint8_t* out, int64_t n, cudaStream_t st) {
  int grid = (int)std::min<int64_t>((n + 255) / 256, 16384);
  pack_e4m3_kernel<<<grid, 256, 0, st>>>(in, out, n);
}

__global__ void pack_bf16_kernel(const float* __restrict__ in, uint16_t* __restrict__ out,
                                 int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = enc_bf16(in[i]);
}

void launch_pack_bf16(const float* in, uint16_t* out, int64_t n, cudaStream_t st) {
  int grid = (int)std::min<int64_t>((n + 255) / 256, 16384);
  pack_bf16_kernel<<<grid, 256, 0, st>>>(in, out, n);
}

__global__ void rtn_groups_kernel(const float* __restrict__ in, float* __restrict__ out,
                                  int64_t group_off, int rows, int cols, int ld, int bits, int qmax) {
  __shared__ double sh[32];
  const int64_t g0 = (int64_t)blockIdx.x * group_off;
  const int64_t n = (int64_t)rows * cols;
  double mx = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t off = g0 + (i / cols) * ld + (i % cols);
    const double a = fabs((double)in[off]);
    mx = (a > mx) ? a : mx;
  }
  mx = block_reduce(mx, MaxOp(), sh, (double)-INFINITY);
  const double delta = (mx == 0.0) ? 0.0 : __ddiv_rn(mx, ldexp(1.0, bits - 1));
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t off = g0 + (i / cols) * ld + (i % cols);
    out[off] = rtn_apply(in[off], delta, qmax);
  }
}

void launch_rtn_groups(const float* in, float* out, int n_groups, int64_t group_off, int rows,
                       int cols, int ld, int bits, cudaStream_t st, int qmax) {
  for (int g0 = 0; g0 < n_groups; g0 += 65535)
    rtn_groups_kernel<<<std::min(65535, n_groups - g0), 256, 0, st>>>(
        in + (int64_t)g0 * group_off, out + (int64_t)g0 * group_off, group_off, rows, cols, ld, bits, qmax);
}

__global__ void rtn_act_kernel(const RtnJob* __restrict__ jobs, int bits, int qmax) {
  __shared__ double sh[32];
  const RtnJob jb = jobs[blockIdx.y];
  float* base = jb.p + (int64_t)blockIdx.x * jb.group_off;
  const int64_t n = (int64_t)jb.rows * jb.cols;
  double mx = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t off = (i / jb.cols) * jb.ld + (i % jb.cols);
    float x = base[off];
    if (jb.gelu) base[off] = x = gelu_ref(x);
    const double a = fabs((double)x);
    mx = (a > mx) ? a : mx;
  }
  mx = block_reduce(mx, MaxOp(), sh, (double)-INFINITY);
  const double delta = (mx == 0.0) ? 0.0 : __ddiv_rn(mx, ldexp(1.0, bits - 1));
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t off = (i / jb.cols) * jb.ld + (i % jb.cols);
    base[off] = rtn_apply(base[off], delta, qmax);
  }
}

// Per-row groups (the INT8 extension's per-token scales): one warp per row
// group (rows = 1), max in double over the warp, then the RTN of the row.
__global__ void rtn_rows_kernel(const RtnJob* __restrict__ jobs, int n_groups, int bits, int qmax) {
  const RtnJob jb = jobs[blockIdx.y];
  const int gi = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (gi >= n_groups) return;
  float* base = jb.p + (int64_t)gi * jb.group_off;
  double mx = 0.0;
  for (int i = lane; i < jb.cols; i += 32) {
    float x = base[i];
    if (jb.gelu) base[i] = x = gelu_ref(x);
    const double a = fabs((double)x);
    mx = (a > mx) ? a : mx;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double y = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = (y > mx) ? y : mx;
  }
  __syncwarp();
  const double delta = (mx == 0.0) ? 0.0 : __ddiv_rn(mx, ldexp(1.0, bits - 1));
  for (int i = lane; i < jb.cols; i += 32) base[i] = rtn_apply(base[i], delta, qmax);
}

void launch_rtn_rows(const RtnJob* d_jobs, int n_jobs, int n_groups, int bits, cudaStream_t st, int qmax) {
  for (int y0 = 0; y0 < n_jobs; y0 += 65535)
    if (n_groups > 0)
      rtn_rows_kernel<<<dim3((n_groups + 7) / 8, std::min(65535, n_jobs - y0)), 256, 0, st>>>(d_jobs + y0, n_groups,
                                                                                              bits, qmax);
}

void launch_rtn_act(const RtnJob* d_jobs, int n_jobs, int n_groups, int bits, cudaStream_t st, int qmax) {
  for (int y0 = 0; y0 < n_jobs; y0 += 65535)
    if (n_groups > 0)
      rtn_act_kernel<<<dim3(n_groups, std::min(65535, n_jobs - y0)), 256, 0, st>>>(d_jobs + y0, bits, qmax);
}

// ---------------------------------------------------------------------------
// exhaustive scalar checks (tests)
// ---------------------------------------------------------------------------
__global__ void e4m3_all_kernel(uint8_t* out, uint32_t lo, uint64_t count) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = enc_e4m3(__uint_as_float(lo + (uint32_t)i));
}
__global__ void bf16_all_kernel(uint16_t* out, uint32_t lo, uint64_t count) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = enc_bf16(__uint_as_float(lo + (uint32_t)i));
}
__global__ void libm_all_kernel(float* out, uint32_t lo, uint64_t count, int which) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const float x = __uint_as_float(lo + (uint32_t)i);
    out[i] = which == 0 ? glibc_expf(x) : (which == 1 ? glibc_erff(x) : gelu_ref(x));
  }
}
void launch_e4m3_all(uint8_t* out, uint32_t lo, uint64_t count, cudaStream_t st) {
  e4m3_all_kernel<<<4096, 256, 0, st>>>(out, lo, count);
}
void launch_bf16_all(uint16_t* out, uint32_t lo, uint64_t count, cudaStream_t st) {
  bf16_all_kernel<<<4096, 256, 0, st>>>(out, lo, count);
}
void launch_libm_all(float* out, uint32_t lo, uint64_t count, int which, cudaStream_t st) {
  libm_all_kernel<<<4096, 256, 0, st>>>(out, lo, count, which);
}

}  // namespace cqg
