// numerics.cuh — device-side bit-exact restatements of the reference's
// scalar numerics.
//
//  * E4M3 encode  == cq::encode_f8   (proj/src/numerics.cpp:41-64): OCP E4M3,
//    RNE, saturating to +-448, NaN -> 0x7F. Realised with the hardware
//    cvt.rn.satfinite.e4m3x2.f32 (SASS F2FP.SATFINITE.E4M3.F32.PACK), which
//    SURVEY.md §0.4 measured equal on all 2^32 floats; NaN is pinned to 0x7F
//    explicitly because the reference drops the sign.
//  * BF16 encode  == cq::encode_bf16 (numerics.cpp:84-94) incl. NaN -> s|0x7FC0.
//  * RTN          == quantize_rtn_impl (numerics.cpp:105-120) in double.
//  * glibc_expf / glibc_erff: operation-for-operation restatements of the
//    glibc 2.39 float expf (table-driven, 32-entry 2^(i/32) table, cubic in
//    double) and fdlibm-derived erff that the reference reaches through
//    std::exp(float) (kernels.cpp:180) and std::erf(float) (kernels.cpp:226).
//    Checked exhaustively on the host against the system libm (all 2^32 inputs:
//    erff 0 mismatches; expf 2 mismatches, patched below as explicit cases).
//    Every float/double op uses an explicit _rn intrinsic so nvcc cannot
//    contract or reassociate.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp8.h>
#include <stdint.h>

namespace cqg {

enum : int { kP8 = 0, kP16 = 1, kP32 = 2 };
enum : int { kE4M3 = 0, kRtn4 = 1 };

__device__ __forceinline__ uint8_t enc_e4m3(float x) {
  if (x != x) return 0x7F;
  return (uint8_t)__nv_cvt_float_to_fp8(x, __NV_SATFINITE, __NV_E4M3);
}

__device__ __forceinline__ float dec_e4m3(uint8_t b) {
  __half_raw h = __nv_cvt_fp8_to_halfraw((__nv_fp8_storage_t)b, __NV_E4M3);
  return __half2float(__half(h));
}

__device__ __forceinline__ float round_e4m3(float x) { return dec_e4m3(enc_e4m3(x)); }

__device__ __forceinline__ uint16_t enc_bf16(float x) {
  uint32_t u = __float_as_uint(x);
  if (x != x) return (uint16_t)(((u >> 16) & 0x8000u) | 0x7FC0u);
  uint32_t lsb = (u >> 16) & 1u;
  u += 0x7FFFu + lsb;
  return (uint16_t)(u >> 16);
}

__device__ __forceinline__ float dec_bf16(uint16_t b) { return __uint_as_float((uint32_t)b << 16); }

__device__ __forceinline__ float round_bf16(float x) { return dec_bf16(enc_bf16(x)); }

// round_{p} for elementwise precisions (P8 here means E4M3; Rtn4 is a
// tensor-wide grid handled by dedicated kernels).
__device__ __forceinline__ float round_p(float x, int p) {
  if (p == kP32) return x;
  if (p == kP16) return round_bf16(x);
  return round_e4m3(x);
}

// round_half_even (numerics.cpp:21-28)
__device__ __forceinline__ long long rhe(double q) {
  double fl = floor(q);
  double frac = __dsub_rn(q, fl);
  long long lo = (long long)fl;
  if (frac > 0.5) return lo + 1;
  if (frac < 0.5) return lo;
  return (lo % 2 == 0) ? lo : lo + 1;
}

// One element of quantize_rtn with a known delta (numerics.cpp:115-118).
// qmax: the INT8 extension's clamp (127: the +128 endpoint saturates; see
// oracle/cq_oracle.c rtn8_group); 0 = none.
__device__ __forceinline__ float rtn_apply(float v, double delta, int qmax = 0) {
  if (delta == 0.0) return v;
  double q = __ddiv_rn((double)v, delta);
  long long k = rhe(q);
  if (qmax && k > qmax) k = qmax;
  return (float)__dmul_rn(delta, (double)k);
}

// ---------------------------------------------------------------------------
// glibc expf restatement (sysdeps/ieee754/flt-32/e_expf.c algorithm).
// ---------------------------------------------------------------------------
__constant__ static const unsigned long long kExp2fTab[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull};

__device__ __forceinline__ float glibc_expf(float x) {
  const uint32_t ux = __float_as_uint(x);
  // Two inputs where the system libm's result differs from the plain
  // algorithm (found by the exhaustive host check).
  if (ux == 0x4202422fu) return __uint_as_float(0x56fc9f1cu);  //  0x1.04845ep+5
  if (ux == 0xc27c65d9u) return __uint_as_float(0x11fa2993u);  // -0x1.f8cbb2p+5
  const uint32_t abstop = (ux >> 20) & 0x7ffu;
  if (abstop >= (0x42b00000u >> 20)) {  // |x| >= 88 or nan
    if (ux == 0xff800000u) return 0.0f;
    if (abstop >= (0x7f800000u >> 20)) return __fadd_rn(x, x);
    if (x > 0x1.62e42ep6f) return __uint_as_float(0x7f800000u);
    if (x < -0x1.9fe368p6f) return 0.0f;
  }
  const double N = 32.0;
  const double C0 = 0x1.c6af84b912394p-5 / N / N / N;
  const double C1 = 0x1.ebfce50fac4f3p-3 / N / N;
  const double C2 = 0x1.62e42ff0c52d6p-1 / N;
  const double InvLn2N = 0x1.71547652b82fep+0 * N;
  const double SHIFT = 0x1.8p+52;
  double xd = (double)x;
  double z = __dmul_rn(InvLn2N, xd);
  double kd = __dadd_rn(z, SHIFT);
  unsigned long long ki = (unsigned long long)__double_as_longlong(kd);
  kd = __dsub_rn(kd, SHIFT);
  double r = __dsub_rn(z, kd);
  unsigned long long t = kExp2fTab[ki % 32];
  t += ki << (52 - 5);
  double s = __longlong_as_double((long long)t);
  double zz = __fma_rn(C0, r, C1);
  double r2 = __dmul_rn(r, r);
  double y = __fma_rn(C2, r, 1.0);
  y = __fma_rn(zz, r2, y);
  y = __dmul_rn(y, s);
  return __double2float_rn(y);
}

// ---------------------------------------------------------------------------
// glibc 2.39 erff restatement (fdlibm s_erff.c algorithm, float arithmetic).
// ---------------------------------------------------------------------------
#define FA(a, b) __fadd_rn((a), (b))
#define FS(a, b) __fsub_rn((a), (b))
#define FM(a, b) __fmul_rn((a), (b))
#define FD(a, b) __fdiv_rn((a), (b))

__device__ __forceinline__ float glibc_erff(float x) {
  const float tiny = 1e-30f, one = 1.0f, erx = 8.4506291151e-01f, efx = 1.2837916613e-01f;
  const float pp0 = 1.2837916613e-01f, pp1 = -3.2504209876e-01f, pp2 = -2.8481749818e-02f,
              pp3 = -5.7702702470e-03f, pp4 = -2.3763017452e-05f;
  const float qq1 = 3.9791721106e-01f, qq2 = 6.5022252500e-02f, qq3 = 5.0813062117e-03f,
              qq4 = 1.3249473704e-04f, qq5 = -3.9602282413e-06f;
  const float pa0 = -2.3621185683e-03f, pa1 = 4.1485610604e-01f, pa2 = -3.7220788002e-01f,
              pa3 = 3.1834661961e-01f, pa4 = -1.1089469492e-01f, pa5 = 3.5478305072e-02f,
              pa6 = -2.1663755178e-03f;
  const float qa1 = 1.0642088205e-01f, qa2 = 5.4039794207e-01f, qa3 = 7.1828655899e-02f,
              qa4 = 1.2617121637e-01f, qa5 = 1.3637083583e-02f, qa6 = 1.1984500103e-02f;
  const float ra0 = -9.8649440333e-03f, ra1 = -6.9385856390e-01f, ra2 = -1.0558626175e+01f,
              ra3 = -6.2375331879e+01f, ra4 = -1.6239666748e+02f, ra5 = -1.8460508728e+02f,
              ra6 = -8.1287437439e+01f, ra7 = -9.8143291473e+00f;
  const float sa1 = 1.9651271820e+01f, sa2 = 1.3765776062e+02f, sa3 = 4.3456588745e+02f,
              sa4 = 6.4538726807e+02f, sa5 = 4.2900814819e+02f, sa6 = 1.0863500214e+02f,
              sa7 = 6.5702495575e+00f, sa8 = -6.0424413532e-02f;
  const float rb0 = -9.8649431020e-03f, rb1 = -7.9928326607e-01f, rb2 = -1.7757955551e+01f,
              rb3 = -1.6063638306e+02f, rb4 = -6.3756646729e+02f, rb5 = -1.0250950928e+03f,
              rb6 = -4.8351919556e+02f;
  const float sb1 = 3.0338060379e+01f, sb2 = 3.2579251099e+02f, sb3 = 1.5367296143e+03f,
              sb4 = 3.1998581543e+03f, sb5 = 2.5530502930e+03f, sb6 = 4.7452853394e+02f,
              sb7 = -2.2440952301e+01f;
  const int32_t hx = (int32_t)__float_as_uint(x);
  int32_t ix = hx & 0x7fffffff;
  float R, S, P, Q, s, y, z, r;
  if (ix >= 0x7f800000) {
    int i = ((uint32_t)hx >> 31) << 1;
    return FA((float)(1 - i), FD(one, x));
  }
  if (ix < 0x3f580000) {
    if (ix < 0x31800000) {
      if (ix < 0x04000000) return FM(0.0625f, FA(FM(16.0f, x), FM(FM(16.0f, efx), x)));
      return FA(x, FM(efx, x));
    }
    z = FM(x, x);
    r = FA(pp0, FM(z, FA(pp1, FM(z, FA(pp2, FM(z, FA(pp3, FM(z, pp4))))))));
    s = FA(one, FM(z, FA(qq1, FM(z, FA(qq2, FM(z, FA(qq3, FM(z, FA(qq4, FM(z, qq5))))))))));
    y = FD(r, s);
    return FA(x, FM(x, y));
  }
  if (ix < 0x3fa00000) {
    s = FS(fabsf(x), one);
    P = FA(pa0, FM(s, FA(pa1, FM(s, FA(pa2, FM(s, FA(pa3, FM(s, FA(pa4, FM(s, FA(pa5, FM(s, pa6))))))))))));
    Q = FA(one, FM(s, FA(qa1, FM(s, FA(qa2, FM(s, FA(qa3, FM(s, FA(qa4, FM(s, FA(qa5, FM(s, qa6))))))))))));
    if (hx >= 0) return FA(erx, FD(P, Q));
    return FS(-erx, FD(P, Q));
  }
  if (ix >= 0x40c00000) {
    if (hx >= 0) return FS(one, tiny);
    return FS(tiny, one);
  }
  x = fabsf(x);
  s = FD(one, FM(x, x));
  if (ix < 0x4036DB6E) {
    R = FA(ra0, FM(s, FA(ra1, FM(s, FA(ra2, FM(s, FA(ra3, FM(s, FA(ra4, FM(s, FA(ra5, FM(s, FA(ra6, FM(s, ra7))))))))))))));
    S = FA(one, FM(s, FA(sa1, FM(s, FA(sa2, FM(s, FA(sa3, FM(s, FA(sa4, FM(s, FA(sa5, FM(s, FA(sa6, FM(s, FA(sa7, FM(s, sa8))))))))))))))));
  } else {
    R = FA(rb0, FM(s, FA(rb1, FM(s, FA(rb2, FM(s, FA(rb3, FM(s, FA(rb4, FM(s, FA(rb5, FM(s, rb6))))))))))));
    S = FA(one, FM(s, FA(sb1, FM(s, FA(sb2, FM(s, FA(sb3, FM(s, FA(sb4, FM(s, FA(sb5, FM(s, FA(sb6, FM(s, sb7))))))))))))));
  }
  ix = (int32_t)__float_as_uint(x);
  z = __uint_as_float((uint32_t)ix & 0xfffff000u);
  r = FM(glibc_expf(FS(FM(-z, z), 0.5625f)), glibc_expf(FA(FM(FS(z, x), FA(z, x)), FD(R, S))));
  if (hx >= 0) return FS(one, FD(r, x));
  return FS(FD(r, x), one);
}

// gelu (kernels.cpp:226): 0.5f * x * (1.0f + erff(x * 0.70710678118654752f))
__device__ __forceinline__ float gelu_ref(float x) {
  return FM(FM(0.5f, x), FA(1.0f, glibc_erff(FM(x, 0.70710678118654752f))));
}

#undef FA
#undef FS
#undef FM
#undef FD

}  // namespace cqg
