// Throughput of fma.rn.f32.bf16 (FHFMA.BF16) vs unpack + FFMA on sm_100a:
// 8 independent chains per thread, 148*8 CTAs x 256 threads.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ float fma_bf16x2(uint32_t a, uint32_t b, float s) {
  asm("{\n.reg .b16 al, ah, bl, bh;\nmov.b32 {al, ah}, %1;\nmov.b32 {bl, bh}, %2;\n"
      "fma.rn.f32.bf16 %0, al, bl, %0;\nfma.rn.f32.bf16 %0, ah, bh, %0;\n}" : "+f"(s) : "r"(a), "r"(b));
  return s;
}
template <int MODE>
__global__ void k(float* out, const uint32_t* in, int iters) {
  uint32_t a[8], b[8];
  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = in[(threadIdx.x + i) & 255]; b[i] = in[(threadIdx.x * 3 + i) & 255]; acc[i] = 0.f; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) acc[i] = fma_bf16x2(a[i], b[i], acc[i]);
      else {
        acc[i] = __fmaf_rn(__uint_as_float(a[i] << 16), __uint_as_float(b[i] << 16), acc[i]);
        acc[i] = __fmaf_rn(__uint_as_float(a[i] & 0xFFFF0000u), __uint_as_float(b[i] & 0xFFFF0000u), acc[i]);
      }
      a[i] ^= b[(i + 1) & 7];  // keep operands live and varying
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o; uint32_t* in; cudaMalloc(&o, 148 * 8 * 256 * 4); cudaMalloc(&in, 1024);
  cudaMemset(in, 0x3f, 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int mode = 0; mode < 2; ++mode) for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    if (mode == 0) k<0><<<148 * 8, 256>>>(o, in, iters); else k<1><<<148 * 8, 256>>>(o, in, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double prods = 148.0 * 8 * 256 * iters * 16;
    printf("mode %d (%s): %.3f ms, %.2f T products/s\n", mode, mode ? "unpack+FFMA" : "FHFMA.BF16", ms, prods / ms / 1e9);
  }
}
