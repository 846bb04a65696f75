// diag.cu — exhaustive-check hooks over the device scalar numerics
// (include/cqg_diag.h). Device-only computation; results copied back.
#include <cuda_runtime.h>

#include <string>

#include "../../include/cqg_diag.h"
#include "kernels.h"

namespace {
template <class T, class L>
int run(uint64_t count, T* out_host, L launch) {
  T* d = nullptr;
  if (cudaMalloc(&d, count * sizeof(T)) != cudaSuccess) return 3;
  launch(d);
  cudaError_t e = cudaMemcpy(out_host, d, count * sizeof(T), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e == cudaSuccess ? 0 : 2;
}
}  // namespace

extern "C" {
int cqg_diag_e4m3_range(uint32_t lo, uint64_t count, uint8_t* out) {
  return run(count, out, [&](uint8_t* d) { cqg::launch_e4m3_all(d, lo, count, 0); });
}
int cqg_diag_bf16_range(uint32_t lo, uint64_t count, uint16_t* out) {
  return run(count, out, [&](uint16_t* d) { cqg::launch_bf16_all(d, lo, count, 0); });
}
int cqg_diag_libm_range(int which, uint32_t lo, uint64_t count, float* out) {
  return run(count, out, [&](float* d) { cqg::launch_libm_all(d, lo, count, which, 0); });
}
}
