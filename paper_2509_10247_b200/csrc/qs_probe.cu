// FP32 peak probe: the denominator of the ray-casting roofline (BASELINE.md §3
// asks for a measured FFMA figure, and FFMA2 if used).  Every thread runs 8
// independent FMA chains (enough ILP to saturate the FMA pipes at full
// occupancy); mode 1 issues the packed sm_100 form fma.rn.f32x2 (SASS FFMA2).
#include "qs_common.cuh"

namespace {

__global__ void __launch_bounds__(256) k_probe_ffma(int iters, float seed, float* out) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = seed + threadIdx.x * 1e-3f + k;
  const float m = 0.999999f, c = 1e-7f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], m, c);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.f) out[blockIdx.x] = s;  // keep the chains live
}

__global__ void __launch_bounds__(256) k_probe_ffma2(int iters, float seed, float* out) {
  unsigned long long a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float lo = seed + threadIdx.x * 1e-3f + k, hi = lo + 0.5f;
    a[k] = ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
  }
  const float mf = 0.999999f, cf = 1e-7f;
  const unsigned long long m = ((unsigned long long)__float_as_uint(mf) << 32) | __float_as_uint(mf);
  const unsigned long long c = ((unsigned long long)__float_as_uint(cf) << 32) | __float_as_uint(cf);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[k]) : "l"(m), "l"(c));
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += __uint_as_float((unsigned)a[k]) + __uint_as_float((unsigned)(a[k] >> 32));
  if (s == 12345.f) out[blockIdx.x] = s;
}

}  // namespace

extern "C" {

int qs_probe_fp32(int32_t mode, int32_t n_blocks, int32_t iters, float* out, void* stream) {
  if (n_blocks <= 0 || iters <= 0) return QS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (mode == 0)
    k_probe_ffma<<<n_blocks, 256, 0, s>>>(iters, 1.f, out);
  else if (mode == 1)
    k_probe_ffma2<<<n_blocks, 256, 0, s>>>(iters, 1.f, out);
  else
    return QS_ERR_BAD_ARGUMENT;
  return cudaGetLastError() == cudaSuccess ? QS_OK : QS_ERR_LAUNCH;
}

}  // extern "C"
