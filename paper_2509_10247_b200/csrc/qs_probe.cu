// FP32 peak probe: the denominator of the ray-casting roofline (BASELINE.md §3
// asks for a measured FFMA figure, and FFMA2 if used).  Every thread runs 8
// independent FMA chains (enough ILP to saturate the FMA pipes at full
// occupancy); mode 1 issues the packed sm_100 form fma.rn.f32x2 (SASS FFMA2).
#include "qs_umma.cuh"

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

// tcgen05 self-test: D (128x128 fp32) = A (128x128) B (128x128) in bf16 on the
// 5th-generation tensor cores, with A and B staged K-major or MN-major
// (mode bit 0 / bit 1) in the blocked no-swizzle layout of qs_umma.cuh --
// pins the descriptor / instruction-descriptor encodings the fused critic
// kernel relies on against a host matmul.
__global__ void __launch_bounds__(128) k_probe_umma(int mode, const float* __restrict__ A,
                                                    const float* __restrict__ B, float* __restrict__ D) {
  constexpr int M = 128, N = 128, K = 128;
  extern __shared__ __align__(1024) unsigned char probe_smem[];
  __nv_bfloat16* sa = reinterpret_cast<__nv_bfloat16*>(probe_smem);
  __nv_bfloat16* sb = sa + M * K;
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const bool a_mn = mode & 1, b_mn = mode & 2;
  for (int i = threadIdx.x; i < M * K; i += blockDim.x) {
    const int m = i / K, k = i % K;  // A[m][k]
    sa[a_mn ? umma::blk_off(k, m, M) : umma::blk_off(m, k, K)] = __float2bfloat16_rn(A[i]);
  }
  for (int i = threadIdx.x; i < K * N; i += blockDim.x) {
    const int k = i / N, n = i % N;  // B[k][n]
    sb[b_mn ? umma::blk_off(k, n, N) : umma::blk_off(n, k, K)] = __float2bfloat16_rn(B[i]);
  }
  if (threadIdx.x < 32) umma::tmem_alloc(&tbase, 128);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  umma::fence_async_smem();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t t0 = tbase;
  if (threadIdx.x == 0) {
    const uint32_t id = umma::idesc_bf16(M, N, a_mn, b_mn);
    for (int ks = 0; ks < K / 16; ++ks) {
      // a K step of 16 = two core matrices along K
      const uint64_t da = a_mn ? umma::desc_mnmajor(sa + ks * 2 * (M / 8) * 64, M) : umma::desc_kmajor(sa + ks * 128, K);
      const uint64_t db = b_mn ? umma::desc_mnmajor(sb + ks * 2 * (N / 8) * 64, N) : umma::desc_kmajor(sb + ks * 128, K);
      umma::mma_bf16(t0, da, db, id, ks > 0);
    }
    umma::commit(&bar);
  }
  umma::mbar_wait_parity(&bar, 0);
  umma::fence_after();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = 0; c < N; c += 16) {
    float v[16];
    umma::tmem_ld16(umma::taddr(t0, 32 * w, c), v);
    for (int j = 0; j < 16; ++j) D[(32 * w + lane) * N + c + j] = v[j];
  }
  umma::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) umma::tmem_free(t0, 128);
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

int qs_probe_umma(int32_t mode, const float* A, const float* B, float* D, void* stream) {
  const int smem = 2 * 128 * 128 * 2;
  if (cudaFuncSetAttribute(k_probe_umma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return QS_ERR_LAUNCH;
  k_probe_umma<<<1, 128, smem, (cudaStream_t)stream>>>(mode, A, B, D);
  return cudaGetLastError() == cudaSuccess ? QS_OK : QS_ERR_LAUNCH;
}

}  // extern "C"
