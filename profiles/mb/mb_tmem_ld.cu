// TMEM -> register load throughput per SM for the tcgen05.ld shapes an
// epilogue can use (4 KB per warp per instruction in every case), with 4 or
// 16 warps.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 mb_tmem_ld.cu
#include <cstdio>
#include <cstdint>

#define LD32(shape, ADDR, R)                                                                                     \
  asm volatile("tcgen05.ld.sync.aligned." shape ".b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"   \
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                        \
               : "=r"(R[0]), "=r"(R[1]), "=r"(R[2]), "=r"(R[3]), "=r"(R[4]), "=r"(R[5]), "=r"(R[6]), "=r"(R[7]), \
                 "=r"(R[8]), "=r"(R[9]), "=r"(R[10]), "=r"(R[11]), "=r"(R[12]), "=r"(R[13]), "=r"(R[14]),        \
                 "=r"(R[15]), "=r"(R[16]), "=r"(R[17]), "=r"(R[18]), "=r"(R[19]), "=r"(R[20]), "=r"(R[21]),      \
                 "=r"(R[22]), "=r"(R[23]), "=r"(R[24]), "=r"(R[25]), "=r"(R[26]), "=r"(R[27]), "=r"(R[28]),      \
                 "=r"(R[29]), "=r"(R[30]), "=r"(R[31])                                                            \
               : "r"(ADDR))

template <int SHAPE>
__global__ void k(int iters, unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t lane0 = 32u * (warp & 3);
  const uint32_t col0 = 32u * (warp >> 2);  // warps sharing a lane quarter read different columns
  const uint32_t addr = base + (lane0 << 16) + col0;
  uint32_t r[32], acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (SHAPE == 0) LD32("32x32b.x32", addr, r);
    if (SHAPE == 1) LD32("16x256b.x8", addr, r);
    if (SHAPE == 2) LD32("16x128b.x16", addr, r);
    if (SHAPE == 3) LD32("16x64b.x32", addr, r);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 32; ++j) acc ^= r[j];
  }
  const unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

int main() {
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 1024 * 8);
  cudaMalloc(&sink, 1024 * 1024 * 4);
  const char* names[4] = {"32x32b.x32", "16x256b.x8", "16x128b.x16", "16x64b.x32"};
  const int iters = 4096;
  for (int warps : {4, 8, 16}) {
    for (int s = 0; s < 4; ++s) {
      for (int rep = 0; rep < 2; ++rep) {
        if (s == 0) k<0><<<148, 32 * warps>>>(iters, cyc, sink);
        if (s == 1) k<1><<<148, 32 * warps>>>(iters, cyc, sink);
        if (s == 2) k<2><<<148, 32 * warps>>>(iters, cyc, sink);
        if (s == 3) k<3><<<148, 32 * warps>>>(iters, cyc, sink);
      }
      cudaDeviceSynchronize();
      unsigned long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double bytes = 4096.0 * warps * iters;
      printf("%-12s warps %2d: %7.1f B/cycle per SM (%llu cycles, err %s)\n", names[s], warps, bytes / c, c,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
