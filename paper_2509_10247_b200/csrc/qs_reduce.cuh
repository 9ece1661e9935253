// Deterministic cross-CTA gradient sums.  A persistent gradient kernel writes
// its CTA's partial sums with plain stores to work[blockIdx.x * P + i]
// (every CTA writes every entry of the segments below); k_sum_partials then
// adds the partials to the outputs in a fixed order (16 strided slices of the
// CTAs, combined by a fixed pairwise tree) -- the same bits
// every run, eager or graph-replayed, unlike float atomics whose order
// follows the schedule.
#pragma once
#include "qs_common.cuh"

namespace red {

constexpr int MAXSEG = 8;
struct Segs {  // out[s][i] (+)= sum_b work[b * P + off[s] + i], i < len[s]
  float* out[MAXSEG];
  int64_t off[MAXSEG];
  int64_t len[MAXSEG];
  int n;
  bool accumulate;  // add to out (else overwrite)
};

constexpr int RED_E = 32, RED_S = 16;  // a block: 32 consecutive entries x 16 CTA slices

static __global__ void __launch_bounds__(RED_E * RED_S)
    k_sum_partials(const float* __restrict__ work, int nblk, int64_t P, Segs s) {
  __shared__ float part[RED_S][RED_E];
  const int e = threadIdx.x % RED_E, sl = threadIdx.x / RED_E;
  int64_t i = (int64_t)blockIdx.x * RED_E + e;
  int k = 0;
  while (k < s.n && i >= s.len[k]) i -= s.len[k++];
  float a = 0.f;
  if (k < s.n) {  // slice sl: CTAs sl, sl + 8, sl + 16, ... in order
    const float* p = work + s.off[k] + i;
    for (int b = sl; b < nblk; b += RED_S) a += __ldg(p + (int64_t)b * P);
  }
  part[sl][e] = a;
  __syncthreads();
  if (sl == 0 && k < s.n) {
    float q[RED_S];  // a fixed pairwise tree over the slices
#pragma unroll
    for (int j = 0; j < RED_S; ++j) q[j] = part[j][e];
#pragma unroll
    for (int w = RED_S / 2; w > 0; w >>= 1) {
#pragma unroll
      for (int j = 0; j < w; ++j) q[j] = q[2 * j] + q[2 * j + 1];
    }
    const float sum = q[0];
    s.out[k][i] = s.accumulate ? s.out[k][i] + sum : sum;
  }
}

// launch the sum over `nblk` partials of width P for the non-null segments
static int sum_partials(const float* work, int nblk, int64_t P, const Segs& segs, cudaStream_t st) {
  Segs s{};
  s.accumulate = segs.accumulate;
  int64_t total = 0;
  for (int k = 0; k < segs.n; ++k) {
    if (!segs.out[k] || segs.len[k] <= 0) continue;
    s.out[s.n] = segs.out[k];
    s.off[s.n] = segs.off[k];
    s.len[s.n] = segs.len[k];
    total += segs.len[k];
    ++s.n;
  }
  if (total == 0) return QS_OK;
  k_sum_partials<<<(unsigned)((total + RED_E - 1) / RED_E), RED_E * RED_S, 0, st>>>(work, nblk, P, s);
  return cudaGetLastError() == cudaSuccess ? QS_OK : QS_ERR_LAUNCH;
}

}  // namespace red
