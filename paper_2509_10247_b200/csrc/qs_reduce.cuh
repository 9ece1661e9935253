// Deterministic cross-CTA gradient sums.  A persistent gradient kernel writes
// its CTA's partial sums with plain stores to work[blockIdx.x * P + i]
// (every CTA writes every entry of the segments below); k_sum_partials then
// adds the partials to the outputs in CTA order 0, 1, ... -- the same bits
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

static __global__ void k_sum_partials(const float* __restrict__ work, int nblk, int64_t P, Segs s) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int k = 0;
  while (k < s.n && i >= s.len[k]) i -= s.len[k++];
  if (k >= s.n) return;
  const float* p = work + s.off[k] + i;
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;  // fixed association: ((b%4 classes) in order) then combined
  int b = 0;
  for (; b + 4 <= nblk; b += 4) {
    a0 += __ldg(p + (int64_t)b * P);
    a1 += __ldg(p + (int64_t)(b + 1) * P);
    a2 += __ldg(p + (int64_t)(b + 2) * P);
    a3 += __ldg(p + (int64_t)(b + 3) * P);
  }
  for (; b < nblk; ++b) a0 += __ldg(p + (int64_t)b * P);
  const float sum = (a0 + a1) + (a2 + a3);
  s.out[k][i] = s.accumulate ? s.out[k][i] + sum : sum;
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
  const int threads = 128;
  k_sum_partials<<<(unsigned)((total + threads - 1) / threads), threads, 0, st>>>(work, nblk, P, s);
  return cudaGetLastError() == cudaSuccess ? QS_OK : QS_ERR_LAUNCH;
}

}  // namespace red
