// The policy's MLP trunk and Gaussian heads on the 5th-generation tensor cores
// (the caller side of config C5; q/nets.py:198-256):
//
//     A1 = tanh(h W0 + b0)    A2 = tanh(A1 W1 + b1)    z = tanh(A2 W2 + b2)
//     y  = z Wh + bh          (Wh = [W_mu | W_sigma | 0], 128 x 8)
//
// for the GRU output h (N x 64), hidden widths 128 (the reference's
// PolicyArch: hidden 64, mlp (128, 128), the trunk's last layer squashed).
//   qs_policy_trunk_fwd  y for every row (the rollout's forward)
//   qs_policy_trunk_bwd  given dL/dy, recompute the forward per tile and
//                        return dL/dh (for the GRU's backward) while
//                        accumulating every weight and bias gradient in TMEM.
// Same machinery as the critic fit (qs_mlp.cu / qs_umma.cuh): one persistent
// 512-thread CTA per SM; thread (warp w, lane l) owns tile row 32 (w % 4) + l
// -- its TMEM lane -- and a quarter of the 128 columns; one elected thread
// issues tcgen05.mma (bf16 operands in the blocked no-swizzle layout, fp32
// accumulators in TMEM) and commits to an mbarrier; every weight matrix is
// staged once and serves as a K-major operand one way and MN-major the other.
#include "qs_umma.cuh"

namespace {

constexpr int PT = 512;     // threads
constexpr int TR = 128;     // rows per tile
constexpr int HI = 64;      // GRU width (trunk input)
constexpr int HW = 128;     // trunk width
constexpr int HY = 16;      // head outputs, padded (mu | log sigma | 0 | ones column for bias sums)

QS_D float tanh_f(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
QS_D uint32_t pk(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
QS_D float2 upk(uint32_t u) { return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u)); }
QS_D void ld32(uint32_t t, float (&v)[32]) {
  float a[16], b[16];
  umma::tmem_ld16(t, a);
  umma::tmem_ld16(t + 16, b);
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    v[j] = a[j];
    v[16 + j] = b[j];
  }
}
// 8 bf16 pairs of row r at columns [c0, c0 + 32) of a blocked [rows][cols] buffer
QS_D void st32(__nv_bfloat16* buf, int r, int c0, int cols, const uint32_t (&w)[16]) {
#pragma unroll
  for (int j = 0; j < 4; ++j)
    *reinterpret_cast<uint4*>(&buf[umma::blk_off(r, c0 + 8 * j, cols)]) =
        make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
}
QS_D void ld32s(const __nv_bfloat16* buf, int r, int c0, int cols, float (&v)[32]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint4 u = *reinterpret_cast<const uint4*>(&buf[umma::blk_off(r, c0 + 8 * j, cols)]);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = upk(w[i]);
      v[8 * j + 2 * i] = f.x;
      v[8 * j + 2 * i + 1] = f.y;
    }
  }
}

struct PolSmem {
  __nv_bfloat16 W0[HI * HW];   // [64][128]   B of h W0 (MN-major) and of gA1 W0^T (K-major)
  __nv_bfloat16 W1[HW * HW];   // [128][128]  B of A1 W1 (MN) and gA2 W1^T (K)
  __nv_bfloat16 W2[HW * HW];   // [128][128]
  __nv_bfloat16 WH[HW * HY];   // [128][16]   B of z Wh (MN) and dY Wh^T (K)
  __nv_bfloat16 H[TR * HI];    // [rows][64]  the tile's GRU output
  __nv_bfloat16 A1[TR * HW];   // A1, then dL/dA1-pre in place
  __nv_bfloat16 A2[TR * HW];   // A2, then dL/dA2-pre in place
  __nv_bfloat16 Z[TR * HW];    // z, then dL/dz-pre in place
  __nv_bfloat16 DY[TR * HY];   // dL/dy (8 columns), column 15 = 1
  float b0[HW], b1[HW], b2[HW], bh[HY];
  float dbh[HY];
  uint64_t bar;
  uint32_t tbase;
};

template <bool BWD>
__global__ void __launch_bounds__(PT, 1)
    k_policy_trunk(int64_t N, int n_out, const float* __restrict__ h, const float* __restrict__ dy,
                   const float* __restrict__ W0, const float* __restrict__ b0, const float* __restrict__ W1,
                   const float* __restrict__ b1, const float* __restrict__ W2, const float* __restrict__ b2,
                   const float* __restrict__ Wh, const float* __restrict__ bh, float* __restrict__ y,
                   float* __restrict__ dh, float* __restrict__ gW0, float* __restrict__ gb0,
                   float* __restrict__ gW1, float* __restrict__ gb1, float* __restrict__ gW2,
                   float* __restrict__ gb2, float* __restrict__ gWh, float* __restrict__ gbh) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  PolSmem& S = *reinterpret_cast<PolSmem*>(smem_raw);
  using umma::blk_off;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = 32 * (warp & 3) + lane, q = warp >> 2, cq = 32 * q;
  // ---- weights (bf16, blocked) and biases
  for (int i = tid; i < HI * HW; i += PT) S.W0[blk_off(i / HW, i % HW, HW)] = __float2bfloat16_rn(W0[i]);
  for (int i = tid; i < HW * HW; i += PT) {
    S.W1[blk_off(i / HW, i % HW, HW)] = __float2bfloat16_rn(W1[i]);
    S.W2[blk_off(i / HW, i % HW, HW)] = __float2bfloat16_rn(W2[i]);
  }
  for (int i = tid; i < HW * HY; i += PT) {
    const int k = i / HY, n = i % HY;  // Wh (128, n_out) row-major, zero-padded to 16 columns
    S.WH[blk_off(k, n, HY)] = __float2bfloat16_rn(n < n_out ? Wh[k * n_out + n] : 0.f);
  }
  for (int i = tid; i < HW; i += PT) {
    S.b0[i] = b0[i];
    S.b1[i] = b1[i];
    S.b2[i] = b2[i];
  }
  if (tid < HY) {
    S.bh[tid] = (bh && tid < n_out) ? bh[tid] : 0.f;  // (the backward takes no bh)
    S.dbh[tid] = 0.f;
  }
  if (warp == 0) umma::tmem_alloc(&S.tbase, 512);
  if (tid == 0) {
    mbar_init(&S.bar, 1);
    fence_barrier_init();
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t T0 = S.tbase;
  // TMEM: tile GEMM [0,128); dW2 [128,256); dW1 [256,384); dW0^T [384,448);
  // dWh [448,464); db2 [464,480); db1 [480,496); db0 [496,512)
  const uint32_t TG = T0, TW2 = T0 + 128, TW1 = T0 + 256, TW0 = T0 + 384, TWH = T0 + 448, TB2 = T0 + 464,
                 TB1 = T0 + 480, TB0 = T0 + 496;
  const uint32_t lanes = umma::taddr(0, 32 * (warp & 3), 0);
  uint32_t phase = 0;
  bool first = true;
  float dbh_acc[HY / 2];  // quarter 0: this row's dL/dy, summed over tiles
#pragma unroll
  for (int j = 0; j < HY / 2; ++j) dbh_acc[j] = 0.f;
  auto to_mma = [&]() {
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
  };
  auto wait = [&]() {
    umma::mbar_wait_parity(&S.bar, phase);
    phase ^= 1u;
    umma::fence_after();
  };
  // K-major A over a blocked [rows][cols] buffer, K step ks (16 columns)
  auto aK = [](const __nv_bfloat16* b, int cols, int ks) { return umma::desc_kmajor(b + ks * 128, cols); };
  // MN-major operand over a blocked [rows=K][cols=MN] buffer, K step ks (16 rows)
  auto mK = [](const __nv_bfloat16* b, int cols, int ks) {
    return umma::desc_mnmajor(b + ks * 2 * (cols / 8) * 64, cols);
  };
  // epilogue: TMEM columns [cq, cq+32) of this row + bias -> tanh -> bf16 row of dst
  auto epi_tanh = [&](const float* bias, __nv_bfloat16* dst) {
    float v[32];
    ld32(TG + lanes + cq, v);
    uint32_t w[16];
#pragma unroll
    for (int j = 0; j < 32; j += 2) w[j / 2] = pk(tanh_f(v[j] + bias[cq + j]), tanh_f(v[j + 1] + bias[cq + j + 1]));
    st32(dst, r, cq, HW, w);
  };
  // epilogue: TMEM columns * (1 - act^2) (act = the bf16 activation row) -> in place over act
  auto epi_dtanh = [&](__nv_bfloat16* act) {
    float v[32], a[32];
    ld32(TG + lanes + cq, v);
    ld32s(act, r, cq, HW, a);
    uint32_t w[16];
#pragma unroll
    for (int j = 0; j < 32; j += 2) w[j / 2] = pk(v[j] * (1.f - a[j] * a[j]), v[j + 1] * (1.f - a[j + 1] * a[j + 1]));
    st32(act, r, cq, HW, w);
  };
  const uint32_t id_mn_b = umma::idesc_bf16(128, 128, false, true);  // A K-major, B MN-major
  const uint32_t id_kk = umma::idesc_bf16(128, 128, false, false);
  const uint32_t id_mm = umma::idesc_bf16(128, 128, true, true);
  const uint32_t id_kk64 = umma::idesc_bf16(128, 64, false, false);
  const uint32_t id_mm64 = umma::idesc_bf16(128, 64, true, true);
  const uint32_t id_mm16 = umma::idesc_bf16(128, 16, true, true);
  const uint32_t id_k_mn16 = umma::idesc_bf16(128, 16, false, true);
  const int64_t ntiles = (N + TR - 1) / TR;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row = tile * TR + r;
    const bool valid = row < N;
    // ---- stage h (quarter q: columns 16q..16q+15) and, backward, dL/dy
    {
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        const float4 t = valid ? __ldg(reinterpret_cast<const float4*>(h + row * HI + 16 * q + j))
                               : make_float4(0.f, 0.f, 0.f, 0.f);
        v[j] = t.x;
        v[j + 1] = t.y;
        v[j + 2] = t.z;
        v[j + 3] = t.w;
      }
#pragma unroll
      for (int j = 0; j < 16; j += 8)
        *reinterpret_cast<uint4*>(&S.H[blk_off(r, 16 * q + j, HI)]) =
            make_uint4(pk(v[j], v[j + 1]), pk(v[j + 2], v[j + 3]), pk(v[j + 4], v[j + 5]), pk(v[j + 6], v[j + 7]));
    }
    if (BWD && q == 0) {
      float g[HY];
#pragma unroll
      for (int j = 0; j < HY; ++j) g[j] = 0.f;
      if (valid) {
#pragma unroll
        for (int j = 0; j < HY / 2; ++j)
          if (j < n_out) g[j] = __ldg(dy + row * n_out + j);
      }
#pragma unroll
      for (int j = 0; j < HY / 2; ++j) dbh_acc[j] += g[j];
      g[HY - 1] = 1.f;  // ones column: the bias gradients' column sums
#pragma unroll
      for (int j = 0; j < HY; j += 8)
        *reinterpret_cast<uint4*>(&S.DY[blk_off(r, j, HY)]) =
            make_uint4(pk(g[j], g[j + 1]), pk(g[j + 2], g[j + 3]), pk(g[j + 4], g[j + 5]), pk(g[j + 6], g[j + 7]));
    }
    to_mma();
    // ---- forward: A1, A2, z
    if (tid == 0) {
#pragma unroll
      for (int ks = 0; ks < HI / 16; ++ks) umma::mma_bf16(TG, aK(S.H, HI, ks), mK(S.W0, HW, ks), id_mn_b, ks > 0);
      umma::commit(&S.bar);
    }
    wait();
    epi_tanh(S.b0, S.A1);
    to_mma();
    if (tid == 0) {
#pragma unroll
      for (int ks = 0; ks < HW / 16; ++ks) umma::mma_bf16(TG, aK(S.A1, HW, ks), mK(S.W1, HW, ks), id_mn_b, ks > 0);
      umma::commit(&S.bar);
    }
    wait();
    epi_tanh(S.b1, S.A2);
    to_mma();
    if (tid == 0) {
#pragma unroll
      for (int ks = 0; ks < HW / 16; ++ks) umma::mma_bf16(TG, aK(S.A2, HW, ks), mK(S.W2, HW, ks), id_mn_b, ks > 0);
      umma::commit(&S.bar);
    }
    wait();
    epi_tanh(S.b2, S.Z);
    to_mma();
    if constexpr (!BWD) {
      // ---- heads: y = z Wh + bh (N = 16, the first n_out columns written)
      if (tid == 0) {
#pragma unroll
        for (int ks = 0; ks < HW / 16; ++ks)
          umma::mma_bf16(TG, aK(S.Z, HW, ks), mK(S.WH, HY, ks), id_k_mn16, ks > 0);
        umma::commit(&S.bar);
      }
      wait();
      if (q == 0) {
        float v[16];
        umma::tmem_ld16(TG + lanes, v);
        if (valid) {
#pragma unroll
          for (int j = 0; j < HY / 2; ++j)
            if (j < n_out) y[row * n_out + j] = v[j] + S.bh[j];
        }
      }
      umma::fence_before();
      __syncthreads();  // the next tile overwrites H, A1, A2, Z
      umma::fence_after();
      continue;
    }
    // ---- backward: dz-pre = dY Wh^T (1 - z^2); dWh += z^T dY
    if (tid == 0) {
      umma::mma_bf16(TG, aK(S.DY, HY, 0), umma::desc_kmajor(S.WH, HY), id_kk, false);
#pragma unroll
      for (int ks = 0; ks < TR / 16; ++ks) umma::mma_bf16(TWH, mK(S.Z, HW, ks), mK(S.DY, HY, ks), id_mm16, !first || ks > 0);
      umma::commit(&S.bar);
    }
    wait();
    epi_dtanh(S.Z);  // Z <- dL/d(z-pre)
    to_mma();
    // dA2-pre = dZ W2^T (1 - A2^2); dW2 += A2^T dZ; db2 += dZ^T 1
    if (tid == 0) {
#pragma unroll
      for (int ks = 0; ks < HW / 16; ++ks) umma::mma_bf16(TG, aK(S.Z, HW, ks), aK(S.W2, HW, ks), id_kk, ks > 0);
#pragma unroll
      for (int ks = 0; ks < TR / 16; ++ks) {
        umma::mma_bf16(TW2, mK(S.A2, HW, ks), mK(S.Z, HW, ks), id_mm, !first || ks > 0);
        umma::mma_bf16(TB2, mK(S.Z, HW, ks), mK(S.DY, HY, ks), id_mm16, !first || ks > 0);
      }
      umma::commit(&S.bar);
    }
    wait();
    epi_dtanh(S.A2);  // A2 <- dL/d(A2-pre)
    to_mma();
    // dA1-pre = dA2 W1^T (1 - A1^2); dW1 += A1^T dA2; db1
    if (tid == 0) {
#pragma unroll
      for (int ks = 0; ks < HW / 16; ++ks) umma::mma_bf16(TG, aK(S.A2, HW, ks), aK(S.W1, HW, ks), id_kk, ks > 0);
#pragma unroll
      for (int ks = 0; ks < TR / 16; ++ks) {
        umma::mma_bf16(TW1, mK(S.A1, HW, ks), mK(S.A2, HW, ks), id_mm, !first || ks > 0);
        umma::mma_bf16(TB1, mK(S.A2, HW, ks), mK(S.DY, HY, ks), id_mm16, !first || ks > 0);
      }
      umma::commit(&S.bar);
    }
    wait();
    epi_dtanh(S.A1);  // A1 <- dL/d(A1-pre)
    to_mma();
    // dh = dA1 W0^T (N = 64); dW0^T += dA1^T h; db0
    if (tid == 0) {
#pragma unroll
      for (int ks = 0; ks < HW / 16; ++ks) umma::mma_bf16(TG, aK(S.A1, HW, ks), aK(S.W0, HW, ks), id_kk64, ks > 0);
#pragma unroll
      for (int ks = 0; ks < TR / 16; ++ks) {
        umma::mma_bf16(TW0, mK(S.A1, HW, ks), mK(S.H, HI, ks), id_mm64, !first || ks > 0);
        umma::mma_bf16(TB0, mK(S.A1, HW, ks), mK(S.DY, HY, ks), id_mm16, !first || ks > 0);
      }
      umma::commit(&S.bar);
    }
    wait();
    first = false;
    {  // dh: quarter q writes columns 16q..16q+15 of its row
      float v[16];
      umma::tmem_ld16(TG + lanes + 16 * q, v);
      if (valid) {
        float4* dst = reinterpret_cast<float4*>(dh + row * HI + 16 * q);
#pragma unroll
        for (int j = 0; j < 4; ++j) dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      }
    }
    umma::fence_before();
    __syncthreads();  // the next tile overwrites H, A1, A2, Z, DY and the tile GEMM columns
    umma::fence_after();
  }
  if constexpr (BWD) {
    if (!first) {  // flush the TMEM accumulators (lane = the gradient's row index)
      float v[32];
      ld32(TW2 + lanes + cq, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) atomicAdd(&gW2[r * HW + cq + j], v[j]);
      ld32(TW1 + lanes + cq, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) atomicAdd(&gW1[r * HW + cq + j], v[j]);
      float u[16];
      umma::tmem_ld16(TW0 + lanes + 16 * q, u);  // dW0^T: lane = trunk unit, column = input
#pragma unroll
      for (int j = 0; j < 16; ++j) atomicAdd(&gW0[(16 * q + j) * HW + r], u[j]);
      if (q == 0) {
        umma::tmem_ld16(TWH + lanes, u);
#pragma unroll
        for (int j = 0; j < HY / 2; ++j)
          if (j < n_out) atomicAdd(&gWh[r * n_out + j], u[j]);
        umma::tmem_ld16(TB2 + lanes, u);
        atomicAdd(&gb2[r], u[HY - 1]);
      } else if (q == 1) {
        umma::tmem_ld16(TB1 + lanes, u);
        atomicAdd(&gb1[r], u[HY - 1]);
      } else if (q == 2) {
        umma::tmem_ld16(TB0 + lanes, u);
        atomicAdd(&gb0[r], u[HY - 1]);
      }
    }
    if (q == 0) {  // dbh: per-row sums of dL/dy, reduced over the warp then the CTA
#pragma unroll
      for (int j = 0; j < HY / 2; ++j) {
        float v = dbh_acc[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) atomicAdd(&S.dbh[j], v);
      }
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free(T0, 512);
  if (BWD && tid < n_out) atomicAdd(&gbh[tid], S.dbh[tid]);
}

template <bool BWD>
int launch_trunk(int64_t n, int32_t n_out, const float* h, const float* dy, const float* W0, const float* b0,
                 const float* W1, const float* b1, const float* W2, const float* b2, const float* Wh,
                 const float* bh, float* y, float* dh, float* gW0, float* gb0, float* gW1, float* gb1,
                 float* gW2, float* gb2, float* gWh, float* gbh, int32_t n_sm, void* stream) {
  if (n <= 0) return QS_OK;
  if (n_out < 1 || n_out > 8 || n_sm < 1) return QS_ERR_BAD_ARGUMENT;
  const size_t smem = sizeof(PolSmem);
  static_assert(sizeof(PolSmem) <= 227 * 1024, "shared memory");
  if (cudaFuncSetAttribute(k_policy_trunk<BWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return QS_ERR_LAUNCH;
  const int64_t ntiles = (n + TR - 1) / TR;
  const int grid = (int)(ntiles < n_sm ? ntiles : n_sm);
  k_policy_trunk<BWD><<<grid, PT, smem, (cudaStream_t)stream>>>(n, n_out, h, dy, W0, b0, W1, b1, W2, b2, Wh, bh, y,
                                                                dh, gW0, gb0, gW1, gb1, gW2, gb2, gWh, gbh);
  return cudaGetLastError() == cudaSuccess ? QS_OK : QS_ERR_LAUNCH;
}

}  // namespace

extern "C" {

int qs_policy_trunk_fwd(int64_t n, int32_t n_out, const float* h, const float* W0, const float* b0, const float* W1,
                        const float* b1, const float* W2, const float* b2, const float* Wh, const float* bh, float* y,
                        int32_t n_sm, void* stream) {
  if (!y) return QS_ERR_BAD_ARGUMENT;
  return launch_trunk<false>(n, n_out, h, nullptr, W0, b0, W1, b1, W2, b2, Wh, bh, y, nullptr, nullptr, nullptr,
                             nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, n_sm, stream);
}

int qs_policy_trunk_bwd(int64_t n, int32_t n_out, const float* h, const float* dy, const float* W0, const float* b0,
                        const float* W1, const float* b1, const float* W2, const float* b2, const float* Wh,
                        float* dh, float* gW0, float* gb0, float* gW1, float* gb1, float* gW2, float* gb2,
                        float* gWh, float* gbh, int32_t n_sm, void* stream) {
  if (!dy || !dh) return QS_ERR_BAD_ARGUMENT;
  return launch_trunk<true>(n, n_out, h, dy, W0, b0, W1, b1, W2, b2, Wh, nullptr, nullptr, dh, gW0, gb0, gW1, gb1,
                            gW2, gb2, gWh, gbh, n_sm, stream);
}

}  // extern "C"
