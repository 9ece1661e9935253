// Fused critic fit step (the caller side of config C5): one
// full-batch gradient of the privileged-state value MLP of q/nets.py:259-274
//
//     pred = tanh(tanh(x W0 + b0) W1 + b1) w2 + b2,   L = mean((pred - y)^2)
//
// (q/learners.py:232-245) over all M = T x N rows in ONE launch, on the
// tensor cores (mma.sync m16n8k16 bf16 -> fp32).  The torch version writes and
// re-reads every 128-wide activation of 2.1M rows (GBs per iteration); here a
// persistent CTA per SM keeps a 128-row tile's activations in shared memory,
// runs forward and backward on it, and accumulates the weight gradients in
// registers across all its tiles -- HBM sees only x, y and the parameters.
//
// Per tile (8 warps, warp w owns rows 16w..16w+15 for the row-parallel GEMMs):
//   G1  H1 = tanh(X W0 + b0)            (128x16 @ 16x128)
//   G2  H2 = tanh(H1 W1 + b1)           (128x128 @ 128x128), pred = H2 w2 + b2
//       dZ2 = (2/M)(pred - y) w2 (1 - H2^2)
//   G3  dZ1 = (dZ2 W1^T)(1 - H1^2)      (128x128 @ 128x128)
//   G4  dW1 += H1^T dZ2                 (warp w owns dW1 rows 16w..: 16x128, K = 128 rows)
//   G5  dW0 += X^T dZ1                  (warp w owns dW0 cols 16w..: 16x16)
// The bias gradients are column sums taken by the same MMAs with an all-ones
// A operand, and the w2 gradient dpred^T H2 by one more MMA per k-step.  Operands are bf16 in shared
// memory (row stride padded by 8 elements: conflict-free ldmatrix); the
// accumulators, biases and all gradients are fp32.
#include <cuda_bf16.h>

#include "qs_reduce.cuh"
#include "qs_umma.cuh"

namespace {

constexpr int HID = 128;       // hidden width (the reference's (128, 128))
constexpr int KIN = 16;        // input features, zero-padded (privileged state: 14)
constexpr int TILE = 128;      // rows per tile
constexpr int NWARP = 8;
constexpr int LDH = HID + 8;   // padded row strides (bf16 elements)
constexpr int LDX = KIN + 8;

struct MlpSmem {
  __nv_bfloat16 X[TILE][LDX];
  __nv_bfloat16 W0[KIN][LDH];
  __nv_bfloat16 W1[HID][LDH];
  __nv_bfloat16 H1[TILE][LDH];
  __nv_bfloat16 D2[TILE][LDH];
  __nv_bfloat16 D1[TILE][LDH];
  __nv_bfloat16 H2[TILE][LDH];
  float b0[HID], b1[HID], w2[HID];
  float dp[TILE];  // dL/dpred of the tile's rows
  float red[4];  // gb2, loss
};

QS_D uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
QS_D void ldsm4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(saddr(p)));
}
QS_D void ldsm4t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(saddr(p)));
}
QS_D void mma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
QS_D float tanh_mufu(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
QS_D uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
QS_D float2 unpack_bf16(uint32_t u) {
  __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&u);
  return __bfloat1622float2(v);
}
// ldmatrix lane addresses: lane l feeds row (l % 8) of 8x8 matrix (l / 8)
// A (16x16) from [m][k] storage: matrices (m0,k0) (m0+8,k0) (m0,k0+8) (m0+8,k0+8)
template <int LD>
QS_D const __nv_bfloat16* a_addr(const __nv_bfloat16* S, int m0, int k0, int lane) {
  const int i = lane & 7, j = lane >> 3;
  return S + (m0 + i + (j & 1) * 8) * LD + k0 + (j >> 1) * 8;
}
// A (16x16) from [k][m] storage with .trans: matrices (k0,m0) (k0,m0+8) (k0+8,m0) (k0+8,m0+8)
template <int LD>
QS_D const __nv_bfloat16* at_addr(const __nv_bfloat16* S, int m0, int k0, int lane) {
  const int i = lane & 7, j = lane >> 3;
  return S + (k0 + i + (j >> 1) * 8) * LD + m0 + (j & 1) * 8;
}
// two B (16x8) tiles n0, n0+8 from [k][n] storage with .trans:
// matrices (k0,n0) (k0+8,n0) (k0,n0+8) (k0+8,n0+8) -> b0,b1 of tile 0, b0,b1 of tile 1
template <int LD>
QS_D const __nv_bfloat16* bt_addr(const __nv_bfloat16* S, int k0, int n0, int lane) {
  const int i = lane & 7, j = lane >> 3;
  return S + (k0 + i + (j & 1) * 8) * LD + n0 + (j >> 1) * 8;
}
// two B tiles from [n][k] storage (no trans): matrices (n0,k0) (n0,k0+8) (n0+8,k0) (n0+8,k0+8)
template <int LD>
QS_D const __nv_bfloat16* bn_addr(const __nv_bfloat16* S, int k0, int n0, int lane) {
  const int i = lane & 7, j = lane >> 3;
  return S + (n0 + i + (j >> 1) * 8) * LD + k0 + (j & 1) * 8;
}

__global__ void __launch_bounds__(NWARP * 32, 1)
    k_mlp3_fit_grad(int64_t M, int K, float inv_m, const float* __restrict__ x, const float* __restrict__ scale,
                    const float* __restrict__ y, const float* __restrict__ W0, const float* __restrict__ b0,
                    const float* __restrict__ W1, const float* __restrict__ b1, const float* __restrict__ w2,
                    const float* __restrict__ b2, float* __restrict__ gW0, float* __restrict__ gb0,
                    float* __restrict__ gW1, float* __restrict__ gb1, float* __restrict__ gw2,
                    float* __restrict__ gb2, float* __restrict__ loss) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MlpSmem& S = *reinterpret_cast<MlpSmem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  // ---- stage the parameters (bf16 operands, fp32 vectors)
  for (int i = tid; i < KIN * HID; i += blockDim.x) {
    const int r = i / HID, c = i % HID;
    S.W0[r][c] = __float2bfloat16_rn(r < K ? W0[r * HID + c] : 0.f);
  }
  for (int i = tid; i < HID * HID; i += blockDim.x) S.W1[i / HID][i % HID] = __float2bfloat16_rn(W1[i]);
  for (int i = tid; i < HID; i += blockDim.x) {
    S.b0[i] = b0[i];
    S.b1[i] = b1[i];
    S.w2[i] = w2[i];
  }
  if (tid < 4) S.red[tid] = 0.f;
  const float bias2 = b2[0];
  float acc4[16][4];  // dW1 rows 16w.. x 128 cols, persistent over tiles
  float acc5[2][4];   // dW0 16 rows x cols 16w..16w+15
  float accb1[2][4];  // db1, db0 for cols 16w..16w+15 (every row of the tile holds the sums)
  float accb0[2][4];
  float accw2[2][4];  // dw2 for cols 16w..16w+15
  const uint32_t kOnes[4] = {0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u};  // bf16 1.0 pairs
#pragma unroll
  for (int j = 0; j < 16; ++j) acc4[j][0] = acc4[j][1] = acc4[j][2] = acc4[j][3] = 0.f;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    acc5[j][0] = acc5[j][1] = acc5[j][2] = acc5[j][3] = 0.f;
    accb1[j][0] = accb1[j][1] = accb1[j][2] = accb1[j][3] = 0.f;
    accb0[j][0] = accb0[j][1] = accb0[j][2] = accb0[j][3] = 0.f;
    accw2[j][0] = accw2[j][1] = accw2[j][2] = accw2[j][3] = 0.f;
  }
  __syncthreads();
  const int r0 = warp * 16;  // this warp's rows within a tile
  const int64_t ntiles = (M + TILE - 1) / TILE;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * TILE;
    // ---- X tile (scaled, zero-padded to 16 features; rows past M are zero)
    for (int i = tid; i < TILE * KIN; i += blockDim.x) {
      const int r = i / KIN, c = i % KIN;
      const int64_t gr = row0 + r;
      float v = 0.f;
      if (c < K && gr < M) v = x[gr * K + c] * scale[c];
      S.X[r][c] = __float2bfloat16_rn(v);
    }
    __syncthreads();
    // ---- G1: H1 = tanh(X W0 + b0), this warp's 16 rows
    float acc[16][4];
    {
      uint32_t a[4];
      ldsm4(a, a_addr<LDX>(&S.X[0][0], r0, 0, lane));
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        uint32_t b[4];
        ldsm4t(b, bt_addr<LDH>(&S.W0[0][0], 0, j * 8, lane));
        acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
        acc[j + 1][0] = acc[j + 1][1] = acc[j + 1][2] = acc[j + 1][3] = 0.f;
        mma(acc[j], a, b[0], b[1]);
        mma(acc[j + 1], a, b[2], b[3]);
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int c = j * 8 + 2 * t4;
        const float h00 = tanh_mufu(acc[j][0] + S.b0[c]), h01 = tanh_mufu(acc[j][1] + S.b0[c + 1]);
        const float h10 = tanh_mufu(acc[j][2] + S.b0[c]), h11 = tanh_mufu(acc[j][3] + S.b0[c + 1]);
        *reinterpret_cast<uint32_t*>(&S.H1[r0 + g][c]) = pack_bf16(h00, h01);
        *reinterpret_cast<uint32_t*>(&S.H1[r0 + g + 8][c]) = pack_bf16(h10, h11);
      }
    }
    __syncwarp();
    // ---- G2: H2 = tanh(H1 W1 + b1); pred; dZ2
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
#pragma unroll
    for (int k0 = 0; k0 < HID; k0 += 16) {
      uint32_t a[4];
      ldsm4(a, a_addr<LDH>(&S.H1[0][0], r0, k0, lane));
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        uint32_t b[4];
        ldsm4t(b, bt_addr<LDH>(&S.W1[0][0], k0, j * 8, lane));
        mma(acc[j], a, b[0], b[1]);
        mma(acc[j + 1], a, b[2], b[3]);
      }
    }
    float p0 = 0.f, p1 = 0.f;  // pred partials, rows g and g+8
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = j * 8 + 2 * t4;
      acc[j][0] = tanh_mufu(acc[j][0] + S.b1[c]);
      acc[j][1] = tanh_mufu(acc[j][1] + S.b1[c + 1]);
      acc[j][2] = tanh_mufu(acc[j][2] + S.b1[c]);
      acc[j][3] = tanh_mufu(acc[j][3] + S.b1[c + 1]);
      p0 = fmaf(acc[j][0], S.w2[c], fmaf(acc[j][1], S.w2[c + 1], p0));
      p1 = fmaf(acc[j][2], S.w2[c], fmaf(acc[j][3], S.w2[c + 1], p1));
    }
    p0 += __shfl_xor_sync(0xffffffffu, p0, 1);
    p0 += __shfl_xor_sync(0xffffffffu, p0, 2);
    p1 += __shfl_xor_sync(0xffffffffu, p1, 1);
    p1 += __shfl_xor_sync(0xffffffffu, p1, 2);
    const int64_t ra = row0 + r0 + g, rb = ra + 8;
    const float e0 = ra < M ? p0 + bias2 - y[ra] : 0.f;
    const float e1 = rb < M ? p1 + bias2 - y[rb] : 0.f;
    const float d0 = 2.f * inv_m * e0, d1 = 2.f * inv_m * e1;  // dL/dpred
    float lsum = t4 == 0 ? e0 * e0 + e1 * e1 : 0.f, gb2s = t4 == 0 ? d0 + d1 : 0.f;
    if (t4 == 0) {
      S.dp[r0 + g] = d0;
      S.dp[r0 + g + 8] = d1;
    }
    // H2 -> smem (for dw2 = H2^T dpred in G4); dZ2 -> D2
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = j * 8 + 2 * t4;
      *reinterpret_cast<uint32_t*>(&S.H2[r0 + g][c]) = pack_bf16(acc[j][0], acc[j][1]);
      *reinterpret_cast<uint32_t*>(&S.H2[r0 + g + 8][c]) = pack_bf16(acc[j][2], acc[j][3]);
      const float z00 = d0 * S.w2[c] * (1.f - acc[j][0] * acc[j][0]);
      const float z01 = d0 * S.w2[c + 1] * (1.f - acc[j][1] * acc[j][1]);
      const float z10 = d1 * S.w2[c] * (1.f - acc[j][2] * acc[j][2]);
      const float z11 = d1 * S.w2[c + 1] * (1.f - acc[j][3] * acc[j][3]);
      *reinterpret_cast<uint32_t*>(&S.D2[r0 + g][c]) = pack_bf16(z00, z01);
      *reinterpret_cast<uint32_t*>(&S.D2[r0 + g + 8][c]) = pack_bf16(z10, z11);
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
      gb2s += __shfl_xor_sync(0xffffffffu, gb2s, o);
    }
    if (lane == 0) {
      atomicAdd(&S.red[0], gb2s);
      atomicAdd(&S.red[1], lsum);
    }
    __syncwarp();
    // ---- G3: dZ1 = (dZ2 W1^T)(1 - H1^2) -> D1; db0 partials
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
#pragma unroll
    for (int k0 = 0; k0 < HID; k0 += 16) {
      uint32_t a[4];
      ldsm4(a, a_addr<LDH>(&S.D2[0][0], r0, k0, lane));
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        uint32_t b[4];
        ldsm4(b, bn_addr<LDH>(&S.W1[0][0], k0, j * 8, lane));  // W1^T: B(k=o, n=i) = W1[i][o]
        mma(acc[j], a, b[0], b[1]);
        mma(acc[j + 1], a, b[2], b[3]);
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = j * 8 + 2 * t4;
      const float2 h0 = unpack_bf16(*reinterpret_cast<const uint32_t*>(&S.H1[r0 + g][c]));
      const float2 h1 = unpack_bf16(*reinterpret_cast<const uint32_t*>(&S.H1[r0 + g + 8][c]));
      const float z00 = acc[j][0] * (1.f - h0.x * h0.x), z01 = acc[j][1] * (1.f - h0.y * h0.y);
      const float z10 = acc[j][2] * (1.f - h1.x * h1.x), z11 = acc[j][3] * (1.f - h1.y * h1.y);
      *reinterpret_cast<uint32_t*>(&S.D1[r0 + g][c]) = pack_bf16(z00, z01);
      *reinterpret_cast<uint32_t*>(&S.D1[r0 + g + 8][c]) = pack_bf16(z10, z11);
    }
    __syncthreads();  // H1, D2, D1, X of every row are in shared memory
    // ---- G4: dW1[16w.., :] += H1^T dZ2 (K = the tile's 128 rows)
#pragma unroll
    for (int k0 = 0; k0 < TILE; k0 += 16) {
      uint32_t a[4];
      ldsm4t(a, at_addr<LDH>(&S.H1[0][0], r0, k0, lane));
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        uint32_t b[4];
        ldsm4t(b, bt_addr<LDH>(&S.D2[0][0], k0, j * 8, lane));
        mma(acc4[j], a, b[0], b[1]);
        mma(acc4[j + 1], a, b[2], b[3]);
        if (j == 2 * warp) {  // db1 = 1^T dZ2: an all-ones A on the same fragments
          mma(accb1[0], kOnes, b[0], b[1]);
          mma(accb1[1], kOnes, b[2], b[3]);
        }
      }
      // dw2 = dpred^T H2 for this warp's columns: A rows all = dpred (k = rows)
      uint32_t ad[4], bh[4];
      const uint32_t lo = pack_bf16(S.dp[k0 + 2 * t4], S.dp[k0 + 2 * t4 + 1]);
      const uint32_t hi = pack_bf16(S.dp[k0 + 8 + 2 * t4], S.dp[k0 + 9 + 2 * t4]);
      ad[0] = ad[1] = lo;
      ad[2] = ad[3] = hi;
      ldsm4t(bh, bt_addr<LDH>(&S.H2[0][0], k0, r0, lane));
      mma(accw2[0], ad, bh[0], bh[1]);
      mma(accw2[1], ad, bh[2], bh[3]);
    }
    // ---- G5: dW0[:, 16w..16w+15] += X^T dZ1
#pragma unroll
    for (int k0 = 0; k0 < TILE; k0 += 16) {
      uint32_t a[4], b[4];
      ldsm4t(a, at_addr<LDX>(&S.X[0][0], 0, k0, lane));
      ldsm4t(b, bt_addr<LDH>(&S.D1[0][0], k0, r0, lane));
      mma(acc5[0], a, b[0], b[1]);
      mma(acc5[1], a, b[2], b[3]);
      mma(accb0[0], kOnes, b[0], b[1]);  // db0 = 1^T dZ1 on the same fragments
      mma(accb0[1], kOnes, b[2], b[3]);
    }
    __syncthreads();  // the next tile overwrites X, H1, D2, D1
  }
  // ---- flush: register / shared partials into the global fp32 gradients
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int c = j * 8 + 2 * t4;
    atomicAdd(&gW1[(r0 + g) * HID + c], acc4[j][0]);
    atomicAdd(&gW1[(r0 + g) * HID + c + 1], acc4[j][1]);
    atomicAdd(&gW1[(r0 + g + 8) * HID + c], acc4[j][2]);
    atomicAdd(&gW1[(r0 + g + 8) * HID + c + 1], acc4[j][3]);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int c = r0 + j * 8 + 2 * t4;
    if (g < K) {
      atomicAdd(&gW0[g * HID + c], acc5[j][0]);
      atomicAdd(&gW0[g * HID + c + 1], acc5[j][1]);
    }
    if (g + 8 < K) {
      atomicAdd(&gW0[(g + 8) * HID + c], acc5[j][2]);
      atomicAdd(&gW0[(g + 8) * HID + c + 1], acc5[j][3]);
    }
  }
  if (g == 0) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int c = r0 + j * 8 + 2 * t4;
      atomicAdd(&gb1[c], accb1[j][0]);
      atomicAdd(&gb1[c + 1], accb1[j][1]);
      atomicAdd(&gb0[c], accb0[j][0]);
      atomicAdd(&gb0[c + 1], accb0[j][1]);
      atomicAdd(&gw2[c], accw2[j][0]);
      atomicAdd(&gw2[c + 1], accw2[j][1]);
    }
  }
  __syncthreads();
  if (tid == 0) {
    atomicAdd(gb2, S.red[0]);
    atomicAdd(loss, S.red[1] * inv_m);
  }
}

// ---------------------------------------------------------------------------
// The same fit step on the 5th-generation tensor cores (tcgen05).  One
// persistent 512-thread CTA per SM walks 128-row tiles; thread (warp w, lane
// l) owns row 32 (w % 4) + l of a tile -- its TMEM lane -- and columns
// 32 (w / 4) .. + 31 of every 128-wide activation.  Operands live in shared memory in the blocked
// no-swizzle layout of qs_umma.cuh, so every activation tile is written once
// and read by the MMAs both as a K-major operand (next layer) and as an
// MN-major one (weight gradients, K = the tile's rows).  Accumulators live in
// TMEM (512 columns):
//   [0,256)   G1 / G2 / G3 results of the tiles in slots 0 and 1 (reused in turn)
//   [256,384) dW1 = sum over tiles of H1^T dZ2          (lane = hid1 row)
//   [384,400) dW0^T | db0 = dZ1^T X                     (lane = hid1; col 15 = db0)
//   [400,416) db1 = dZ2^T X, column 15                  (lane = hid2)
// Tiles run in pairs through two operand slots: while the epilogue threads
// work on one slot's tile, the tensor cores run the other slot's GEMMs; the
// next pair's x / y rows stream into the slots with cp.async meanwhile.
// X's padding column 15 is all ones, so the bias gradients are column sums
// taken by the same MMAs; dw2 = dpred^T H2 is accumulated in fp32 registers
// by the epilogue threads (each owns 32 columns).  K <= 14 input features
// (the privileged state has 14).
// Per tile, one thread issues: G1 (X W0), G2 (H1 W1), then G3 (dZ2 W1^T), G4
// (H1^T dZ2), db1, then G5 (dZ1^T X); tcgen05.commit -> mbarrier hands each
// group to the 128 epilogue threads (TMEM -> registers -> bias / tanh / chain
// rule -> bf16 -> shared memory).

constexpr int TC_THREADS = 512;  // 16 warps: warp w reads TMEM lanes 32 (w % 4).., columns 32 (w / 4)..
constexpr int TC_KMAX = 14;
constexpr int TC_QC = HID / 4;   // columns per thread (a quarter of a row)

// one tile's operands; two slots let the tensor cores run one tile's GEMMs
// while the epilogue threads work on the other's
struct TcSlot {
  __nv_bfloat16 X[TILE * KIN];     // [rows][16]   blocked
  __nv_bfloat16 H1[TILE * HID];    // [rows][hid1]  H1, then dZ1 in place (epilogue 3)
  __nv_bfloat16 D2[TILE * HID];    // [rows][hid2]  dZ2
  float predq[4][TILE];            // per-quarter partial dot products H2 . w2
  // raw fp32 rows of the NEXT pair's tile for this slot, prefetched with
  // cp.async while the current pair computes (x: 128 rows x K floats, y)
  float xraw[TILE * TC_KMAX];
  float yraw[TILE];
};
struct TcSmem {
  TcSlot slot[2];
  __nv_bfloat16 W0T[HID * KIN];    // [hid1][16]   blocked (K-major B of G1)
  __nv_bfloat16 W1T[HID * HID];    // [hid2][hid1] blocked (K-major B of G2, MN-major B of G3)
  float b0[HID], b1[HID], w2[HID];
  float red[2];                    // db2, loss
  float w2p[4][HID];               // dw2 per row quarter (warp % 4)
  float redp[4][2];                // db2, loss per row quarter
  uint64_t bar[2];
  uint32_t tbase;
};
// per-CTA gradient partials of the tcgen05 fit (qs_reduce.cuh)
constexpr int64_t CK_W1 = 0, CK_W0 = CK_W1 + HID * HID, CK_B0 = CK_W0 + 16 * HID, CK_B1 = CK_B0 + HID,
                  CK_W2 = CK_B1 + HID, CK_B2 = CK_W2 + HID, CK_L = CK_B2 + 1,
                  CK_P = (CK_L + 1 + 31) / 32 * 32;  // rows 128-byte aligned (float4 stores)

// 32 consecutive columns of this thread's TMEM lane
QS_D void tmem_ld32(uint32_t t, float (&v)[32]) { umma::tmem_ld32(t, v); }
// tanh of a bf16 pair (MUFU, one op for two values): torch's bf16 autocast
// rounds the linear layer's output to bf16 before its tanh, so does this
QS_D uint32_t tanh_bf16x2(uint32_t x) {
  uint32_t y;
  asm("tanh.approx.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
// 8 bf16 pairs -> one 16-byte store at (row, c0) of a blocked [rows][HID] buffer
QS_D void st_row8(__nv_bfloat16* buf, int row, int c0, const uint32_t* w) {
  *reinterpret_cast<uint4*>(&buf[umma::blk_off(row, c0, HID)]) = make_uint4(w[0], w[1], w[2], w[3]);
}

// FWD: forward only -- pred (the value) of every row into `pred_out`, no
// backward GEMMs (the TD-lambda targets' values and bootstrap, q/learners.py:286-292)
template <bool FWD>
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_mlp3_fit_grad_tc(int64_t M, int K, float inv_m, const float* __restrict__ x, const float* __restrict__ scale,
                       const float* __restrict__ y, const float* __restrict__ W0, const float* __restrict__ b0,
                       const float* __restrict__ W1, const float* __restrict__ b1, const float* __restrict__ w2,
                       const float* __restrict__ b2, float* __restrict__ gW0, float* __restrict__ gb0,
                       float* __restrict__ gW1, float* __restrict__ gb1, float* __restrict__ gw2,
                       float* __restrict__ gb2, float* __restrict__ loss, float* __restrict__ pred_out,
                       float* __restrict__ work) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  TcSmem& S = *reinterpret_cast<TcSmem*>(smem_raw);
  using umma::blk_off;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = 32 * (warp & 3) + lane;  // this thread's tile row == TMEM lane
  const int q = warp >> 2;               // its column quarter
  const int cq = q * TC_QC;
  // ---- parameters -> shared memory (bf16 operands, fp32 vectors)
  for (int i = tid; i < HID * KIN; i += TC_THREADS) {
    const int n = i / KIN, k = i % KIN;  // W0T[n][k] = W0[k][n]; column 15 = b0 (X's ones column adds it)
    S.W0T[blk_off(n, k, KIN)] = __float2bfloat16_rn(k < K ? W0[k * HID + n] : k == KIN - 1 ? b0[n] : 0.f);
  }
  for (int i = tid; i < HID * HID; i += TC_THREADS) {
    const int k = i / HID, n = i % HID;  // W1[k][n] -> W1T[n][k]
    S.W1T[blk_off(n, k, HID)] = __float2bfloat16_rn(W1[i]);
  }
  for (int i = tid; i < HID; i += TC_THREADS) {
    S.b0[i] = b0[i];
    S.b1[i] = b1[i];
    S.w2[i] = w2[i];
  }
  if (tid < 2) S.red[tid] = 0.f;
  if (warp == 0) umma::tmem_alloc(&S.tbase, 512);
  if (tid == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    fence_barrier_init();
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t T0 = S.tbase;
  // TMEM: G accumulator per slot [0,128) [128,256); dW1 [256,384); dW0^T|db0 [384,400); db1 [400,416)
  const uint32_t T_W1 = T0 + 256, T_W0 = T0 + 384, T_B1 = T0 + 400;
  const uint32_t id_128 = umma::idesc_bf16(128, 128, false, false);
  const uint32_t id_128_bmn = umma::idesc_bf16(128, 128, false, true);
  const uint32_t id_128_mn = umma::idesc_bf16(128, 128, true, true);
  const uint32_t id_16_mn = umma::idesc_bf16(128, 16, true, true);
  const uint32_t my = umma::taddr(0, 32 * (warp & 3), cq);  // this thread's lanes / columns
  const float bias2 = b2[0];
  uint32_t phase[2] = {0u, 0u};
  bool first = true;   // no dW1 / db1 MMA issued yet (the first one overwrites TMEM)
  bool first5 = true;  // no dW0 / db0 MMA issued yet
  float gb2_acc = 0.f, loss_acc = 0.f;
  float gw2p[32];  // this thread's columns of dw2, summed over its rows
#pragma unroll
  for (int j = 0; j < 32; ++j) gw2p[j] = 0.f;
  auto sync_to_mma = [&]() {  // epilogue writes -> visible to the tensor cores, then hand over
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
  };
  auto wait_mma = [&](int sl) {
    umma::mbar_wait_parity(&S.bar[sl], phase[sl]);
    phase[sl] ^= 1u;
    umma::fence_after();
  };
  // ---- the phases of one tile in slot sl
  // the tile's raw x / y rows -> slot staging (contiguous blocks, 16-byte
  // cp.async chunks; the tail tile's bytes past row M are zero-filled)
  auto prefetch = [&](int sl, int64_t tile) {
    if (tile >= (M + TILE - 1) / TILE) return;
    const int64_t r0 = tile * TILE;
    const int64_t nrows = M - r0 < TILE ? M - r0 : TILE;
    const char* xs = reinterpret_cast<const char*>(x + r0 * K);
    char* xd = reinterpret_cast<char*>(S.slot[sl].xraw);
    const int xbytes = (int)(nrows * K * 4), xcap = TILE * K * 4;
    for (int b = tid * 16; b < xcap; b += TC_THREADS * 16) {
      const int n = xbytes - b >= 16 ? 16 : (xbytes > b ? xbytes - b : 0);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(xd + b)), "l"(xs + (n ? b : 0)),
                   "r"(n)
                   : "memory");
    }
    const char* ys = reinterpret_cast<const char*>(y + r0);
    char* yd = reinterpret_cast<char*>(S.slot[sl].yraw);
    const int ybytes = (int)(nrows * 4);
    if (!FWD && tid * 16 < TILE * 4) {
      const int b = tid * 16, n = ybytes - b >= 16 ? 16 : (ybytes > b ? ybytes - b : 0);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(yd + b)), "l"(ys + (n ? b : 0)),
                   "r"(n)
                   : "memory");
    }
  };
  auto stage_x = [&](int sl, int64_t tile) {  // quarter q stages columns 4q..4q+3 of its row
    const int64_t row = tile * TILE + r;
    float v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = 4 * q + j;
      v[j] = (row < M && c < K) ? S.slot[sl].xraw[r * K + c] * __ldg(scale + c) : (c == KIN - 1 ? 1.f : 0.f);
    }  // column 15: ones (the bias / bias-gradient column)
    *reinterpret_cast<uint2*>(&S.slot[sl].X[blk_off(r, 4 * q, KIN)]) =
        make_uint2(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]));
  };
  auto issue_g1 = [&](int sl) {  // X W0
    TcSlot& T = S.slot[sl];
    umma::mma_bf16(T0 + 128 * sl, umma::desc_kmajor(T.X, KIN), umma::desc_kmajor(S.W0T, KIN), id_128, false);
    umma::commit(&S.bar[sl]);
  };
  auto issue_g2 = [&](int sl) {  // H1 W1
    TcSlot& T = S.slot[sl];
#pragma unroll
    for (int ks = 0; ks < HID / 16; ++ks)
      umma::mma_bf16(T0 + 128 * sl, umma::desc_kmajor(T.H1 + ks * 128, HID), umma::desc_kmajor(S.W1T + ks * 128, HID),
                     id_128, ks > 0);
    umma::commit(&S.bar[sl]);
  };
  auto issue_g34 = [&](int sl) {  // dZ2 W1^T;  dW1 += H1^T dZ2;  db1 += dZ2^T 1
    TcSlot& T = S.slot[sl];
#pragma unroll
    for (int ks = 0; ks < HID / 16; ++ks)
      umma::mma_bf16(T0 + 128 * sl, umma::desc_kmajor(T.D2 + ks * 128, HID),
                     umma::desc_mnmajor(S.W1T + ks * 2048, HID), id_128_bmn, ks > 0);
#pragma unroll
    for (int ks = 0; ks < TILE / 16; ++ks) {
      const bool acc = !first || ks > 0;
      umma::mma_bf16(T_W1, umma::desc_mnmajor(T.H1 + ks * 2048, HID), umma::desc_mnmajor(T.D2 + ks * 2048, HID),
                     id_128_mn, acc);
      umma::mma_bf16(T_B1, umma::desc_mnmajor(T.D2 + ks * 2048, HID), umma::desc_mnmajor(T.X + ks * 256, KIN),
                     id_16_mn, acc);
    }
    umma::commit(&S.bar[sl]);
  };
  auto issue_g5 = [&](int sl) {  // dW0^T | db0 += dZ1^T X
    TcSlot& T = S.slot[sl];
#pragma unroll
    for (int ks = 0; ks < TILE / 16; ++ks)
      umma::mma_bf16(T_W0, umma::desc_mnmajor(T.H1 + ks * 2048, HID), umma::desc_mnmajor(T.X + ks * 256, KIN),
                     id_16_mn, !first5 || ks > 0);
    umma::commit(&S.bar[sl]);
  };
  auto epi1 = [&](int sl) {  // H1 = tanh(X W0 + b0) (b0 entered through X's ones column)
    float v[32];
    tmem_ld32(T0 + 128 * sl + my, v);
    uint32_t w[16];
#pragma unroll
    for (int j = 0; j < 32; j += 2) w[j / 2] = tanh_bf16x2(pack_bf16(v[j], v[j + 1]));
#pragma unroll
    for (int j = 0; j < 4; ++j) st_row8(S.slot[sl].H1, r, cq + 8 * j, w + 4 * j);
  };
  auto epi2 = [&](int sl, int64_t tile) {  // H2, pred, dL/dpred, dZ2 = dpred w2 (1 - H2^2), dw2
    TcSlot& T = S.slot[sl];
    float h[32];
    tmem_ld32(T0 + 128 * sl + my, h);
    float part = 0.f;
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      const float2 t = unpack_bf16(tanh_bf16x2(pack_bf16(h[j] + S.b1[cq + j], h[j + 1] + S.b1[cq + j + 1])));
      h[j] = t.x;
      h[j + 1] = t.y;
      part = fmaf(h[j], S.w2[cq + j], fmaf(h[j + 1], S.w2[cq + j + 1], part));
    }
    T.predq[q][r] = part;
    // only the four warps sharing these rows (warp % 4) exchange partials
    asm volatile("bar.sync %0, 128;" ::"r"(1 + (warp & 3)) : "memory");
    const int64_t row = tile * TILE + r;
    const float pred = bias2 + T.predq[0][r] + T.predq[1][r] + T.predq[2][r] + T.predq[3][r];
    if constexpr (FWD) {
      if (q == 0 && row < M) pred_out[row] = pred;
      return;
    }
    const float e = row < M ? pred - T.yraw[r] : 0.f;
    const float dp = 2.f * inv_m * e;
    if (q == 0) {
      loss_acc += e * e;
      gb2_acc += dp;
    }
    uint32_t w[16];
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      gw2p[j] = fmaf(dp, h[j], gw2p[j]);  // dw2 = dpred^T H2, fp32 in registers
      gw2p[j + 1] = fmaf(dp, h[j + 1], gw2p[j + 1]);
      w[j / 2] = pack_bf16(dp * S.w2[cq + j] * (1.f - h[j] * h[j]), dp * S.w2[cq + j + 1] * (1.f - h[j + 1] * h[j + 1]));
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) st_row8(T.D2, r, cq + 8 * j, w + 4 * j);
  };
  auto epi3 = [&](int sl) {  // dZ1 = (dZ2 W1^T)(1 - H1^2), in place over H1
    TcSlot& T = S.slot[sl];
    float v[32];
    tmem_ld32(T0 + 128 * sl + my, v);
    uint32_t w[16];
#pragma unroll
    for (int j8 = 0; j8 < 32; j8 += 8) {
      const uint4 hh = *reinterpret_cast<const uint4*>(&T.H1[blk_off(r, cq + j8, HID)]);
      const uint32_t hw[4] = {hh.x, hh.y, hh.z, hh.w};
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        const float2 hv = unpack_bf16(hw[j / 2]);
        w[(j8 + j) / 2] = pack_bf16(v[j8 + j] * (1.f - hv.x * hv.x), v[j8 + j + 1] * (1.f - hv.y * hv.y));
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) st_row8(T.H1, r, cq + 8 * j, w + 4 * j);
  };
  // ---- tiles in pairs (slot 0, slot 1): each epilogue overlaps the other
  //      slot's GEMMs on the tensor cores
  const int64_t ntiles = (M + TILE - 1) / TILE;
  prefetch(0, blockIdx.x);
  prefetch(1, blockIdx.x + gridDim.x);
  cp_async_commit();
  for (int64_t ta = blockIdx.x; ta < ntiles; ta += 2 * (int64_t)gridDim.x) {
    const int64_t tb = ta + gridDim.x;
    const bool two = tb < ntiles;
    cp_async_wait<0>();
    __syncthreads();  // this pair's raw rows have landed
    stage_x(0, ta);
    if (two) stage_x(1, tb);
    sync_to_mma();
    if (tid == 0) {
      issue_g1(0);
      if (two) issue_g1(1);
    }
    wait_mma(0);
    epi1(0);
    sync_to_mma();
    if (tid == 0) issue_g2(0);
    if (two) {
      wait_mma(1);
      epi1(1);
      sync_to_mma();
      if (tid == 0) issue_g2(1);
    }
    if constexpr (FWD) {
      wait_mma(0);
      epi2(0, ta);
      if (two) {
        wait_mma(1);
        epi2(1, tb);
      }
      __syncthreads();  // every thread is past this pair's slot reads
      prefetch(0, ta + 2 * (int64_t)gridDim.x);
      prefetch(1, tb + 2 * (int64_t)gridDim.x);
      cp_async_commit();
      continue;
    }
    wait_mma(0);
    epi2(0, ta);
    sync_to_mma();  // (also: every thread is past its reads of this pair's xraw / yraw)
    if (tid == 0) issue_g34(0);
    first = false;
    if (two) {
      wait_mma(1);
      epi2(1, tb);
      sync_to_mma();
      if (tid == 0) issue_g34(1);
    }
    prefetch(0, ta + 2 * (int64_t)gridDim.x);  // the next pair's rows, behind this pair's GEMMs
    prefetch(1, tb + 2 * (int64_t)gridDim.x);
    cp_async_commit();
    wait_mma(0);
    epi3(0);
    sync_to_mma();
    if (tid == 0) issue_g5(0);
    first5 = false;
    if (two) {
      wait_mma(1);
      epi3(1);
      sync_to_mma();
      if (tid == 0) issue_g5(1);
    }
    wait_mma(0);  // both slots' buffers are free for the next pair
    if (two) wait_mma(1);
  }
  cp_async_wait<0>();
  if constexpr (FWD) {
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_free(T0, 512);
    return;
  }
  // ---- this CTA's partial gradients (TMEM lane = hid row) -> work; summed
  // over the CTAs in a fixed order by red::sum_partials
  float* wk = work + (int64_t)blockIdx.x * CK_P;
  {
    float v[32];
    if (!first) {
      tmem_ld32(T_W1 + my, v);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < 32; j += 4)
      *reinterpret_cast<float4*>(wk + CK_W1 + r * HID + cq + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    if (q < 2) {
      float u[16];
      if (!first) {
        umma::tmem_ld16(umma::taddr(q == 0 ? T_W0 : T_B1, 32 * (warp & 3), 0), u);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) u[j] = 0.f;
      }
      if (q == 0) {
#pragma unroll
        for (int k = 0; k < TC_KMAX; ++k)
          if (k < K) wk[CK_W0 + k * HID + r] = u[k];
        wk[CK_B0 + r] = u[KIN - 1];
      } else {
        wk[CK_B1 + r] = u[KIN - 1];
      }
    }
  }
  // dw2: each column reduced over the warp's 32 rows, then over the 4 row quarters in order
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    float v = gw2p[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == j) S.w2p[warp & 3][cq + j] = v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    gb2_acc += __shfl_xor_sync(0xffffffffu, gb2_acc, o);
    loss_acc += __shfl_xor_sync(0xffffffffu, loss_acc, o);
  }
  if (lane == 0 && q == 0) {
    S.redp[warp & 3][0] = gb2_acc;
    S.redp[warp & 3][1] = loss_acc;
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free(T0, 512);
  if (tid < HID) wk[CK_W2 + tid] = (S.w2p[0][tid] + S.w2p[1][tid]) + (S.w2p[2][tid] + S.w2p[3][tid]);
  if (tid == 0) {
    wk[CK_B2] = (S.redp[0][0] + S.redp[1][0]) + (S.redp[2][0] + S.redp[3][0]);
    wk[CK_L] = ((S.redp[0][1] + S.redp[1][1]) + (S.redp[2][1] + S.redp[3][1])) * inv_m;
  }
}

}  // namespace

extern "C" {

int64_t qs_mlp3_work_floats(int32_t n_sm) { return n_sm < 1 ? -1 : (int64_t)n_sm * CK_P; }

int qs_mlp3_fit_grad_tc(int64_t m, int32_t k, const float* x, const float* scale, const float* y, const float* W0,
                        const float* b0, const float* W1, const float* b1, const float* w2, const float* b2,
                        float* gW0, float* gb0, float* gW1, float* gb1, float* gw2, float* gb2, float* loss,
                        float* work, int64_t work_floats, int32_t n_sm, void* stream) {
  if (m <= 0) return QS_OK;
  if (k < 1 || k > TC_KMAX || n_sm < 1) return QS_ERR_BAD_ARGUMENT;
  if (!work || work_floats < (int64_t)n_sm * CK_P) return QS_ERR_BAD_ARGUMENT;
  const size_t smem = sizeof(TcSmem);
  static_assert(sizeof(TcSmem) <= 227 * 1024, "shared memory");
  if (cudaFuncSetAttribute(k_mlp3_fit_grad_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return QS_ERR_LAUNCH;
  const int64_t ntiles = (m + TILE - 1) / TILE;
  const int grid = (int)(ntiles < n_sm ? ntiles : n_sm);
  k_mlp3_fit_grad_tc<false><<<grid, TC_THREADS, smem, (cudaStream_t)stream>>>(
      m, k, 1.f / (float)m, x, scale, y, W0, b0, W1, b1, w2, b2, gW0, gb0, gW1, gb1, gw2, gb2, loss, nullptr, work);
  if (cudaGetLastError() != cudaSuccess) return QS_ERR_LAUNCH;
  red::Segs sg{{gW1, gW0, gb0, gb1, gw2, gb2, loss},
               {CK_W1, CK_W0, CK_B0, CK_B1, CK_W2, CK_B2, CK_L},
               {HID * HID, (int64_t)k * HID, HID, HID, HID, 1, 1},
               7,
               true};
  return red::sum_partials(work, grid, CK_P, sg, (cudaStream_t)stream);
}

int qs_mlp3_forward_tc(int64_t m, int32_t k, const float* x, const float* scale, const float* W0, const float* b0,
                       const float* W1, const float* b1, const float* w2, const float* b2, float* pred,
                       int32_t n_sm, void* stream) {
  if (m <= 0) return QS_OK;
  if (k < 1 || k > TC_KMAX || n_sm < 1 || !pred) return QS_ERR_BAD_ARGUMENT;
  const size_t smem = sizeof(TcSmem);
  if (cudaFuncSetAttribute(k_mlp3_fit_grad_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return QS_ERR_LAUNCH;
  const int64_t ntiles = (m + TILE - 1) / TILE;
  const int grid = (int)(ntiles < n_sm ? ntiles : n_sm);
  k_mlp3_fit_grad_tc<true><<<grid, TC_THREADS, smem, (cudaStream_t)stream>>>(
      m, k, 1.f, x, scale, nullptr, W0, b0, W1, b1, w2, b2, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
      nullptr, pred, nullptr);
  return cudaGetLastError() == cudaSuccess ? QS_OK : QS_ERR_LAUNCH;
}

int qs_mlp3_fit_grad(int64_t m, int32_t k, const float* x, const float* scale, const float* y, const float* W0,
                     const float* b0, const float* W1, const float* b1, const float* w2, const float* b2,
                     float* gW0, float* gb0, float* gW1, float* gb1, float* gw2, float* gb2, float* loss,
                     int32_t n_sm, void* stream) {
  if (m <= 0) return QS_OK;
  if (k < 1 || k > KIN || n_sm < 1) return QS_ERR_BAD_ARGUMENT;
  const size_t smem = sizeof(MlpSmem);
  static_assert(sizeof(MlpSmem) <= 227 * 1024, "shared memory");
  if (cudaFuncSetAttribute(k_mlp3_fit_grad, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return QS_ERR_LAUNCH;
  const int64_t ntiles = (m + TILE - 1) / TILE;
  const int grid = (int)(ntiles < n_sm ? ntiles : n_sm);
  k_mlp3_fit_grad<<<grid, NWARP * 32, smem, (cudaStream_t)stream>>>(m, k, 1.f / (float)m, x, scale, y, W0, b0, W1,
                                                                     b1, w2, b2, gW0, gb0, gW1, gb1, gw2, gb2,
                                                                     loss);
  return cudaGetLastError() == cudaSuccess ? QS_OK : QS_ERR_LAUNCH;
}

}  // extern "C"
