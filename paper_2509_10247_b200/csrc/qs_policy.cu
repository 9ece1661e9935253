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
//   qs_policy_gru_fwd    the GRU cell (q/nets.py:107-132, gates r, z, n) fused
//                        in front of the trunk: h' and y from (x, h) in one pass
//                        (k_policy_fwd2: two 8-warp groups, two tiles in flight)
//   qs_policy_gru_bwd    the GRU cell's backward: recompute the gates, return
//                        dL/dx and dL/dh for dL/dh' (trunk + carried), and
//                        accumulate dWi, dWh, dbi, dbh in TMEM.
//   qs_policy_pack_image the weights as one bf16 operand image every CTA stages
//                        with bulk copies.
// Same machinery as the critic fit (qs_mlp.cu / qs_umma.cuh): one persistent
// 512-thread CTA per SM; thread (warp w, lane l) owns tile row 32 (w % 4) + l
// -- its TMEM lane -- and a slice of the columns; one elected thread issues
// tcgen05.mma (bf16 operands in the blocked no-swizzle layout, fp32
// accumulators in TMEM) and commits to an mbarrier; every weight matrix is
// staged once and serves as a K-major operand one way and MN-major the other.
// Weight gradients leave as per-CTA partials summed in a fixed order
// (qs_reduce.cuh): bitwise reproducible.
#include "qs_reduce.cuh"
#include "qs_umma.cuh"

namespace {

constexpr int PT = 512;     // threads
constexpr int TR = 128;     // rows per tile
constexpr int HI = 64;      // GRU width (trunk input)
constexpr int HW = 128;     // trunk width
constexpr int HY = 16;      // head outputs, padded (mu | log sigma | 0 | ones column for bias sums)
constexpr int XI = 16;      // GRU input width, padded (proprio features)
constexpr int G3 = 3 * HI;  // GRU gate columns (r | z | n)
// logistic sigmoid as 0.5 tanh(x / 2) + 0.5: one MUFU op (an IEEE 1 / (1 + e^-x)
// is a multi-instruction software divide: it was a third of the policy
// kernels' instructions)
QS_D float tanh_f(float x);
QS_D float sigm_f(float x) { return fmaf(0.5f, tanh_f(0.5f * x), 0.5f); }
// tanh of a bf16 pair in one MUFU op; the trunk's activations are bf16 (and
// torch's bf16 autocast rounds the linear output to bf16 before its tanh)
QS_D uint32_t tanh_bf16x2(uint32_t x) {
  uint32_t y;
  asm("tanh.approx.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
// per-CTA gradient partials (qs_reduce.cuh): the trunk backward's layout
constexpr int64_t TK_W0 = 0, TK_B0 = TK_W0 + HI * HW, TK_W1 = TK_B0 + HW, TK_B1 = TK_W1 + HW * HW,
                  TK_W2 = TK_B1 + HW, TK_B2 = TK_W2 + HW * HW, TK_WH = TK_B2 + HW, TK_BH = TK_WH + HW * 8,
                  TK_P = (TK_BH + 8 + 31) / 32 * 32;
// ... and the GRU backward's
constexpr int64_t GK_WI = 0, GK_BI = GK_WI + XI * G3, GK_WG = GK_BI + G3, GK_BG = GK_WG + HI * G3,
                  GK_P = (GK_BG + G3 + 31) / 32 * 32;
// the bf16 weight image (qs_policy_pack_image): W0 | W1 | W2 | WH | WI | WG, each
// in the blocked operand layout -- byte for byte the kernels' shared-memory
// weight section, so a CTA stages it with bulk copies instead of converting
constexpr int IMG_W0 = 0, IMG_W1 = IMG_W0 + HI * HW, IMG_W2 = IMG_W1 + HW * HW, IMG_WH = IMG_W2 + HW * HW,
              IMG_WI = IMG_WH + HW * HY, IMG_WG = IMG_WI + XI * G3, IMG_N = IMG_WG + HI * G3;  // bf16 elements
// one thread: bulk-copy `bytes` of the image (from element `off`) to smem, in <= 32 KB pieces
QS_D void load_image(void* dst, const __nv_bfloat16* img, int off, int elems, uint64_t* bar) {
  const uint32_t bytes = (uint32_t)elems * 2u;
  tma_expect(bar, bytes);
  const char* src = reinterpret_cast<const char*>(img + off);
  char* d = reinterpret_cast<char*>(dst);
  for (uint32_t o = 0; o < bytes; o += 32768u)
    tma_copy_1d(d + o, src + o, bytes - o < 32768u ? bytes - o : 32768u, bar);
}

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

// fp32 row-major [rows][COLS] (rows >= valid read as 0) -> bf16 blocked [rows][COLS]:
// 16-byte loads, four in flight per thread before any conversion
template <int COLS>
QS_D void stage_w(const float* __restrict__ src, int rows, int valid, __nv_bfloat16* dst, int tid) {
  constexpr int C4 = COLS / 4;
  const int total = rows * C4;
  for (int i0 = tid; i0 < total; i0 += 4 * PT) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * PT, rr = i / C4;
      v[u] = (i < total && rr < valid) ? __ldg(reinterpret_cast<const float4*>(src) + i)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * PT;
      if (i < total)
        *reinterpret_cast<uint2*>(&dst[umma::blk_off(i / C4, (i % C4) * 4, COLS)]) =
            make_uint2(pk(v[u].x, v[u].y), pk(v[u].z, v[u].w));
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
  __nv_bfloat16 Z[TR * HW];    // z, then (backward) dL/dz-pre in place
  __nv_bfloat16 DY[TR * HY];   // dL/dy (8 columns), column 15 = 1
  float b0[HW], b1[HW], b2[HW], bh[HY];
  float dbh[4][HY];             // per-warp dL/dbh sums (warps 0-3)
  uint64_t bar, wbar;
  uint32_t tbase;
};

// head output j of row `row` in y: row-major (n, n_out), or planar (2, n, n_out / 2)
// -- the mu block then the log-sigma block, each contiguous
QS_D int wh_at(int k, int n, int n_out, int planar) {  // Wh (128, n_out), or planar (2, 128, n_out / 2)
  const int half = n_out >> 1;
  return planar ? (n >= half ? 128 * half : 0) + k * half + (n >= half ? n - half : n) : k * n_out + n;
}
QS_D int64_t y_at(int64_t row, int j, int64_t N, int n_out, int planar) {
  const int half = n_out >> 1;
  return planar ? (j >= half ? N * half : 0) + row * half + (j >= half ? j - half : j) : row * n_out + j;
}

struct GruArgs {  // the GRU cell of the forward (k_policy_fwd2)
  int n_in;
  const float *x, *xs, *hp, *Wi, *bi, *Wg, *bg;  // xs: per-feature input scale, or null
  const uint8_t* reset;  // rows whose carried h restarts at 0 (episode reset), or null
  float* h_out;
};

template <bool BWD>
__global__ void __launch_bounds__(PT, 1)
    k_policy_trunk(int64_t N, int n_out, int planar, const __nv_bfloat16* __restrict__ img,
                   const float* __restrict__ h, const float* __restrict__ dy,
                   const float* __restrict__ W0, const float* __restrict__ b0, const float* __restrict__ W1,
                   const float* __restrict__ b1, const float* __restrict__ W2, const float* __restrict__ b2,
                   const float* __restrict__ Wh, const float* __restrict__ bh, float* __restrict__ y,
                   float* __restrict__ dh, float* __restrict__ work) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  PolSmem& S = *reinterpret_cast<PolSmem*>(smem_raw);
  using umma::blk_off;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = 32 * (warp & 3) + lane, q = warp >> 2, cq = 32 * q;
  // ---- weights (bf16, blocked) and biases
  if (img) {  // pre-converted image: W0 | W1 | W2 | WH are the first members of PolSmem
    if (tid == 0) {
      mbar_init(&S.wbar, 1);
      fence_barrier_init();
      load_image(S.W0, img, IMG_W0, IMG_WI - IMG_W0, &S.wbar);
    }
  } else {
    stage_w<HW>(W0, HI, HI, S.W0, tid);
    stage_w<HW>(W1, HW, HW, S.W1, tid);
    stage_w<HW>(W2, HW, HW, S.W2, tid);
    for (int i = tid; i < HW * HY; i += PT) {
      const int k = i / HY, n = i % HY;  // Wh (128, n_out) row-major, zero-padded to 16 columns
      S.WH[blk_off(k, n, HY)] = __float2bfloat16_rn(n < n_out ? Wh[wh_at(k, n, n_out, planar)] : 0.f);
    }
  }
  for (int i = tid; i < HW; i += PT) {
    S.b0[i] = b0[i];
    S.b1[i] = b1[i];
    S.b2[i] = b2[i];
  }
  if (tid < HY) S.bh[tid] = (bh && tid < n_out) ? bh[tid] : 0.f;  // (the backward takes no bh)
  if (warp == 0) umma::tmem_alloc(&S.tbase, 512);
  if (tid == 0) {
    mbar_init(&S.bar, 1);
    fence_barrier_init();
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  if (img) mbar_wait(&S.wbar, 0);  // (initialised before the barrier above)
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
  // the same from MN column c0 (a multiple of 8)
  auto mKc = [](const __nv_bfloat16* b, int cols, int ks, int c0) {
    return umma::desc_mnmajor(b + ks * 2 * (cols / 8) * 64 + (c0 / 8) * 64, cols);
  };
  // epilogue: TMEM columns [cq, cq+32) of this row + bias -> tanh -> bf16 row of dst
  auto epi_tanh = [&](const float* bias, __nv_bfloat16* dst) {
    float v[32];
    ld32(TG + lanes + cq, v);
    uint32_t w[16];
#pragma unroll
    for (int j = 0; j < 32; j += 2) w[j / 2] = tanh_bf16x2(pk(v[j] + bias[cq + j], v[j + 1] + bias[cq + j + 1]));
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
  // the next tile's h row quarter and dL/dy, loaded one tile ahead (registers)
  float hv_n[16], gy_n[HY / 2];
  auto fetch = [&](int64_t t) {
    const int64_t rw = t * TR + r;
    const bool vd = t < ntiles && rw < N;
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      const float4 u = vd ? __ldg(reinterpret_cast<const float4*>(h + rw * HI + 16 * q + j))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
      hv_n[j] = u.x;
      hv_n[j + 1] = u.y;
      hv_n[j + 2] = u.z;
      hv_n[j + 3] = u.w;
    }
    if constexpr (BWD) {
      if (q == 0) {
#pragma unroll
        for (int j = 0; j < HY / 2; ++j) gy_n[j] = (vd && j < n_out) ? __ldg(dy + y_at(rw, j, N, n_out, planar)) : 0.f;
      }
    }
  };
  fetch(blockIdx.x);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row = tile * TR + r;
    const bool valid = row < N;
    float v[16], gyc[HY / 2];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = hv_n[j];
#pragma unroll
    for (int j = 0; j < HY / 2; ++j) gyc[j] = gy_n[j];
    fetch(tile + gridDim.x);
    {  // ---- stage h (quarter q: columns 16q..16q+15)
#pragma unroll
      for (int j = 0; j < 16; j += 8)
        *reinterpret_cast<uint4*>(&S.H[blk_off(r, 16 * q + j, HI)]) =
            make_uint4(pk(v[j], v[j + 1]), pk(v[j + 2], v[j + 3]), pk(v[j + 4], v[j + 5]), pk(v[j + 6], v[j + 7]));
    }
    if (BWD && q == 0) {  // dL/dy
      float g[HY];
#pragma unroll
      for (int j = 0; j < HY; ++j) g[j] = j < HY / 2 ? gyc[j] : 0.f;
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
    __nv_bfloat16* const ZB = S.Z;
    epi_tanh(S.b2, ZB);
    to_mma();
    if constexpr (!BWD) {
      // ---- heads: y = z Wh + bh (N = 16, the first n_out columns written)
      if (tid == 0) {
#pragma unroll
        for (int ks = 0; ks < HW / 16; ++ks)
          umma::mma_bf16(TG, aK(ZB, HW, ks), mK(S.WH, HY, ks), id_k_mn16, ks > 0);
        umma::commit(&S.bar);
      }
      wait();
      if (q == 0) {
        float v[16];
        umma::tmem_ld16(TG + lanes, v);
        if (valid) {
#pragma unroll
          for (int j = 0; j < HY / 2; ++j)
            if (j < n_out) y[y_at(row, j, N, n_out, planar)] = v[j] + S.bh[j];
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
    // this CTA's partial gradients (lane = the gradient's row index) -> work;
    // summed over the CTAs in a fixed order by red::sum_partials
    float* wk = work + (int64_t)blockIdx.x * TK_P;
    auto ld32z = [&](uint32_t t, float (&v)[32]) {
      if (!first) {
        ld32(t, v);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.f;
      }
    };
    auto ld16z = [&](uint32_t t, float (&v)[16]) {
      if (!first) {
        umma::tmem_ld16(t, v);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0.f;
      }
    };
    float v[32];
    ld32z(TW2 + lanes + cq, v);
#pragma unroll
    for (int j = 0; j < 32; j += 4)
      *reinterpret_cast<float4*>(wk + TK_W2 + r * HW + cq + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    ld32z(TW1 + lanes + cq, v);
#pragma unroll
    for (int j = 0; j < 32; j += 4)
      *reinterpret_cast<float4*>(wk + TK_W1 + r * HW + cq + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    float u[16];
    ld16z(TW0 + lanes + 16 * q, u);  // dW0^T: lane = trunk unit, column = input
#pragma unroll
    for (int j = 0; j < 16; ++j) wk[TK_W0 + (16 * q + j) * HW + r] = u[j];
    if (q == 0) {
      ld16z(TWH + lanes, u);
#pragma unroll
      for (int j = 0; j < HY / 2; ++j)
        if (j < n_out) wk[TK_WH + wh_at(r, j, n_out, planar)] = u[j];
      ld16z(TB2 + lanes, u);
      wk[TK_B2 + r] = u[HY - 1];
      // dbh: per-row sums of dL/dy over the tiles, reduced over the warp
#pragma unroll
      for (int j = 0; j < HY / 2; ++j) {
        float t = dbh_acc[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) S.dbh[warp][j] = t;
      }
    } else if (q == 1) {
      ld16z(TB1 + lanes, u);
      wk[TK_B1 + r] = u[HY - 1];
    } else if (q == 2) {
      ld16z(TB0 + lanes, u);
      wk[TK_B0 + r] = u[HY - 1];
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free(T0, 512);
  if (BWD && tid < n_out)
    work[(int64_t)blockIdx.x * TK_P + TK_BH + tid] = (S.dbh[0][tid] + S.dbh[1][tid]) + (S.dbh[2][tid] + S.dbh[3][tid]);
}

// ---- the policy step's forward with two tiles in flight (qs_policy_gru_fwd).
// The forward keeps no activation after the next layer's GEMM read it, so a
// tile needs ONE 32 KB activation buffer, overwritten layer by layer (h, then
// A1, A2, z in place: each epilogue runs after the GEMM that read the previous
// activation completed).  That leaves room for two tiles next to the 114 KB of
// weights: the CTA's 16 warps form two independent groups of 8 (256 threads,
// thread = TMEM lane x column half), each with its own tile, TMEM half
// (256 columns), mbarrier and named barrier -- one group's epilogues fill the
// other's GEMM and memory latencies.
struct Fwd2Smem {
  __nv_bfloat16 W0[HI * HW], W1[HW * HW], W2[HW * HW], WH[HW * HY];
  __nv_bfloat16 WI[XI * G3], WG[HI * G3];
  __nv_bfloat16 ACT[2][TR * HW];  // per group: h (prev, bf16) -> h' -> A1 -> A2 -> z
  __nv_bfloat16 XS[2][TR * XI];   // per group: the input rows
  float b0[HW], b1[HW], b2[HW], bh[HY], bg[4 * HI];
  float xs[XI];  // the input scale (1 past n_in / when absent)
  uint64_t bar[2], wbar;
  uint32_t tbase;
};

QS_D void group_sync(int g) { asm volatile("bar.sync %0, 256;" ::"r"(1 + g) : "memory"); }

__global__ void __launch_bounds__(PT, 1)
    k_policy_fwd2(int64_t N, int n_out, int planar, const __nv_bfloat16* __restrict__ img, GruArgs ga,
                  const float* __restrict__ W0, const float* __restrict__ b0,
                  const float* __restrict__ W1, const float* __restrict__ b1, const float* __restrict__ W2,
                  const float* __restrict__ b2, const float* __restrict__ Wh, const float* __restrict__ bh,
                  float* __restrict__ y) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Fwd2Smem& S = *reinterpret_cast<Fwd2Smem*>(smem_raw);
  using umma::blk_off;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = warp >> 3, gw = warp & 7;          // group, warp within the group
  const int r = 32 * (gw & 3) + lane, hh = gw >> 2;  // tile row (TMEM lane), column half
  if (img) {  // pre-converted image == the weight section of Fwd2Smem
    if (tid == 0) {
      mbar_init(&S.wbar, 1);
      fence_barrier_init();
      load_image(S.W0, img, 0, IMG_N, &S.wbar);
    }
  } else {
    stage_w<HW>(W0, HI, HI, S.W0, tid);
    stage_w<HW>(W1, HW, HW, S.W1, tid);
    stage_w<HW>(W2, HW, HW, S.W2, tid);
    stage_w<G3>(ga.Wi, XI, ga.n_in, S.WI, tid);
    stage_w<G3>(ga.Wg, HI, HI, S.WG, tid);
    for (int i = tid; i < HW * HY; i += PT) {
      const int k = i / HY, n = i % HY;
      S.WH[blk_off(k, n, HY)] = __float2bfloat16_rn(n < n_out ? Wh[wh_at(k, n, n_out, planar)] : 0.f);
    }
  }
  for (int i = tid; i < HW; i += PT) {
    S.b0[i] = b0[i];
    S.b1[i] = b1[i];
    S.b2[i] = b2[i];
  }
  for (int i = tid; i < 4 * HI; i += PT)
    S.bg[i] = i < 2 * HI ? ga.bi[i] + ga.bg[i] : i < 3 * HI ? ga.bi[i] : ga.bg[i - HI];
  if (tid < HY) S.bh[tid] = tid < n_out ? bh[tid] : 0.f;
  if (tid < XI) S.xs[tid] = (ga.xs && tid < ga.n_in) ? ga.xs[tid] : 1.f;
  if (warp == 0) umma::tmem_alloc(&S.tbase, 512);
  if (tid == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    fence_barrier_init();
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  if (img) mbar_wait(&S.wbar, 0);
  // this group's TMEM: r|z [0,128) (then the trunk accumulator), x Wi_n [128,192), h Wh_n [192,256)
  const uint32_t TB = S.tbase + 256 * g, TRZ = TB, TGN = TB + 128, THN = TB + 192;
  const uint32_t lanes = umma::taddr(0, 32 * (gw & 3), 0);
  __nv_bfloat16* const ACT = S.ACT[g];
  __nv_bfloat16* const XS = S.XS[g];
  const bool issuer = (tid & 255) == 0;
  uint32_t phase = 0;
  auto to_mma = [&]() {
    umma::fence_async_smem();
    umma::fence_before();
    group_sync(g);
    umma::fence_after();
  };
  auto wait = [&]() {
    umma::mbar_wait_parity(&S.bar[g], phase);
    phase ^= 1u;
    umma::fence_after();
  };
  auto aK = [](const __nv_bfloat16* b, int cols, int ks) { return umma::desc_kmajor(b + ks * 128, cols); };
  auto mKc = [](const __nv_bfloat16* b, int cols, int ks, int c0) {
    return umma::desc_mnmajor(b + ks * 2 * (cols / 8) * 64 + (c0 / 8) * 64, cols);
  };
  const uint32_t id128 = umma::idesc_bf16(128, 128, false, true), id64 = umma::idesc_bf16(128, 64, false, true),
                 id16 = umma::idesc_bf16(128, 16, false, true);
  // trunk layer epilogue: TMEM columns [64 hh, 64 hh + 64) + bias -> tanh -> ACT (in place)
  auto epi_tanh = [&](const float* bias) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int c0 = 64 * hh + 32 * c;
      float v[32];
      umma::tmem_ld32(TRZ + lanes + c0, v);
      uint32_t w[16];
#pragma unroll
      for (int j = 0; j < 32; j += 2) w[j / 2] = tanh_bf16x2(pk(v[j] + bias[c0 + j], v[j + 1] + bias[c0 + j + 1]));
      st32(ACT, r, c0, HW, w);
    }
  };
  const int64_t ntiles = (N + TR - 1) / TR;
  for (int64_t tile = 2 * (int64_t)blockIdx.x + g; tile < ntiles; tile += 2 * (int64_t)gridDim.x) {
    const int64_t row = tile * TR + r;
    const bool valid = row < N;
    const bool live = valid && !(ga.reset && ga.reset[row]);
    // ---- stage the carried h (units 32 hh .. 32 hh + 31; 0 on a reset row) and the input row
    float hp[32];
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      const float4 t = live ? __ldg(reinterpret_cast<const float4*>(ga.hp + row * HI + 32 * hh + j))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
      hp[j] = t.x;
      hp[j + 1] = t.y;
      hp[j + 2] = t.z;
      hp[j + 3] = t.w;
    }
#pragma unroll
    for (int j = 0; j < 32; j += 8)
      *reinterpret_cast<uint4*>(&ACT[blk_off(r, 32 * hh + j, HI)]) =
          make_uint4(pk(hp[j], hp[j + 1]), pk(hp[j + 2], hp[j + 3]), pk(hp[j + 4], hp[j + 5]), pk(hp[j + 6], hp[j + 7]));
    if (hh == 0) {
      float xv[XI];
#pragma unroll
      for (int j = 0; j < XI; ++j)
        xv[j] = (valid && j < ga.n_in) ? __ldg(ga.x + row * ga.n_in + j) * S.xs[j] : 0.f;
#pragma unroll
      for (int j = 0; j < XI; j += 8)
        *reinterpret_cast<uint4*>(&XS[blk_off(r, j, XI)]) = make_uint4(
            pk(xv[j], xv[j + 1]), pk(xv[j + 2], xv[j + 3]), pk(xv[j + 4], xv[j + 5]), pk(xv[j + 6], xv[j + 7]));
    }
    to_mma();
    if (issuer) {  // gate pre-activations: r|z (x Wi + h Wh), x Wi_n, h Wh_n
      umma::mma_bf16(TRZ, aK(XS, XI, 0), mKc(S.WI, G3, 0, 0), id128, false);
#pragma unroll
      for (int ks = 0; ks < HI / 16; ++ks) umma::mma_bf16(TRZ, aK(ACT, HI, ks), mKc(S.WG, G3, ks, 0), id128, true);
      umma::mma_bf16(TGN, aK(XS, XI, 0), mKc(S.WI, G3, 0, 2 * HI), id64, false);
#pragma unroll
      for (int ks = 0; ks < HI / 16; ++ks)
        umma::mma_bf16(THN, aK(ACT, HI, ks), mKc(S.WG, G3, ks, 2 * HI), id64, ks > 0);
      umma::commit(&S.bar[g]);
    }
    wait();
#pragma unroll
    for (int c = 0; c < 2; ++c) {  // h' = n + z (h - n), units 32 hh + 16 c .. + 15
      const int u0 = 32 * hh + 16 * c;
      float gr[16], gz[16], gn[16], hn[16];
      umma::tmem_ld16(TRZ + lanes + u0, gr);
      umma::tmem_ld16(TRZ + lanes + HI + u0, gz);
      umma::tmem_ld16(TGN + lanes + u0, gn);
      umma::tmem_ld16(THN + lanes + u0, hn);
      float o[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int u = u0 + j;
        const float rr = sigm_f(gr[j] + S.bg[u]), zz = sigm_f(gz[j] + S.bg[HI + u]);
        const float nn = tanh_f(gn[j] + S.bg[2 * HI + u] + rr * (hn[j] + S.bg[3 * HI + u]));
        o[j] = nn + zz * (hp[16 * c + j] - nn);
      }
      if (valid) {
        float4* dst = reinterpret_cast<float4*>(ga.h_out + row * HI + u0);
#pragma unroll
        for (int j = 0; j < 4; ++j) dst[j] = make_float4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
      }
#pragma unroll
      for (int j = 0; j < 16; j += 8)
        *reinterpret_cast<uint4*>(&ACT[blk_off(r, u0 + j, HI)]) =
            make_uint4(pk(o[j], o[j + 1]), pk(o[j + 2], o[j + 3]), pk(o[j + 4], o[j + 5]), pk(o[j + 6], o[j + 7]));
    }
    to_mma();
    if (issuer) {  // A1 = tanh(h' W0 + b0)
#pragma unroll
      for (int ks = 0; ks < HI / 16; ++ks) umma::mma_bf16(TRZ, aK(ACT, HI, ks), mKc(S.W0, HW, ks, 0), id128, ks > 0);
      umma::commit(&S.bar[g]);
    }
    wait();
    epi_tanh(S.b0);
    to_mma();
    if (issuer) {
#pragma unroll
      for (int ks = 0; ks < HW / 16; ++ks) umma::mma_bf16(TRZ, aK(ACT, HW, ks), mKc(S.W1, HW, ks, 0), id128, ks > 0);
      umma::commit(&S.bar[g]);
    }
    wait();
    epi_tanh(S.b1);
    to_mma();
    if (issuer) {
#pragma unroll
      for (int ks = 0; ks < HW / 16; ++ks) umma::mma_bf16(TRZ, aK(ACT, HW, ks), mKc(S.W2, HW, ks, 0), id128, ks > 0);
      umma::commit(&S.bar[g]);
    }
    wait();
    epi_tanh(S.b2);
    to_mma();
    if (issuer) {  // heads: y = z Wh + bh (N = 16)
#pragma unroll
      for (int ks = 0; ks < HW / 16; ++ks) umma::mma_bf16(TRZ, aK(ACT, HW, ks), mKc(S.WH, HY, ks, 0), id16, ks > 0);
      umma::commit(&S.bar[g]);
    }
    wait();
    if (hh == 0) {
      float v[16];
      umma::tmem_ld16(TRZ + lanes, v);
      if (valid) {
#pragma unroll
        for (int j = 0; j < HY / 2; ++j)
          if (j < n_out) y[y_at(row, j, N, n_out, planar)] = v[j] + S.bh[j];
      }
    }
    umma::fence_before();
    group_sync(g);  // the next tile overwrites ACT / XS and the accumulators
    umma::fence_after();
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free(S.tbase, 512);
}

// ---- the GRU cell's backward (q/nets.py:107-132 differentiated):
//   r = s(ar), z = s(az), n = tanh(an), an = xWi_n + bi_n + r (hWh_n + bh_n),
//   h' = n + z (h - n);  for g = dL/dh':
//   dn = g (1 - z), dz = g (h - n), dan = dn (1 - n^2), dr = dan (hWh_n + bh_n)
//   dar = dr r (1 - r), daz = dz z (1 - z)
//   dgi = [dar | daz | dan], dgh = [dar | daz | dan r]
//   dx = dgi Wi^T, dh = g z + dgh Wh^T, dWi = x^T dgi, dWh = h^T dgh
// Weight gradients as (gate units) x [x | h | 1]: two M = 128 GEMMs per tile
// over B = [x | h | 1] (96 columns) -- rows r|z of dgi^T (= dgh^T), and
// [dan | dan r]^T (rows 0-63 give dWi_n, dbi_n; rows 64-127 dWh_n, dbh_n).
struct GruSmem {
  __nv_bfloat16 WI[XI * G3];   // [16][192]  MN-major B of x Wi, K-major B of dgi Wi^T
  __nv_bfloat16 WG[HI * G3];   // [64][192]
  __nv_bfloat16 B[TR * 96];    // [rows][x 0-15 | h 16-79 | 1 80 | 0]
  __nv_bfloat16 GRZ[TR * HW];  // [rows][dar | daz]
  __nv_bfloat16 GN[TR * HW];   // [rows][dan | dan r]
  // the next tile's raw rows, streamed in by cp.async while this tile computes:
  // h, dL/dh' (a, b) as 16-byte chunks XOR-swizzled by row (conflict-free row reads)
  float HR[TR * HI], AR[TR * HI], BR[TR * HI];
  float XR[TR * XI];           // x rows (n_in floats each, contiguous)
  uint8_t RR[TR];              // reset bytes
  float xs[XI];                // the input scale (1 past n_in / when absent)
  float bg[4 * HI];
  uint64_t bar, wbar;
  uint32_t tbase;
};
static_assert(sizeof(GruSmem) <= 227 * 1024, "GRU backward shared memory");

__global__ void __launch_bounds__(PT, 1)
    k_gru_bwd(int64_t N, int n_in, const __nv_bfloat16* __restrict__ img, const float* __restrict__ x,
              const float* __restrict__ xs, const float* __restrict__ hp,
              const uint8_t* __restrict__ rst, const float* __restrict__ dha, const float* __restrict__ dhb, const float* __restrict__ Wi,
              const float* __restrict__ bi, const float* __restrict__ Wg, const float* __restrict__ bgv,
              float* __restrict__ dx, float* __restrict__ dhp, float* __restrict__ work) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  GruSmem& S = *reinterpret_cast<GruSmem*>(smem_raw);
  using umma::blk_off;
  constexpr int BC = 96;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = 32 * (warp & 3) + lane, q = warp >> 2;
  if (img) {  // WI | WG: the image's tail, the first members of GruSmem
    if (tid == 0) {
      mbar_init(&S.wbar, 1);
      fence_barrier_init();
      load_image(S.WI, img, IMG_WI, IMG_N - IMG_WI, &S.wbar);
    }
  } else {
    stage_w<G3>(Wi, XI, n_in, S.WI, tid);
    stage_w<G3>(Wg, HI, HI, S.WG, tid);
  }
  for (int i = tid; i < 4 * HI; i += PT) S.bg[i] = i < 2 * HI ? bi[i] + bgv[i] : i < 3 * HI ? bi[i] : bgv[i - HI];
  if (tid < XI) S.xs[tid] = (xs && tid < n_in) ? xs[tid] : 1.f;
  if (warp == 0) umma::tmem_alloc(&S.tbase, 512);
  if (tid == 0) {
    mbar_init(&S.bar, 1);
    fence_barrier_init();
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  if (img) mbar_wait(&S.wbar, 0);
  const uint32_t T0 = S.tbase;
  // TMEM: r|z [0,128), x Wi_n [128,192), h Wh_n [192,256) -- then dx [0,16),
  // dgh Wh^T [64,128); dW r|z [256,352); dW n [352,448)
  const uint32_t TRZ = T0, TGN = T0 + 128, THN = T0 + 192, TDX = T0, TDH = T0 + 64, TWR = T0 + 256,
                 TWN = T0 + 352;
  const uint32_t lanes = umma::taddr(0, 32 * (warp & 3), 0);
  uint32_t phase = 0;
  bool first = true;
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
  auto aK = [](const __nv_bfloat16* b, int cols, int ks) { return umma::desc_kmajor(b + ks * 128, cols); };
  auto mKc = [](const __nv_bfloat16* b, int cols, int ks, int c0) {
    return umma::desc_mnmajor(b + ks * 2 * (cols / 8) * 64 + (c0 / 8) * 64, cols);
  };
  const int64_t ntiles = (N + TR - 1) / TR;
  const bool rst_bulk = rst && (reinterpret_cast<uintptr_t>(rst) & 15) == 0;
  auto cp16 = [](void* dst, const void* src, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes)
                 : "memory");
  };
  auto prefetch = [&](int64_t t) {  // all threads: tile t's raw rows -> HR / AR / BR / XR / RR
    if (t >= ntiles) return;
    const int64_t r0 = t * TR;
    const int nrows = (int)(N - r0 < TR ? N - r0 : TR);
    for (int i = tid; i < TR * 16; i += PT) {
      const int rr = i >> 4, c = i & 15, ok = rr < nrows;
      const int dst = rr * HI + ((c ^ (rr & 15)) << 2);
      const int64_t src = ok ? (r0 + rr) * HI + 4 * c : 0;
      cp16(&S.HR[dst], hp + src, ok ? 16 : 0);
      cp16(&S.AR[dst], dha + src, ok ? 16 : 0);
      if (dhb) cp16(&S.BR[dst], dhb + src, ok ? 16 : 0);
    }
    const int xbytes = nrows * n_in * 4;
    const char* xs = reinterpret_cast<const char*>(x + r0 * n_in);
    for (int b = tid * 16; b < TR * n_in * 4; b += PT * 16) {
      const int nb = xbytes - b >= 16 ? 16 : (xbytes > b ? xbytes - b : 0);
      cp16(reinterpret_cast<char*>(S.XR) + b, xs + (nb ? b : 0), nb);
    }
    if (rst_bulk && tid < TR / 16) {
      const int nb = nrows - 16 * tid >= 16 ? 16 : (nrows > 16 * tid ? nrows - 16 * tid : 0);
      cp16(&S.RR[16 * tid], rst + r0 + (nb ? 16 * tid : 0), nb);
    }
    cp_async_commit();
  };
  prefetch(blockIdx.x);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row = tile * TR + r;
    const bool valid = row < N;
    cp_async_wait<0>();
    __syncthreads();  // this tile's raw rows have landed
    float h0[16], g[16];  // h (0 on a reset row) and dL/dh', units 16q..16q+15
    const bool live = valid && !(rst && (rst_bulk ? S.RR[r] : rst[row]));
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      const int off = r * HI + (((4 * q + j / 4) ^ (r & 15)) << 2);
      const float4 t = live ? *reinterpret_cast<const float4*>(&S.HR[off]) : make_float4(0.f, 0.f, 0.f, 0.f);
      float4 a = valid ? *reinterpret_cast<const float4*>(&S.AR[off]) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (valid && dhb) {
        const float4 b = *reinterpret_cast<const float4*>(&S.BR[off]);
        a = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
      }
      h0[j] = t.x;
      h0[j + 1] = t.y;
      h0[j + 2] = t.z;
      h0[j + 3] = t.w;
      g[j] = a.x;
      g[j + 1] = a.y;
      g[j + 2] = a.z;
      g[j + 3] = a.w;
    }
#pragma unroll
    for (int j = 0; j < 16; j += 8)
      *reinterpret_cast<uint4*>(&S.B[blk_off(r, 16 + 16 * q + j, BC)]) =
          make_uint4(pk(h0[j], h0[j + 1]), pk(h0[j + 2], h0[j + 3]), pk(h0[j + 4], h0[j + 5]), pk(h0[j + 6], h0[j + 7]));
    if (q == 0) {
      float xv[XI];
#pragma unroll
      for (int j = 0; j < XI; ++j) xv[j] = (valid && j < n_in) ? S.XR[r * n_in + j] * S.xs[j] : 0.f;
#pragma unroll
      for (int j = 0; j < XI; j += 8)
        *reinterpret_cast<uint4*>(&S.B[blk_off(r, j, BC)]) = make_uint4(
            pk(xv[j], xv[j + 1]), pk(xv[j + 2], xv[j + 3]), pk(xv[j + 4], xv[j + 5]), pk(xv[j + 6], xv[j + 7]));
    } else if (q == 1) {
      const uint32_t one = pk(valid ? 1.f : 0.f, 0.f), zero = pk(0.f, 0.f);
      *reinterpret_cast<uint4*>(&S.B[blk_off(r, 80, BC)]) = make_uint4(one, zero, zero, zero);
      *reinterpret_cast<uint4*>(&S.B[blk_off(r, 88, BC)]) = make_uint4(zero, zero, zero, zero);
    }
    to_mma();                         // (every thread is past its raw reads)
    prefetch(tile + gridDim.x);       // the next tile's rows stream in behind this one
    if (tid == 0) {  // recompute the gate pre-activations
      const uint32_t id128 = umma::idesc_bf16(128, 128, false, true), id64 = umma::idesc_bf16(128, 64, false, true);
      umma::mma_bf16(TRZ, aK(S.B, BC, 0), mKc(S.WI, G3, 0, 0), id128, false);
#pragma unroll
      for (int ks = 0; ks < HI / 16; ++ks) umma::mma_bf16(TRZ, aK(S.B, BC, 1 + ks), mKc(S.WG, G3, ks, 0), id128, true);
      umma::mma_bf16(TGN, aK(S.B, BC, 0), mKc(S.WI, G3, 0, 2 * HI), id64, false);
#pragma unroll
      for (int ks = 0; ks < HI / 16; ++ks)
        umma::mma_bf16(THN, aK(S.B, BC, 1 + ks), mKc(S.WG, G3, ks, 2 * HI), id64, ks > 0);
      umma::commit(&S.bar);
    }
    wait();
    float dd[16];  // g z: the direct part of dL/dh
    {
      float gr[16], gz[16], gn[16], hn[16];
      umma::tmem_ld16(TRZ + lanes + 16 * q, gr);
      umma::tmem_ld16(TRZ + lanes + HI + 16 * q, gz);
      umma::tmem_ld16(TGN + lanes + 16 * q, gn);
      umma::tmem_ld16(THN + lanes + 16 * q, hn);
      uint32_t wr[8], wz[8], wn[8], wnr[8];
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        float ar[2], az[2], an[2], anr[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int u = 16 * q + j + e;
          const float rr = sigm_f(gr[j + e] + S.bg[u]), zz = sigm_f(gz[j + e] + S.bg[HI + u]);
          const float hb = hn[j + e] + S.bg[3 * HI + u];
          const float nn = tanh_f(gn[j + e] + S.bg[2 * HI + u] + rr * hb);
          const float gg = g[j + e];
          dd[j + e] = gg * zz;
          const float dan = gg * (1.f - zz) * (1.f - nn * nn);
          ar[e] = dan * hb * rr * (1.f - rr);
          az[e] = gg * (h0[j + e] - nn) * zz * (1.f - zz);
          an[e] = dan;
          anr[e] = dan * rr;
        }
        wr[j / 2] = pk(ar[0], ar[1]);
        wz[j / 2] = pk(az[0], az[1]);
        wn[j / 2] = pk(an[0], an[1]);
        wnr[j / 2] = pk(anr[0], anr[1]);
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        *reinterpret_cast<uint4*>(&S.GRZ[blk_off(r, 16 * q + 8 * j, HW)]) =
            make_uint4(wr[4 * j], wr[4 * j + 1], wr[4 * j + 2], wr[4 * j + 3]);
        *reinterpret_cast<uint4*>(&S.GRZ[blk_off(r, HI + 16 * q + 8 * j, HW)]) =
            make_uint4(wz[4 * j], wz[4 * j + 1], wz[4 * j + 2], wz[4 * j + 3]);
        *reinterpret_cast<uint4*>(&S.GN[blk_off(r, 16 * q + 8 * j, HW)]) =
            make_uint4(wn[4 * j], wn[4 * j + 1], wn[4 * j + 2], wn[4 * j + 3]);
        *reinterpret_cast<uint4*>(&S.GN[blk_off(r, HI + 16 * q + 8 * j, HW)]) =
            make_uint4(wnr[4 * j], wnr[4 * j + 1], wnr[4 * j + 2], wnr[4 * j + 3]);
      }
    }
    to_mma();
    if (tid == 0) {
      const uint32_t id16 = umma::idesc_bf16(128, 16, false, false), id64 = umma::idesc_bf16(128, 64, false, false);
      const uint32_t idw = umma::idesc_bf16(128, BC, true, true);
      // dx = [dar | daz | dan] Wi^T; dh = [dar | daz | dan r] Wh^T
#pragma unroll
      for (int ks = 0; ks < HW / 16; ++ks) {
        umma::mma_bf16(TDX, aK(S.GRZ, HW, ks), aK(S.WI, G3, ks), id16, ks > 0);
        umma::mma_bf16(TDH, aK(S.GRZ, HW, ks), aK(S.WG, G3, ks), id64, ks > 0);
      }
#pragma unroll
      for (int ks = 0; ks < HI / 16; ++ks) {
        umma::mma_bf16(TDX, aK(S.GN, HW, ks), aK(S.WI, G3, 8 + ks), id16, true);
        umma::mma_bf16(TDH, aK(S.GN, HW, 4 + ks), aK(S.WG, G3, 8 + ks), id64, true);
      }
      // weight gradients: (gate units) x [x | h | 1], summed over the tile rows
#pragma unroll
      for (int ks = 0; ks < TR / 16; ++ks) {
        umma::mma_bf16(TWR, mKc(S.GRZ, HW, ks, 0), mKc(S.B, BC, ks, 0), idw, !first || ks > 0);
        umma::mma_bf16(TWN, mKc(S.GN, HW, ks, 0), mKc(S.B, BC, ks, 0), idw, !first || ks > 0);
      }
      umma::commit(&S.bar);
    }
    wait();
    first = false;
    {
      float v[16];
      umma::tmem_ld16(TDH + lanes + 16 * q, v);
      if (valid) {  // a reset row's carried h was replaced by 0: no gradient reaches it
        float4* dst = reinterpret_cast<float4*>(dhp + row * HI + 16 * q);
        const float m = live ? 1.f : 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          dst[j] = make_float4(m * (v[4 * j] + dd[4 * j]), m * (v[4 * j + 1] + dd[4 * j + 1]),
                               m * (v[4 * j + 2] + dd[4 * j + 2]), m * (v[4 * j + 3] + dd[4 * j + 3]));
      }
      if (q == 0) {
        umma::tmem_ld16(TDX + lanes, v);
        if (valid) {
#pragma unroll
          for (int j = 0; j < XI; ++j)
            if (j < n_in) dx[row * n_in + j] = v[j] * S.xs[j];  // d/dx = d/d(x * xs) * xs
        }
      }
    }
    umma::fence_before();
    __syncthreads();  // the next tile overwrites B, GRZ, GN and the gate columns
    umma::fence_after();
  }
  {  // this CTA's partials -> work (TMEM lane = gate unit; columns [x 0-15 | h 16-79 | 1 80])
    float* wk = work + (int64_t)blockIdx.x * GK_P;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int chunk = q + 4 * c;  // 16-column chunks 0..5 of each 96-column accumulator
      if (chunk >= 6) continue;
      float a[16], b[16];
      if (!first) {
        umma::tmem_ld16(TWR + lanes + 16 * chunk, a);
        umma::tmem_ld16(TWN + lanes + 16 * chunk, b);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] = b[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int col = 16 * chunk + j;
        if (col < XI) {
          if (col < n_in) {
            wk[GK_WI + col * G3 + r] = a[j];
            if (r < HI) wk[GK_WI + col * G3 + 2 * HI + r] = b[j];
          }
        } else if (col < XI + HI) {
          wk[GK_WG + (col - XI) * G3 + r] = a[j];
          if (r >= HI) wk[GK_WG + (col - XI) * G3 + HI + r] = b[j];
        } else if (col == XI + HI) {
          wk[GK_BI + r] = a[j];
          wk[GK_BG + r] = a[j];
          if (r < HI)
            wk[GK_BI + 2 * HI + r] = b[j];
          else
            wk[GK_BG + HI + r] = b[j];
        }
      }
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free(T0, 512);
}

template <bool BWD>
int launch_trunk(int64_t n, int32_t n_out, int32_t planar, const void* img, const float* h, const float* dy,
                 const float* W0, const float* b0,
                 const float* W1, const float* b1, const float* W2, const float* b2, const float* Wh,
                 const float* bh, float* y, float* dh, float* gW0, float* gb0, float* gW1, float* gb1,
                 float* gW2, float* gb2, float* gWh, float* gbh, float* work, int64_t work_floats, int32_t n_sm,
                 void* stream) {
  if (n <= 0) return QS_OK;
  if (n_out < 1 || n_out > 8 || n_sm < 1 || (planar && (n_out & 1))) return QS_ERR_BAD_ARGUMENT;
  if (BWD && (!work || work_floats < (int64_t)n_sm * TK_P)) return QS_ERR_BAD_ARGUMENT;
  const size_t smem = sizeof(PolSmem);
  static_assert(sizeof(PolSmem) <= 227 * 1024, "shared memory");
  if (cudaFuncSetAttribute(k_policy_trunk<BWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return QS_ERR_LAUNCH;
  const int64_t ntiles = (n + TR - 1) / TR;
  const int grid = (int)(ntiles < n_sm ? ntiles : n_sm);
  k_policy_trunk<BWD><<<grid, PT, smem, (cudaStream_t)stream>>>(n, n_out, planar,
                                                                reinterpret_cast<const __nv_bfloat16*>(img), h, dy, W0, b0, W1, b1, W2, b2, Wh, bh, y,
                                                                     dh, work);
  if (cudaGetLastError() != cudaSuccess) return QS_ERR_LAUNCH;
  if (!BWD) return QS_OK;
  red::Segs sg{{gW0, gb0, gW1, gb1, gW2, gb2, gWh, gbh},
               {TK_W0, TK_B0, TK_W1, TK_B1, TK_W2, TK_B2, TK_WH, TK_BH},
               {HI * HW, HW, HW * HW, HW, HW * HW, HW, (int64_t)HW * n_out, n_out},
               8,
               false};
  return red::sum_partials(work, grid, TK_P, sg, (cudaStream_t)stream);
}

__global__ void k_pack_image(int n_in, int n_out, int planar, const float* __restrict__ Wi, const float* __restrict__ Wg,
                             const float* __restrict__ W0, const float* __restrict__ W1, const float* __restrict__ W2,
                             const float* __restrict__ Wh, __nv_bfloat16* __restrict__ img) {
  using umma::blk_off;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < IMG_N; i += gridDim.x * blockDim.x) {
    float v;
    if (i < IMG_W1) {
      const int e = i - IMG_W0;  // element e of the blocked W0: find (k, n) by inverting blk_off
      const int k = e / HW, n = e % HW;
      v = W0[k * HW + n];
      img[IMG_W0 + blk_off(k, n, HW)] = __float2bfloat16_rn(v);
    } else if (i < IMG_W2) {
      const int e = i - IMG_W1, k = e / HW, n = e % HW;
      img[IMG_W1 + blk_off(k, n, HW)] = __float2bfloat16_rn(W1[e]);
    } else if (i < IMG_WH) {
      const int e = i - IMG_W2, k = e / HW, n = e % HW;
      img[IMG_W2 + blk_off(k, n, HW)] = __float2bfloat16_rn(W2[e]);
    } else if (i < IMG_WI) {
      const int e = i - IMG_WH, k = e / HY, n = e % HY;
      img[IMG_WH + blk_off(k, n, HY)] = __float2bfloat16_rn(n < n_out ? Wh[wh_at(k, n, n_out, planar)] : 0.f);
    } else if (i < IMG_WG) {
      const int e = i - IMG_WI, k = e / G3, n = e % G3;
      img[IMG_WI + blk_off(k, n, G3)] = __float2bfloat16_rn(k < n_in ? Wi[k * G3 + n] : 0.f);
    } else {
      const int e = i - IMG_WG, k = e / G3, n = e % G3;
      img[IMG_WG + blk_off(k, n, G3)] = __float2bfloat16_rn(Wg[e]);
    }
  }
}

}  // namespace

extern "C" {

int64_t qs_policy_image_bytes(void) { return (int64_t)IMG_N * 2; }

int qs_policy_pack_image(int32_t n_in, int32_t n_out, const float* Wi, const float* Wh_g, const float* W0,
                         const float* W1, const float* W2, const float* Wh, int32_t wh_planar, void* w_image,
                         void* stream) {
  if (!Wi || !Wh_g || !W0 || !W1 || !W2 || !Wh || !w_image || n_in < 1 || n_in > XI || n_out < 1 || n_out > 8 ||
      (wh_planar && (n_out & 1)))
    return QS_ERR_BAD_ARGUMENT;
  if (reinterpret_cast<uintptr_t>(w_image) % 16) return QS_ERR_BAD_ARGUMENT;
  k_pack_image<<<(IMG_N + 255) / 256, 256, 0, (cudaStream_t)stream>>>(n_in, n_out, wh_planar, Wi, Wh_g, W0, W1, W2, Wh,
                                                                     reinterpret_cast<__nv_bfloat16*>(w_image));
  return cudaGetLastError() == cudaSuccess ? QS_OK : QS_ERR_LAUNCH;
}

int64_t qs_policy_work_floats(int32_t which, int32_t n_sm) {
  if (n_sm < 1) return -1;
  return which == 0 ? (int64_t)n_sm * TK_P : which == 1 ? (int64_t)n_sm * GK_P : -1;
}

int qs_policy_trunk_fwd(int64_t n, int32_t n_out, const float* h, const float* W0, const float* b0, const float* W1,
                        const float* b1, const float* W2, const float* b2, const float* Wh, const float* bh, float* y,
                        int32_t n_sm, void* stream) {
  if (!y || !h) return QS_ERR_BAD_ARGUMENT;
  return launch_trunk<false>(n, n_out, 0, nullptr, h, nullptr, W0, b0, W1, b1, W2, b2, Wh, bh, y, nullptr, nullptr,
                             nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0, n_sm, stream);
}

int qs_policy_trunk_bwd(int64_t n, int32_t n_out, const void* w_image, const float* h, const float* dy,
                        int32_t dy_planar, const float* W0, const float* b0,
                        const float* W1, const float* b1, const float* W2, const float* b2, const float* Wh,
                        float* dh, float* gW0, float* gb0, float* gW1, float* gb1, float* gW2, float* gb2,
                        float* gWh, float* gbh, float* work, int64_t work_floats, int32_t n_sm, void* stream) {
  if (!h || !dy || !dh) return QS_ERR_BAD_ARGUMENT;
  return launch_trunk<true>(n, n_out, dy_planar, w_image, h, dy, W0, b0, W1, b1, W2, b2, Wh, nullptr, nullptr, dh, gW0, gb0,
                            gW1, gb1, gW2, gb2, gWh, gbh, work, work_floats, n_sm, stream);
}

int qs_policy_gru_fwd(int64_t n, int32_t n_in, int32_t n_out, const void* w_image, const float* x,
                      const float* x_scale, const float* h, const uint8_t* h_reset,
                      const float* Wi, const float* bi, const float* Wh_g, const float* bh_g, const float* W0,
                      const float* b0, const float* W1, const float* b1, const float* W2, const float* b2,
                      const float* Wh, const float* bh, float* h_out, float* y, int32_t y_planar, int32_t n_sm,
                      void* stream) {
  if (!y || !h_out || !x || !h || n_in < 1 || n_in > XI) return QS_ERR_BAD_ARGUMENT;
  if (n <= 0) return QS_OK;
  if (n_out < 1 || n_out > 8 || n_sm < 1 || (y_planar && (n_out & 1))) return QS_ERR_BAD_ARGUMENT;
  const GruArgs ga{n_in, x, x_scale, h, Wi, bi, Wh_g, bh_g, h_reset, h_out};
  const size_t smem = sizeof(Fwd2Smem);
  static_assert(sizeof(Fwd2Smem) <= 227 * 1024, "shared memory");
  if (cudaFuncSetAttribute(k_policy_fwd2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return QS_ERR_LAUNCH;
  const int64_t npairs = ((n + TR - 1) / TR + 1) / 2;
  const int grid = (int)(npairs < n_sm ? npairs : n_sm);
  k_policy_fwd2<<<grid, PT, smem, (cudaStream_t)stream>>>(n, n_out, y_planar,
                                                          reinterpret_cast<const __nv_bfloat16*>(w_image),
                                                          ga, W0, b0, W1, b1, W2, b2, Wh, bh, y);
  return cudaGetLastError() == cudaSuccess ? QS_OK : QS_ERR_LAUNCH;
}

int qs_policy_gru_bwd(int64_t n, int32_t n_in, const void* w_image, const float* x, const float* x_scale,
                      const float* h, const uint8_t* h_reset,
                      const float* dh_out_a,
                      const float* dh_out_b, const float* Wi, const float* bi, const float* Wh_g, const float* bh_g,
                      float* dx, float* dh, float* gWi, float* gbi, float* gWh_g, float* gbh_g, float* work,
                      int64_t work_floats, int32_t n_sm, void* stream) {
  if (n <= 0) return QS_OK;
  if (!x || !h || !dh_out_a || !dx || !dh || n_in < 1 || n_in > XI || n_sm < 1) return QS_ERR_BAD_ARGUMENT;
  if (!work || work_floats < (int64_t)n_sm * GK_P) return QS_ERR_BAD_ARGUMENT;
  const size_t smem = sizeof(GruSmem);
  if (cudaFuncSetAttribute(k_gru_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return QS_ERR_LAUNCH;
  const int64_t ntiles = (n + TR - 1) / TR;
  const int grid = (int)(ntiles < n_sm ? ntiles : n_sm);
  k_gru_bwd<<<grid, PT, smem, (cudaStream_t)stream>>>(n, n_in, reinterpret_cast<const __nv_bfloat16*>(w_image), x,
                                                      x_scale, h, h_reset, dh_out_a, dh_out_b, Wi, bi, Wh_g, bh_g, dx, dh,
                                                      work);
  if (cudaGetLastError() != cudaSuccess) return QS_ERR_LAUNCH;
  red::Segs sg{{gWi, gbi, gWh_g, gbh_g}, {GK_WI, GK_BI, GK_WG, GK_BG}, {(int64_t)n_in * G3, G3, HI * G3, G3}, 4, false};
  return red::sum_partials(work, grid, GK_P, sg, (cudaStream_t)stream);
}

}  // extern "C"
