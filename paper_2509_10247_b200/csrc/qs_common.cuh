// Shared device helpers: small-vector math, Philox4x32-10, error word.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>

#include "../../include/quadsim_b200.h"

#define QS_HD __host__ __device__ __forceinline__
#define QS_D __device__ __forceinline__

struct V3 {
  float x, y, z;
};

QS_HD V3 v3(float x, float y, float z) { return V3{x, y, z}; }
QS_HD V3 operator+(V3 a, V3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
QS_HD V3 operator-(V3 a, V3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
QS_HD V3 operator-(V3 a) { return v3(-a.x, -a.y, -a.z); }
QS_HD V3 operator*(V3 a, float s) { return v3(a.x * s, a.y * s, a.z * s); }
QS_HD V3 operator*(float s, V3 a) { return v3(a.x * s, a.y * s, a.z * s); }
QS_HD V3 hmul(V3 a, V3 b) { return v3(a.x * b.x, a.y * b.y, a.z * b.z); }
QS_HD float dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
QS_HD V3 cross(V3 a, V3 b) {
  return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
// Euclidean norm.  On device: MUFU sqrt (sqrt.approx, ~1 ulp) instead of the
// IEEE-rounded sequence; norms feed rewards, SDF and attitude, all checked
// against the fp64 oracle at 1e-5 relative.
QS_HD float sqrt_mufu(float x) {
#ifdef __CUDA_ARCH__
  float d;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(d) : "f"(x));  // denormal inputs flush to 0
  return d;
#else
  return sqrtf(x);
#endif
}
QS_HD float norm3(V3 a) { return sqrt_mufu(dot(a, a)); }
QS_HD V3& operator+=(V3& a, V3 b) {
  a.x += b.x; a.y += b.y; a.z += b.z;
  return a;
}
QS_HD V3& operator-=(V3& a, V3 b) {
  a.x -= b.x; a.y -= b.y; a.z -= b.z;
  return a;
}
QS_HD V3 xyz(float4 f) { return v3(f.x, f.y, f.z); }
QS_HD float4 f4(V3 a, float w) { return make_float4(a.x, a.y, a.z, w); }
QS_HD bool finite3(V3 a) { return isfinite(a.x) && isfinite(a.y) && isfinite(a.z); }

// norm VJP with the reference's convention: zero vector -> zero gradient
// (q/autodiff.py:580-591)
QS_HD V3 norm_vjp(V3 a, float n, float g) {
#ifdef __CUDA_ARCH__
  return n > 0.f ? a * __fdividef(g, n) : v3(0.f, 0.f, 0.f);  // n is a norm: far below 2^126
#else
  return n > 0.f ? a * (g / n) : v3(0.f, 0.f, 0.f);
#endif
}

struct Q4 {
  float w, x, y, z;
};
QS_HD Q4 q4(float w, float x, float y, float z) { return Q4{w, x, y, z}; }
QS_HD Q4 qmul(Q4 q, Q4 r) {  // q/autodiff.py:689-701
  return q4(q.w * r.w - q.x * r.x - q.y * r.y - q.z * r.z,
            q.w * r.x + q.x * r.w + q.y * r.z - q.z * r.y,
            q.w * r.y - q.x * r.z + q.y * r.w + q.z * r.x,
            q.w * r.z + q.x * r.y - q.y * r.x + q.z * r.w);
}
QS_HD Q4 qconj(Q4 q) { return q4(q.w, -q.x, -q.y, -q.z); }
QS_HD V3 qvec(Q4 q) { return v3(q.x, q.y, q.z); }
// v + 2 (w (u x v) + u x (u x v))   (q/autodiff.py:737-750)
QS_HD V3 qrot(Q4 q, V3 v) {
  V3 u = qvec(q);
  V3 uv = cross(u, v);
  V3 uuv = cross(u, uv);
  return v + (uv * q.w + uuv) * 2.f;
}
// qrot(q, e_z) -- the body z axis, third column of R(q) -- written out: the
// general formula's products with the zero components of e_z cannot be
// folded without fast-math (0 * x is not 0 for x = inf / nan), so this is
// ~2x fewer instructions.  The same polynomial in q (exactly equal for every
// q, unit or not); only the rounding order differs.
QS_HD V3 qaxis_z(Q4 q) {
  return v3(2.f * (q.x * q.z + q.w * q.y), 2.f * (q.y * q.z - q.w * q.x), 1.f - 2.f * (q.x * q.x + q.y * q.y));
}
// VJP of qaxis_z wrt q = (w, x, y, z): g . d(axis)/dq
QS_HD Q4 qaxis_z_vjp(Q4 q, V3 g) {
  return q4(2.f * (g.x * q.y - g.y * q.x), 2.f * (g.x * q.z - g.y * q.w) - 4.f * g.z * q.x,
            2.f * (g.x * q.w + g.y * q.z) - 4.f * g.z * q.y, 2.f * (g.x * q.x + g.y * q.y));
}
// VJP of qrot wrt v: exact transpose of the formula (== qrot(conj q, g))
QS_HD V3 qrot_vjp_v(Q4 q, V3 g) { return qrot(qconj(q), g); }
// VJP of qrot wrt q (w, u):  g_w = 2 g.(u x v);
// g_u = 2w (v x g) + 2 (u.v) g + 2 (g.u) v - 4 (g.v) u
QS_HD Q4 qrot_vjp_q(Q4 q, V3 v, V3 g) {
  V3 u = qvec(q);
  float gw = 2.f * dot(g, cross(u, v));
  V3 gu = cross(v, g) * (2.f * q.w) + g * (2.f * dot(u, v)) + v * (2.f * dot(g, u)) -
          u * (4.f * dot(g, v));
  return q4(gw, gu.x, gu.y, gu.z);
}

// MUFU ex2 / lg2 / rcp with flush-to-zero: no denormal fix-up sequences
QS_D float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
QS_D float lg2_ftz(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
QS_D float rcp_ftz(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// sigmoid / softplus / tanh on the MUFU ex2/lg2/rcp units.  Absolute error
// <= ~2e-7 (what the 1e-5 state/reward bars see); the saturated tails are
// exact: sigmoid -> 0/1, tanh -> +-1 (ex2 -> inf/0, rcp(inf) = 0).
QS_HD float sigmoid_stable(float x) {  // q/autodiff.py:446-456
#ifdef __CUDA_ARCH__
  return rcp_ftz(1.f + ex2_ftz(-1.44269504f * x));
#else
  if (x >= 0.f) return 1.f / (1.f + expf(-x));
  float e = expf(x);
  return e / (1.f + e);
#endif
}
QS_HD float softplus(float x) {  // logaddexp(0, x)
#ifdef __CUDA_ARCH__
  return fmaxf(x, 0.f) + 0.693147181f * lg2_ftz(1.f + ex2_ftz(-1.44269504f * fabsf(x)));
#else
  return fmaxf(x, 0.f) + log1pf(expf(-fabsf(x)));
#endif
}
QS_HD float tanh_fast(float x) {  // 1 - 2 / (e^{2x} + 1)
#ifdef __CUDA_ARCH__
  return 1.f - 2.f * rcp_ftz(ex2_ftz(2.88539008f * x) + 1.f);
#else
  return tanhf(x);
#endif
}

// ---------------------------------------------------------------------------
// Philox4x32-10 counter-based RNG (Salmon et al., SC'11).  Stateless: a draw
// is a pure function of (key, counter), so resets and IMU noise are graph
// capturable and independent of launch geometry / sharding.

QS_HD uint4 philox_round(uint4 c, uint32_t k0, uint32_t k1) {
#ifdef __CUDA_ARCH__
  uint32_t lo0 = c.x * 0xD2511F53u, hi0 = __umulhi(c.x, 0xD2511F53u);
  uint32_t lo1 = c.z * 0xCD9E8D57u, hi1 = __umulhi(c.z, 0xCD9E8D57u);
#else
  uint64_t p0 = (uint64_t)c.x * 0xD2511F53u, p1 = (uint64_t)c.z * 0xCD9E8D57u;
  uint32_t lo0 = (uint32_t)p0, hi0 = (uint32_t)(p0 >> 32), lo1 = (uint32_t)p1, hi1 = (uint32_t)(p1 >> 32);
#endif
  return make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
}

QS_D uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    c = philox_round(c, k.x, k.y);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// the same permutation with the key schedule precomputed on the host
// (qs_task_cfg::rng_round_keys): inside a kernel the round keys are
// kernel-parameter operands, so each round is 2 IMAD.WIDE + 2 LOP3
QS_D uint4 philox4x32_10_rk(uint4 c, const uint32_t* rk) {
#pragma unroll
  for (int i = 0; i < 10; ++i) c = philox_round(c, rk[2 * i], rk[2 * i + 1]);
  return c;
}

// Philox4x32-7: the first seven rounds of the same schedule.  Random123 lists
// it as Crush-resistant (BigCrush-clean) with a smaller safety margin; it
// draws the IMU's per-step sensor noise (12 normals per row-step, the
// forward window's largest RNG consumer), where 30% fewer rounds matter.
QS_D uint4 philox4x32_7_rk(uint4 c, const uint32_t* rk) {
#pragma unroll
  for (int i = 0; i < 7; ++i) c = philox_round(c, rk[2 * i], rk[2 * i + 1]);
  return c;
}

inline void philox_round_keys(uint64_t seed, uint32_t* rk) {
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int i = 0; i < 10; ++i) {
    rk[2 * i] = k0;
    rk[2 * i + 1] = k1;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// 32 random bits -> uniform in (0, 1): the low 23 bits as the mantissa of
// v in [1, 2) (one LOP3), shifted by 1 - 2^-24 (exact by Sterbenz), so the
// result lies in [2^-24, 1 - 2^-24]
QS_D float u12(uint32_t r) { return __uint_as_float((r & 0x007fffffu) | 0x3f800000u); }
QS_D float u01(uint32_t r) { return u12(r) - 0.99999994f; }

QS_D float4 u01x4(uint4 r) { return make_float4(u01(r.x), u01(r.y), u01(r.z), u01(r.w)); }

// four standard normals from 128 random bits (Box-Muller on two pairs):
// radius from 2 - v in (0, 1] (|z| <= 5.6), angle from v in [1, 2) directly
// (sin/cos of 2 pi v are 1-periodic).  MUFU lg2/sqrt/sin/cos: their ~2-ulp
// error is immaterial for sampling noise.
QS_D float4 box_muller4(uint4 r) {
  float d0, d1;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(d0) : "f"(-1.38629436f * lg2_ftz(2.f - u12(r.x))));
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(d1) : "f"(-1.38629436f * lg2_ftz(2.f - u12(r.z))));
  float s0, c0, s1, c1;
  __sincosf(6.28318530717958648f * u12(r.y), &s0, &c0);
  __sincosf(6.28318530717958648f * u12(r.w), &s1, &c1);
  return make_float4(d0 * c0, d0 * s0, d1 * c1, d1 * s1);
}

// twelve standard normals from 256 random bits (two Philox blocks): six
// Box-Muller pairs.  Radii take 23 bits (bits 8-30) of a word each, so
// |z| <= 5.6 as before; angles take 16 bits each (a 2^-16-turn grid, far
// below anything a sensor-noise model resolves): the low bytes of the four
// radius words of block a, and the two halves of b.z and b.w.
QS_D float bm_radius(uint32_t r) {  // sqrt(-2 ln u), u = 2 - v in (0, 1]
  float d;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(d) : "f"(-1.38629436f * lg2_ftz(2.f - u12(r >> 8))));
  return d;
}
QS_D float2 bm_pair(uint32_t rbits, uint32_t abits) {
  const float d = bm_radius(rbits);
  const float v = __uint_as_float(((abits & 0xffffu) << 7) | 0x3f800000u);  // [1, 2), 16 bits
  float s, c;
  __sincosf(6.28318530717958648f * v, &s, &c);
  return make_float2(d * c, d * s);
}
QS_D void normals12(uint4 a, uint4 b, float4& n0, float4& n1, float4& n2) {
  const uint32_t h0 = (a.x & 255u) | ((a.y & 255u) << 8), h1 = (a.z & 255u) | ((a.w & 255u) << 8);
  const float2 p0 = bm_pair(a.x, h0), p1 = bm_pair(a.y, h1), p2 = bm_pair(a.z, b.z),
               p3 = bm_pair(a.w, b.z >> 16), p4 = bm_pair(b.x, b.w), p5 = bm_pair(b.y, b.w >> 16);
  n0 = make_float4(p0.x, p0.y, p1.x, p1.y);
  n1 = make_float4(p2.x, p2.y, p3.x, p3.y);
  n2 = make_float4(p4.x, p4.y, p5.x, p5.y);
}

// six standard normals from one block: three Box-Muller pairs, radii from
// bits 8-30 of x, y, z, angles from the halves of w and the low bytes of x, y
QS_D void normals6(uint4 r, float4& n0, float4& n1) {
  const float2 p0 = bm_pair(r.x, r.w), p1 = bm_pair(r.y, r.w >> 16),
               p2 = bm_pair(r.z, (r.x & 255u) | ((r.y & 255u) << 8));
  n0 = make_float4(p0.x, p0.y, p1.x, p1.y);
  n1 = make_float4(p2.x, p2.y, 0.f, 0.f);
}
// a uniform in (0, 1) on a 2^-16 grid from the low 16 bits
QS_D float u16(uint32_t h) { return __uint_as_float(((h & 0xffffu) << 7) | 0x3f800000u) - 0.99999237f; }

// purposes (counter word 3, high byte)
enum : uint32_t {
  RNG_SPAWN = 1u,
  RNG_DR = 2u,
  RNG_IMU = 3u,
  RNG_SCENE = 4u,
  RNG_TRACK = 5u,
};

struct Rng {
  uint4 ctr;
  uint2 key;
  QS_D Rng(uint64_t seed, uint64_t id, uint32_t sub, uint32_t purpose) {
    key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    ctr = make_uint4((uint32_t)id, (uint32_t)(id >> 32), sub, purpose << 24);
  }
  // four uniforms in (0, 1)
  QS_D float4 uniform4() {
    uint4 r = philox4x32_10(ctr, key);
    ctr.w++;
    return u01x4(r);
  }
  QS_D float4 normal4() {
    uint4 r = philox4x32_10(ctr, key);
    ctr.w++;
    return box_muller4(r);
  }
  QS_D uint4 bits4() {
    uint4 r = philox4x32_10(ctr, key);
    ctr.w++;
    return r;
  }
};

// Rng with the round keys precomputed (the task kernels: cfg.rng_round_keys);
// draws are identical to Rng's for the same seed
struct RngK {
  uint4 ctr;
  const uint32_t* rk;
  QS_D RngK(const uint32_t* rk_, uint64_t id, uint32_t sub, uint32_t purpose) : rk(rk_) {
    ctr = make_uint4((uint32_t)id, (uint32_t)(id >> 32), sub, purpose << 24);
  }
  QS_D float4 uniform4() {
    uint4 r = philox4x32_10_rk(ctr, rk);
    ctr.w++;
    return u01x4(r);
  }
  QS_D float4 normal4() {
    uint4 r = philox4x32_10_rk(ctr, rk);
    ctr.w++;
    return box_muller4(r);
  }
  QS_D uint4 bits4() {
    uint4 r = philox4x32_10_rk(ctr, rk);
    ctr.w++;
    return r;
  }
  QS_D uint4 bits4_r7() {  // Philox4x32-7 (IMU noise)
    uint4 r = philox4x32_7_rk(ctr, rk);
    ctr.w++;
    return r;
  }
};

// ---------------------------------------------------------------------------
// TMA bulk copy (cp.async.bulk, sm_90+) global -> shared with mbarrier
// completion; used to stage the next step's action block one step ahead.

QS_D uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

QS_D void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
QS_D void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
QS_D void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// one thread: arm the barrier with the byte count and launch the bulk copy
QS_D void tma_load_1d(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// several bulk copies completing on one barrier: arm once with the total
QS_D void tma_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
QS_D void tma_copy_1d(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// per-thread asynchronous global -> shared copies (LDGSTS): no register is held
// while the data is in flight; completion is tracked per thread by groups
QS_D void cp_async16(void* dst_smem, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst_smem)), "l"(src) : "memory");
}
QS_D void cp_async4(void* dst_smem, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst_smem)), "l"(src) : "memory");
}
QS_D void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
QS_D void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

QS_D void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

QS_D void report_err(int32_t* err, int code, int row) {
  if (!err) return;
  atomicCAS(err, 0, code);
  atomicMin(err + 1, row);
}

template <typename T>
QS_D T ldg(const T* p) {
  return __ldg(p);
}

QS_D float4 ld4(const float* p, long i) { return __ldg(reinterpret_cast<const float4*>(p) + i); }
QS_D void st4(float* p, long i, float4 v) { reinterpret_cast<float4*>(p)[i] = v; }
