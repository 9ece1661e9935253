// Standalone kernels behind the reference's module-level API: sdf_np/sdf_var,
// ImuModel.read, DynamicsModel.step (+VJP for rollout_grad) and
// reconstruct_attitude.
#include "qs_dynamics.cuh"
#include "qs_geom.cuh"

namespace {

inline int grid_for(long n, int b) { return (int)((n + b - 1) / b); }
inline int status() { return cudaGetLastError() == cudaSuccess ? QS_OK : QS_ERR_LAUNCH; }

__global__ void k_sdf(const qs_scene sc, int n, int na, const float* __restrict__ pts,
                      float* __restrict__ out, float* __restrict__ grad) {
  long row = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  SceneView sv = scene_view(sc, row / na);
  V3 p = xyz(ld4(pts, row));
  int code;
  float d = sdf_eval(sv, p, code);
  out[row] = d;
  if (grad) st4(grad, row, f4(code ? sdf_grad(sv, p, code) : v3(0.f, 0.f, 0.f), 0.f));
}

__global__ void k_imu(int n, const float* __restrict__ R, const float* __restrict__ w,
                      const float* __restrict__ vdot, V3 g, float dt, float sa, float sg, float ra,
                      float rg, uint64_t seed, int64_t tick, const float* __restrict__ noise,
                      float* __restrict__ bias, float* __restrict__ out) {
  long row = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  V3 nba, nbg, na, ng;
  if (noise) {
    const long N = n;
    nba = v3(noise[3 * row], noise[3 * row + 1], noise[3 * row + 2]);
    nbg = v3(noise[3 * (N + row)], noise[3 * (N + row) + 1], noise[3 * (N + row) + 2]);
    na = v3(noise[3 * (2 * N + row)], noise[3 * (2 * N + row) + 1], noise[3 * (2 * N + row) + 2]);
    ng = v3(noise[3 * (3 * N + row)], noise[3 * (3 * N + row) + 1], noise[3 * (3 * N + row) + 2]);
  } else {
    Rng rng(seed, (uint64_t)row, (uint32_t)tick, RNG_IMU);
    const uint4 ua = rng.bits4(), ub = rng.bits4();
    float4 a, b, c;
    normals12(ua, ub, a, b, c);  // the same 12 normals as the fused step's IMU
    nba = v3(a.x, a.y, a.z);
    nbg = v3(a.w, b.x, b.y);
    na = v3(b.z, b.w, c.x);
    ng = v3(c.y, c.z, c.w);
  }
  float sq = sqrtf(dt);
  V3 ba = xyz(ld4(bias, 2 * row)) + nba * (ra * sq);
  V3 bg = xyz(ld4(bias, 2 * row + 1)) + nbg * (rg * sq);
  const float* r = R + 9 * row;  // row-major body->world; accel = R^T (vdot - g)
  V3 s = xyz(ld4(vdot, row)) - g;
  V3 acc = v3(r[0] * s.x + r[3] * s.y + r[6] * s.z, r[1] * s.x + r[4] * s.y + r[7] * s.z,
              r[2] * s.x + r[5] * s.y + r[8] * s.z) + ba;
  if (sa != 0.f) acc += na * sa;
  V3 gy = (w ? xyz(ld4(w, row)) : v3(0.f, 0.f, 0.f)) + bg;
  if (sg != 0.f) gy += ng * sg;
  st4(bias, 2 * row, f4(ba, 0.f));
  st4(bias, 2 * row + 1, f4(bg, 0.f));
  float* o = out + 6 * row;
  o[0] = acc.x; o[1] = acc.y; o[2] = acc.z;
  o[3] = gy.x; o[4] = gy.y; o[5] = gy.z;
}

template <int M>
__global__ void k_dyn_fwd(int n, const float* __restrict__ S, const float* __restrict__ act,
                          const float* __restrict__ dr, const qs_task_cfg cfg, float* __restrict__ So,
                          int32_t* err) {
  long row = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  constexpr int A = ModelTraits<M>::A;
  State s = load_state<M>(S, n, row);
  if (!state_finite<M>(s)) report_err(err, QS_ERR_NONFINITE_STATE, (int)row);
  const float* a = act + row * A;
  float4 c = make_float4(a[0], a[1], a[2], A == 4 ? a[3] : 0.f);
  RowPrm rp = row_params<M>(cfg, dr, row);
  State o = model_step<M>(s, c, rp, dyn_consts(cfg));
  store_state<M>(So, n, row, o);
}

template <int M>
__global__ void k_dyn_bwd(int n, const float* __restrict__ S, const float* __restrict__ act,
                          const float* __restrict__ dr, const qs_task_cfg cfg,
                          const float* __restrict__ gSo, float* __restrict__ gS,
                          float* __restrict__ gact) {
  long row = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  constexpr int A = ModelTraits<M>::A;
  State s = load_state<M>(S, n, row);
  const float* a = act + row * A;
  float4 c = make_float4(a[0], a[1], a[2], A == 4 ? a[3] : 0.f);
  RowPrm rp = row_params<M>(cfg, dr, row);
  State gi;
  float4 gc;
  model_step_vjp<M>(s, c, rp, dyn_consts(cfg), load_grad<M>(gSo, n, row), gi, gc);
  store_state<M>(gS, n, row, gi);
  float* ga = gact + row * A;
  ga[0] = gc.x; ga[1] = gc.y; ga[2] = gc.z;
  if (A == 4) ga[3] = gc.w;
}

__global__ void k_attitude(int n, const float* __restrict__ a, const float* __restrict__ ve,
                           float* __restrict__ R) {
  long row = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  V3 xb, yb, zb;
  attitude_pm(xyz(ld4(a, row)), xyz(ld4(ve, row)), xb, yb, zb);
  float* r = R + 9 * row;  // columns x_b, y_b, z_b
  r[0] = xb.x; r[1] = yb.x; r[2] = zb.x;
  r[3] = xb.y; r[4] = yb.y; r[5] = zb.y;
  r[6] = xb.z; r[7] = yb.z; r[8] = zb.z;
}

__global__ void k_philox(int n, const uint32_t* __restrict__ ck, uint32_t* __restrict__ out, int rounds) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t* p = ck + 6 * i;
  const uint4 c = make_uint4(p[0], p[1], p[2], p[3]);
  uint32_t rk[20];
  uint32_t k0 = p[4], k1 = p[5];
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    rk[2 * r] = k0;
    rk[2 * r + 1] = k1;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  const uint4 a = rounds == 7 ? philox4x32_7_rk(c, rk) : philox4x32_10(c, make_uint2(p[4], p[5]));
  const uint4 b = rounds == 7 ? philox4x32_7_rk(c, rk) : philox4x32_10_rk(c, rk);
  uint32_t* o = out + 8 * i;
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
  o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}

}  // namespace

// TD(lambda) targets with termination cuts (q/learners.py:78-94, the full
// window): one thread per env walks the window backwards,
//   G_t = r_t + (gamma cont_t) ((1 - lam) V_{t+1} + lam G_{t+1}),  G_T = V_T = bootstrap,
// with every multiply / add rounded separately in the order torch evaluates
// train.td_lambda_targets, and 1 - lam rounded from double as torch's scalar
// is, so both give the same bits.
__global__ void k_td_lambda(int T, int64_t N, const float* __restrict__ r, const float* __restrict__ v,
                            const float* __restrict__ boot, const uint8_t* __restrict__ done, float gamma, float lam,
                            float oml, float* __restrict__ G) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const float b = boot[n];
  float nxt = b;
  for (int t = T - 1; t >= 0; --t) {
    const int64_t i = (int64_t)t * N + n;
    const float v_next = t + 1 < T ? v[i + N] : b;
    const float cont = done[i] ? 0.f : 1.f;
    const float mix = __fadd_rn(__fmul_rn(oml, v_next), __fmul_rn(lam, nxt));
    const float g = __fadd_rn(r[i], __fmul_rn(__fmul_rn(gamma, cont), mix));
    G[i] = g;
    nxt = g;
  }
}

extern "C" {

int qs_philox4x32_10(int32_t n, const uint32_t* ctr_key, uint32_t* out, void* stream) {
  if (n <= 0) return QS_OK;
  k_philox<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(n, ctr_key, out, 10);
  return status();
}

int qs_philox4x32_7(int32_t n, const uint32_t* ctr_key, uint32_t* out, void* stream) {
  if (n <= 0) return QS_OK;
  k_philox<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(n, ctr_key, out, 7);
  return status();
}

int qs_sdf(const qs_scene* scene, int32_t n_rows, int32_t n_agents, const float* pts, float* out,
           float* grad, void* stream) {
  if (n_rows <= 0) return QS_OK;
  k_sdf<<<grid_for(n_rows, 128), 128, 0, (cudaStream_t)stream>>>(*scene, n_rows, n_agents, pts, out,
                                                                  grad);
  return status();
}

int qs_imu_read(int32_t n_rows, const float* R, const float* w, const float* vdot, const float* g,
                float dt, float sa, float sg, float ra, float rg, uint64_t seed, int64_t tick,
                const float* noise, float* bias, float* out, void* stream) {
  if (n_rows <= 0) return QS_OK;
  k_imu<<<grid_for(n_rows, 128), 128, 0, (cudaStream_t)stream>>>(
      n_rows, R, w, vdot, v3(g[0], g[1], g[2]), dt, sa, sg, ra, rg, seed, tick, noise, bias, out);
  return status();
}

int qs_dyn_step_fwd(int32_t model, int32_t n, const float* S_in, const float* act, const float* dr,
                    const qs_task_cfg* cfg, float* S_out, int32_t* err, void* stream) {
  if (n <= 0) return QS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int g = grid_for(n, 128);
  if (model == QS_MODEL_FULL) k_dyn_fwd<QS_MODEL_FULL><<<g, 128, 0, s>>>(n, S_in, act, dr, *cfg, S_out, err);
  else if (model == QS_MODEL_PM_CONTINUOUS)
    k_dyn_fwd<QS_MODEL_PM_CONTINUOUS><<<g, 128, 0, s>>>(n, S_in, act, dr, *cfg, S_out, err);
  else if (model == QS_MODEL_PM_DISCRETE)
    k_dyn_fwd<QS_MODEL_PM_DISCRETE><<<g, 128, 0, s>>>(n, S_in, act, dr, *cfg, S_out, err);
  else if (model == QS_MODEL_SIMPLIFIED)
    k_dyn_fwd<QS_MODEL_SIMPLIFIED><<<g, 128, 0, s>>>(n, S_in, act, dr, *cfg, S_out, err);
  else return QS_ERR_BAD_ARGUMENT;
  return status();
}

int qs_dyn_step_bwd(int32_t model, int32_t n, const float* S_in, const float* act, const float* dr,
                    const qs_task_cfg* cfg, const float* g_S_out, float* g_S_in, float* g_act,
                    void* stream) {
  if (n <= 0) return QS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int g = grid_for(n, 128);
  if (model == QS_MODEL_FULL)
    k_dyn_bwd<QS_MODEL_FULL><<<g, 128, 0, s>>>(n, S_in, act, dr, *cfg, g_S_out, g_S_in, g_act);
  else if (model == QS_MODEL_PM_CONTINUOUS)
    k_dyn_bwd<QS_MODEL_PM_CONTINUOUS><<<g, 128, 0, s>>>(n, S_in, act, dr, *cfg, g_S_out, g_S_in, g_act);
  else if (model == QS_MODEL_PM_DISCRETE)
    k_dyn_bwd<QS_MODEL_PM_DISCRETE><<<g, 128, 0, s>>>(n, S_in, act, dr, *cfg, g_S_out, g_S_in, g_act);
  else if (model == QS_MODEL_SIMPLIFIED)
    k_dyn_bwd<QS_MODEL_SIMPLIFIED><<<g, 128, 0, s>>>(n, S_in, act, dr, *cfg, g_S_out, g_S_in, g_act);
  else return QS_ERR_BAD_ARGUMENT;
  return status();
}

int qs_reconstruct_attitude(int32_t n, const float* a, const float* v_ema, float* R, void* stream) {
  if (n <= 0) return QS_OK;
  k_attitude<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(n, a, v_ema, R);
  return status();
}

int qs_td_lambda(int32_t T, int64_t n, const float* r, const float* values, const float* bootstrap,
                 const uint8_t* done, float gamma, float lam, float one_minus_lam, float* targets, void* stream) {
  if (T <= 0 || n <= 0) return QS_OK;
  if (!r || !values || !bootstrap || !done || !targets) return QS_ERR_BAD_ARGUMENT;
  k_td_lambda<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(T, n, r, values, bootstrap, done, gamma,
                                                                             lam, one_minus_lam, targets);
  return status();
}

}  // extern "C"
