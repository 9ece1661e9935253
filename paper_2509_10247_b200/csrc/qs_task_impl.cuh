// Fused env step (forward + analytic VJP), spawn and observe kernels.
//
// One thread owns one agent ROW; an env's rows sit in adjacent lanes (a lane
// group), so every per-env coupling of the reference step -- success needs all
// agents, bounds/collision any agent, the formation penalty, the shared reset
// -- is a shuffle within the group, and single-agent envs need none.  Reference: q/tasks.py:549-763, 817-844,
// 925-972; q/dynamics.py; q/sensors.py:417-611; q/world.py:409-448.
#pragma once
#include "qs_dynamics.cuh"
#include "qs_geom.cuh"

namespace qs {

constexpr int FLAG_DONE = 1;
constexpr int FLAG_CLAMP_SHIFT = 1;  // 9 bits: goal(3) gate0(3) gate1(3)
constexpr int FLAG_CLAMP_MASK = 0x1FF << FLAG_CLAMP_SHIFT;
constexpr int FLAG_SDF_SHIFT = 10;

template <int M, int TASK>
struct TaskTraits {
  static constexpr int A = ModelTraits<M>::A;
  static constexpr int P = ModelTraits<M>::P + (TASK == QS_TASK_RACING ? 9 : 0);
};

struct GateV {
  V3 c, n;
  float inner, frame;
};

QS_D GateV load_gate(const qs_scene& sc, const qs_task_cfg& cfg, long e, int g) {
  const float* p = sc.gates + (e * cfg.n_gates + g) * 8;
  float4 a = ld4(p, 0), b = ld4(p, 1);
  return GateV{xyz(a), xyz(b), a.w, b.w};
}

QS_D V3 load3(const float* p, long row) { return xyz(ld4(p, row)); }

QS_D V3 head_xy(V3 d) {  // q/tasks.py:705-708
  d.z = 0.f;
  float n = norm3(d);
  return d * (1.f / fmaxf(n, 1e-9f));
}

QS_D bool in_range(float x, float lo, float hi) { return x >= lo && x <= hi; }
QS_D float clampf(float x, float lo, float hi) { return fminf(fmaxf(x, lo), hi); }

// ---------------------------------------------------------------------------
// observation (q/tasks.py:415-442, racing extras :904-915)

template <int M, int TASK>
QS_D int observe_row(const qs_task_cfg& cfg, const State& s, float2 cs, V3 goal, const GateV* g0,
                     const GateV* g1, float* o) {
  const float clip = cfg.obs_clip;
  int bits = 0;
  V3 off = unrotz(cs, goal - s.p);
  o[0] = clampf(off.x, -clip, clip);
  o[1] = clampf(off.y, -clip, clip);
  o[2] = clampf(off.z, -clip, clip);
  bits |= (in_range(off.x, -clip, clip) ? 1 : 0) | (in_range(off.y, -clip, clip) ? 2 : 0) |
          (in_range(off.z, -clip, clip) ? 4 : 0);
  V3 vl = unrotz(cs, s.v);
  o[3] = vl.x;
  o[4] = vl.y;
  o[5] = vl.z;
  int k = 6;
  if (M == QS_MODEL_SIMPLIFIED) {  // body z axis = third column of R (q/tasks.py:431-432)
    V3 zl = unrotz(cs, s.r2);
    o[6] = zl.x;
    o[7] = zl.y;
    o[8] = zl.z;
    k = 9;
  } else if (M == QS_MODEL_FULL) {
    V3 zl = unrotz(cs, qaxis_z(s.q));
    o[6] = zl.x;
    o[7] = zl.y;
    o[8] = zl.z;
    o[9] = s.w.x;
    o[10] = s.w.y;
    o[11] = s.w.z;
    k = 12;
  } else {
    V3 xl = unrotz(cs, s.x);
    o[6] = xl.x;
    o[7] = xl.y;
    o[8] = xl.z;
    k = 9;
  }
  if (TASK == QS_TASK_RACING) {
    V3 a = unrotz(cs, g0->c - s.p);
    V3 nl = unrotz(cs, g0->n);
    V3 b = unrotz(cs, g1->c - s.p);
    o[k + 0] = clampf(a.x, -clip, clip);
    o[k + 1] = clampf(a.y, -clip, clip);
    o[k + 2] = clampf(a.z, -clip, clip);
    o[k + 3] = nl.x;
    o[k + 4] = nl.y;
    o[k + 5] = nl.z;
    o[k + 6] = clampf(b.x, -clip, clip);
    o[k + 7] = clampf(b.y, -clip, clip);
    o[k + 8] = clampf(b.z, -clip, clip);
    bits |= (in_range(a.x, -clip, clip) ? 8 : 0) | (in_range(a.y, -clip, clip) ? 16 : 0) |
            (in_range(a.z, -clip, clip) ? 32 : 0) | (in_range(b.x, -clip, clip) ? 64 : 0) |
            (in_range(b.y, -clip, clip) ? 128 : 0) | (in_range(b.z, -clip, clip) ? 256 : 0);
  }
  return bits << FLAG_CLAMP_SHIFT;
}

template <int M, int TASK>
QS_D void write_obs(const qs_task_cfg& cfg, const qs_step_io& io, long row, const float* o) {
  constexpr int P = TaskTraits<M, TASK>::P;
  float* dst = io.obs + row * P;
#pragma unroll
  for (int k = 0; k < P; ++k) dst[k] = o[k];
}

// ---------------------------------------------------------------------------
// lane groups.  An env's agent rows live in G adjacent lanes (G = 1, 2, 4, 8,
// the power of two >= n_agents); lane g of a group owns agent row g, so each
// thread carries ONE row's registers.  Per-env couplings (all-agent success,
// any-agent bounds/collision, the formation penalty and its VJP, the shared
// reset) are group shuffles.  Lanes g >= n_agents (padding, when n_agents is
// not a power of two) mirror agent 0, contribute neutral values and write
// nothing.  G = 1 compiles every group operation away.

template <int G>
struct Grp {
  unsigned mask;  // this group's lanes in the warp
  int g;          // agent index of this lane
  bool real;      // g < n_agents
  QS_D static Grp make(int na) {
    Grp r;
    const int lane = threadIdx.x & 31;
    r.g = G == 1 ? 0 : (lane & (G - 1));
    r.mask = G == 1 ? 0u : (((1u << G) - 1u) << (lane & ~(G - 1)));
    r.real = r.g < na;
    return r;
  }
  QS_D float sum(float v) const {
#pragma unroll
    for (int o = 1; o < G; o <<= 1) v += __shfl_xor_sync(mask, v, o, G);
    return v;
  }
  QS_D bool any(bool b) const {
    int v = b;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) v |= __shfl_xor_sync(mask, v, o, G);
    return v != 0;
  }
  QS_D bool all(bool b) const {
    int v = b;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) v &= __shfl_xor_sync(mask, v, o, G);
    return v != 0;
  }
  QS_D float bcast(float v, int src) const { return G == 1 ? v : __shfl_sync(mask, v, src, G); }
  QS_D V3 bcast(V3 v, int src) const { return v3(bcast(v.x, src), bcast(v.y, src), bcast(v.z, src)); }
};

// ---------------------------------------------------------------------------
// resets: in-kernel Philox sampling (q/tasks.py:676-710, 789-815, 873-902;
// q/world.py:130-137, 409-448).  Keys: (seed, global env id, episode index).
// One stream per env; the agents' draws sit at fixed counter offsets, so each
// lane computes exactly the draws its agent takes in the reference's order.

// blo/bhi: the env's bounds shrunk by 1e-6 (EnvRegs keeps them in registers;
// the spawn margins below are taken from the shrunk bounds, so every caller
// draws identical spawns without a global load on the reset path)
template <int M, int TASK, int G>
QS_D bool spawn_sample(const qs_task_cfg& cfg, const qs_scene& sc, long e, int episode, int na, V3 blo,
                       V3 bhi, const Grp<G>& grp, V3& p, V3& v, V3& goal, V3& head, int& next_gate) {
  const uint64_t gid = (uint64_t)(e + cfg.env_offset);
  RngK rng(cfg.rng_round_keys, gid, (uint32_t)episode, RNG_SPAWN);
  const uint32_t c0 = rng.ctr.w;
  const V3 lo = blo, hi = bhi;
  const int ag = grp.real ? grp.g : 0;
  const V3 f = v3(cfg.formation[ag][0], cfg.formation[ag][1], cfg.formation[ag][2]);
  bool ok = true;
  next_gate = 0;
  if (TASK == QS_TASK_POSITION) {
    // the shared spawn/goal pair: every lane runs the same rejection loop
    V3 l8 = lo + v3(0.8f, 0.8f, 0.8f), h8 = hi - v3(0.8f, 0.8f, 0.8f);
    V3 sp = l8, gl = l8;
    ok = false;
    // one Philox block per candidate pair: six 16-bit uniforms (a 2^-16 grid,
    // ~0.2 mm over these courses), so a rejection try costs one block
    for (int t = 0; t < 100 && !ok; ++t) {
      const uint4 r = rng.bits4();
      sp = l8 + hmul(h8 - l8, v3(u16(r.x), u16(r.x >> 16), u16(r.y)));
      gl = l8 + hmul(h8 - l8, v3(u16(r.y >> 16), u16(r.z), u16(r.z >> 16)));
      float d = norm3(gl - sp);
      ok = d >= 2.5f && d <= cfg.goal_dist;
    }
    rng.ctr.w += (uint32_t)ag;  // agent a's six spawn normals: block a after the pair
    float4 n0, n1;
    normals6(rng.bits4(), n0, n1);
    p = sp + f + v3(n0.x, n0.y, n0.z) * 0.1f;
    v = v3(n0.w, n1.x, n1.y) * 0.3f;
    goal = gl + f;
    head = head_xy(gl - sp);
  } else if (TASK == QS_TASK_AVOIDANCE) {
    V3 ssp = load3(sc.spawn_goal, 2 * e), sgl = load3(sc.spawn_goal, 2 * e + 1);
    SceneView sv = scene_view(sc, e);
    ok = false;
    int t = 0;
    for (; t < 100 && !ok; ++t) {
      rng.ctr.w = c0 + (uint32_t)(t * na + ag);  // try t: one normal4 per agent, in agent order
      float4 n0 = rng.normal4();
      V3 q = ssp + f + v3(n0.x, n0.y, n0.z) * 0.15f;
      q.z = clampf(q.z, lo.z + 0.3f, hi.z - 0.3f);
      p = q;
      bool good = true;
      if (G > 1) {  // pairwise separation (q/world.py:433-437)
#pragma unroll
        for (int j = 0; j < G; ++j) {
          V3 pj = grp.bcast(q, j);
          if (j > grp.g && j < na) good = good && norm3(q - pj) >= cfg.d_min;
        }
      }
      int code;
      good = good && sdf_eval(sv, q, code) > cfg.collision_radius + 0.3f;
      good = good && q.x > lo.x + 0.2f && q.y > lo.y + 0.2f && q.z > lo.z + 0.2f && q.x < hi.x - 0.2f &&
             q.y < hi.y - 0.2f && q.z < hi.z - 0.2f;
      ok = grp.all(good || !grp.real);
    }
    rng.ctr.w = c0 + (uint32_t)(t * na);
    float4 nj = rng.normal4();  // shared goal jitter
    V3 jit = v3(nj.x, nj.y, nj.z) * 0.2f;
    rng.ctr.w = c0 + (uint32_t)(t * na + 1 + ag);
    float4 n1 = rng.normal4();
    v = v3(n1.x, n1.y, n1.z) * 0.2f;
    goal = sgl + f + jit;
    head = head_xy(sgl - ssp);
  } else {  // racing, single agent
    V3 ssp = load3(sc.spawn_goal, 2 * e);
    float4 n0 = rng.normal4(), n1 = rng.normal4();
    p = ssp + v3(n0.x, n0.y, n0.z) * 0.2f;
    v = v3(n0.w, n1.x, n1.y) * 0.2f;
    GateV g0 = load_gate(sc, cfg, e, 0);
    goal = g0.c;
    head = head_xy(g0.c - ssp);
  }
  return ok;
}

QS_D float4 dr_sample(const qs_task_cfg& cfg, long row, int episode) {
  RngK rng(cfg.rng_round_keys, (uint64_t)(row + cfg.env_offset * cfg.n_agents), (uint32_t)episode, RNG_DR);
  float4 u = rng.uniform4();
  float drag = cfg.dr_drag[0] + (cfg.dr_drag[1] - cfg.dr_drag[0]) * u.x;
  float lat = cfg.dr_latency[0] + (cfg.dr_latency[1] - cfg.dr_latency[0]) * u.y;
  float scale = cfg.dr_scale[0] + (cfg.dr_scale[1] - cfg.dr_scale[0]) * u.z;
  return make_float4(drag, expf(-lat * cfg.dt), scale, lat);
}

// ---------------------------------------------------------------------------
// IMU read (q/sensors.py:540-555) on the post-dynamics state.  Bias state lives
// in registers (ba, bg); noise is injected (noise != NULL, (4,N,3)) or Philox.

// the 12 Philox normals of one row-step: bias walks (accel, gyro), then white
// noise (accel, gyro).  Independent of the state, so the window kernel draws
// them at the top of the step where they fill the dynamics' dependency stalls.
struct ImuNoise {
  float4 a, b, c;
};
QS_D ImuNoise imu_draw(const qs_task_cfg& cfg, long row, int tick) {
  RngK rng(cfg.rng_round_keys, (uint64_t)(row + cfg.env_offset * cfg.n_agents), (uint32_t)tick, RNG_IMU);
  ImuNoise z;
  const uint4 a = rng.bits4_r7(), b = rng.bits4_r7();  // Philox4x32-7: sensor noise
  normals12(a, b, z.a, z.b, z.c);
  return z;
}

template <int M>
QS_D void imu_apply_z(const qs_task_cfg& cfg, long row, const State& s2, V3 vdot, V3 g, float4& b0, float4& b1,
                      V3 nba, V3 nbg, V3 na, V3 ng, float* out);

template <int M>
QS_D void imu_apply(const qs_task_cfg& cfg, long row, long N, int tick, const State& s2, V3 vdot, V3 g,
                    float4& b0, float4& b1, const float* noise, float* out) {
  V3 nba, nbg, na, ng;
  if (noise) {
    const float* z = noise;
    nba = v3(z[3 * row], z[3 * row + 1], z[3 * row + 2]);
    nbg = v3(z[3 * (N + row)], z[3 * (N + row) + 1], z[3 * (N + row) + 2]);
    na = v3(z[3 * (2 * N + row)], z[3 * (2 * N + row) + 1], z[3 * (2 * N + row) + 2]);
    ng = v3(z[3 * (3 * N + row)], z[3 * (3 * N + row) + 1], z[3 * (3 * N + row) + 2]);
  } else {
    ImuNoise z = imu_draw(cfg, row, tick);
    nba = v3(z.a.x, z.a.y, z.a.z);
    nbg = v3(z.a.w, z.b.x, z.b.y);
    na = v3(z.b.z, z.b.w, z.c.x);
    ng = v3(z.c.y, z.c.z, z.c.w);
  }
  imu_apply_z<M>(cfg, row, s2, vdot, g, b0, b1, nba, nbg, na, ng, out);
}

template <int M>
QS_D void imu_apply_z(const qs_task_cfg& cfg, long row, const State& s2, V3 vdot, V3 g, float4& b0, float4& b1,
                      V3 nba, V3 nbg, V3 na, V3 ng, float* out) {
  V3 ba = xyz(b0), bg = xyz(b1);
  const float sq = cfg.imu_sqrt_dt;
  ba += nba * (cfg.imu_accel_rw * sq);
  bg += nbg * (cfg.imu_gyro_rw * sq);
  V3 xb, yb, zb;
  V3 w = v3(0.f, 0.f, 0.f);
  if (M == QS_MODEL_FULL) {  // columns of quat_to_matrix (q/dynamics.py:448-460)
    const Q4 q = s2.q;
    const float xx = q.x * q.x, yy = q.y * q.y, zz = q.z * q.z;
    const float xy = q.x * q.y, xz = q.x * q.z, yz = q.y * q.z;
    const float wx = q.w * q.x, wy = q.w * q.y, wz = q.w * q.z;
    xb = v3(1.f - 2.f * (yy + zz), 2.f * (xy + wz), 2.f * (xz - wy));
    yb = v3(2.f * (xy - wz), 1.f - 2.f * (xx + zz), 2.f * (yz + wx));
    zb = v3(2.f * (xz + wy), 2.f * (yz - wx), 1.f - 2.f * (xx + yy));
    w = s2.w;
  } else if (M == QS_MODEL_SIMPLIFIED) {  // no rate state: gyro reads bias + noise
    xb = s2.r0;
    yb = s2.r1;
    zb = s2.r2;
  } else {
    attitude_pm(thrust_of<M>(s2, g), s2.ve, xb, yb, zb);
  }
  V3 sp = vdot - g;
  V3 acc = v3(dot(xb, sp), dot(yb, sp), dot(zb, sp)) + ba;
  if (cfg.imu_accel_std != 0.f) acc += na * cfg.imu_accel_std;
  V3 gy = w + bg;
  if (cfg.imu_gyro_std != 0.f) gy += ng * cfg.imu_gyro_std;
  b0 = f4(ba, 0.f);
  b1 = f4(bg, 0.f);
  float* o = out;  // 6 floats: accel xyz, gyro xyz
  o[0] = acc.x; o[1] = acc.y; o[2] = acc.z;
  o[3] = gy.x; o[4] = gy.y; o[5] = gy.z;
}


// ---------------------------------------------------------------------------
// rewards (q/tasks.py:144-170, 625-637, 744-763, 817-844)

struct RewardFwd {
  float r, dist, speed, nearv, track;
};

QS_D RewardFwd reward_ctrl(const qs_weights& w, V3 off, V3 v, float effn, float deffn) {
  float dist = norm3(off);
  float speed = norm3(v);
  float nearv = sigmoid_stable((w.near_radius - dist) * (1.f / w.near_width));
  float sd = fminf(dist * w.track_gain, w.v_max);
  V3 vdes = off * __fdividef(sd, fmaxf(dist, 1e-9f));
  float track = norm3(v - vdes);
  float pen = dist * w.w_p;
  pen = pen + (speed * nearv) * w.w_v;
  pen = pen + effn * w.w_a;
  pen = pen + deffn * w.w_s;
  pen = pen + track * w.w_t;
  return RewardFwd{-pen, dist, speed, nearv, track};
}

// RL scalar (q/tasks.py:744-763): never differentiated, so the divisions use
// the 2-ulp fast path
QS_D float reward_rl(const qs_weights& w, float clip, V3 off, V3 v, float effn, float deffn) {
  float dist = norm3(off);
  float speed = norm3(v);
  float nearv = sigmoid_stable((w.near_radius - dist) * (1.f / w.near_width));  // exp overflow -> 0
  float sd = fminf(dist * w.track_gain, w.v_max);
  V3 vdes = off * __fdividef(sd, fmaxf(dist, 1e-9f));
  float track = norm3(v - vdes);
  float dist_c = fminf(dist, clip);
  return -(w.w_p * dist_c + w.w_v * speed * nearv + w.w_a * effn + w.w_s * deffn + w.w_t * track);
}

// the same RL scalar from reward_ctrl's terms: when the RL weights share the
// control weights' shape parameters (near radius/width, tracking gain, v_max
// -- the reference's defaults), dist, speed, near and track are the identical
// fp32 values, so only the weighted sum is recomputed
QS_D bool rl_shares_shape(const qs_weights& w, const qs_weights& wr) {
  return w.near_radius == wr.near_radius && w.near_width == wr.near_width && w.track_gain == wr.track_gain &&
         w.v_max == wr.v_max;
}
QS_D float reward_rl_from(const qs_weights& w, float clip, const RewardFwd& rf, float effn, float deffn) {
  const float dist_c = fminf(rf.dist, clip);
  return -(w.w_p * dist_c + w.w_v * rf.speed * rf.nearv + w.w_a * effn + w.w_s * deffn + w.w_t * rf.track);
}

// VJP of reward_ctrl: returns grads wrt off, v, effort vec, d_effort vec
QS_D void reward_ctrl_vjp(const qs_weights& w, V3 off, V3 v, float4 eff, float4 deff, int A, float g,
                          V3& g_off, V3& g_v, float4& g_eff) {
  float dist = norm3(off);
  float speed = norm3(v);
  float x = (w.near_radius - dist) * (1.f / w.near_width);
  float nearv = sigmoid_stable(x);
  float m = fmaxf(dist, 1e-9f);
  float sd = fminf(dist * w.track_gain, w.v_max);
  const float im = __fdividef(1.f, m);
  float kk = sd * im;
  V3 vdes = off * kk;
  V3 ev = v - vdes;
  float track = norm3(ev);
  float gp = -g;  // r = -pen
  float g_dist = gp * w.w_p;
  float g_speed = gp * w.w_v * nearv;
  float g_near = gp * w.w_v * speed;
  g_dist += g_near * nearv * (1.f - nearv) * (-1.f / w.near_width);
  float g_track = gp * w.w_t;
  // track = |v - off*k|
  V3 gev = norm_vjp(ev, track, g_track);
  g_v = gev + norm_vjp(v, speed, g_speed);
  V3 g_vdes = -gev;
  g_off = g_vdes * kk;
  float g_k = dot(g_vdes, off);
  float g_sd = g_k * im;
  float g_m = -g_k * kk * im;
  if (dist * w.track_gain <= w.v_max) g_dist += g_sd * w.track_gain;  // minimum: tie -> first
  if (dist >= 1e-9f) g_dist += g_m;                                   // maximum: tie -> first
  g_off += norm_vjp(off, dist, g_dist);
  // effort norms
  float en = sqrt_mufu(eff.x * eff.x + eff.y * eff.y + eff.z * eff.z + (A == 4 ? eff.w * eff.w : 0.f));
  float dn = sqrt_mufu(deff.x * deff.x + deff.y * deff.y + deff.z * deff.z +
                       (A == 4 ? deff.w * deff.w : 0.f));
  float ca = en > 0.f ? __fdividef(gp * w.w_a, en) : 0.f;
  float cs = dn > 0.f ? __fdividef(gp * w.w_s, dn) : 0.f;
  g_eff = make_float4(eff.x * ca + deff.x * cs, eff.y * ca + deff.y * cs, eff.z * ca + deff.z * cs,
                      A == 4 ? eff.w * ca + deff.w * cs : 0.f);
}

QS_D float f4get(float4 v, int k) { return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w; }
QS_D void f4set(float4& v, int k, float x) {
  if (k == 0) v.x = x; else if (k == 1) v.y = x; else if (k == 2) v.z = x; else v.w = x;
}

template <int A>
QS_D float4 load_act(const float* raw, long row) {
  if (A == 4) return ld4(raw, row);  // 16-byte rows: one vector load
  const float* p = raw + row * A;
  return make_float4(__ldg(p), __ldg(p + 1), __ldg(p + 2), 0.f);
}

template <int A>
QS_D bool act_finite(float4 a) {
  return isfinite(a.x) && isfinite(a.y) && isfinite(a.z) && (A < 4 || isfinite(a.w));
}

struct Squash {
  float4 t, sq, eff;
};

template <int A>
QS_D Squash squash(float4 raw, const RowPrm& rp) {  // q/dynamics.py:277-284
  Squash s;
  s.t = make_float4(tanh_fast(raw.x), tanh_fast(raw.y), tanh_fast(raw.z), A == 4 ? tanh_fast(raw.w) : 0.f);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k < A) {
      float sq = rp.center[k] + rp.half[k] * f4get(s.t, k);
      f4set(s.sq, k, sq);
      f4set(s.eff, k, sq - rp.center[k]);  // q/tasks.py:568
    } else {
      f4set(s.sq, k, 0.f);
      f4set(s.eff, k, 0.f);
    }
  }
  return s;
}

template <int M>
QS_D float4 world_cmd(const State& s, float4 sq, V3 g, float2& cs) {  // q/tasks.py:613-618
  if (M == QS_MODEL_FULL || M == QS_MODEL_SIMPLIFIED) {  // only point-mass commands are yaw-local
    cs = make_float2(1.f, 0.f);
    return sq;
  }
  cs = yaw_cs<M>(s, g);
  V3 c = rotz(cs, v3(sq.x, sq.y, sq.z));
  return make_float4(c.x, c.y, c.z, 0.f);
}

QS_D float effnorm(float4 e, int A) {
  return sqrt_mufu(e.x * e.x + e.y * e.y + e.z * e.z + (A == 4 ? e.w * e.w : 0.f));
}

QS_D void warp_stats(bool active, bool done, int term, float ret, double* stats) {
  unsigned m = __ballot_sync(0xffffffffu, active && done);
  if (!m) return;
  unsigned ms = __ballot_sync(0xffffffffu, active && done && term == 1);
  unsigned mc = __ballot_sync(0xffffffffu, active && done && term == 2);
  double r = (active && done) ? (double)ret : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  if ((threadIdx.x & 31) == 0 && stats) {
    atomicAdd(stats + 0, (double)__popc(m));
    atomicAdd(stats + 1, (double)__popc(ms));
    atomicAdd(stats + 2, (double)__popc(mc));
    atomicAdd(stats + 3, r);
  }
}

// ---------------------------------------------------------------------------
// per-row register file: everything one agent row carries from step to step
// (meta / ep_ret / bounds are the env's, replicated across its group)

struct EnvRegs {
  State s;
  float4 goal, peff, dr;
  float4 ba, bg;  // IMU bias (accel, gyro)
  int4 meta;      // steps_in_episode, episode, tick, next_gate
  float ep_ret;
  V3 blo, bhi;    // bounds shrunk by 1e-6 (q/tasks.py:673-674)
};

// pointers of one step's outputs (rows are env-major, N = n_envs * n_agents)
struct StepOut {
  float* obs;
  float* r_ctrl;
  float* r_goal;
  float* r_rl;
  int8_t* term;
  uint8_t* trunc;
  int32_t* flags;
  float* cam;
  float* imu_out;
  const float* imu_noise;
};

template <int M>
QS_D RowPrm row_params_v(const qs_task_cfg& cfg, bool has_dr, float4 d) {
  RowPrm r;
  float scale = 1.f;
  r.drag = cfg.drag_coeff;
  r.decay = cfg.lag_decay;
  if (has_dr) {
    r.drag = d.x;
    r.decay = d.y;
    scale = d.z;
  }
#pragma unroll
  for (int k = 0; k < ModelTraits<M>::A; ++k) {
    if (has_dr) {  // q/tasks.py:370-375
      const float c = cfg.act_center[k], h = cfg.act_half[k];
      const float lo = c - h * scale, hi = c + h * scale;
      r.center[k] = (lo + hi) * 0.5f;
      r.half[k] = (hi - lo) * 0.5f;
    } else {  // host-precomputed: no per-step arithmetic
      r.center[k] = cfg.act_center[k];
      r.half[k] = cfg.act_half[k];
    }
  }
  return r;
}

template <int M>
QS_D void env_load(const float* sc_bounds, long e, long row, long N, EnvRegs& R, const float* S,
                   const float* goal, const float* peff, const float* dr, const int32_t* meta,
                   const float* ep_ret, const float* bias) {
  R.meta = reinterpret_cast<const int4*>(meta)[e];
  R.ep_ret = ep_ret[e];
  R.blo = xyz(ld4(sc_bounds, 2 * e)) + v3(1e-6f, 1e-6f, 1e-6f);
  R.bhi = xyz(ld4(sc_bounds, 2 * e + 1)) - v3(1e-6f, 1e-6f, 1e-6f);
  R.s = load_state<M>(S, N, row);
  R.goal = ld4(goal, row);
  R.peff = ld4(peff, row);
  R.dr = dr ? ld4(dr, row) : make_float4(0.f, 0.f, 0.f, 0.f);
  if (bias) {
    R.ba = ld4(bias, 2 * row);
    R.bg = ld4(bias, 2 * row + 1);
  }
}

// the functional (checkpointed) part of the register file
template <int M>
QS_D void env_store_ckpt(long row, long N, const EnvRegs& R, float* S, float* goal, float* peff, float* dr) {
  store_state<M>(S, N, row, R.s);
  st4(goal, row, R.goal);
  st4(peff, row, R.peff);
  if (dr) st4(dr, row, R.dr);
}

// the in-place part (env counters by the group's lane 0)
QS_D void env_store_inplace(long e, long row, bool lead, const EnvRegs& R, int32_t* meta, float* ep_ret,
                            float* bias) {
  if (lead) {
    reinterpret_cast<int4*>(meta)[e] = R.meta;
    ep_ret[e] = R.ep_ret;
  }
  if (bias) {
    st4(bias, 2 * row, R.ba);
    st4(bias, 2 * row + 1, R.bg);
  }
}

struct StepStat {
  bool done;
  int term;
  float ret;
  float rc;  // this row's r_ctrl (0 for padding lanes)
};

// spawn-ahead (fused windows): a row's NEXT reset sample -- spawn, velocity,
// goal, heading, DR draw for episode meta.y + 1 -- is drawn before the window's
// step loop, with every lane of the warp in lockstep, and parked in shared
// memory.  The draw is a pure function of (seed, global env, episode), so the
// in-loop reset reads exactly the values the inline draw would produce, while
// the warp no longer runs the divergent rejection-sampling path whenever one
// of its lanes resets.  A second reset of the same row inside the window
// (episode no longer matches) falls back to the inline draw.
struct SpawnAhead {
  float4* slot;  // 4 float4 with stride `stride`: (p, head.x) (v, head.y) (goal, ok) (dr)
  int stride;
  int episode;   // episode index the slot holds; -1 once consumed
};

// ---------------------------------------------------------------------------
// one fused env step of one agent row (FlightTask.step, q/tasks.py:549-600);
// IMU: 0 = decided at run time by has_imu / out.imu_noise; 1 = Philox IMU on
// (compile time), its normals drawn at the top of the step

template <int M, int TASK, int G, bool INLINE, int IMU = 0>
QS_D StepStat env_step_fwd(const qs_task_cfg& cfg, const qs_scene& sc, long e, long row, int na, long N,
                           const Grp<G>& grp, EnvRegs& R, float4 raw, const StepOut& out, int32_t* err,
                           bool has_dr, bool has_imu, SpawnAhead* ahead = nullptr, float* obs_stage = nullptr) {
  constexpr int A = ModelTraits<M>::A;
  constexpr int P = TaskTraits<M, TASK>::P;
  const DynK k = dyn_consts(cfg);
  if (IMU == 1) has_imu = true;
  const bool real = grp.real;
  SceneView sv;
  if (TASK == QS_TASK_AVOIDANCE) sv = scene_view(sc, e);
  const V3 blo = R.blo, bhi = R.bhi;
  const State& s = R.s;
  RowPrm rp = row_params_v<M>(cfg, has_dr, R.dr);
  ImuNoise z;
  if (IMU == 1) z = imu_draw(cfg, row, R.meta.z);
  {
    const int c = !act_finite<A>(raw) ? QS_ERR_NONFINITE_ACTION
                                      : (!state_finite<M>(s) ? QS_ERR_NONFINITE_STATE : 0);
    if (c != 0 && real) report_err(err, c, (int)row);
  }
  Squash q = squash<A>(raw, rp);
  float2 cs;
  float4 cmd = world_cmd<M>(s, q.sq, k.g, cs);
  State n = model_step<M>(s, cmd, rp, k);
  n.ve = s.ve * (1.f - cfg.yaw_ema_alpha) + n.v * cfg.yaw_ema_alpha;  // q/sensors.py:566
  float4 ba = R.ba, bg = R.bg;
  float imu[6];
  if (IMU == 1)
    imu_apply_z<M>(cfg, row, n, (n.v - s.v) * (1.f / cfg.dt), k.g, ba, bg, v3(z.a.x, z.a.y, z.a.z),
                   v3(z.a.w, z.b.x, z.b.y), v3(z.b.z, z.b.w, z.c.x), v3(z.c.y, z.c.z, z.c.w), imu);
  else if (has_imu)
    imu_apply<M>(cfg, row, N, R.meta.z, n, (n.v - s.v) * (1.f / cfg.dt), k.g, ba, bg, out.imu_noise, imu);
  if (has_imu && real) {
    float* o = out.imu_out + 6 * row;
    if ((reinterpret_cast<uintptr_t>(o) & 7) == 0) {  // 3 x 8-byte stores
      float2* o2 = reinterpret_cast<float2*>(o);
      o2[0] = make_float2(imu[0], imu[1]);
      o2[1] = make_float2(imu[2], imu[3]);
      o2[2] = make_float2(imu[4], imu[5]);
    } else {
      o[0] = imu[0]; o[1] = imu[1]; o[2] = imu[2];
      o[3] = imu[3]; o[4] = imu[4]; o[5] = imu[5];
    }
  }
  R.ba = ba;
  R.bg = bg;
  const float4 pe = R.peff;
  float4 de = make_float4(q.eff.x - pe.x, q.eff.y - pe.y, q.eff.z - pe.z, q.eff.w - pe.w);
  float en = effnorm(q.eff, A), dn = effnorm(de, A);
  R.peff = q.eff;  // q/tasks.py:570
  int code = 0;
  float rc = 0.f, rl = 0.f;
  bool goal_ok = true, coll = false;
  if (TASK != QS_TASK_RACING) {
    V3 off = xyz(R.goal) - n.p;
    RewardFwd rf = reward_ctrl(cfg.w, off, n.v, en, dn);
    float extra = 0.f;
    if (TASK == QS_TASK_AVOIDANCE) {
      float sd = sdf_eval(sv, n.p, code);
      rf.r -= cfg.w.w_o * softplus((cfg.d_safe - sd) * (1.f / cfg.w.sdf_sharpness));
      coll = sd <= cfg.collision_radius;
      extra = -(cfg.w_rl.w_o * softplus((cfg.d_safe - sd) / cfg.w_rl.sdf_sharpness));
    }
    rc = rf.r;
    rl = (rl_shares_shape(cfg.w, cfg.w_rl) ? reward_rl_from(cfg.w_rl, cfg.obs_clip, rf, en, dn)
                                           : reward_rl(cfg.w_rl, cfg.obs_clip, off, n.v, en, dn)) +
         extra;
    goal_ok = (rf.dist < cfg.success_radius) && (rf.speed < cfg.hover_speed);
  }
  const bool oob = n.p.x < blo.x || n.p.y < blo.y || n.p.z < blo.z || n.p.x > bhi.x || n.p.y > bhi.y ||
                   n.p.z > bhi.z;
  // ---- per-env couplings
  int term_env = 0;
  float r_goal = 0.f;
  int next_gate = R.meta.w;
  if (TASK == QS_TASK_RACING) {  // q/tasks.py:925-972 (single agent)
    const qs_weights& w = cfg.w_rl;
    const V3 p0 = s.p;
    GateV gt = load_gate(sc, cfg, e, next_gate);
    V3 p1 = n.p;
    float r = w.w_g * (norm3(p0 - gt.c) - norm3(p1 - gt.c));
    float sa = dot(p0 - gt.c, gt.n), sb = dot(p1 - gt.c, gt.n);
    if (sa < 0.f && sb >= 0.f) {
      float frac = -sa / fmaxf(sb - sa, 1e-12f);
      V3 x = p0 + (p1 - p0) * frac;
      V3 xc = x - gt.c;
      float radial = norm3(xc - gt.n * dot(xc, gt.n));
      bool passed = radial < gt.inner;
      bool crashed = !passed && radial < gt.inner + gt.frame;
      if (passed) r += w.gate_pass_bonus;
      if (crashed) {
        r -= w.gate_crash_penalty;
        term_env = 2;
        r_goal = -1.f;
      }
      bool finished = passed && next_gate == cfg.n_gates - 1;
      if (finished) {
        term_env = 1;
        r_goal = 1.f;
      }
      if (passed && !finished) {
        next_gate += 1;
        R.goal = f4(load_gate(sc, cfg, e, next_gate).c, 0.f);
      }
    }
    if (oob && term_env == 0) {
      term_env = 3;
      r_goal = -1.f;
      r -= w.goal_bonus;
    }
    rc = 0.f;
    rl = r;
  } else {
    bool all_goal = grp.all(goal_ok || !real);
    bool any_oob = grp.any(oob && real);
    bool any_coll = grp.any(coll && real);
    if (G > 1 && na > 1) {  // formation penalty + inter-agent collision (q/tasks.py:173-192)
      float part = 0.f;
      bool close = false;
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const V3 pj = grp.bcast(n.p, j);
        if (real && j > grp.g && j < na) {
          float dij = norm3(n.p - pj);
          float t = dij - cfg.form_ref[grp.g][j];
          part = part + t * t;
          close = close || dij < cfg.d_min;
        }
      }
      const float pen = grp.sum(part) * cfg.w.w_f;
      any_coll = any_coll || grp.any(close);
      rc -= pen;
    }
    // precedence: success, then bounds, then collision overwrite (q/tasks.py:734-737)
    if (all_goal) term_env = 1;
    if (any_oob) term_env = 3;
    if (any_coll) term_env = 2;
    r_goal = term_env == 1 ? 1.f : (term_env != 0 ? -1.f : 0.f);
    rl = rl + cfg.w_rl.goal_bonus * r_goal;
  }
  // ---- counters, truncation (q/tasks.py:574-591, 606-611); the return is agent 0's
  int steps = R.meta.x + 1;
  const bool trunc = steps >= cfg.episode_len && term_env == 0;
  const bool done = term_env != 0 || trunc;
  const float ret = R.ep_ret + grp.bcast(rl, 0);
  int episode = R.meta.y;
  if (done) {
    steps = 0;
    episode += 1;
    R.ep_ret = 0.f;
    next_gate = 0;
  } else {
    R.ep_ret = ret;
  }
  R.meta = make_int4(steps, episode, R.meta.z + 1, next_gate);
  // ---- auto-reset (inline Philox) or keep
  State so = n;
  if (done) {
    R.peff = make_float4(0.f, 0.f, 0.f, 0.f);
    if (has_imu) {
      R.ba = make_float4(0.f, 0.f, 0.f, 0.f);
      R.bg = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (INLINE) {
      V3 sp, sv_, sg, head;
      bool ok;
      const bool dr_new = cfg.dr_enabled && cfg.dr_per_episode;
      if (ahead && ahead->episode == episode) {  // env-uniform: the group takes the same branch
        const float4 a = ahead->slot[0], b = ahead->slot[ahead->stride], c = ahead->slot[2 * ahead->stride];
        sp = xyz(a);
        sv_ = xyz(b);
        sg = xyz(c);
        head = v3(a.w, b.w, 0.f);
        ok = c.w != 0.f;
        if (dr_new) R.dr = ahead->slot[3 * ahead->stride];
        ahead->episode = -1;
      } else {
        int ng0;
        ok = spawn_sample<M, TASK, G>(cfg, sc, e, episode, na, R.blo, R.bhi, grp, sp, sv_, sg, head, ng0);
        if (dr_new) R.dr = dr_sample(cfg, row, episode);
      }
      if (!ok && grp.g == 0) report_err(err, QS_ERR_GENERATION, (int)(e * na));
      so = init_state<M>(sp, sv_, head, k.g);
      R.goal = f4(sg, 0.f);
    }
  }
  R.s = so;
  int fl = (done ? FLAG_DONE : 0) | (code << FLAG_SDF_SHIFT);
  if (INLINE && out.obs) {
    GateV g0, g1;
    if (TASK == QS_TASK_RACING) {
      int ngate = done ? 0 : next_gate;
      g0 = load_gate(sc, cfg, e, ngate);
      g1 = load_gate(sc, cfg, e, min(ngate + 1, cfg.n_gates - 1));
    }
    float o[P];
    float2 cs2 = yaw_cs<M>(so, k.g);
    fl |= observe_row<M, TASK>(cfg, so, cs2, xyz(R.goal), &g0, &g1, o);
    if (real) {
      float* dst = out.obs + row * P;
      if (P % 4 == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {  // 16-byte stores
        float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
        for (int kk = 0; kk < P / 4; ++kk) d4[kk] = make_float4(o[4 * kk], o[4 * kk + 1], o[4 * kk + 2], o[4 * kk + 3]);
      } else if (G == 1 && obs_stage) {
        // rows of P (not a multiple of 4) floats: through this warp's shared
        // staging buffer, so the warp's consecutive rows leave as one coalesced
        // run (per-lane scalar rows touched ~8x the sectors they wrote)
        // the lanes stepping rows are the prefix of the warp with row < N
        const int lane = threadIdx.x & 31;
        const long left = N - (row - lane);
        const unsigned m = left >= 32 ? 0xffffffffu : ((1u << left) - 1u);
#pragma unroll
        for (int kk = 0; kk < P; ++kk) obs_stage[lane * P + kk] = o[kk];
        __syncwarp(m);
        float* base = out.obs + (row - lane) * P;
        const int nl = __popc(m), nv = nl * P;  // only the nl stepping lanes copy
        for (int i = lane; i < nv; i += nl) base[i] = obs_stage[i];
        __syncwarp(m);  // the buffer is reused by the next step
      } else {
#pragma unroll
        for (int kk = 0; kk < P; ++kk) dst[kk] = o[kk];
      }
      if (out.cam) reinterpret_cast<float2*>(out.cam)[row] = cs2;
    }
  }
  if (real) {
    out.r_ctrl[row] = rc;
    out.r_goal[row] = r_goal;
    out.r_rl[row] = rl;
    out.term[row] = (int8_t)term_env;
    out.trunc[row] = trunc ? 1 : 0;
    out.flags[row] = fl;
  }
  return StepStat{done, term_env, ret, real ? rc : 0.f};
}

// ---------------------------------------------------------------------------
// analytic VJP of one agent row's step.  Inputs: the step's checkpoint
// (pre-step state s, raw action, goal, previous effort, per-row params,
// flags), the upstream grad of the post-step state (gS, in/out: replaced by
// the grad of s), of the observation (g_obs, may be NULL) and of r_ctrl (per
// row or a scalar).  The formation penalty's VJP is the group's only coupling.

template <int M, int TASK, int G>
QS_D void env_step_bwd(const qs_task_cfg& cfg, const qs_scene& sc, long e, long row, int na, long N,
                       const Grp<G>& grp, const State& s, float4 raw, float4 goal, float4 peff, float4 dr,
                       bool has_dr, int fl, const float* g_obs, const float* g_r_rows, float g_r_scalar, State& gS,
                       float* g_raw_t, const State* s2_known = nullptr) {
  constexpr int A = ModelTraits<M>::A;
  constexpr int P = TaskTraits<M, TASK>::P;
  const DynK k = dyn_consts(cfg);
  const bool real = grp.real;
  SceneView sv;
  if (TASK == QS_TASK_AVOIDANCE) sv = scene_view(sc, e);
  RowPrm rp = row_params_v<M>(cfg, has_dr, dr);
  Squash q = squash<A>(raw, rp);
  float2 cs;
  float4 c = world_cmd<M>(s, q.sq, k.g, cs);
  const bool done = fl & FLAG_DONE;
  State n;
  if (s2_known && !done) {
    n = *s2_known;  // the next checkpoint is this step's post-dynamics state
  } else {  // reset rows: the checkpoint holds the respawned state, recompute
    n = model_step<M>(s, c, rp, k);
    n.ve = s.ve * (1.f - cfg.yaw_ema_alpha) + n.v * cfg.yaw_ema_alpha;
  }
  State g = done ? zero_state() : gS;
  g.ve = v3(0.f, 0.f, 0.f);
  // observation path (only rows that were not reset; q/tasks.py:584-594)
  if (!done && g_obs) {
    const float* go = g_obs + row * P;
    float2 cs2 = yaw_cs<M>(n, k.g);
    V3 gg = v3(go[0], go[1], go[2]);
    int cb = fl >> FLAG_CLAMP_SHIFT;
    gg = v3((cb & 1) ? gg.x : 0.f, (cb & 2) ? gg.y : 0.f, (cb & 4) ? gg.z : 0.f);
    g.p -= rotz(cs2, gg);  // unrot^T = rot
    g.v += rotz(cs2, v3(go[3], go[4], go[5]));
    if (M == QS_MODEL_SIMPLIFIED) {
      g.r2 += rotz(cs2, v3(go[6], go[7], go[8]));
    } else if (M == QS_MODEL_FULL) {
      V3 gz = rotz(cs2, v3(go[6], go[7], go[8]));
      Q4 gq = qaxis_z_vjp(n.q, gz);
      g.q = q4(g.q.w + gq.w, g.q.x + gq.x, g.q.y + gq.y, g.q.z + gq.z);
      g.w += v3(go[9], go[10], go[11]);
    } else {
      g.x += rotz(cs2, v3(go[6], go[7], go[8]));
    }
    if (TASK == QS_TASK_RACING) {
      const int kk = ModelTraits<M>::P;
      V3 ga = v3((cb & 8) ? go[kk] : 0.f, (cb & 16) ? go[kk + 1] : 0.f, (cb & 32) ? go[kk + 2] : 0.f);
      V3 gb = v3((cb & 64) ? go[kk + 6] : 0.f, (cb & 128) ? go[kk + 7] : 0.f, (cb & 256) ? go[kk + 8] : 0.f);
      g.p -= rotz(cs2, ga + gb);
    }
  }
  const float grr = g_r_rows ? g_r_rows[row] : g_r_scalar;
  float4 ge = make_float4(0.f, 0.f, 0.f, 0.f);
  if (TASK != QS_TASK_RACING && grr != 0.f) {
    float4 de = make_float4(q.eff.x - peff.x, q.eff.y - peff.y, q.eff.z - peff.z, q.eff.w - peff.w);
    V3 off = xyz(goal) - n.p;
    V3 goff, gv;
    reward_ctrl_vjp(cfg.w, off, n.v, q.eff, de, A, grr, goff, gv, ge);
    g.p -= goff;
    g.v += gv;
    if (TASK == QS_TASK_AVOIDANCE) {
      const int code = fl >> FLAG_SDF_SHIFT;  // argmin recorded by the forward
      if (code != 0) {
        float sd = sdf_prim(sv, n.p, code);
        float arg = (cfg.d_safe - sd) * (1.f / cfg.w.sdf_sharpness);
        float gsd = grr * cfg.w.w_o * sigmoid_stable(arg) * (1.f / cfg.w.sdf_sharpness);
        g.p += sdf_grad(sv, n.p, code) * gsd;
      }
    }
  }
  if (TASK != QS_TASK_RACING && G > 1 && na > 1) {  // formation penalty VJP
    // pen is subtracted from every agent's r_ctrl: dL/dpen = -sum_a dL/dr_a
    const float gpen = -grp.sum(real ? grr : 0.f) * cfg.w.w_f;
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const V3 pj = grp.bcast(n.p, j);
      if (real && j != grp.g && j < na) {
        V3 d = n.p - pj;
        float dij = norm3(d);
        const int a0 = min(grp.g, j), a1 = max(grp.g, j);
        float gd = gpen * 2.f * (dij - cfg.form_ref[a0][a1]);
        g.p += norm_vjp(d, dij, gd);
      }
    }
  }
  State gi;
  float4 gc;
  model_step_vjp<M>(s, c, rp, k, g, gi, gc);
  float4 gsq;
  if (M == QS_MODEL_FULL || M == QS_MODEL_SIMPLIFIED) {
    gsq = gc;
  } else {
    V3 u = unrotz(cs, v3(gc.x, gc.y, gc.z));  // Rz^T g
    gsq = make_float4(u.x, u.y, u.z, 0.f);
  }
  gsq = make_float4(gsq.x + ge.x, gsq.y + ge.y, gsq.z + ge.z, gsq.w + ge.w);
  if (real) {
    float* gout = g_raw_t + row * A;
#pragma unroll
    for (int kk = 0; kk < A; ++kk) {
      const float t = f4get(q.t, kk);  // tanh(raw), from the squash above
      gout[kk] = f4get(gsq, kk) * rp.half[kk] * (1.f - t * t);
    }
  }
  gS = gi;
}

// ---------------------------------------------------------------------------
// thread -> (env, agent row): G lanes per env, padding lanes read agent 0

template <int G>
struct RowMap {
  long e, row;
  bool active;  // e < n_envs (group-uniform)
  QS_D static RowMap make(long t, int n_envs, int na) {
    RowMap m;
    m.e = G == 1 ? t : t / G;
    const int g = G == 1 ? 0 : (int)(t & (G - 1));
    m.row = m.e * na + (g < na ? g : 0);
    m.active = m.e < n_envs;
    return m;
  }
};

// ---------------------------------------------------------------------------
// per-step kernels (FlightTask.step and its autograd node)

template <int M, int TASK, int G, bool INLINE>
__global__ void __launch_bounds__(128) k_task_fwd(const qs_task_cfg cfg, const qs_scene sc,
                                                  const qs_step_io io) {
  const int na = G == 1 ? 1 : cfg.n_agents;
  const RowMap<G> rm = RowMap<G>::make((long)blockIdx.x * blockDim.x + threadIdx.x, cfg.n_envs, na);
  const Grp<G> grp = Grp<G>::make(na);
  const long N = (long)cfg.n_envs * na;
  if (cfg.guard && io.err && io.err[2] != INT_MAX) return;  // rejected by qs_task_validate: mutate nothing
  StepStat st{false, 0, 0.f, 0.f};
  constexpr int P = TaskTraits<M, TASK>::P;
  __shared__ float s_obs[4][32 * P];  // per-warp observation staging (128-thread CTA)
  if (rm.active) {
    EnvRegs R;
    const float4 raw = load_act<ModelTraits<M>::A>(io.raw, rm.row);
    env_load<M>(sc.bounds, rm.e, rm.row, N, R, io.S_in, io.goal_in, io.peff_in, io.dr_in, io.meta,
                io.ep_return, io.imu_bias);
    StepOut o{io.obs, io.r_ctrl, io.r_goal, io.r_rl, io.terminated, io.truncated, io.flags, io.cam,
              io.imu_out, io.imu_noise};
    st = env_step_fwd<M, TASK, G, INLINE>(cfg, sc, rm.e, rm.row, na, N, grp, R, raw, o, io.err,
                                          io.dr_in != nullptr, io.imu_out != nullptr, nullptr,
                                          s_obs[threadIdx.x >> 5]);
    if (grp.real) {
      env_store_ckpt<M>(rm.row, N, R, io.S_out, io.goal_out, io.peff_out, io.dr_out);
      env_store_inplace(rm.e, rm.row, grp.g == 0, R, io.meta, io.ep_return, io.imu_out ? io.imu_bias : nullptr);
    }
  }
  warp_stats(rm.active && grp.g == 0, st.done, st.term, st.ret, io.stats);
}

template <int M, int TASK, int G>
__global__ void __launch_bounds__(128) k_task_bwd(const qs_task_cfg cfg, const qs_scene sc,
                                                  const qs_step_grad gr) {
  const int na = G == 1 ? 1 : cfg.n_agents;
  const RowMap<G> rm = RowMap<G>::make((long)blockIdx.x * blockDim.x + threadIdx.x, cfg.n_envs, na);
  if (!rm.active) return;
  const Grp<G> grp = Grp<G>::make(na);
  const long N = (long)cfg.n_envs * na;
  const long row = rm.row;
  const State s_in = load_state<M>(gr.S_in, N, row);
  const float4 goal = ld4(gr.goal_in, row), peff = ld4(gr.peff_in, row);
  const float4 dr = gr.dr_in ? ld4(gr.dr_in, row) : make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 raw = load_act<ModelTraits<M>::A>(gr.raw, row);
  const int fl = __ldg(gr.flags + row);
  State gS = load_grad<M>(gr.g_S_out, N, row);
  env_step_bwd<M, TASK, G>(cfg, sc, rm.e, row, na, N, grp, s_in, raw, goal, peff, dr, gr.dr_in != nullptr, fl,
                           gr.g_obs, gr.g_rctrl, 0.f, gS, gr.g_raw);
  if (grp.real) store_state<M>(gr.g_S_in, N, row, gS);
}

// ---------------------------------------------------------------------------
// fused T-step windows (open-loop actions): each row's register file stays on
// chip for the whole window; only the per-step outputs and the backward's
// checkpoints go to HBM, and the backward carries dL/dS in registers.

// 64-thread CTAs, >= 7 resident per SM: 65,536 envs = 1,024 CTAs = one wave
// on 148 SMs with <= 144 registers per thread
#ifndef QS_WIN_BLOCK
#define QS_WIN_BLOCK 64
#endif
#ifndef QS_WIN_MINB
#define QS_WIN_MINB 7
#endif
#ifndef QS_BWD_NST
#define QS_BWD_NST 2  // ring depth of the bwd checkpoint stream: 2 beats 3 (52.5 vs 54.6 us at C2) and 4 (70 us)
#endif
constexpr int WIN_BLOCK = QS_WIN_BLOCK;

template <int M, int TASK, int G, int IMU>
__global__ void __launch_bounds__(WIN_BLOCK, QS_WIN_MINB) k_window_fwd(const qs_task_cfg cfg, const qs_scene sc,
                                                    const qs_window_io w) {
  constexpr int A = ModelTraits<M>::A;
  constexpr int P = TaskTraits<M, TASK>::P;
  const int na = G == 1 ? 1 : cfg.n_agents;
  const RowMap<G> rm = RowMap<G>::make((long)blockIdx.x * blockDim.x + threadIdx.x, cfg.n_envs, na);
  const Grp<G> grp = Grp<G>::make(na);
  const bool active = rm.active;
  const long e = rm.e, row = rm.row;
  const long N = (long)cfg.n_envs * na;
  const int NP = ModelTraits<M>::NP;
  const bool has_dr = w.dr != nullptr, has_imu = IMU == 1 || w.imu_out != nullptr;
  EnvRegs R;
  int n_done = 0, n_succ = 0, n_coll = 0;
  float ret_sum = 0.f;
  double loss_sum = 0.0;
  float gpow = 1.f;
  // The CTA's action block of a step (its envs' rows x A floats, contiguous) is
  // staged in shared memory by a TMA bulk copy into a 4-deep ring, 4 steps
  // ahead, so the action latency never sits on the step's critical path and
  // costs no registers.  Partial tail CTAs load directly.
  constexpr int NB = 4;  // ring depth: step t+NB is in flight during step t
  __shared__ __align__(128) float s_raw[NB][WIN_BLOCK * 4];
  __shared__ __align__(8) uint64_t s_bar[NB];
  __shared__ int s_free[NB];  // warps done with each buffer this round
  const int epc = blockDim.x / G;  // envs per CTA
  const long e0 = (long)blockIdx.x * epc;
  const uint32_t blk_bytes = (uint32_t)(epc * na * A * 4);
  const bool use_tma = (e0 + epc <= cfg.n_envs) && (blk_bytes % 16 == 0) && ((N * A) % 4 == 0) &&
                       ((reinterpret_cast<uintptr_t>(w.actions) & 15) == 0);
  if (use_tma && threadIdx.x == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(&s_bar[b], 1);
      s_free[b] = 0;
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (use_tma && threadIdx.x == 0) {
    for (int b = 0; b < NB && b < w.T; ++b)
      tma_load_1d(s_raw[b], w.actions + ((long)b * N + e0 * na) * A, blk_bytes, &s_bar[b]);
  }
  if (active)
    env_load<M>(sc.bounds, e, row, N, R, w.S, w.goal, w.peff, w.dr, w.meta, w.ep_return, w.imu_bias);
  // spawn-ahead: this row's next reset sample, drawn by the whole warp at once
  __shared__ float4 s_ahead[4][WIN_BLOCK];
  SpawnAhead ahead{&s_ahead[0][threadIdx.x], WIN_BLOCK, -1};
  if (active) {
    const int ep = R.meta.y + 1;
    V3 sp, sv_, sg, head;
    int ng0;
    const bool ok = spawn_sample<M, TASK, G>(cfg, sc, e, ep, na, R.blo, R.bhi, grp, sp, sv_, sg, head, ng0);
    s_ahead[0][threadIdx.x] = f4(sp, head.x);
    s_ahead[1][threadIdx.x] = f4(sv_, head.y);
    s_ahead[2][threadIdx.x] = f4(sg, ok ? 1.f : 0.f);
    if (has_dr && cfg.dr_per_episode) s_ahead[3][threadIdx.x] = dr_sample(cfg, row, ep);
    ahead.episode = ep;
  }
  const int lrow = (int)(row - e0 * na);  // this row's slot in the CTA's action block
  for (int t = 0; t < w.T; ++t) {
    float4 raw = make_float4(0.f, 0.f, 0.f, 0.f);
    if (use_tma) {
      mbar_wait(&s_bar[t % NB], (t / NB) & 1);
      const float* p = s_raw[t % NB] + lrow * A;
      raw = make_float4(p[0], p[1], p[2], A == 4 ? p[3] : 0.f);
    } else if (active) {
      raw = load_act<A>(w.actions + (long)t * N * A, row);
    }
    if (active) {
      StepOut o{w.obs ? w.obs + (long)t * N * P : nullptr, w.r + (long)t * 3 * N, w.r + (long)t * 3 * N + N,
                w.r + (long)t * 3 * N + 2 * N, w.terminated + (long)t * N, w.truncated + (long)t * N,
                w.flags + (long)t * N, nullptr, has_imu ? w.imu_out + (long)t * N * 6 : nullptr,
                w.imu_noise ? w.imu_noise + (long)t * 4 * N * 3 : nullptr};
      // (no observation staging here: at C1's 1,024 rows the window is latency-bound
      // and the staging's warp syncs cost more than the coalescing saves, measured)
      StepStat st = env_step_fwd<M, TASK, G, true, IMU>(cfg, sc, e, row, na, N, grp, R, raw, o, w.err, has_dr,
                                                        has_imu, &ahead);
      if (st.done && grp.g == 0) {
        n_done++;
        n_succ += st.term == 1;
        n_coll += st.term == 2;
        ret_sum += st.ret;
      }
      loss_sum += (double)(gpow * st.rc);
      gpow *= w.gamma;
      if (grp.real)
        env_store_ckpt<M>(row, N, R, w.S + (long)(t + 1) * NP * N * 4, w.goal + (long)(t + 1) * N * 4,
                          w.peff + (long)(t + 1) * N * 4, has_dr ? w.dr + (long)(t + 1) * N * 4 : nullptr);
    }
    if (use_tma) {
      // No CTA barrier: the last warp to finish with buffer t%NB (its lanes'
      // actions have fed this step) refills it with step t+NB, so warps drift
      // freely by up to a few steps instead of meeting every step.
      __syncwarp();
      if ((threadIdx.x & 31) == 0) {
        __threadfence_block();
        if (atomicAdd(&s_free[t % NB], 1) == (int)(blockDim.x >> 5) - 1) {
          atomicExch(&s_free[t % NB], 0);
          if (t + NB < w.T) {
            fence_proxy_async();
            tma_load_1d(s_raw[t % NB], w.actions + ((long)(t + NB) * N + e0 * na) * A, blk_bytes,
                        &s_bar[t % NB]);
          }
        }
      }
    }
  }
  if (active && grp.real)
    env_store_inplace(e, row, grp.g == 0, R, w.meta, w.ep_return, has_imu ? w.imu_bias : nullptr);
  // episode statistics and the BPTT loss: one warp reduction for the window
  double r = ret_sum;
  double ls = loss_sum;
  int c0 = n_done, c1 = n_succ, c2 = n_coll;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r += __shfl_xor_sync(0xffffffffu, r, o);
    ls += __shfl_xor_sync(0xffffffffu, ls, o);
    c0 += __shfl_xor_sync(0xffffffffu, c0, o);
    c1 += __shfl_xor_sync(0xffffffffu, c1, o);
    c2 += __shfl_xor_sync(0xffffffffu, c2, o);
  }
  if ((threadIdx.x & 31) == 0 && w.loss) atomicAdd(w.loss, ls * (double)w.g_rctrl_scale);
  if ((threadIdx.x & 31) == 0 && w.stats && c0) {
    atomicAdd(w.stats + 0, (double)c0);
    atomicAdd(w.stats + 1, (double)c1);
    atomicAdd(w.stats + 2, (double)c2);
    atomicAdd(w.stats + 3, r);
  }
}

template <int M, int TASK, int G>
__global__ void __launch_bounds__(WIN_BLOCK, QS_WIN_MINB) k_window_bwd(const qs_task_cfg cfg, const qs_scene sc,
                                                    const qs_window_io w) {
  constexpr int A = ModelTraits<M>::A;
  const int na = G == 1 ? 1 : cfg.n_agents;
  const RowMap<G> rm = RowMap<G>::make((long)blockIdx.x * blockDim.x + threadIdx.x, cfg.n_envs, na);
  if (!rm.active) return;  // group-uniform
  const Grp<G> grp = Grp<G>::make(na);
  const long e = rm.e, row = rm.row;
  const long N = (long)cfg.n_envs * na;
  const int NP = ModelTraits<M>::NP;
  const bool has_dr = w.dr != nullptr;
  State gS = load_grad<M>(w.g_S_final, N, row);
  // Each thread streams its row's checkpoints through a private cp.async ring
  // in shared memory, NST steps ahead: the loads hold no registers while in
  // flight and each thread waits only for its own copies (no barrier).
  constexpr int NST = QS_BWD_NST;
  constexpr int NPL = ModelTraits<M>::NP;
  constexpr int NREC = NPL + 4;  // state planes, goal, peff, dr, raw
  __shared__ __align__(16) float4 ring[NST][NREC][WIN_BLOCK];
  __shared__ int ring_fl[NST][WIN_BLOCK];
  const int tx = threadIdx.x;
  auto issue = [&](int t, int b) {  // this thread's row of step t -> stage b
    if (t >= 0) {
#pragma unroll
      for (int k = 0; k < NPL; ++k) cp_async16(&ring[b][k][tx], w.S + (((long)t * NP + k) * N + row) * 4);
      cp_async16(&ring[b][NPL][tx], w.goal + ((long)t * N + row) * 4);
      cp_async16(&ring[b][NPL + 1][tx], w.peff + ((long)t * N + row) * 4);
      if (has_dr) cp_async16(&ring[b][NPL + 2][tx], w.dr + ((long)t * N + row) * 4);
      const float* ra = w.actions + ((long)t * N + row) * A;
      float* rd = &ring[b][NPL + 3][tx].x;
#pragma unroll
      for (int k = 0; k < A; ++k) cp_async4(rd + k, ra + k);
      cp_async4(&ring_fl[b][tx], w.flags + (long)t * N + row);
    }
    cp_async_commit();  // one group per step, possibly empty, keeps the count uniform
  };
  for (int k = 0; k < NST; ++k) issue(w.T - 1 - k, k);
  // checkpoint t+1 = post-dynamics state of step t (non-reset rows)
  State s2 = load_state<M>(w.S + (long)w.T * NP * N * 4, N, row);
  const float lg_gamma = log2f(w.gamma);  // gamma^t = 2^(t lg): one MUFU.EX2 per step
  for (int t = w.T - 1; t >= 0; --t) {
    const float gscale = w.g_rctrl_scale * (t == 0 ? 1.f : exp2f((float)t * lg_gamma));
    const int kk = w.T - 1 - t;
    const int b = kk % NST;
    cp_async_wait<NST - 1>();  // this thread's copies of step t have landed
    const State s_in = load_state<M, true>(&ring[b][0][0].x, WIN_BLOCK, tx);
    const float4 goal = ring[b][NPL][tx], peff = ring[b][NPL + 1][tx];
    const float4 dr = has_dr ? ring[b][NPL + 2][tx] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 rr = ring[b][NPL + 3][tx];
    const float4 raw = make_float4(rr.x, rr.y, rr.z, A == 4 ? rr.w : 0.f);
    const int fl = ring_fl[b][tx];
    env_step_bwd<M, TASK, G>(cfg, sc, e, row, na, N, grp, s_in, raw, goal, peff, dr, has_dr, fl, nullptr,
                             w.g_rctrl ? w.g_rctrl + (long)t * N : nullptr, gscale, gS,
                             w.g_actions + (long)t * N * A, &s2);
    s2 = s_in;
    issue(t - NST, b);  // the stage just consumed takes step t - NST
  }
  if (!grp.real) return;
  if (w.g_S0) store_state<M>(w.g_S0, N, row, gS);
  if (w.carry) {  // this thread's row only: slot 0 was its last checkpoint read
    const long T = w.T;
#pragma unroll
    for (int k = 0; k < NP; ++k) st4(w.S, (long)k * N + row, ld4(w.S + T * NP * N * 4, (long)k * N + row));
    st4(w.goal, row, ld4(w.goal + T * N * 4, row));
    st4(w.peff, row, ld4(w.peff + T * N * 4, row));
    if (has_dr) st4(w.dr, row, ld4(w.dr + T * N * 4, row));
  }
}

// ---------------------------------------------------------------------------
// spawn (reset of masked envs), observe

template <int M, int TASK, int G>
__global__ void __launch_bounds__(128) k_task_spawn(const qs_task_cfg cfg, const qs_scene sc,
                                                    const qs_step_io io, const uint8_t* mask,
                                                    const qs_reset_table tab, bool use_tab) {
  const int na = G == 1 ? 1 : cfg.n_agents;
  const RowMap<G> rm = RowMap<G>::make((long)blockIdx.x * blockDim.x + threadIdx.x, cfg.n_envs, na);
  if (!rm.active) return;
  const long e = rm.e, row = rm.row;
  if (mask && !mask[e]) return;  // env-uniform
  const Grp<G> grp = Grp<G>::make(na);
  const long N = (long)cfg.n_envs * na;
  const DynK k = dyn_consts(cfg);
  int4 meta = reinterpret_cast<int4*>(io.meta)[e];
  V3 p, v, gl, ve = v3(0.f, 0.f, 0.f);
  int ng0 = 0;
  if (!use_tab) {
    const V3 blo = xyz(ld4(sc.bounds, 2 * e)) + v3(1e-6f, 1e-6f, 1e-6f);  // as env_load
    const V3 bhi = xyz(ld4(sc.bounds, 2 * e + 1)) - v3(1e-6f, 1e-6f, 1e-6f);
    bool ok = spawn_sample<M, TASK, G>(cfg, sc, e, meta.y, na, blo, bhi, grp, p, v, gl, ve, ng0);
    if (!ok && grp.g == 0) report_err(io.err, QS_ERR_GENERATION, (int)(e * na));
  } else {
    if (tab.next_gate) ng0 = tab.next_gate[e];
    p = load3(tab.p, row);
    v = load3(tab.v, row);
    gl = load3(tab.goal, row);
    ve = load3(tab.v_ema, row);
  }
  if (!grp.real) return;
  if (grp.g == 0) {
    meta.w = ng0;
    reinterpret_cast<int4*>(io.meta)[e] = meta;
  }
  store_state<M>(io.S_out, N, row, init_state<M>(p, v, ve, k.g));
  st4(io.goal_out, row, f4(gl, 0.f));
  st4(io.peff_out, row, make_float4(0.f, 0.f, 0.f, 0.f));
  if (io.dr_out && cfg.dr_enabled) {
    float4 d = use_tab && tab.dr ? ld4(tab.dr, row) : dr_sample(cfg, row, meta.y);
    st4(io.dr_out, row, d);
  }
  if (io.imu_bias) {
    st4(io.imu_bias, 2 * row, make_float4(0.f, 0.f, 0.f, 0.f));
    st4(io.imu_bias, 2 * row + 1, make_float4(0.f, 0.f, 0.f, 0.f));
  }
}

template <int M, int TASK, int G>
__global__ void __launch_bounds__(128) k_task_observe(const qs_task_cfg cfg, const qs_scene sc,
                                                      const qs_step_io io) {
  constexpr int P = TaskTraits<M, TASK>::P;
  const int na = G == 1 ? 1 : cfg.n_agents;
  const RowMap<G> rm = RowMap<G>::make((long)blockIdx.x * blockDim.x + threadIdx.x, cfg.n_envs, na);
  const Grp<G> grp = Grp<G>::make(na);
  if (!rm.active || !grp.real) return;
  const long e = rm.e, row = rm.row;
  const long N = (long)cfg.n_envs * na;
  const DynK k = dyn_consts(cfg);
  GateV g0, g1;
  if (TASK == QS_TASK_RACING) {
    int ng = io.meta[4 * e + 3];
    g0 = load_gate(sc, cfg, e, ng);
    g1 = load_gate(sc, cfg, e, min(ng + 1, cfg.n_gates - 1));
  }
  State s = load_state<M>(io.S_out, N, row);
  V3 goal = load3(io.goal_out, row);
  float o[P];
  float2 cs = yaw_cs<M>(s, k.g);
  int bits = observe_row<M, TASK>(cfg, s, cs, goal, &g0, &g1, o);
  write_obs<M, TASK>(cfg, io, row, o);
  if (io.cam) reinterpret_cast<float2*>(io.cam)[row] = cs;
  if (io.flags) io.flags[row] = (io.flags[row] & ~FLAG_CLAMP_MASK) | bits;
}

// critic features of the current state (q/tasks.py:500-545, the no-grad
// FlightTask.privileged_state): yaw-local goal offset, velocity and thrust,
// sdf clamped to +-5, yaw-local clearance direction (the sdf's analytic
// gradient at its first argmin), goal distance -- 14 floats per row, written
// to io.obs (stride 14).  One launch instead of the ~30 torch ops + 2 sdf
// launches of the differentiable twin (privileged_var), which stays in torch.
template <int M, int TASK, int G>
__global__ void __launch_bounds__(128) k_task_privileged(const qs_task_cfg cfg, const qs_scene sc,
                                                         const qs_step_io io) {
  // the CTA's rows are consecutive: their 14 features go out through shared
  // memory as one contiguous, coalesced block (per-thread 56-byte rows of scalar
  // stores touched 8x the sectors they wrote)
  __shared__ float s_out[128 * 14];
  const int na = G == 1 ? 1 : cfg.n_agents;
  const RowMap<G> rm = RowMap<G>::make((long)blockIdx.x * blockDim.x + threadIdx.x, cfg.n_envs, na);
  const Grp<G> grp = Grp<G>::make(na);
  const bool contiguous = G == 1;  // one row per thread, rows = global thread ids
  if (!contiguous && (!rm.active || !grp.real)) return;
  const long e = rm.e, row = rm.row;
  if (rm.active) {  // (contiguous: every thread reaches the one barrier below)
  const long N = (long)cfg.n_envs * na;
  const DynK k = dyn_consts(cfg);
  const State s = load_state<M>(io.S_out, N, row);
  const V3 off = load3(io.goal_out, row) - s.p;
  const float2 cs = yaw_cs<M>(s, k.g);
  V3 th;  // FlightTask._thrust (q/tasks.py:479-498)
  if (M == QS_MODEL_FULL) {
    const Q4 q = s.q;
    th = v3(2.f * (q.x * q.z + q.w * q.y), 2.f * (q.y * q.z - q.w * q.x), 1.f - 2.f * (q.x * q.x + q.y * q.y)) * 9.81f;
  } else if (M == QS_MODEL_SIMPLIFIED) {
    th = s.r2 * 9.81f;
  } else {
    th = thrust_of<M>(s, k.g);
  }
  const SceneView sv = scene_view(sc, e);
  int code;
  const float sd = sdf_eval(sv, s.p, code);
  const V3 gd = code ? sdf_grad(sv, s.p, code) : v3(0.f, 0.f, 0.f);
  const V3 a = unrotz(cs, off), b = unrotz(cs, s.v), c = unrotz(cs, th), d = unrotz(cs, gd);
  float* o = contiguous ? s_out + threadIdx.x * 14 : io.obs + row * 14;
  o[0] = a.x; o[1] = a.y; o[2] = a.z;
  o[3] = b.x; o[4] = b.y; o[5] = b.z;
  o[6] = c.x; o[7] = c.y; o[8] = c.z;
  o[9] = clampf(sd, -5.f, 5.f);
  o[10] = d.x; o[11] = d.y; o[12] = d.z;
  o[13] = sqrtf(dot(off, off));
  }
  if (!contiguous) return;
  __syncthreads();
  {
    const long NR = (long)cfg.n_envs * na, r0 = (long)blockIdx.x * blockDim.x;
    const long nrows = NR - r0 < (long)blockDim.x ? NR - r0 : (long)blockDim.x;
    float* dst = io.obs + r0 * 14;
    for (int i = threadIdx.x; i < nrows * 14; i += blockDim.x) dst[i] = s_out[i];
  }
}

// ---------------------------------------------------------------------------
// per-task launchers (one translation unit per task keeps builds parallel)

inline int grid_for(long n, int block) { return (int)((n + block - 1) / block); }
inline int launch_status() { return cudaGetLastError() == cudaSuccess ? QS_OK : QS_ERR_LAUNCH; }

// per-step kernels: 128-thread CTAs, or 32 when too few rows to fill the SMs
inline int step_block(long threads) { return threads >= 148 * 2 * 128 ? 128 : 32; }

template <int M, int T, int G>
int run_fwd(const qs_task_cfg* cfg, const qs_scene* sc, const qs_step_io* io, cudaStream_t s) {
  const long th = (long)cfg->n_envs * G;
  const int b = step_block(th);
  if (cfg->reset_mode == 0)
    k_task_fwd<M, T, G, true><<<grid_for(th, b), b, 0, s>>>(*cfg, *sc, *io);
  else
    k_task_fwd<M, T, G, false><<<grid_for(th, b), b, 0, s>>>(*cfg, *sc, *io);
  return launch_status();
}
template <int M, int T, int G>
int run_bwd(const qs_task_cfg* cfg, const qs_scene* sc, const qs_step_grad* g, cudaStream_t s) {
  const long th = (long)cfg->n_envs * G;
  const int b = step_block(th);
  k_task_bwd<M, T, G><<<grid_for(th, b), b, 0, s>>>(*cfg, *sc, *g);
  return launch_status();
}
template <int M, int T, int G>
int run_spawn(const qs_task_cfg* cfg, const qs_scene* sc, const qs_step_io* io, const uint8_t* mask,
              const qs_reset_table* tab, cudaStream_t s) {
  qs_reset_table t{};
  if (tab) t = *tab;
  const long th = (long)cfg->n_envs * G;
  k_task_spawn<M, T, G><<<grid_for(th, 128), 128, 0, s>>>(*cfg, *sc, *io, mask, t, tab != nullptr);
  return launch_status();
}
template <int M, int T, int G>
int run_observe(const qs_task_cfg* cfg, const qs_scene* sc, const qs_step_io* io, cudaStream_t s) {
  const long th = (long)cfg->n_envs * G;
  k_task_observe<M, T, G><<<grid_for(th, 128), 128, 0, s>>>(*cfg, *sc, *io);
  return launch_status();
}

template <int M, int T, int G>
int run_privileged(const qs_task_cfg* cfg, const qs_scene* sc, const qs_step_io* io, cudaStream_t s) {
  const long th = (long)cfg->n_envs * G;
  k_task_privileged<M, T, G><<<grid_for(th, 128), 128, 0, s>>>(*cfg, *sc, *io);
  return launch_status();
}

template <int M, int T, int G>
int run_window(int op, const qs_task_cfg* cfg, const qs_scene* sc, const qs_window_io* w, cudaStream_t s) {
  if (w->T <= 0) return QS_OK;
  if (op == 4 && w->loss) cudaMemsetAsync(w->loss, 0, sizeof(double), s);
  // 64-thread CTAs when there are enough rows for >= 4 CTAs per SM; otherwise
  // 32-thread CTAs spread the (few, latency-bound) rows over twice the SMs
  const long th = (long)cfg->n_envs * G;
  const int blk = th >= 148 * 4 * WIN_BLOCK ? WIN_BLOCK : 32;
  const dim3 grid(grid_for(th, blk));
  if (op == 4 && G == 1 && w->imu_out && !w->imu_noise)  // Philox IMU specialisation
    k_window_fwd<M, T, G, G == 1 ? 1 : 0><<<grid, blk, 0, s>>>(*cfg, *sc, *w);
  else if (op == 4)
    k_window_fwd<M, T, G, 0><<<grid, blk, 0, s>>>(*cfg, *sc, *w);
  else
    k_window_bwd<M, T, G><<<grid, blk, 0, s>>>(*cfg, *sc, *w);
  return launch_status();
}

// op: 0 fwd, 1 bwd, 2 spawn, 3 observe, 4 window fwd, 5 window bwd, 7 critic features.
// One translation unit per (task, single / multi agent) keeps the build
// parallel; multi-agent picks the lane-group width G from n_agents.
template <int T, int NA>
int task_dispatch_na(int op, const qs_task_cfg* cfg, const qs_scene* sc, const void* p,
                     const uint8_t* mask, const qs_reset_table* tab, cudaStream_t s);

template <int T, int M, int G>
int task_op(int op, const qs_task_cfg* cfg, const qs_scene* sc, const void* p, const uint8_t* mask,
            const qs_reset_table* tab, cudaStream_t s) {
  switch (op) {
    case 0: return run_fwd<M, T, G>(cfg, sc, static_cast<const qs_step_io*>(p), s);
    case 1: return run_bwd<M, T, G>(cfg, sc, static_cast<const qs_step_grad*>(p), s);
    case 2: return run_spawn<M, T, G>(cfg, sc, static_cast<const qs_step_io*>(p), mask, tab, s);
    case 3: return run_observe<M, T, G>(cfg, sc, static_cast<const qs_step_io*>(p), s);
    case 4:
    case 5: return run_window<M, T, G>(op, cfg, sc, static_cast<const qs_window_io*>(p), s);
    case 7: return run_privileged<M, T, G>(cfg, sc, static_cast<const qs_step_io*>(p), s);
  }
  return QS_ERR_BAD_ARGUMENT;
}

template <int T, int M, int NA>
int task_op_groups(int op, const qs_task_cfg* cfg, const qs_scene* sc, const void* p, const uint8_t* mask,
                   const qs_reset_table* tab, cudaStream_t s) {
  if constexpr (NA == 1) {
    return task_op<T, M, 1>(op, cfg, sc, p, mask, tab, s);
  } else {
    const int na = cfg->n_agents;
    if (na <= 2) return task_op<T, M, 2>(op, cfg, sc, p, mask, tab, s);
    if (na <= 4) return task_op<T, M, 4>(op, cfg, sc, p, mask, tab, s);
    return task_op<T, M, 8>(op, cfg, sc, p, mask, tab, s);
  }
}

#define QS_DEFINE_TASK_DISPATCH(T, NA)                                                          \
  template <>                                                                                  \
  int task_dispatch_na<T, NA>(int op, const qs_task_cfg* cfg, const qs_scene* sc, const void* p, \
                              const uint8_t* mask, const qs_reset_table* tab, cudaStream_t s) { \
    switch (cfg->model) {                                                                      \
      case QS_MODEL_FULL: return task_op_groups<T, QS_MODEL_FULL, NA>(op, cfg, sc, p, mask, tab, s); \
      case QS_MODEL_PM_CONTINUOUS:                                                             \
        return task_op_groups<T, QS_MODEL_PM_CONTINUOUS, NA>(op, cfg, sc, p, mask, tab, s);    \
      case QS_MODEL_PM_DISCRETE:                                                               \
        return task_op_groups<T, QS_MODEL_PM_DISCRETE, NA>(op, cfg, sc, p, mask, tab, s);      \
      case QS_MODEL_SIMPLIFIED:                                                                \
        return task_op_groups<T, QS_MODEL_SIMPLIFIED, NA>(op, cfg, sc, p, mask, tab, s);       \
    }                                                                                          \
    return QS_ERR_BAD_ARGUMENT;                                                                \
  }

}  // namespace qs
