// Dynamics models, attitude/yaw frames and their analytic VJPs (per row, in
// registers).  Reference: q/dynamics.py:140-284, q/sensors.py:562-611,
// q/tasks.py:129-137, 400-418, 613-618.
#pragma once
#include "qs_common.cuh"

// State held in registers.  In HBM it is (NP, N, 4) float planes:
//   pm:   P0 = (p, vema.x)  P1 = (v, vema.y)  P2 = (a_lat | u_prev, vema.z)
//   full: P0 = (p, vema.x)  P1 = (v, vema.y)  P2 = q (w,x,y,z)  P3 = (w, vema.z)
// so every row is 3 or 4 coalesced 16-byte loads and v_ema (non-differentiable,
// q/tasks.py:566) rides in the pad lanes for free.
//   simplified (NP = 5): P0 = (p, vema.x)  P1 = (v, vema.y)  P2 = (R col0, vema.z)
//                        P3 = (R col1, _)  P4 = (R col2, _)
struct State {
  V3 p, v, x;  // x: a_lat (pm_continuous) / u_prev (pm_discrete)
  Q4 q;        // full
  V3 w;        // full: body rates
  V3 ve;       // velocity EMA (not differentiated)
  V3 r0, r1, r2;  // simplified: rotation-matrix columns (body x, y, z in world)
};

QS_D State zero_state() {
  State z;
  z.p = z.v = z.x = z.w = z.ve = z.r0 = z.r1 = z.r2 = v3(0.f, 0.f, 0.f);
  z.q = q4(0.f, 0.f, 0.f, 0.f);
  return z;
}
QS_D State zero_state_like() { return zero_state(); }

template <int M>
struct ModelTraits;
template <>
struct ModelTraits<QS_MODEL_FULL> {
  static constexpr int NP = 4, A = 4, P = 12;
};
template <>
struct ModelTraits<QS_MODEL_PM_CONTINUOUS> {
  static constexpr int NP = 3, A = 3, P = 9;
};
template <>
struct ModelTraits<QS_MODEL_PM_DISCRETE> {
  static constexpr int NP = 3, A = 3, P = 9;
};
template <>
struct ModelTraits<QS_MODEL_SIMPLIFIED> {
  static constexpr int NP = 5, A = 4, P = 9;
};

template <int M, bool GENERIC = false>  // GENERIC: plain loads (shared-memory staging)
QS_D State load_state(const float* S, long N, long row) {
  auto ld = [](const float* p, long i) { return GENERIC ? reinterpret_cast<const float4*>(p)[i] : ld4(p, i); };
  State s;
  float4 a = ld(S, row), b = ld(S, N + row), c = ld(S, 2 * N + row);
  s.p = xyz(a);
  s.v = xyz(b);
  s.r0 = s.r1 = s.r2 = v3(0.f, 0.f, 0.f);
  if (M == QS_MODEL_SIMPLIFIED) {
    s.r0 = xyz(c);
    s.r1 = xyz(ld(S, 3 * N + row));
    s.r2 = xyz(ld(S, 4 * N + row));
    s.ve = v3(a.w, b.w, c.w);
    s.x = v3(0.f, 0.f, 0.f);
    s.q = q4(1.f, 0.f, 0.f, 0.f);
    s.w = v3(0.f, 0.f, 0.f);
  } else if (M == QS_MODEL_FULL) {
    float4 d = ld(S, 3 * N + row);
    s.q = q4(c.x, c.y, c.z, c.w);
    s.w = xyz(d);
    s.ve = v3(a.w, b.w, d.w);
    s.x = v3(0.f, 0.f, 0.f);
  } else {
    s.x = xyz(c);
    s.ve = v3(a.w, b.w, c.w);
    s.q = q4(1.f, 0.f, 0.f, 0.f);
    s.w = v3(0.f, 0.f, 0.f);
  }
  return s;
}

template <int M>
QS_D void store_state(float* S, long N, long row, const State& s) {
  st4(S, row, f4(s.p, s.ve.x));
  st4(S, N + row, f4(s.v, s.ve.y));
  if (M == QS_MODEL_SIMPLIFIED) {
    st4(S, 2 * N + row, f4(s.r0, s.ve.z));
    st4(S, 3 * N + row, f4(s.r1, 0.f));
    st4(S, 4 * N + row, f4(s.r2, 0.f));
  } else if (M == QS_MODEL_FULL) {
    st4(S, 2 * N + row, make_float4(s.q.w, s.q.x, s.q.y, s.q.z));
    st4(S, 3 * N + row, f4(s.w, s.ve.z));
  } else {
    st4(S, 2 * N + row, f4(s.x, s.ve.z));
  }
}

template <int M>
QS_D bool state_finite(const State& s) {
  bool ok = finite3(s.p) && finite3(s.v);
  if (M == QS_MODEL_SIMPLIFIED)
    ok = ok && finite3(s.r0) && finite3(s.r1) && finite3(s.r2);
  else if (M == QS_MODEL_FULL)
    ok = ok && isfinite(s.q.w) && isfinite(s.q.x) && isfinite(s.q.y) && isfinite(s.q.z) &&
         finite3(s.w);
  else
    ok = ok && finite3(s.x);
  return ok;
}

// init_state (q/dynamics.py:324-330, 386-390, 412-416)
template <int M>
QS_D State init_state(V3 p, V3 v, V3 ve, V3 g) {
  State s;
  s.p = p;
  s.v = v;
  s.ve = ve;
  s.q = q4(1.f, 0.f, 0.f, 0.f);
  s.w = v3(0.f, 0.f, 0.f);
  s.x = (M == QS_MODEL_PM_CONTINUOUS) ? -g : v3(0.f, 0.f, 0.f);
  s.r0 = v3(1.f, 0.f, 0.f);  // q/dynamics.py:356-360 (R = I)
  s.r1 = v3(0.f, 1.f, 0.f);
  s.r2 = v3(0.f, 0.f, 1.f);
  return s;
}

// Per-row physical parameters (domain randomisation makes them per row).
struct RowPrm {
  float drag, decay;
  float center[4], half[4];  // squash box after the action-scale draw
};

template <int M>
QS_D RowPrm row_params(const qs_task_cfg& cfg, const float* dr, long row) {
  RowPrm r;
  float scale = 1.f;
  r.drag = cfg.drag_coeff;
  r.decay = cfg.lag_decay;
  if (dr) {
    float4 d = ld4(dr, row);
    r.drag = d.x;
    r.decay = d.y;
    scale = d.z;
  }
#pragma unroll
  for (int k = 0; k < ModelTraits<M>::A; ++k) {
    float lo = cfg.act_lo[k], hi = cfg.act_hi[k];
    if (dr) {  // q/tasks.py:370-375
      float c = (lo + hi) * 0.5f, h = (hi - lo) * 0.5f;
      lo = c - h * scale;
      hi = c + h * scale;
    }
    r.center[k] = (lo + hi) * 0.5f;
    r.half[k] = (hi - lo) * 0.5f;
  }
  return r;
}

// ---------------------------------------------------------------------------
// attitude / yaw

// reconstruct_attitude (q/sensors.py:569-606): columns x_b, y_b, z_b
QS_D void attitude_pm(V3 a, V3 ve, V3& xb, V3& yb, V3& zb) {
  float tn = norm3(a);
  zb = tn > 1e-6f ? a * (1.f / fmaxf(tn, 1e-12f)) : v3(0.f, 0.f, 1.f);
  V3 h = v3(ve.x, ve.y, 0.f);
  float hn = norm3(h);
  V3 xr = hn > 1e-3f ? h * (1.f / fmaxf(hn, 1e-12f)) : v3(1.f, 0.f, 0.f);
  float zz = zb.z;
  bool upright = fabsf(zz) > 0.1f;
  V3 xraw;
  if (upright) {
    xraw = v3(xr.x, xr.y, -(xr.x * zb.x + xr.y * zb.y) / zz);
  } else {
    xraw = xr - zb * dot(xr, zb);
  }
  float xn = norm3(xraw);
  if (xn > 1e-9f) {
    xb = xraw * (1.f / fmaxf(xn, 1e-12f));
  } else {
    V3 fb = v3(zb.z, 0.f, -zb.x);  // e_y x z_b
    float fn = norm3(fb);
    xb = fb * (1.f / fmaxf(fn, 1e-12f));
  }
  yb = cross(zb, xb);
}

// (cos, sin) of atan2(y, x) without the transcendental; exact zeros keep the
// atan2 signed-zero semantics (q/sensors.py:609-611).
QS_D float2 yaw_cs_from(float x, float y) {
  float m = fmaxf(fabsf(x), fabsf(y));
  if (m > 1e-18f && m < 1e18f) {  // no under/overflow in x^2 + y^2
    float r = rsqrtf(x * x + y * y);
    return make_float2(x * r, y * r);
  }
  if (m == 0.f) {
    float yaw = atan2f(y, x), s, c;
    sincosf(yaw, &s, &c);
    return make_float2(c, s);
  }
  float im = 1.f / m;
  x *= im;
  y *= im;
  float r = rsqrtf(x * x + y * y);
  return make_float2(x * r, y * r);
}

template <int M>
QS_D V3 thrust_of(const State& s, V3 g) {  // q/dynamics.py:406, 430
  return (M == QS_MODEL_PM_CONTINUOUS) ? s.x : s.x - g;
}

template <int M>
QS_D float2 yaw_cs(const State& s, V3 g) {  // q/tasks.py:400-413
  if (M == QS_MODEL_SIMPLIFIED) return yaw_cs_from(s.r0.x, s.r0.y);  // R00, R10
  if (M == QS_MODEL_FULL) {
    const Q4 q = s.q;  // R00, R10 of q/dynamics.py:448-460
    return yaw_cs_from(1.f - 2.f * (q.y * q.y + q.z * q.z), 2.f * (q.x * q.y + q.w * q.z));
  } else {
    V3 xb, yb, zb;
    attitude_pm(thrust_of<M>(s, g), s.ve, xb, yb, zb);
    return yaw_cs_from(xb.x, xb.y);
  }
}

// Rz(yaw) v and Rz(-yaw) v   (q/tasks.py:129-137)
QS_HD V3 rotz(float2 cs, V3 v) { return v3(cs.x * v.x - cs.y * v.y, cs.y * v.x + cs.x * v.y, v.z); }
QS_HD V3 unrotz(float2 cs, V3 v) { return v3(cs.x * v.x + cs.y * v.y, -cs.y * v.x + cs.x * v.y, v.z); }

// ---------------------------------------------------------------------------
// model steps (explicit Euler), cmd in world frame after squash/yaw rotation

struct DynK {  // per-launch constants
  float dt;
  V3 g, D, K;
  bool has_drag;
};

QS_D DynK dyn_consts(const qs_task_cfg& c) {
  DynK k;
  k.dt = c.dt;
  k.g = v3(c.g[0], c.g[1], c.g[2]);
  k.D = v3(c.drag_diag[0], c.drag_diag[1], c.drag_diag[2]);
  k.K = v3(c.rate_gains[0], c.rate_gains[1], c.rate_gains[2]);
  k.has_drag = (k.D.x != 0.f) || (k.D.y != 0.f) || (k.D.z != 0.f);
  return k;
}

// step_full (q/dynamics.py:155-186).  The rate loop's tau = J(K(wc-w)) + w x Jw
// followed by J^-1(tau - w x Jw) is K(wc-w) in exact arithmetic
// (q/dynamics.py:171-174); the gyroscopic terms cancel, so J drops out.
QS_D State step_full(const State& s, float4 cmd, const DynK& k) {
  const float dt = k.dt;
  const Q4 q = s.q;
  V3 zb = qaxis_z(q);
  V3 vdot = k.g + zb * cmd.x;
  if (k.has_drag) {
    V3 vb = qrot(qconj(q), s.v);
    vdot -= qrot(q, hmul(k.D, vb));
  }
  V3 wc = v3(cmd.y, cmd.z, cmd.w);
  V3 wdot = hmul(k.K, wc - s.w);
  Q4 qd = qmul(q, q4(0.f, s.w.x, s.w.y, s.w.z));
  Q4 qn = q4(q.w + qd.w * 0.5f * dt, q.x + qd.x * 0.5f * dt, q.y + qd.y * 0.5f * dt,
             q.z + qd.z * 0.5f * dt);
  // |qn| ~ 1: rsqrt (<= 2 ulp) instead of IEEE sqrt + divide
  float inv = rsqrtf(qn.w * qn.w + qn.x * qn.x + qn.y * qn.y + qn.z * qn.z);
  State o;
  o.p = s.p + s.v * dt;
  o.v = s.v + vdot * dt;
  o.q = q4(qn.w * inv, qn.x * inv, qn.y * inv, qn.z * inv);
  o.w = s.w + wdot * dt;
  o.x = s.x;
  o.ve = s.ve;
  return o;
}

// VJP of step_full.  gs: upstream grads of (p', v', q', w'); returns grads of
// (p, v, q, w) in gi and of cmd (c, wc) in gc.
QS_D void step_full_vjp(const State& s, float4 cmd, const DynK& k, const State& gs, State& gi,
                        float4& gc) {
  const float dt = k.dt;
  const Q4 q = s.q;
  // recompute
  Q4 qd = qmul(q, q4(0.f, s.w.x, s.w.y, s.w.z));
  Q4 qn = q4(q.w + qd.w * 0.5f * dt, q.x + qd.x * 0.5f * dt, q.y + qd.y * 0.5f * dt,
             q.z + qd.z * 0.5f * dt);
  float inv = rsqrtf(qn.w * qn.w + qn.x * qn.x + qn.y * qn.y + qn.z * qn.z);
  Q4 qo = q4(qn.w * inv, qn.x * inv, qn.y * inv, qn.z * inv);
  // normalize VJP: (g - q'(q'.g)) / |qn|
  const Q4 gq = gs.q;
  float pr = qo.w * gq.w + qo.x * gq.x + qo.y * gq.y + qo.z * gq.z;
  Q4 gqn = q4((gq.w - qo.w * pr) * inv, (gq.x - qo.x * pr) * inv, (gq.y - qo.y * pr) * inv,
              (gq.z - qo.z * pr) * inv);
  // qn = q + 0.5 dt (q x (0,w))
  Q4 gqd = q4(gqn.w * 0.5f * dt, gqn.x * 0.5f * dt, gqn.y * 0.5f * dt, gqn.z * 0.5f * dt);
  Q4 gq_from_qd = qmul(gqd, q4(0.f, -s.w.x, -s.w.y, -s.w.z));  // g (x) conj(r)
  Q4 gw_q = qmul(qconj(q), gqd);                               // conj(q) (x) g
  Q4 gq_tot = q4(gqn.w + gq_from_qd.w, gqn.x + gq_from_qd.x, gqn.y + gq_from_qd.y,
                 gqn.z + gq_from_qd.z);
  // w' = w + K (wc - w) dt
  V3 gwdot = gs.w * dt;
  V3 gKw = hmul(k.K, gwdot);
  gi.w = gs.w - gKw + v3(gw_q.x, gw_q.y, gw_q.z);
  // v' = v + vdot dt ; p' = p + v dt
  V3 gvdot = gs.v * dt;
  gi.p = gs.p;
  gi.v = gs.v + gs.p * dt;
  V3 zb = qaxis_z(q);
  float gcx = dot(gvdot, zb);
  Q4 gzq = qaxis_z_vjp(q, gvdot * cmd.x);
  gq_tot = q4(gq_tot.w + gzq.w, gq_tot.x + gzq.x, gq_tot.y + gzq.y, gq_tot.z + gzq.z);
  if (k.has_drag) {
    // drag = rot(q, D (.) rot(conj q, v)); vdot -= drag
    V3 vb = qrot(qconj(q), s.v);
    V3 dv = hmul(k.D, vb);
    V3 gdrag = -gvdot;
    Q4 g1 = qrot_vjp_q(q, dv, gdrag);
    V3 gdv = qrot_vjp_v(q, gdrag);
    V3 gvb = hmul(k.D, gdv);
    Q4 qc = qconj(q);
    gi.v += qrot_vjp_v(qc, gvb);
    Q4 g2 = qrot_vjp_q(qc, s.v, gvb);  // grad wrt conj(q)
    gq_tot = q4(gq_tot.w + g1.w + g2.w, gq_tot.x + g1.x - g2.x, gq_tot.y + g1.y - g2.y,
                gq_tot.z + g1.z - g2.z);
  }
  gi.q = gq_tot;
  gi.x = v3(0.f, 0.f, 0.f);
  gi.ve = v3(0.f, 0.f, 0.f);
  gc = make_float4(gcx, gKw.x, gKw.y, gKw.z);
}

// step_pm_continuous (q/dynamics.py:237-258)
QS_D State step_pmc(const State& s, V3 u, float drag, float decay, const DynK& k) {
  State o = s;
  V3 an = u + (s.x - u) * decay;
  V3 vdot = (an + k.g) - s.v * drag;
  o.p = s.p + s.v * k.dt;
  o.v = s.v + vdot * k.dt;
  o.x = an;
  return o;
}
QS_D void step_pmc_vjp(const State& gs, float drag, float decay, const DynK& k, State& gi, V3& gu) {
  V3 ga = gs.x + gs.v * k.dt;
  gi.p = gs.p;
  gi.v = gs.v - gs.v * (k.dt * drag) + gs.p * k.dt;
  gi.x = ga * decay;
  gu = ga - ga * decay;
  gi.q = q4(0.f, 0.f, 0.f, 0.f);
  gi.w = gi.ve = v3(0.f, 0.f, 0.f);
}

// step_pm_discrete (q/dynamics.py:261-274)
QS_D State step_pmd(const State& s, V3 u, const DynK& k) {
  State o = s;
  const float dt = k.dt;
  o.p = s.p + (s.v * dt + u * (0.5f * dt * dt));
  o.v = s.v + (s.x + u) * (0.5f * dt);
  o.x = u;
  return o;
}
QS_D void step_pmd_vjp(const State& gs, const DynK& k, State& gi, V3& gu) {
  const float dt = k.dt;
  gi.p = gs.p;
  gi.v = gs.v + gs.p * dt;
  gi.x = gs.v * (0.5f * dt);
  gu = gs.p * (0.5f * dt * dt) + gs.v * (0.5f * dt) + gs.x;
  gi.q = q4(0.f, 0.f, 0.f, 0.f);
  gi.w = gi.ve = v3(0.f, 0.f, 0.f);
}

// step_simplified (q/dynamics.py:189-234): v' = v + (R e_z c + g) dt,
// R' = GramSchmidt(R + R [w]x dt) on columns 0,1 (z = x cross y), body rates
// are the command (cmd = (c, wx, wy, wz)).
struct GsFwd {
  V3 m0, m1, xn, yn, yo;
  float n0, n1, s;
};
QS_D GsFwd simplified_gs(const State& s, float4 cmd, float dt) {
  GsFwd f;
  const float wx = cmd.y, wy = cmd.z, wz = cmd.w;
  f.m0 = s.r0 + (s.r1 * wz - s.r2 * wy) * dt;  // column 0 of R + R S dt
  f.m1 = s.r1 + (s.r2 * wx - s.r0 * wz) * dt;  // column 1
  f.n0 = norm3(f.m0);
  f.xn = f.m0 * (1.f / f.n0);
  f.s = dot(f.m1, f.xn);
  f.yo = f.m1 - f.xn * f.s;
  f.n1 = norm3(f.yo);
  f.yn = f.yo * (1.f / f.n1);
  return f;
}

QS_D State step_simplified(const State& s, float4 cmd, const DynK& k) {
  const float dt = k.dt;
  GsFwd f = simplified_gs(s, cmd, dt);
  State o = s;
  V3 vdot = s.r2 * cmd.x + k.g;
  o.p = s.p + s.v * dt;
  o.v = s.v + vdot * dt;
  o.r0 = f.xn;
  o.r1 = f.yn;
  o.r2 = cross(f.xn, f.yn);
  return o;
}

QS_D void step_simplified_vjp(const State& s, float4 cmd, const DynK& k, const State& gs, State& gi,
                              float4& gc) {
  const float dt = k.dt;
  GsFwd f = simplified_gs(s, cmd, dt);
  gi = zero_state_like();
  gi.p = gs.p;
  gi.v = gs.v + gs.p * dt;
  V3 gvdot = gs.v * dt;
  float g_c = dot(gvdot, s.r2);
  V3 g_r2 = gvdot * cmd.x;
  // z' = xn x yn
  V3 g_xn = gs.r0 + cross(f.yn, gs.r2);
  V3 g_yn = gs.r1 + cross(gs.r2, f.xn);
  // yn = yo / |yo|
  V3 g_yo = (g_yn - f.yn * dot(f.yn, g_yn)) * (1.f / f.n1);
  // yo = m1 - xn (m1 . xn)
  V3 g_m1 = g_yo;
  g_xn -= g_yo * f.s;
  float g_s = -dot(f.xn, g_yo);
  g_m1 += f.xn * g_s;
  g_xn += f.m1 * g_s;
  // xn = m0 / |m0|
  V3 g_m0 = (g_xn - f.xn * dot(f.xn, g_xn)) * (1.f / f.n0);
  const float wx = cmd.y, wy = cmd.z, wz = cmd.w;
  gi.r0 = g_m0 - g_m1 * (dt * wz);
  gi.r1 = g_m1 + g_m0 * (dt * wz);
  gi.r2 = g_r2 + (g_m1 * wx - g_m0 * wy) * dt;
  gc = make_float4(g_c, dt * dot(s.r2, g_m1), -dt * dot(s.r2, g_m0), dt * (dot(s.r1, g_m0) - dot(s.r0, g_m1)));
}

template <int M>
QS_D State model_step(const State& s, float4 cmd, const RowPrm& rp, const DynK& k) {
  if (M == QS_MODEL_SIMPLIFIED) return step_simplified(s, cmd, k);
  if (M == QS_MODEL_FULL) return step_full(s, cmd, k);
  V3 u = v3(cmd.x, cmd.y, cmd.z);
  if (M == QS_MODEL_PM_CONTINUOUS) return step_pmc(s, u, rp.drag, rp.decay, k);
  return step_pmd(s, u, k);
}

template <int M>
QS_D void model_step_vjp(const State& s, float4 cmd, const RowPrm& rp, const DynK& k,
                         const State& gs, State& gi, float4& gc) {
  if (M == QS_MODEL_SIMPLIFIED) {
    step_simplified_vjp(s, cmd, k, gs, gi, gc);
  } else if (M == QS_MODEL_FULL) {
    step_full_vjp(s, cmd, k, gs, gi, gc);
  } else {
    V3 gu;
    if (M == QS_MODEL_PM_CONTINUOUS)
      step_pmc_vjp(gs, rp.drag, rp.decay, k, gi, gu);
    else
      step_pmd_vjp(gs, k, gi, gu);
    gc = make_float4(gu.x, gu.y, gu.z, 0.f);
  }
}


template <int M>
QS_D State load_grad(const float* G, long N, long row) {
  if (!G) return zero_state();
  State g = load_state<M>(G, N, row);
  g.ve = v3(0.f, 0.f, 0.f);
  return g;
}
