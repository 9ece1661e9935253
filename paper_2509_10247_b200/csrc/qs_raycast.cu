// Per-ray ray casting against analytic obstacles: depth camera, LiDAR and
// generic rays (q/sensors.py:131-269, 276-410), plus the opt-in analytic
// depth VJP (new; no reference counterpart, q/sensors.py:4-6).
//
// Layout: one CTA per (row, ray chunk).  The CTA stages its env's obstacles
// in shared memory ONCE, hoisting every ray-invariant term (o - c, |o-c|^2 - r^2,
// slab offsets, ...) and dropping obstacles the conservative frustum /
// range-ball test proves unreachable (never changes the image, q/sensors.py:
// 338-374); each thread then owns RPT rays and keeps its running min-t in
// registers, reading obstacle records as shared-memory broadcasts.
#include "qs_dynamics.cuh"
#include "qs_geom.cuh"

namespace {

constexpr int RAY_BLOCK = 256;
constexpr float INF = __builtin_huge_valf();

// NaN-propagating min/max (PTX min.NaN/max.NaN, sm_80+): a NaN slab term makes
// the whole box test fail exactly like the reference's nan_to_num dance
// (q/sensors.py:157-159).
QS_D float fmin_nan(float a, float b) {
  float d;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}
QS_D float fmax_nan(float a, float b) {
  float d;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}
QS_D float sqrt_approx(float x) {
  float d;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(d) : "f"(x));
  return d;
}

// conservative keep tests (fp32 margins absorb rounding; the reference uses
// 1e-9 in fp64)
QS_D bool keep_camera(const qs_ray_cfg& rc, float2 cs, V3 o, V3 c, float rad) {
  V3 l = unrotz(cs, c - o);  // camera-frame centre (yaw-only attitude)
  const float m = 1e-3f * (1.f + fabsf(l.x) + fabsf(l.y) + fabsf(l.z));
  const float nh = rsqrtf(rc.tan_h * rc.tan_h + 1.f), nv = rsqrtf(rc.tan_v * rc.tan_v + 1.f);
  bool in = (rc.tan_h * l.x - l.y) * nh >= -rad - m;
  in = in && (rc.tan_h * l.x + l.y) * nh >= -rad - m;
  in = in && (rc.tan_v * l.x - l.z) * nv >= -rad - m;
  in = in && (rc.tan_v * l.x + l.z) * nv >= -rad - m;
  in = in && l.x >= -rad - m;
  in = in && norm3(l) - rad <= rc.max_range + m;
  return in;
}
QS_D bool keep_ball(const qs_ray_cfg& rc, V3 o, V3 c, float rad) {
  V3 l = c - o;
  const float m = 1e-3f * (1.f + fabsf(l.x) + fabsf(l.y) + fabsf(l.z));
  return norm3(l) - rad <= rc.max_range + m;
}

// --- ray-primitive tests on hoisted records ---------------------------------
// One arithmetic core per primitive, shared by the untiled kernel (float
// min-t, argmin for the depth VJP) and the tiled one (min-t in IEEE bit
// order, below), so both kernels produce identical images.

QS_D float rcp_fast(float x) {  // one MUFU.RCP; 1/(+-0) = +-inf, 1/(+-inf) = +-0
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
QS_D float pos0(float x) { return __fadd_rn(x, 0.f); }  // -0 -> +0, else x
// yaw rotation and |d_xy|^2 with explicit FMAs, so every kernel (and every
// tile width) rounds them identically
QS_D V3 rotz_f(float2 cs, V3 v) { return v3(fmaf(cs.x, v.x, -cs.y * v.y), fmaf(cs.y, v.x, cs.x * v.y), v.z); }
QS_D float dxy2(V3 d) { return fmaf(d.x, d.x, d.y * d.y); }

// sphere record: (oc.xyz, r^2), oc = o - c.  Robust discriminant
// r^2 - |oc - b d|^2 (== b^2 - (|oc|^2 - r^2) in exact arithmetic); its sqrt is
// NaN when it is negative (a miss), so both roots are NaN then.  t1 <= t2.
QS_D float2 sphere_roots(float4 s, V3 d) {
  const float b = fmaf(d.x, s.x, fmaf(d.y, s.y, d.z * s.z));
  const float vx = fmaf(-b, d.x, s.x), vy = fmaf(-b, d.y, s.y), vz = fmaf(-b, d.z, s.z);
  const float disc = fmaf(-vx, vx, fmaf(-vy, vy, fmaf(-vz, vz, s.w)));
  const float sq = sqrt_approx(disc);
  return make_float2(-b - sq, sq - b);
}
QS_D float hit_sphere(float4 s, V3 d) {
  const float2 r = sphere_roots(s, d);
  return r.x >= 0.f ? r.x : (r.y >= 0.f ? r.y : INF);  // NaN compares false
}

// box record: lo - o, hi - o.  Slab entry/exit with NaN-propagating min/max.
QS_D void box_slab(float4 lo, float4 hi, V3 inv, float& tn, float& tf, int* axis) {
  const float t1x = lo.x * inv.x, t2x = hi.x * inv.x;
  const float t1y = lo.y * inv.y, t2y = hi.y * inv.y;
  const float t1z = lo.z * inv.z, t2z = hi.z * inv.z;
  const float nx = fmin_nan(t1x, t2x), fx = fmax_nan(t1x, t2x);
  const float ny = fmin_nan(t1y, t2y), fy = fmax_nan(t1y, t2y);
  const float nz = fmin_nan(t1z, t2z), fz = fmax_nan(t1z, t2z);
  tn = fmax_nan(fmax_nan(nx, ny), nz);
  tf = fmin_nan(fmin_nan(fx, fy), fz);
  if (axis) {  // face normal axis of the returned root (depth VJP)
    if (tn >= 0.f)
      *axis = (tn == nx) ? 0 : (tn == ny ? 1 : 2);
    else
      *axis = (tf == fx) ? 0 : (tf == fy ? 1 : 2);
  }
}
QS_D float hit_box(float4 lo, float4 hi, V3 inv, int* axis) {
  float tn, tf;
  box_slab(lo, hi, inv, tn, tf, axis);
  const bool hit = (tn <= tf) && (tf >= 0.f);
  return hit ? (tn >= 0.f ? tn : tf) : INF;
}

// capped z-cylinder: record (o - c, r^2) and the cap planes relative to o
// (ztop = hh - (o-c).z, zbot = -hh - (o-c).z).  Robust side discriminant
// a r^2 - (ox dy - oy dx)^2 (Lagrange identity).  Side roots count within
// |z| <= hh, cap roots within the disc; degenerate rays give NaN roots
// (a = 0: 0 * inf; dz = 0: inf - inf in the cap point) that fail every test.
struct CylRoots {
  float ts1, ts2, tt, tb;
  bool z1, z2, ct, cb;
};
QS_D CylRoots cyl_roots(float4 c, float hh, float ztop, float zbot, V3 d, float a, float inv_a, float inv_dz) {
  CylRoots r;
  const float b = fmaf(c.x, d.x, c.y * d.y);
  const float cr = fmaf(c.x, d.y, -c.y * d.x);
  const float disc = fmaf(a, c.w, -cr * cr);
  const float sq = sqrt_approx(disc);
  r.ts1 = (-b - sq) * inv_a;  // -0 only together with ts2 = +0
  r.ts2 = (sq - b) * inv_a;
  r.z1 = fabsf(fmaf(r.ts1, d.z, c.z)) <= hh;
  r.z2 = fabsf(fmaf(r.ts2, d.z, c.z)) <= hh;
  r.tt = pos0(ztop * inv_dz);
  r.tb = pos0(zbot * inv_dz);
  const float xt = fmaf(r.tt, d.x, c.x), yt = fmaf(r.tt, d.y, c.y);
  const float xb = fmaf(r.tb, d.x, c.x), yb = fmaf(r.tb, d.y, c.y);
  r.ct = fmaf(xt, xt, yt * yt) <= c.w;  // false for inf / NaN cap points
  r.cb = fmaf(xb, xb, yb * yb) <= c.w;
  return r;
}
QS_D float hit_cyl(float4 c, float hh, float ztop, float zbot, V3 d, float a, float inv_a, float inv_dz, int* part) {
  const CylRoots r = cyl_roots(c, hh, ztop, zbot, d, a, inv_a, inv_dz);
  const float ts = (r.z1 && r.ts1 >= 0.f) ? r.ts1 : ((r.z2 && r.ts2 >= 0.f) ? r.ts2 : INF);
  const float tc = fminf((r.ct && r.tt >= 0.f) ? r.tt : INF, (r.cb && r.tb >= 0.f) ? r.tb : INF);
  if (part) *part = (ts <= tc) ? 0 : 1;
  return fminf(ts, tc);
}

template <int KIND, bool GRAD>
__global__ void __launch_bounds__(RAY_BLOCK) k_raycast(const qs_ray_cfg rc, const qs_scene sc,
                                                       int n_rows, const float* __restrict__ pos,
                                                       int pos_stride, const float* __restrict__ cam_cs,
                                                       const float* __restrict__ dirs_body,
                                                       const float* __restrict__ dirs_world,
                                                       float* __restrict__ out, uint8_t* __restrict__ hitm,
                                                       float* __restrict__ dT_dO, int rays_per_cta) {
  extern __shared__ float4 sm[];
  __shared__ int cnt[3];
  const long row = blockIdx.y;
  const long e = row / rc.n_agents;
  const int r0 = blockIdx.x * rays_per_cta;
  const int r1 = min(rc.n_rays, r0 + rays_per_cta);
  float2 cs = make_float2(1.f, 0.f);
  if (cam_cs) cs = reinterpret_cast<const float2*>(cam_cs)[row];
  const float* pp = pos + row * pos_stride;
  V3 off = rotz_f(cs, v3(rc.offset[0], rc.offset[1], rc.offset[2]));
  V3 o = v3(pp[0], pp[1], pp[2]) + off;
  SceneView sv = scene_view(sc, e);
  float4* s_sph = sm;
  float4* s_box = sm + sc.Sm;
  float4* s_cyl = s_box + 2 * sc.Bm;
  float* s_cyl_hh = reinterpret_cast<float*>(s_cyl + sc.Cm);
  if (threadIdx.x < 3) cnt[threadIdx.x] = 0;
  __syncthreads();
  // stage + cull; compaction order is arbitrary, which is fine: min-t is
  // order independent (fminf is exact), so the image is deterministic
  const int tot = sv.ns + sv.nb + sv.nc;
  for (int i = threadIdx.x; i < tot; i += blockDim.x) {
    if (i < sv.ns) {
      float4 s = ld4(sv.sph, i);
      V3 c = xyz(s);
      bool keep = !(rc.cull & 1) || (KIND == 0 ? keep_camera(rc, cs, o, c, s.w) : keep_ball(rc, o, c, s.w));
      if (keep) {
        int k = atomicAdd(&cnt[0], 1);
        V3 oc = o - c;
        s_sph[k] = f4(oc, s.w * s.w);
      }
    } else if (i < sv.ns + sv.nb) {
      int j = i - sv.ns;
      float4 c = ld4(sv.box, 2 * j), h = ld4(sv.box, 2 * j + 1);
      float rad = norm3(xyz(h));
      bool keep = !(rc.cull & 1) ||
                  (KIND == 0 ? keep_camera(rc, cs, o, xyz(c), rad) : keep_ball(rc, o, xyz(c), rad));
      if (keep) {
        int k = atomicAdd(&cnt[1], 1);
        s_box[2 * k] = f4(xyz(c) - xyz(h) - o, 0.f);
        s_box[2 * k + 1] = f4(xyz(c) + xyz(h) - o, 0.f);
      }
    } else {
      int j = i - sv.ns - sv.nb;
      float4 c = ld4(sv.cyl, 2 * j);
      float hh = __ldg(sv.cyl + 8 * j + 4);
      float rad = sqrtf(c.w * c.w + hh * hh);
      bool keep = !(rc.cull & 1) ||
                  (KIND == 0 ? keep_camera(rc, cs, o, xyz(c), rad) : keep_ball(rc, o, xyz(c), rad));
      if (keep) {
        int k = atomicAdd(&cnt[2], 1);
        s_cyl[k] = make_float4(o.x - c.x, o.y - c.y, o.z - c.z, c.w * c.w);
        s_cyl_hh[k] = hh;
      }
    }
  }
  __syncthreads();
  const int ns = cnt[0], nb = cnt[1], nc = cnt[2];
  const bool ground = sv.ground;
  const float gdz = sv.gz - o.z;
  for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    V3 d;
    if (KIND == 2) {
      d = xyz(ld4(dirs_world, row * rc.n_rays + r));
    } else {
      d = rotz_f(cs, xyz(ld4(dirs_body, r)));
    }
    const V3 inv = v3(rcp_fast(d.x), rcp_fast(d.y), rcp_fast(d.z));
    const float a = dxy2(d);
    const float inv_a = rcp_fast(a);
    float best = INF;
    int code = 0, bidx = 0;  // kind | detail, shared-memory index of the argmin
    for (int i = 0; i < ns; ++i) {
      float t = hit_sphere(s_sph[i], d);
      if (GRAD) {
        if (t < best) { best = t; code = 1; bidx = i; }
      } else {
        best = fminf(best, t);
      }
    }
    for (int i = 0; i < nb; ++i) {
      int ax = 0;
      float t = hit_box(s_box[2 * i], s_box[2 * i + 1], inv, GRAD ? &ax : nullptr);
      if (GRAD) {
        if (t < best) { best = t; code = 2 | (ax << 4); bidx = i; }
      } else {
        best = fminf(best, t);
      }
    }
    for (int i = 0; i < nc; ++i) {
      int part = 0;
      const float4 c = s_cyl[i];
      const float hh = s_cyl_hh[i];
      float t = hit_cyl(c, hh, hh - c.z, -hh - c.z, d, a, inv_a, inv.z, GRAD ? &part : nullptr);
      if (GRAD) {
        if (t < best) { best = t; code = 3 | (part << 4); bidx = i; }
      } else {
        best = fminf(best, t);
      }
    }
    if (ground) {
      float t = gdz * inv.z;
      bool ok = t >= 0.f && t < INF;  // isfinite(t) && t >= 0
      if (ok && t < best) { best = t; code = 4; }
    }
    float tout = fminf(best, rc.max_range);
    const long oi = row * rc.n_rays + r;
    out[oi] = tout;
    if (hitm) hitm[oi] = best < rc.max_range ? 1 : 0;
    if (GRAD) {
      // d t / d o = -n / (n . d) at the hit surface; 0 when clamped / missed
      V3 n = v3(0.f, 0.f, 0.f);
      if (best < rc.max_range) {
        int kind = code & 15;
        if (kind == 1) {
          n = xyz(s_sph[bidx]) + d * best;  // x - c = oc + t d
        } else if (kind == 2) {
          int ax = code >> 4;
          n = v3(ax == 0 ? 1.f : 0.f, ax == 1 ? 1.f : 0.f, ax == 2 ? 1.f : 0.f);
        } else if (kind == 3) {
          if ((code >> 4) == 0) {
            float4 c = s_cyl[bidx];
            n = v3(c.x + best * d.x, c.y + best * d.y, 0.f);
          } else {
            n = v3(0.f, 0.f, 1.f);
          }
        } else if (kind == 4) {
          n = v3(0.f, 0.f, 1.f);
        }
      }
      float nd = dot(n, d);
      V3 g = nd != 0.f ? n * (-1.f / nd) : v3(0.f, 0.f, 0.f);
      reinterpret_cast<float4*>(dT_dO)[oi] = f4(g, 0.f);
    }
  }
}

// ---------------------------------------------------------------------------
// tiled variant: rays are grouped host-side into tiles of 32 angularly compact
// rays (8x4 pixel blocks for cameras, 2 azimuths x 16 elevations for LiDAR);
// each tile carries a bounding cone (axis, cos/sin of its half-angle, body
// frame).  A warp owns a tile: lane j tests staged obstacle j's bounding
// sphere against the cone, one ballot per 32 obstacles gives the warp-uniform
// candidate mask, and every lane intersects its ray with the candidates only.
// The surviving set is a superset of the obstacles any ray of the tile can
// hit, so the image is identical to the untiled kernel's.

// bounding-sphere record, hoisted once per (env, obstacle):
//   b = (u = c - o, Q)  with Q = sqrt(|u|^2 - r^2) the tangent length (-1: o inside)
//   e = (r, slack)      slack = 1e-4 (1 + |u|) absorbs fp32 round-off
// keep iff angle(u, axis) <= half-angle + asin(r/|u|)
//      <=> u . axis >= cos(th) Q - sin(th) r           (times |u| on both sides)
QS_D float4 bsphere(V3 u, float r, float2& e) {
  float L2 = dot(u, u);
  float L = sqrtf(L2);
  e = make_float2(r, 1e-4f * (1.f + L));
  return f4(u, L2 <= r * r ? -1.f : sqrtf(L2 - r * r));
}
QS_D bool cone_keeps(float4 b, float2 e, V3 ax, float cth, float sth) {
  if (b.w < 0.f) return true;
  return dot(xyz(b), ax) >= cth * b.w - sth * e.x - e.y;
}
// azimuth record of an obstacle's horizontal footprint seen from o: the unit
// centre direction and cos/sin of the half-width of the angular interval it
// covers (ch < -1.5: o is inside the footprint, keep for every azimuth).
// Circles (spheres, cylinders) are exact; a box's footprint rectangle uses the
// extreme corners.  Every ray that hits the obstacle crosses its footprint, so
// its azimuth lies in that interval; a tile whose azimuth sector misses the
// interval cannot hit it.
QS_D float4 az_circle(V3 u, float r2) {
  const float L2 = u.x * u.x + u.y * u.y;
  if (L2 <= r2 * r2 * (1.f + 1e-4f) + 1e-8f) return make_float4(1.f, 0.f, -2.f, 0.f);
  const float il = rsqrtf(L2), sh = fminf(r2 * il, 1.f);
  return make_float4(u.x * il, u.y * il, sqrtf(fmaxf(1.f - sh * sh, 0.f)), sh);
}
// horizontal footprint circle record (u2 = (c - o).xy, Q2 = tangent length, r2 =
// radius; Q2 = -1: o is inside) and its sector test in distance units
QS_D float4 footprint(V3 u, float r2) {
  float L2 = u.x * u.x + u.y * u.y;
  return make_float4(u.x, u.y, L2 <= r2 * r2 ? -1.f : sqrtf(L2 - r2 * r2), r2);
}
QS_D bool circle_sector_keeps(float4 h, float slack, float2 az, float cw, float sw) {
  if (h.z < 0.f || cw < -1.5f) return true;
  return h.x * az.x + h.y * az.y >= cw * h.z - sw * h.w - slack;
}
// pseudo-angle of (x, y): strictly increasing in atan2(y, x) over (-pi, pi]
QS_D float pseudo_angle(float x, float y) {
  const float q = __fdividef(y, fabsf(x) + fabsf(y));
  return x >= 0.f ? q : (y >= 0.f ? 2.f - q : -2.f - q);
}
QS_D float4 az_rect(V3 u, float hx, float hy) {
  const float m = 1e-4f * (1.f + fabsf(u.x) + fabsf(u.y));
  if (fabsf(u.x) <= hx + m && fabsf(u.y) <= hy + m) return make_float4(1.f, 0.f, -2.f, 0.f);
  const float il = rsqrtf(u.x * u.x + u.y * u.y);
  const float cx = u.x * il, cy = u.y * il;  // frame: c along +x
  float plo = 3.f, phi = -3.f;
  float2 e1 = make_float2(cx, cy), e2 = e1;
#pragma unroll
  for (int k = 0; k < 4; ++k) {  // the corners with the extreme angles about c
    const float kx = u.x + ((k & 1) ? hx : -hx), ky = u.y + ((k & 2) ? hy : -hy);
    const float pa = pseudo_angle(cx * kx + cy * ky, cx * ky - cy * kx);
    const float ik = rsqrtf(kx * kx + ky * ky);
    if (pa < plo) { plo = pa; e1 = make_float2(kx * ik, ky * ik); }
    if (pa > phi) { phi = pa; e2 = make_float2(kx * ik, ky * ik); }
  }
  const float sx = e1.x + e2.x, sy = e1.y + e2.y, s2 = sx * sx + sy * sy;
  if (s2 < 0.05f) return make_float4(1.f, 0.f, -2.f, 0.f);  // interval close to a half-turn
  const float is = rsqrtf(s2);
  const float ax = sx * is, ay = sy * is;
  const float ch = fmaxf(ax * e1.x + ay * e1.y - 1e-4f, 0.f);  // widened by ~1e-4 for round-off
  return make_float4(ax, ay, ch, sqrtf(fmaxf(1.f - ch * ch, 0.f)));
}
// angle(az, centre) <= w + h  <=>  az . centre >= cos(w + h)   (w, h <= pi/2)
QS_D bool sector_keeps(float4 h, float2 az, float cw, float sw) {
  if (h.z < -1.5f || cw < -1.5f) return true;
  return h.x * az.x + h.y * az.y >= cw * h.z - sw * h.w - 1e-4f;
}
// vertical flags: a ray that never rises (d.z <= 0) cannot reach an obstacle
// entirely above o, nor one that never falls an obstacle entirely below it

// --- min-t in IEEE bit order (tiled kernel) ----------------------------------
// Non-negative floats order as their bit patterns read as unsigned ints, and
// every negative float and every NaN reads as a larger unsigned than +inf.  So
// one integer min over the candidate roots keeps exactly the roots the
// reference accepts (finite or +inf, t >= 0; q/sensors.py:139-216) and drops
// roots behind the origin and NaN roots (missed discriminant -> sqrt of a
// negative; 0 * inf slab terms) with no compares or selects.  A -0 root (the
// origin exactly on a surface plane) is canonicalised to +0 where one can
// arise, because the reference counts t = -0.0 as t >= 0.
constexpr unsigned INF_BITS = 0x7f800000u;
QS_D unsigned fbits(float x) { return __float_as_uint(x); }
QS_D unsigned umin3(unsigned a, unsigned b, unsigned c) { return min(a, min(b, c)); }

QS_D unsigned hit_sphere_u(unsigned best, float4 s, V3 d) {
  const float2 r = sphere_roots(s, d);  // t1 <= t2: the min non-negative root is the reference's
  return umin3(best, fbits(r.x), fbits(r.y));  // -0 t1 comes with +0 t2
}
QS_D unsigned hit_box_u(unsigned best, float4 lo, float4 hi, V3 inv) {
  float tn, tf;  // hit iff tn <= tf and tf >= 0, at tn if tn >= 0 else tf
  box_slab(lo, hi, inv, tn, tf, nullptr);
  const unsigned c = min(fbits(pos0(tn)), fbits(pos0(tf)));
  return tn <= tf ? min(best, c) : best;
}
QS_D unsigned hit_cyl_u(unsigned best, float4 c, float4 h, V3 d, float a, float inv_a, float inv_dz) {
  const CylRoots r = cyl_roots(c, h.x, h.y, h.z, d, a, inv_a, inv_dz);
  unsigned m = best;
  m = r.z1 ? min(m, fbits(r.ts1)) : m;
  m = r.z2 ? min(m, fbits(r.ts2)) : m;
  m = r.ct ? min(m, fbits(r.tt)) : m;
  m = r.cb ? min(m, fbits(r.tb)) : m;
  return m;
}
// --- packed ray pairs (FFMA2/FMUL2/FADD2, sm_100) -----------------------------
// Two rays of a lane run each test as f32x2 instructions with the obstacle
// record as a broadcast scalar operand.  Every packed op is the same IEEE
// rn op the scalar cores above perform, in the same order, so a pair's depths
// are bit-identical to the scalar (and untiled) kernels'.
struct RayPair {
  float2 dx, dy, dz;  // directions
  float2 ix, iy, iz;  // reciprocal components
  float2 a, ia;       // dx^2 + dy^2 and its reciprocal
};
QS_D float2 bc(float x) { return make_float2(x, x); }
QS_D float2 neg2(float2 v) { return make_float2(-v.x, -v.y); }
QS_D void hit_sphere_p(unsigned& b0, unsigned& b1, float4 s, const RayPair& r) {
  const float2 b = __ffma2_rn(r.dx, bc(s.x), __ffma2_rn(r.dy, bc(s.y), __fmul2_rn(r.dz, bc(s.z))));
  const float2 nb = neg2(b);
  const float2 vx = __ffma2_rn(nb, r.dx, bc(s.x)), vy = __ffma2_rn(nb, r.dy, bc(s.y)),
               vz = __ffma2_rn(nb, r.dz, bc(s.z));
  const float2 disc = __ffma2_rn(neg2(vx), vx, __ffma2_rn(neg2(vy), vy, __ffma2_rn(neg2(vz), vz, bc(s.w))));
  const float2 sq = make_float2(sqrt_approx(disc.x), sqrt_approx(disc.y));
  const float2 t1 = __fadd2_rn(nb, neg2(sq)), t2 = __fadd2_rn(sq, nb);
  b0 = umin3(b0, fbits(t1.x), fbits(t2.x));
  b1 = umin3(b1, fbits(t1.y), fbits(t2.y));
}
QS_D unsigned box_u(unsigned best, float t1x, float t2x, float t1y, float t2y, float t1z, float t2z) {
  const float tn = fmax_nan(fmax_nan(fmin_nan(t1x, t2x), fmin_nan(t1y, t2y)), fmin_nan(t1z, t2z));
  const float tf = fmin_nan(fmin_nan(fmax_nan(t1x, t2x), fmax_nan(t1y, t2y)), fmax_nan(t1z, t2z));
  const unsigned c = min(fbits(pos0(tn)), fbits(pos0(tf)));
  return tn <= tf ? min(best, c) : best;
}
QS_D void hit_box_p(unsigned& b0, unsigned& b1, float4 lo, float4 hi, const RayPair& r) {
  const float2 t1x = __fmul2_rn(bc(lo.x), r.ix), t2x = __fmul2_rn(bc(hi.x), r.ix);
  const float2 t1y = __fmul2_rn(bc(lo.y), r.iy), t2y = __fmul2_rn(bc(hi.y), r.iy);
  const float2 t1z = __fmul2_rn(bc(lo.z), r.iz), t2z = __fmul2_rn(bc(hi.z), r.iz);
  b0 = box_u(b0, t1x.x, t2x.x, t1y.x, t2y.x, t1z.x, t2z.x);
  b1 = box_u(b1, t1x.y, t2x.y, t1y.y, t2y.y, t1z.y, t2z.y);
}
QS_D unsigned cyl_u(unsigned m, float ts1, float ts2, float zs1, float zs2, float tt, float tb, float rt2,
                    float rb2, float hh, float r2) {
  m = fabsf(zs1) <= hh ? min(m, fbits(ts1)) : m;
  m = fabsf(zs2) <= hh ? min(m, fbits(ts2)) : m;
  m = rt2 <= r2 ? min(m, fbits(tt)) : m;
  m = rb2 <= r2 ? min(m, fbits(tb)) : m;
  return m;
}
QS_D void hit_cyl_p(unsigned& b0, unsigned& b1, float4 c, float4 h, const RayPair& r) {
  const float2 b = __ffma2_rn(bc(c.x), r.dx, __fmul2_rn(bc(c.y), r.dy));
  const float2 cr = __ffma2_rn(bc(c.x), r.dy, neg2(__fmul2_rn(bc(c.y), r.dx)));
  const float2 disc = __ffma2_rn(r.a, bc(c.w), neg2(__fmul2_rn(cr, cr)));
  const float2 sq = make_float2(sqrt_approx(disc.x), sqrt_approx(disc.y));
  const float2 nb = neg2(b);
  const float2 ts1 = __fmul2_rn(__fadd2_rn(nb, neg2(sq)), r.ia), ts2 = __fmul2_rn(__fadd2_rn(sq, nb), r.ia);
  const float2 zs1 = __ffma2_rn(ts1, r.dz, bc(c.z)), zs2 = __ffma2_rn(ts2, r.dz, bc(c.z));
  const float2 tt = __fadd2_rn(__fmul2_rn(bc(h.y), r.iz), bc(0.f));  // pos0
  const float2 tb = __fadd2_rn(__fmul2_rn(bc(h.z), r.iz), bc(0.f));
  const float2 xt = __ffma2_rn(tt, r.dx, bc(c.x)), yt = __ffma2_rn(tt, r.dy, bc(c.y));
  const float2 xb = __ffma2_rn(tb, r.dx, bc(c.x)), yb = __ffma2_rn(tb, r.dy, bc(c.y));
  const float2 rt2 = __ffma2_rn(xt, xt, __fmul2_rn(yt, yt)), rb2 = __ffma2_rn(xb, xb, __fmul2_rn(yb, yb));
  b0 = cyl_u(b0, ts1.x, ts2.x, zs1.x, zs2.x, tt.x, tb.x, rt2.x, rb2.x, h.x, c.w);
  b1 = cyl_u(b1, ts1.y, ts2.y, zs1.y, zs2.y, tt.y, tb.y, rt2.y, rb2.y, h.x, c.w);
}

// lanes [0, k) of a warp, k clamped to [0, 32]
QS_D unsigned lanes_below(int k) { return k >= 32 ? 0xffffffffu : (k <= 0 ? 0u : (1u << k) - 1u); }

#ifndef QS_TILED_BLOCK
// one warp per env: staging needs no CTA barrier and its latency is spread
// over all of the env's tiles; 24+ resident CTAs per SM cap the registers so
// that ~32 warps fit (measured best: profiles/README.md)
#define QS_TILED_BLOCK 32
#endif
#ifndef QS_TILED_MINB
#define QS_TILED_MINB 24
#endif
constexpr int TILED_BLOCK = QS_TILED_BLOCK;

// EXT (qs_ray_cfg.cull bit 1): box footprints use their exact azimuth interval
// and every obstacle carries vertical flags.  That costs a third record load
// per (tile, obstacle) and pays off when large boxes (indoor shells: walls,
// ceiling) would otherwise be candidates for every tile.
// RPL rays per lane: a tile holds 32 * RPL rays (lane j owns rays j, j + 32,
// ...), so the tile's cone test, ballot, candidate loop and obstacle-record
// loads are shared by RPL rays, and each candidate runs RPL independent tests.
//
// GRAD: the depth VJP by recasting (no per-ray dT/dO in HBM).  The same tiles
// and culls, but each lane tracks the argmin primitive of its rays with the
// untiled kernel's float tests (same cores, same first-wins tie rule within the
// kind order), then accumulates g_depth[ray] * dt/do = -n/(n.d) of the hit
// surface; one warp reduction per row adds the sum into g_pos.
template <int KIND, bool EXT, int RPL, bool GRAD = false>
__global__ void __launch_bounds__(TILED_BLOCK, QS_TILED_MINB) k_raycast_tiled(
    const qs_ray_cfg rc, const qs_scene sc, int n_rows, const float* __restrict__ pos, int pos_stride,
    const float* __restrict__ cam_cs, const float* __restrict__ tile_dirs, const float* __restrict__ tile_cones,
    int n_tiles, int tiles_per_cta, float* __restrict__ out, uint8_t* __restrict__ hitm,
    const float* __restrict__ g_depth = nullptr, float* __restrict__ g_pos = nullptr, int gpos_stride = 4) {
  extern __shared__ float4 sm[];
  __shared__ int cnt[3];
  const long row = blockIdx.y;
  const long e = row / rc.n_agents;
  float2 cs = make_float2(1.f, 0.f);
  if (cam_cs) cs = reinterpret_cast<const float2*>(cam_cs)[row];
  const float* pp = pos + row * pos_stride;
  V3 o = v3(pp[0], pp[1], pp[2]) + rotz_f(cs, v3(rc.offset[0], rc.offset[1], rc.offset[2]));
  SceneView sv = scene_view(sc, e);
  // One list of kept obstacles in input order (spheres, boxes, cylinders, so
  // the list stays kind-sorted), each with two intersection records
  //   sphere (o - c, r^2) | box (lo - o), (hi - o) | cylinder (o - c, r^2), (hh)
  // plus its bounding sphere, horizontal footprint and slack.  Warp 0 builds it
  // with ballot compaction (no atomics, one CTA barrier); a single ballot per 32
  // entries then culls every kind at once for a tile.
  const int cap = sc.Sm + sc.Bm + sc.Cm;
  float4* r0 = sm;
  float4* r1 = r0 + cap;
  float4* b_all = r1 + cap;  // bounding sphere (u = c - o, Q)
  // EXT: a_all = azimuth interval of the footprint; f_all.xy = (r, slack) with
  // the sign bits as vertical flags (r < 0: entirely above o, slack < 0:
  // entirely below).  Otherwise f_all = (r, slack, Q2, r2): the footprint
  // circle's tangent length and radius for the sector test, a_all unused.
  float4* a_all = b_all + cap;
  float4* f_all = a_all + (EXT ? cap : 0);
  uint2* kmask = reinterpret_cast<uint2*>(f_all + cap);  // per 32-chunk: (sphere lanes, sphere|box lanes)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  if (warp == 0) {
    const int tot_in = sv.ns + sv.nb + sv.nc;
    int run = 0, ks = 0, kb = 0;
    for (int c0 = 0; c0 < tot_in; c0 += 32) {
      const int i = c0 + lane;
      bool keep = false;
      float4 q0, q1, bs, az;
      float2 ee;
      float zl, zh;
      if (i < sv.ns) {
        float4 sp = ld4(sv.sph, i);
        V3 c = xyz(sp);
        keep = !(rc.cull & 1) || (KIND == 0 ? keep_camera(rc, cs, o, c, sp.w) : keep_ball(rc, o, c, sp.w));
        q0 = f4(o - c, sp.w * sp.w);
        q1 = make_float4(0.f, 0.f, 0.f, 0.f);
        bs = bsphere(c - o, sp.w, ee);
        az = EXT ? az_circle(c - o, sp.w) : footprint(c - o, sp.w);
        zl = c.z - sp.w - o.z;
        zh = c.z + sp.w - o.z;
      } else if (i < sv.ns + sv.nb) {
        int j = i - sv.ns;
        float4 c = ld4(sv.box, 2 * j), h = ld4(sv.box, 2 * j + 1);
        float rad = norm3(xyz(h));
        keep = !(rc.cull & 1) || (KIND == 0 ? keep_camera(rc, cs, o, xyz(c), rad) : keep_ball(rc, o, xyz(c), rad));
        q0 = f4(xyz(c) - xyz(h) - o, 0.f);
        q1 = f4(xyz(c) + xyz(h) - o, 0.f);
        bs = bsphere(xyz(c) - o, rad, ee);
        az = EXT ? az_rect(xyz(c) - o, h.x, h.y) : footprint(xyz(c) - o, sqrtf(h.x * h.x + h.y * h.y));
        zl = c.z - h.z - o.z;
        zh = c.z + h.z - o.z;
      } else if (i < tot_in) {
        int j = i - sv.ns - sv.nb;
        float4 c = ld4(sv.cyl, 2 * j);
        float hh = __ldg(sv.cyl + 8 * j + 4);
        float rad = sqrtf(c.w * c.w + hh * hh);
        keep = !(rc.cull & 1) || (KIND == 0 ? keep_camera(rc, cs, o, xyz(c), rad) : keep_ball(rc, o, xyz(c), rad));
        q0 = make_float4(o.x - c.x, o.y - c.y, o.z - c.z, c.w * c.w);
        q1 = make_float4(hh, hh - (o.z - c.z), -hh - (o.z - c.z), 0.f);  // cap planes relative to o
        bs = bsphere(xyz(c) - o, rad, ee);
        az = EXT ? az_circle(xyz(c) - o, c.w) : footprint(xyz(c) - o, c.w);
        zl = c.z - hh - o.z;
        zh = c.z + hh - o.z;
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const int p = run + __popc(m & ((1u << lane) - 1u));
        r0[p] = q0;
        r1[p] = q1;
        b_all[p] = bs;
        if (EXT) {
          const float zs = 1e-4f * (1.f + fabsf(zl) + fabsf(zh));  // fp32 slack
          f_all[p] = make_float4(zl - zs > 0.f ? -ee.x : ee.x, zh + zs < 0.f ? -ee.y : ee.y, 0.f, 0.f);
          a_all[p] = az;
        } else {
          f_all[p] = make_float4(ee.x, ee.y, az.z, az.w);
        }
      }
      run += __popc(m);
      ks += __popc(__ballot_sync(0xffffffffu, keep && i < sv.ns));
      kb += __popc(__ballot_sync(0xffffffffu, keep && i >= sv.ns && i < sv.ns + sv.nb));
    }
    if (lane == 0) {
      cnt[0] = ks;
      cnt[1] = kb;
      cnt[2] = run - ks - kb;
    }
    for (int c = lane; c * 32 < run; c += 32)
      kmask[c] = make_uint2(lanes_below(ks - 32 * c), lanes_below(ks + kb - 32 * c));
  }
  __syncthreads();
  const int ns = cnt[0], nb = cnt[1], nc = cnt[2];
  const int tot = ns + nb + nc;
  const bool ground = sv.ground;
  const float gdz = sv.gz - o.z;
  const int t0 = blockIdx.x * tiles_per_cta, t1 = min(n_tiles, t0 + tiles_per_cta);
  float* out_row = GRAD ? nullptr : out + row * rc.n_rays;
  uint8_t* hitm_row = hitm && !GRAD ? hitm + row * rc.n_rays : nullptr;
  const float* g_row = GRAD ? g_depth + row * rc.n_rays : nullptr;
  V3 gacc = v3(0.f, 0.f, 0.f);  // GRAD: this lane's share of d loss / d origin
  // vector stores of a lane's consecutive rays need rows that keep their alignment
  const bool vec_ok = RPL > 1 && !GRAD && (rc.n_rays % RPL) == 0 &&
                      (reinterpret_cast<uintptr_t>(out) % (4 * RPL)) == 0 &&
                      (!hitm || (reinterpret_cast<uintptr_t>(hitm) % RPL) == 0);
  for (int tile = t0 + warp; tile < t1; tile += nwarps) {
    // tile record (12 floats): cone axis xyz, cos, sin | azimuth centre xy, cos, sin of the sector
    const float4 c0 = ld4(tile_cones, 3 * tile), c1 = ld4(tile_cones, 3 * tile + 1);
    const float4 c2 = ld4(tile_cones, 3 * tile + 2);  // sin(sector half-width), dz range
    const float sw = c2.x;
    const bool down = c2.z <= 0.f, up = c2.y >= 0.f;  // the tile never rises / never falls
    const V3 ax = rotz(cs, xyz(c0));
    const float cth = c0.w, sth = c1.x;
    const float2 azw = make_float2(cs.x * c1.y - cs.y * c1.z, cs.y * c1.y + cs.x * c1.z);
    const float cw = c1.w;
    // lane's rays: body-frame direction + ray index from the tile-ordered table
    constexpr int NP = GRAD ? 0 : RPL / 2;  // packed pairs (RPL >= 2; GRAD tracks argmins per ray)
    int ray[RPL];
    V3 d[RPL];
    unsigned best[RPL];
    float bestf[RPL];  // GRAD: float min-t, argmin code (kind | detail << 4) and list index
    int code[RPL], bidx[RPL];
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      const float4 td = ld4(tile_dirs, (tile * RPL + k) * 32 + lane);
      ray[k] = __float_as_int(td.w);  // the ray index's int32 bits (no conversion)
      d[k] = rotz_f(cs, xyz(td));
      best[k] = INF_BITS;
      bestf[k] = INF;
      code[k] = 0;
      bidx[k] = 0;
    }
    V3 inv[RPL];
    float a[RPL], inv_a[RPL];
    RayPair rp[NP > 0 ? NP : 1];
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      inv[k] = v3(rcp_fast(d[k].x), rcp_fast(d[k].y), rcp_fast(d[k].z));
      a[k] = dxy2(d[k]);
      inv_a[k] = rcp_fast(a[k]);
    }
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const int k0 = 2 * p, k1 = 2 * p + 1;
      rp[p].dx = make_float2(d[k0].x, d[k1].x);
      rp[p].dy = make_float2(d[k0].y, d[k1].y);
      rp[p].dz = make_float2(d[k0].z, d[k1].z);
      rp[p].ix = make_float2(inv[k0].x, inv[k1].x);
      rp[p].iy = make_float2(inv[k0].y, inv[k1].y);
      rp[p].iz = make_float2(inv[k0].z, inv[k1].z);
      rp[p].a = make_float2(a[k0], a[k1]);
      rp[p].ia = make_float2(inv_a[k0], inv_a[k1]);
    }
    for (int base = 0; base < tot; base += 32) {
      const int j = base + lane;
      const uint2 km = kmask[base >> 5];  // (loaded ahead of the cone test that hides its latency)
      bool keep = false;
      if (j < tot) {
        const float4 bj = b_all[j], fj = f_all[j];
        if (EXT) {
          const bool above = __float_as_int(fj.x) < 0, below = __float_as_int(fj.y) < 0;
          keep = !((above && down) || (below && up)) &&
                 cone_keeps(bj, make_float2(fabsf(fj.x), fabsf(fj.y)), ax, cth, sth) &&
                 sector_keeps(a_all[j], azw, cw, sw);
        } else {
          keep = cone_keeps(bj, make_float2(fj.x, fj.y), ax, cth, sth) &&
                 circle_sector_keeps(make_float4(bj.x, bj.y, fj.z, fj.w), fj.y, azw, cw, sw);
        }
      }
      // warp-uniform candidate masks, split by kind (the list is kind-sorted:
      // spheres, boxes, cylinders), so each loop runs one test with no dispatch
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      unsigned ms = m & km.x, mb = m & km.y & ~km.x, mc = m & ~km.y;
      if constexpr (!GRAD && NP > 0) {
        // software-pipelined candidate loops: the next candidate's record is
        // read from shared memory while the current one is tested
        if (ms) {
          int i = base + __ffs(ms) - 1;
          ms &= ms - 1;
          float4 q = r0[i];
          for (;;) {
            const int i2 = ms ? base + __ffs(ms) - 1 : i;
            const float4 qn = r0[i2];
#pragma unroll
            for (int p = 0; p < NP; ++p) hit_sphere_p(best[2 * p], best[2 * p + 1], q, rp[p]);
            if (!ms) break;
            ms &= ms - 1;
            q = qn;
          }
        }
        if (mb) {
          int i = base + __ffs(mb) - 1;
          mb &= mb - 1;
          float4 lo = r0[i], hi = r1[i];
          for (;;) {
            const int i2 = mb ? base + __ffs(mb) - 1 : i;
            const float4 lon = r0[i2], hin = r1[i2];
#pragma unroll
            for (int p = 0; p < NP; ++p) hit_box_p(best[2 * p], best[2 * p + 1], lo, hi, rp[p]);
            if (!mb) break;
            mb &= mb - 1;
            lo = lon;
            hi = hin;
          }
        }
        if (mc) {
          int i = base + __ffs(mc) - 1;
          mc &= mc - 1;
          float4 q = r0[i], h = r1[i];
          for (;;) {
            const int i2 = mc ? base + __ffs(mc) - 1 : i;
            const float4 qn = r0[i2], hn = r1[i2];
#pragma unroll
            for (int p = 0; p < NP; ++p) hit_cyl_p(best[2 * p], best[2 * p + 1], q, h, rp[p]);
            if (!mc) break;
            mc &= mc - 1;
            q = qn;
            h = hn;
          }
        }
        continue;
      }
      while (ms) {
        const int i = base + __ffs(ms) - 1;
        ms &= ms - 1;
        const float4 q = r0[i];
        if constexpr (GRAD) {
#pragma unroll
          for (int k = 0; k < RPL; ++k) {
            const float t = hit_sphere(q, d[k]);
            if (t < bestf[k]) { bestf[k] = t; code[k] = 1; bidx[k] = i; }
          }
        } else if constexpr (NP > 0) {
#pragma unroll
          for (int p = 0; p < NP; ++p) hit_sphere_p(best[2 * p], best[2 * p + 1], q, rp[p]);
        } else {
          best[0] = hit_sphere_u(best[0], q, d[0]);
        }
      }
      while (mb) {
        const int i = base + __ffs(mb) - 1;
        mb &= mb - 1;
        const float4 lo = r0[i], hi = r1[i];
        if constexpr (GRAD) {
#pragma unroll
          for (int k = 0; k < RPL; ++k) {
            int axk = 0;
            const float t = hit_box(lo, hi, inv[k], &axk);
            if (t < bestf[k]) { bestf[k] = t; code[k] = 2 | (axk << 4); bidx[k] = i; }
          }
        } else if constexpr (NP > 0) {
#pragma unroll
          for (int p = 0; p < NP; ++p) hit_box_p(best[2 * p], best[2 * p + 1], lo, hi, rp[p]);
        } else {
          best[0] = hit_box_u(best[0], lo, hi, inv[0]);
        }
      }
      while (mc) {
        const int i = base + __ffs(mc) - 1;
        mc &= mc - 1;
        const float4 q = r0[i], h = r1[i];
        if constexpr (GRAD) {
#pragma unroll
          for (int k = 0; k < RPL; ++k) {
            int part = 0;
            const float t = hit_cyl(q, h.x, h.y, h.z, d[k], a[k], inv_a[k], inv[k].z, &part);
            if (t < bestf[k]) { bestf[k] = t; code[k] = 3 | (part << 4); bidx[k] = i; }
          }
        } else if constexpr (NP > 0) {
#pragma unroll
          for (int p = 0; p < NP; ++p) hit_cyl_p(best[2 * p], best[2 * p + 1], q, h, rp[p]);
        } else {
          best[0] = hit_cyl_u(best[0], q, h, d[0], a[0], inv_a[0], inv[0].z);
        }
      }
    }
    if constexpr (GRAD) {
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        if (ground) {
          const float t = gdz * inv[k].z;
          if (t >= 0.f && t < INF && t < bestf[k]) { bestf[k] = t; code[k] = 4; }
        }
        if (ray[k] < 0 || !(bestf[k] < rc.max_range)) continue;  // clamped / missed: zero gradient
        V3 n = v3(0.f, 0.f, 0.f);
        const int kind = code[k] & 15;
        if (kind == 1) {
          n = xyz(r0[bidx[k]]) + d[k] * bestf[k];  // x - c = oc + t d
        } else if (kind == 2) {
          const int axk = code[k] >> 4;
          n = v3(axk == 0 ? 1.f : 0.f, axk == 1 ? 1.f : 0.f, axk == 2 ? 1.f : 0.f);
        } else if (kind == 3) {
          if ((code[k] >> 4) == 0) {
            const float4 c = r0[bidx[k]];
            n = v3(c.x + bestf[k] * d[k].x, c.y + bestf[k] * d[k].y, 0.f);
          } else {
            n = v3(0.f, 0.f, 1.f);
          }
        } else if (kind == 4) {
          n = v3(0.f, 0.f, 1.f);
        }
        const float nd = dot(n, d[k]);
        const V3 gv = nd != 0.f ? n * (-1.f / nd) : v3(0.f, 0.f, 0.f);
        gacc += gv * g_row[ray[k]];
      }
      continue;
    }
    float tk[RPL];
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      if (ground) best[k] = min(best[k], fbits(pos0(gdz * inv[k].z)));  // +inf / NaN / t < 0 drop out
      tk[k] = __uint_as_float(best[k]);
    }
    // the host table gives a lane consecutive rays (sensors._tile_table): one
    // vector store of the depths and one of the hit bytes
    bool vec = vec_ok && ray[0] >= 0 && (ray[0] % RPL) == 0;
#pragma unroll
    for (int k = 1; k < RPL; ++k) vec = vec && ray[k] == ray[0] + k;
    if (vec) {
      if constexpr (RPL == 2) {
        *reinterpret_cast<float2*>(out_row + ray[0]) =
            make_float2(fminf(tk[0], rc.max_range), fminf(tk[1], rc.max_range));
        if (hitm)
          *reinterpret_cast<uint16_t*>(hitm_row + ray[0]) =
              (uint16_t)((tk[0] < rc.max_range ? 1u : 0u) | (tk[1] < rc.max_range ? 0x100u : 0u));
      } else if constexpr (RPL == 4) {
        *reinterpret_cast<float4*>(out_row + ray[0]) =
            make_float4(fminf(tk[0], rc.max_range), fminf(tk[1], rc.max_range), fminf(tk[2], rc.max_range),
                        fminf(tk[3], rc.max_range));
        if (hitm)
          *reinterpret_cast<uint32_t*>(hitm_row + ray[0]) =
              (tk[0] < rc.max_range ? 1u : 0u) | (tk[1] < rc.max_range ? 0x100u : 0u) |
              (tk[2] < rc.max_range ? 0x10000u : 0u) | (tk[3] < rc.max_range ? 0x1000000u : 0u);
      }
    } else {
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        if (ray[k] >= 0) {
          out_row[ray[k]] = fminf(tk[k], rc.max_range);
          if (hitm) hitm_row[ray[k]] = tk[k] < rc.max_range ? 1 : 0;
        }
      }
    }
  }
  if constexpr (GRAD) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      gacc.x += __shfl_xor_sync(0xffffffffu, gacc.x, off);
      gacc.y += __shfl_xor_sync(0xffffffffu, gacc.y, off);
      gacc.z += __shfl_xor_sync(0xffffffffu, gacc.z, off);
    }
    if (lane == 0) {
      float* gp = g_pos + row * gpos_stride;
      atomicAdd(gp + 0, gacc.x);
      atomicAdd(gp + 1, gacc.y);
      atomicAdd(gp + 2, gacc.z);
    }
  }
}

// g_pos[row] += sum_r g_depth[row, r] * dT_dO[row, r]   (one CTA per row)
__global__ void __launch_bounds__(256) k_raycast_vjp(int n_rays, const float* __restrict__ g_depth,
                                                     const float* __restrict__ dT_dO,
                                                     float* __restrict__ g_pos, int pos_stride) {
  const long row = blockIdx.x;
  V3 acc = v3(0.f, 0.f, 0.f);
  for (int r = threadIdx.x; r < n_rays; r += blockDim.x) {
    long i = row * n_rays + r;
    float g = g_depth[i];
    acc += xyz(ld4(dT_dO, i)) * g;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
  }
  __shared__ V3 part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    V3 s = v3(0.f, 0.f, 0.f);
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += part[w];
    float* gp = g_pos + row * pos_stride;
    gp[0] += s.x;
    gp[1] += s.y;
    gp[2] += s.z;
  }
}

}  // namespace

extern "C" {

int qs_raycast(const qs_ray_cfg* cfg, const qs_scene* scene, int32_t n_rows, const float* pos,
               int32_t pos_stride, const float* cam_cs, const float* dirs_body,
               const float* dirs_world, float* out, uint8_t* hit, float* dT_dO, void* stream) {
  if (n_rows <= 0 || cfg->n_rays <= 0) return QS_OK;
  if (cfg->kind < 0 || cfg->kind > 2 || cfg->n_agents < 1) return QS_ERR_BAD_ARGUMENT;
  const int rpc = cfg->n_rays <= 4096 ? cfg->n_rays : 4096;
  dim3 grid((cfg->n_rays + rpc - 1) / rpc, n_rows);
  size_t smem = (size_t)(scene->Sm + 2 * scene->Bm + scene->Cm) * 16 + scene->Cm * 4;
  cudaStream_t s = (cudaStream_t)stream;
  const bool g = dT_dO != nullptr;
#define QS_RC(K, G)                                                                           \
  k_raycast<K, G><<<grid, RAY_BLOCK, smem, s>>>(*cfg, *scene, n_rows, pos, pos_stride, cam_cs, \
                                                dirs_body, dirs_world, out, hit, dT_dO, rpc)
  if (cfg->kind == 0) { if (g) QS_RC(0, true); else QS_RC(0, false); }
  else if (cfg->kind == 1) { if (g) QS_RC(1, true); else QS_RC(1, false); }
  else { if (g) QS_RC(2, true); else QS_RC(2, false); }
#undef QS_RC
  return cudaGetLastError() == cudaSuccess ? QS_OK : QS_ERR_LAUNCH;
}

int qs_raycast_tiled(const qs_ray_cfg* cfg, const qs_scene* scene, int32_t n_rows, const float* pos,
                     int32_t pos_stride, const float* cam_cs, const float* tile_dirs,
                     const float* tile_cones, int32_t n_tiles, int32_t tile_width,
                     float* out, uint8_t* hit, void* stream) {
  if (n_rows <= 0 || cfg->n_rays <= 0) return QS_OK;
  if (cfg->kind < 0 || cfg->kind > 1 || cfg->n_agents < 1 || n_tiles <= 0) return QS_ERR_BAD_ARGUMENT;
  if (tile_width != 32 && tile_width != 64 && tile_width != 128) return QS_ERR_BAD_ARGUMENT;
  const int tpc = n_tiles;  // one CTA per row: the staged obstacles serve every tile
  dim3 grid((n_tiles + tpc - 1) / tpc, n_rows);
  const bool ext = (cfg->cull & 2) != 0;
  const int cap = scene->Sm + scene->Bm + scene->Cm;
  size_t smem = (size_t)cap * ((ext ? 5 : 4) * 16) + (size_t)((cap + 31) / 32 + 1) * 8;
  cudaStream_t s = (cudaStream_t)stream;
#define QS_RT(K, X, R)                                                                                  \
  k_raycast_tiled<K, X, R><<<grid, TILED_BLOCK, smem, s>>>(*cfg, *scene, n_rows, pos, pos_stride, cam_cs, \
                                                           tile_dirs, tile_cones, n_tiles, tpc, out, hit)
#define QS_RT_W(K, X)                 \
  if (tile_width == 32) QS_RT(K, X, 1); \
  else if (tile_width == 64) QS_RT(K, X, 2); \
  else QS_RT(K, X, 4)
  if (cfg->kind == 0) { if (ext) { QS_RT_W(0, true); } else { QS_RT_W(0, false); } }
  else { if (ext) { QS_RT_W(1, true); } else { QS_RT_W(1, false); } }
#undef QS_RT_W
#undef QS_RT
  return cudaGetLastError() == cudaSuccess ? QS_OK : QS_ERR_LAUNCH;
}

int qs_raycast_tiled_vjp(const qs_ray_cfg* cfg, const qs_scene* scene, int32_t n_rows, const float* pos,
                         int32_t pos_stride, const float* cam_cs, const float* tile_dirs, const float* tile_cones,
                         int32_t n_tiles, int32_t tile_width, const float* g_depth, float* g_pos,
                         int32_t gpos_stride, void* stream) {
  if (n_rows <= 0 || cfg->n_rays <= 0) return QS_OK;
  if (cfg->kind < 0 || cfg->kind > 1 || cfg->n_agents < 1 || n_tiles <= 0 || !g_depth || !g_pos)
    return QS_ERR_BAD_ARGUMENT;
  if (tile_width != 32 && tile_width != 64 && tile_width != 128) return QS_ERR_BAD_ARGUMENT;
  dim3 grid(1, n_rows);
  const bool ext = (cfg->cull & 2) != 0;
  const int cap = scene->Sm + scene->Bm + scene->Cm;
  size_t smem = (size_t)cap * ((ext ? 5 : 4) * 16) + (size_t)((cap + 31) / 32 + 1) * 8;
  cudaStream_t s = (cudaStream_t)stream;
#define QS_RV(K, X, R)                                                                                     \
  k_raycast_tiled<K, X, R, true><<<grid, TILED_BLOCK, smem, s>>>(*cfg, *scene, n_rows, pos, pos_stride, cam_cs, \
                                                                 tile_dirs, tile_cones, n_tiles, n_tiles, nullptr, \
                                                                 nullptr, g_depth, g_pos, gpos_stride)
#define QS_RV_W(K, X)                 \
  if (tile_width == 32) QS_RV(K, X, 1); \
  else if (tile_width == 64) QS_RV(K, X, 2); \
  else QS_RV(K, X, 4)
  if (cfg->kind == 0) { if (ext) { QS_RV_W(0, true); } else { QS_RV_W(0, false); } }
  else { if (ext) { QS_RV_W(1, true); } else { QS_RV_W(1, false); } }
#undef QS_RV_W
#undef QS_RV
  return cudaGetLastError() == cudaSuccess ? QS_OK : QS_ERR_LAUNCH;
}

int qs_raycast_vjp(int32_t n_rows, int32_t n_rays, const float* g_depth, const float* dT_dO,
                   float* g_pos, int32_t pos_stride, void* stream) {
  if (n_rows <= 0) return QS_OK;
  k_raycast_vjp<<<n_rows, 256, 0, (cudaStream_t)stream>>>(n_rays, g_depth, dT_dO, g_pos, pos_stride);
  return cudaGetLastError() == cudaSuccess ? QS_OK : QS_ERR_LAUNCH;
}

}  // extern "C"
