// Analytic obstacle geometry: signed distance with first-argmin subgradient
// (q/sensors.py:417-501) and ray-primitive intersections (q/sensors.py:131-216).
#pragma once
#include "qs_common.cuh"

#define QS_FAR 1e9f

// argmin code: bits 0-1 kind (0 none/sphere?,...), bits 2.. index
enum : int { SDF_NONE = 0, SDF_SPH = 1, SDF_BOX = 2, SDF_CYL = 3, SDF_GND = 4 };

QS_D int sdf_code(int kind, int idx) { return kind | (idx << 3); }

struct SceneView {  // one env's obstacles
  const float* sph;
  const float* box;
  const float* cyl;
  int ns, nb, nc;
  bool ground;
  float gz;
};

QS_D SceneView scene_view(const qs_scene& sc, long e) {
  SceneView v;
  int4 c = __ldg(reinterpret_cast<const int4*>(sc.counts) + e);
  v.ns = c.x;
  v.nb = c.y;
  v.nc = c.z;
  v.ground = c.w != 0;
  v.gz = v.ground ? __ldg(sc.ground_z + e) : 0.f;
  v.sph = sc.spheres + e * (long)sc.Sm * 4;
  v.box = sc.boxes + e * (long)sc.Bm * 8;
  v.cyl = sc.cylinders + e * (long)sc.Cm * 8;
  return v;
}

QS_D float sdf_sphere(V3 p, float4 s) { return norm3(p - xyz(s)) - s.w; }

QS_D float sdf_box(V3 p, float4 c, float4 h) {
  V3 d = p - xyz(c);
  V3 q = v3(fabsf(d.x) - h.x, fabsf(d.y) - h.y, fabsf(d.z) - h.z);
  float out = norm3(v3(fmaxf(q.x, 0.f), fmaxf(q.y, 0.f), fmaxf(q.z, 0.f)));
  float m = fmaxf(fmaxf(q.x, q.y), q.z);
  return out + fminf(m, 0.f);
}

QS_D float sdf_cyl(V3 p, float4 c, float hh) {
  float dxy = sqrtf((p.x - c.x) * (p.x - c.x) + (p.y - c.y) * (p.y - c.y)) - c.w;
  float dz = fabsf(p.z - c.z) - hh;
  float a = fmaxf(dxy, 0.f), b = fmaxf(dz, 0.f);
  return sqrtf(a * a + b * b) + fminf(fmaxf(dxy, dz), 0.f);
}

// min over [spheres, boxes, cylinders, ground]; strict < keeps the FIRST argmin
// (q/autodiff.py:545-560)
QS_D float sdf_eval(const SceneView& s, V3 p, int& code) {
  float best = QS_FAR;
  code = SDF_NONE;
  for (int i = 0; i < s.ns; ++i) {
    float d = sdf_sphere(p, ld4(s.sph, i));
    if (d < best) { best = d; code = sdf_code(SDF_SPH, i); }
  }
  for (int i = 0; i < s.nb; ++i) {
    float d = sdf_box(p, ld4(s.box, 2 * i), ld4(s.box, 2 * i + 1));
    if (d < best) { best = d; code = sdf_code(SDF_BOX, i); }
  }
  for (int i = 0; i < s.nc; ++i) {
    float4 c = ld4(s.cyl, 2 * i);
    float hh = __ldg(s.cyl + 8 * i + 4);
    float d = sdf_cyl(p, c, hh);
    if (d < best) { best = d; code = sdf_code(SDF_CYL, i); }
  }
  if (s.ground) {
    float d = p.z - s.gz;
    if (d < best) { best = d; code = sdf_code(SDF_GND, 0); }
  }
  return best;
}

// distance to the primitive selected by `code`
QS_D float sdf_prim(const SceneView& s, V3 p, int code) {
  int kind = code & 7, i = code >> 3;
  if (kind == SDF_SPH) return sdf_sphere(p, ld4(s.sph, i));
  if (kind == SDF_BOX) return sdf_box(p, ld4(s.box, 2 * i), ld4(s.box, 2 * i + 1));
  if (kind == SDF_CYL) return sdf_cyl(p, ld4(s.cyl, 2 * i), __ldg(s.cyl + 8 * i + 4));
  if (kind == SDF_GND) return p.z - s.gz;
  return QS_FAR;
}

// gradient of the selected primitive's distance wrt p, with the reference's
// subgradient choices: norm(0)->0, abs'(0)=0, maximum/minimum ties -> first
QS_D V3 sdf_grad(const SceneView& s, V3 p, int code) {
  int kind = code & 7, i = code >> 3;
  V3 z = v3(0.f, 0.f, 0.f);
  if (kind == SDF_SPH) {
    V3 d = p - xyz(ld4(s.sph, i));
    return norm_vjp(d, norm3(d), 1.f);
  }
  if (kind == SDF_GND) return v3(0.f, 0.f, 1.f);
  if (kind == SDF_BOX) {
    float4 c = ld4(s.box, 2 * i), h = ld4(s.box, 2 * i + 1);
    V3 d = p - xyz(c);
    V3 q = v3(fabsf(d.x) - h.x, fabsf(d.y) - h.y, fabsf(d.z) - h.z);
    V3 mq = v3(fmaxf(q.x, 0.f), fmaxf(q.y, 0.f), fmaxf(q.z, 0.f));
    V3 go = norm_vjp(mq, norm3(mq), 1.f);  // d outside / d max(q,0)
    V3 gq = v3(q.x >= 0.f ? go.x : 0.f, q.y >= 0.f ? go.y : 0.f, q.z >= 0.f ? go.z : 0.f);
    // inside = min(max(max(q0,q1),q2), 0)
    float m01 = q.x >= q.y ? q.x : q.y;
    float m = m01 >= q.z ? m01 : q.z;
    if (m <= 0.f) {
      if (m01 >= q.z) {
        if (q.x >= q.y) gq.x += 1.f; else gq.y += 1.f;
      } else {
        gq.z += 1.f;
      }
    }
    auto sgn = [](float x) { return x > 0.f ? 1.f : (x < 0.f ? -1.f : 0.f); };
    return v3(gq.x * sgn(d.x), gq.y * sgn(d.y), gq.z * sgn(d.z));
  }
  if (kind == SDF_CYL) {
    float4 c = ld4(s.cyl, 2 * i);
    float hh = __ldg(s.cyl + 8 * i + 4);
    V3 dxyv = v3(p.x - c.x, p.y - c.y, 0.f);
    float rxy = norm3(dxyv);
    float dxy = rxy - c.w;
    float dzr = p.z - c.z;
    float dz = fabsf(dzr) - hh;
    float a = fmaxf(dxy, 0.f), b = fmaxf(dz, 0.f);
    float out = sqrtf(a * a + b * b);
    float g_dxy = 0.f, g_dz = 0.f;
    if (out > 0.f) {  // fp64 reference adds 1e-300 under the sqrt: same limit
      if (dxy >= 0.f) g_dxy += a / out;
      if (dz >= 0.f) g_dz += b / out;
    }
    float mx = dxy >= dz ? dxy : dz;
    if (mx <= 0.f) {
      if (dxy >= dz) g_dxy += 1.f; else g_dz += 1.f;
    }
    V3 gxy = norm_vjp(dxyv, rxy, g_dxy);
    float sz = dzr > 0.f ? 1.f : (dzr < 0.f ? -1.f : 0.f);
    return v3(gxy.x, gxy.y, g_dz * sz);
  }
  return z;
}
