// In-kernel obstacle-course generation with grid-BFS feasibility
// (q/world.py:207-340, 144-179), one CTA per env.
//
// Obstacles are drawn from Philox keyed by (seed, global env id, attempt,
// obstacle index) with the reference's distributions (corridor box around the
// spawn->goal segment, SPHERE_R/BOX_HALF/CYL_R/CYL_HH ranges, trunks standing
// on the ground, indoor shell).  Feasibility is the reference's 6-connected
// BFS over the 0.25 m occupancy grid with obstacles inflated by r_quad+0.05,
// run as bit-parallel dilation over a shared-memory bitmap.
#include <climits>

#include "qs_geom.cuh"

namespace {

#ifndef QS_GEN_BLOCK
#define QS_GEN_BLOCK 256
#endif
constexpr int GEN_BLOCK = QS_GEN_BLOCK;

struct Frame {
  V3 spawn, goal, fwd, left, lo, hi;
  float dist, height;
  int dims[3];
};

QS_D Frame make_frame(const qs_gen_cfg& c) {
  Frame f;
  f.spawn = v3(c.spawn[0], c.spawn[1], c.spawn[2]);
  f.goal = v3(c.goal[0], c.goal[1], c.goal[2]);
  V3 span = f.goal - f.spawn;
  f.dist = norm3(span);
  V3 fw = span * (1.f / f.dist);
  V3 fh = v3(fw.x, fw.y, 0.f);
  fh = fh * (1.f / fmaxf(norm3(fh), 1e-9f));
  f.fwd = fh;
  f.left = v3(-fh.y, fh.x, 0.f);
  f.height = c.indoor ? 3.f : 4.f;
  const float pad = 1.5f;
  float xs[4], ys[4];
  int k = 0;
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) {
      float a = i ? f.dist + pad : -pad;
      float b = j ? c.corridor_halfwidth + pad : -c.corridor_halfwidth - pad;
      V3 p = f.spawn + fh * a + f.left * b;
      xs[k] = p.x;
      ys[k] = p.y;
      ++k;
    }
  f.lo = v3(fminf(fminf(xs[0], xs[1]), fminf(xs[2], xs[3])), fminf(fminf(ys[0], ys[1]), fminf(ys[2], ys[3])), 0.f);
  f.hi = v3(fmaxf(fmaxf(xs[0], xs[1]), fmaxf(xs[2], xs[3])), fmaxf(fmaxf(ys[0], ys[1]), fmaxf(ys[2], ys[3])), f.height);
  f.dims[0] = max(2, (int)ceilf((f.hi.x - f.lo.x) / 0.25f));
  f.dims[1] = max(2, (int)ceilf((f.hi.y - f.lo.y) / 0.25f));
  f.dims[2] = max(2, (int)ceilf((f.hi.z - f.lo.z) / 0.25f));
  return f;
}

// signed distance of the reference's clearance test (q/world.py:309-323)
QS_D float end_dist_sphere(V3 e, float4 s) { return norm3(e - xyz(s)) - s.w; }
QS_D float end_dist_box(V3 e, float4 c, float4 h) { return sdf_box(e, c, h); }
QS_D float end_dist_cyl(V3 e, float4 c, float hh) { return sdf_cyl(e, c, hh); }

QS_D uint32_t bits_at(const uint32_t* a, long nbits, long pos) {
  // 32 bits starting at bit `pos` (bits outside [0, nbits) read as 0)
  uint32_t out = 0;
  long w = pos >> 5;
  int sh = (int)(pos & 31);
  long nw = (nbits + 31) >> 5;
  if (pos >= 0) {
    uint32_t lo = (w < nw) ? a[w] : 0u;
    uint32_t hi = (w + 1 < nw) ? a[w + 1] : 0u;
    out = sh ? (lo >> sh) | (hi << (32 - sh)) : lo;
  } else {
    long p = pos + 32;  // partially negative
    if (p > 0) {
      uint32_t lo = a[0];
      out = lo << (32 - (int)p);
    }
  }
  return out;
}

// bits [a, b] of a 32-bit word, clamped to [0, 31]
QS_D uint32_t span32(int a, int b) {
  a = a > 0 ? a : 0;
  b = b < 31 ? b : 31;
  if (a > b) return 0u;
  const uint32_t upto = b == 31 ? 0xffffffffu : ((1u << (b + 1)) - 1u);
  return upto & ~((1u << a) - 1u);
}
// bits b of a word whose first cell has residue r (mod period) such that the
// cell's residue (r + b) mod period lies in [r0, r1]
QS_D uint32_t residue_mask(int r, int period, int r0, int r1) {
  uint32_t m = 0u;
  for (int s = -r; s < 32; s += period) m |= span32(s + r0, s + r1);
  return m;
}

__global__ void __launch_bounds__(GEN_BLOCK) k_gen(const qs_gen_cfg cfg, int n_envs, float* bounds,
                                                   float* spawn_goal, float* spheres, float* boxes,
                                                   float* cylinders, int32_t* counts, float* ground_z,
                                                   int32_t* err) {
  extern __shared__ uint32_t smem[];
  __shared__ float4 s_sph[64];
  __shared__ float4 s_box[2 * 72];
  __shared__ float4 s_cyl[64];
  __shared__ float s_cyl_hh[64];
  __shared__ int s_cnt[3];
  __shared__ int s_done;
  __shared__ int s_vlo, s_vhi;  // visited word range of the BFS
  const long e = blockIdx.x;
  if (e >= n_envs) return;
  if (cfg.env_mask && !cfg.env_mask[e]) return;  // re-randomise only the masked envs
  const uint32_t episode = cfg.episode ? (uint32_t)cfg.episode[e * cfg.episode_stride] : 0u;
  const Frame F = make_frame(cfg);
  const long cells = (long)F.dims[0] * F.dims[1] * F.dims[2];
  const long nw = (cells + 31) >> 5;
  uint32_t* freeb = smem;
  uint32_t* vis = smem + nw;
  uint32_t* nxt = smem + 2 * nw;
  const int nz = F.dims[2], ny = F.dims[1];
  const int P = ny * nz;  // cells per x slab
  // residue steps of a thread's word start i0 = 32 wi between its words
  const int dz32 = (int)((blockDim.x * 32L) % nz), dy32 = (int)((blockDim.x * 32L) % P);
  const int n_total = (int)rintf(cfg.density * F.dist * 2.f * cfg.corridor_halfwidth);
  const int n_cyl = (int)rintf(0.4f * n_total), n_sph = (int)rintf(0.3f * n_total);
  const int n_box = n_total - n_cyl - n_sph;
  const float keep_min = cfg.r_quad + cfg.clearance;
  const uint64_t gid = (uint64_t)(e + cfg.env_offset);
  bool feasible = false;
  for (int attempt = 0; attempt < cfg.max_attempts && !feasible; ++attempt) {
    if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    // ---- sample + clearance filter (order within a type preserved by index)
    for (int i = threadIdx.x; i < n_total; i += blockDim.x) {
      Rng rng(cfg.seed, gid, (uint32_t)attempt, RNG_SCENE);
      rng.ctr.z = (uint32_t)attempt * 4096u + (uint32_t)i;
      rng.ctr.w |= (episode & 0xFFFFu) << 8;  // purpose byte stays on top
      float4 u = rng.uniform4(), w = rng.uniform4();
      float along = u.x * F.dist;
      float lat = -cfg.corridor_halfwidth + 2.f * cfg.corridor_halfwidth * u.y;
      float z = 0.3f + (F.height - 0.6f) * u.z;
      V3 c = F.spawn + F.fwd * along + F.left * lat;
      c.z = z;
      V3 ends[2] = {F.spawn, F.goal};
      if (i < n_sph) {
        float4 s = f4(c, 0.3f + 0.7f * u.w);
        float d = fminf(end_dist_sphere(ends[0], s), end_dist_sphere(ends[1], s));
        if (d > keep_min) s_sph[i] = s; else s_sph[i] = make_float4(0.f, 0.f, 0.f, -1.f);
      } else if (i < n_sph + n_box) {
        int j = i - n_sph;
        float4 cc = f4(c, 0.f), hh = make_float4(0.2f + 0.8f * u.w, 0.2f + 0.8f * w.x, 0.2f + 0.8f * w.y, 0.f);
        float d = fminf(end_dist_box(ends[0], cc, hh), end_dist_box(ends[1], cc, hh));
        if (!(d > keep_min)) hh.w = -1.f;
        s_box[2 * j] = cc;
        s_box[2 * j + 1] = hh;
      } else {
        int j = i - n_sph - n_box;
        float r = 0.2f + 0.4f * u.w, hh = 0.5f + 1.5f * w.x;
        c.z = hh;  // trunks stand on the ground
        float4 cc = f4(c, r);
        float d = fminf(end_dist_cyl(ends[0], cc, hh), end_dist_cyl(ends[1], cc, hh));
        s_cyl[j] = cc;
        s_cyl_hh[j] = d > keep_min ? hh : -1.f;
      }
    }
    __syncthreads();
    // compact kept obstacles in order (single thread: <= 64 items)
    if (threadIdx.x == 0) {
      int k = 0;
      for (int i = 0; i < n_sph; ++i)
        if (s_sph[i].w > 0.f) s_sph[k++] = s_sph[i];
      s_cnt[0] = k;
      k = 0;
      for (int j = 0; j < n_box; ++j)
        if (s_box[2 * j + 1].w == 0.f) {
          s_box[2 * k] = s_box[2 * j];
          s_box[2 * k + 1] = s_box[2 * j + 1];
          ++k;
        }
      if (cfg.indoor) {  // shell: ceiling + 4 walls (q/world.py:284-296), always kept
        float cx = (F.lo.x + F.hi.x) * 0.5f, cy = (F.lo.y + F.hi.y) * 0.5f;
        float sx = (F.hi.x - F.lo.x) * 0.5f, sy = (F.hi.y - F.lo.y) * 0.5f, wt = 0.1f, h = F.height;
        float sh[5][6] = {{cx, cy, h + wt, sx + 1, sy + 1, wt},
                          {F.lo.x - wt, cy, h / 2, wt, sy + 1, h},
                          {F.hi.x + wt, cy, h / 2, wt, sy + 1, h},
                          {cx, F.lo.y - wt, h / 2, sx + 1, wt, h},
                          {cx, F.hi.y + wt, h / 2, sx + 1, wt, h}};
        for (int q = 0; q < 5; ++q) {
          s_box[2 * k] = make_float4(sh[q][0], sh[q][1], sh[q][2], 0.f);
          s_box[2 * k + 1] = make_float4(sh[q][3], sh[q][4], sh[q][5], 0.f);
          ++k;
        }
      }
      s_cnt[1] = k;
      k = 0;
      for (int j = 0; j < n_cyl; ++j)
        if (s_cyl_hh[j] > 0.f) {
          s_cyl[k] = s_cyl[j];
          s_cyl_hh[k] = s_cyl_hh[j];
          ++k;
        }
      s_cnt[2] = k;
    }
    __syncthreads();
    const int ns = s_cnt[0], nb = s_cnt[1], nc = s_cnt[2];
    // ---- occupancy: free iff sdf(cell centre) > r_quad + 0.05 (ground at z=0).
    // The ground rule fills the bitmap; then every obstacle blocks the cells of
    // its thr-inflated bounding box whose centre lies within thr of it.  Blocked
    // iff some distance <= thr is exactly "min over all distances <= thr" (each
    // distance is the same fp32 value as in a full min), at ~1% of the work.
    const float thr = cfg.r_quad + 0.05f;
    auto centre = [&](int ix, int iy, int iz) {
      return v3(F.lo.x + (ix + 0.5f) * (F.hi.x - F.lo.x) / F.dims[0],
                F.lo.y + (iy + 0.5f) * (F.hi.y - F.lo.y) / F.dims[1],
                F.lo.z + (iz + 0.5f) * (F.hi.z - F.lo.z) / F.dims[2]);
    };
    int izmin = nz;  // the ground rule: free iff the centre's z > thr, monotone in iz
    for (int iz = 0; iz < nz; ++iz)
      if (F.lo.z + (iz + 0.5f) * (F.hi.z - F.lo.z) / F.dims[2] > thr) {
        izmin = iz;
        break;
      }
    {
      int rz = (int)((threadIdx.x * 32L) % nz);
      for (long wi = threadIdx.x; wi < nw; wi += blockDim.x) {
        uint32_t word = residue_mask(rz, nz, izmin, nz - 1);
        if (wi * 32 + 32 > cells) word &= span32(0, (int)(cells - wi * 32) - 1);  // no cells past the grid
        freeb[wi] = word;
        vis[wi] = 0u;
        rz += dz32;
        if (rz >= nz) rz -= nz;
      }
    }
    __syncthreads();
    const int n_obs = ns + nb + nc;
    for (int q = 0; q < n_obs; ++q) {
      V3 c, ext;  // centre and thr-inflated half-extent of the obstacle's box
      if (q < ns) {
        c = xyz(s_sph[q]);
        ext = v3(s_sph[q].w, s_sph[q].w, s_sph[q].w);
      } else if (q < ns + nb) {
        c = xyz(s_box[2 * (q - ns)]);
        ext = xyz(s_box[2 * (q - ns) + 1]);
      } else {
        c = xyz(s_cyl[q - ns - nb]);
        ext = v3(s_cyl[q - ns - nb].w, s_cyl[q - ns - nb].w, s_cyl_hh[q - ns - nb]);
      }
      int lo_i[3], n_i[3];
      const float clo[3] = {F.lo.x, F.lo.y, F.lo.z}, chi[3] = {F.hi.x, F.hi.y, F.hi.z};
      const float cc[3] = {c.x, c.y, c.z}, ee[3] = {ext.x + thr, ext.y + thr, ext.z + thr};
#pragma unroll
      for (int a = 0; a < 3; ++a) {  // cell index range, one cell of slack each side
        const float inv = F.dims[a] / (chi[a] - clo[a]);
        const int i0 = max(0, (int)floorf((cc[a] - ee[a] - clo[a]) * inv - 0.5f) - 1);
        const int i1 = min(F.dims[a] - 1, (int)ceilf((cc[a] + ee[a] - clo[a]) * inv - 0.5f) + 1);
        lo_i[a] = i0;
        n_i[a] = max(0, i1 - i0 + 1);
      }
      const int tot = n_i[0] * n_i[1] * n_i[2];
      for (int k = threadIdx.x; k < tot; k += blockDim.x) {
        const int iz = lo_i[2] + k % n_i[2], iy = lo_i[1] + (k / n_i[2]) % n_i[1], ix = lo_i[0] + k / (n_i[2] * n_i[1]);
        const V3 p = centre(ix, iy, iz);
        float d;
        if (q < ns) d = norm3(p - xyz(s_sph[q])) - s_sph[q].w;
        else if (q < ns + nb) d = sdf_box(p, s_box[2 * (q - ns)], s_box[2 * (q - ns) + 1]);
        else d = sdf_cyl(p, s_cyl[q - ns - nb], s_cyl_hh[q - ns - nb]);
        if (!(d > thr)) {
          const long i = ((long)ix * ny + iy) * nz + iz;
          atomicAnd(&freeb[i >> 5], ~(1u << (i & 31)));
        }
      }
    }
    __syncthreads();
    auto cell_of = [&](V3 p) -> long {
      int ix = min(max((int)((p.x - F.lo.x) / (F.hi.x - F.lo.x) * F.dims[0]), 0), F.dims[0] - 1);
      int iy = min(max((int)((p.y - F.lo.y) / (F.hi.y - F.lo.y) * F.dims[1]), 0), F.dims[1] - 1);
      int iz = min(max((int)((p.z - F.lo.z) / (F.hi.z - F.lo.z) * F.dims[2]), 0), F.dims[2] - 1);
      return ((long)ix * ny + iy) * nz + iz;
    };
    const long start = cell_of(F.spawn), target = cell_of(F.goal);
    const bool s_ok = (freeb[start >> 5] >> (start & 31)) & 1u;
    const bool t_ok = (freeb[target >> 5] >> (target & 31)) & 1u;
    bool ok = false;
    if (s_ok && t_ok) {
      if (threadIdx.x == 0) {
        vis[start >> 5] |= 1u << (start & 31);
        s_vlo = s_vhi = (int)(start >> 5);
      }
      __syncthreads();
      // ---- bit-parallel BFS: grown = (v | 6 shifted copies) & free, over the
      // window of words within one x-slab (P bits) of the visited words --
      // nothing outside it can change this iteration
      const int margin = P / 32 + 2;
      for (int it = 0; it < (int)cells; ++it) {
        int changed = 0;
        const long wlo = max(0, s_vlo - margin), whi = min((long)nw - 1, (long)s_vhi + margin);
        int my_lo = INT_MAX, my_hi = -1;
        long w0 = wlo + threadIdx.x;
        int rz = (int)((w0 * 32) % nz), ry = (int)((w0 * 32) % P);  // residues of i0 = 32 wi
        for (long wi = w0; wi <= whi; wi += blockDim.x) {
          uint32_t v = vis[wi];
          uint32_t g = v;
          // neighbour bit i-1 / i+1 (z), i-nz / i+nz (y), i-ny*nz / i+ny*nz (x)
          uint32_t zm = bits_at(vis, cells, wi * 32 - 1), zp = bits_at(vis, cells, wi * 32 + 1);
          uint32_t ym = bits_at(vis, cells, wi * 32 - nz), yp = bits_at(vis, cells, wi * 32 + nz);
          uint32_t xm = bits_at(vis, cells, wi * 32 - (long)ny * nz);
          uint32_t xp = bits_at(vis, cells, wi * 32 + (long)ny * nz);
          // boundary masks: receive from iz-1 only if iz>0, etc. (bits past
          // `cells` are masked by freeb below)
          const uint32_t mzlo = ~residue_mask(rz, nz, 0, 0), mzhi = ~residue_mask(rz, nz, nz - 1, nz - 1);
          const uint32_t mylo = ~residue_mask(ry, P, 0, nz - 1), myhi = ~residue_mask(ry, P, P - nz, P - 1);
          rz += dz32;
          if (rz >= nz) rz -= nz;
          ry += dy32;
          if (ry >= P) ry -= P;
          g |= (zm & mzlo) | (zp & mzhi) | (ym & mylo) | (yp & myhi) | xm | xp;
          g &= freeb[wi];
          nxt[wi] = g;
          changed |= (g != v);
          if (g) {
            my_lo = min(my_lo, (int)wi);
            my_hi = max(my_hi, (int)wi);
          }
        }
        changed = __syncthreads_or(changed);  // every thread has read this iteration's window
        if (my_hi >= 0) {
          atomicMin(&s_vlo, my_lo);
          atomicMax(&s_vhi, my_hi);
        }
        for (long wi = wlo + threadIdx.x; wi <= whi; wi += blockDim.x) vis[wi] = nxt[wi];
        __syncthreads();
        if ((vis[target >> 5] >> (target & 31)) & 1u) {
          ok = true;
          break;
        }
        if (!changed) break;
      }
    }
    if (threadIdx.x == 0) s_done = ok ? 1 : 0;
    __syncthreads();
    feasible = s_done != 0;
    if (feasible) {
      for (int i = threadIdx.x; i < cfg.Sm; i += blockDim.x)
        reinterpret_cast<float4*>(spheres)[e * cfg.Sm + i] = i < ns ? s_sph[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      for (int i = threadIdx.x; i < cfg.Bm; i += blockDim.x) {
        float4* b = reinterpret_cast<float4*>(boxes) + 2 * (e * cfg.Bm + i);
        b[0] = i < nb ? s_box[2 * i] : make_float4(0.f, 0.f, 0.f, 0.f);
        b[1] = i < nb ? s_box[2 * i + 1] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      for (int i = threadIdx.x; i < cfg.Cm; i += blockDim.x) {
        float4* c = reinterpret_cast<float4*>(cylinders) + 2 * (e * cfg.Cm + i);
        c[0] = i < nc ? s_cyl[i] : make_float4(0.f, 0.f, 0.f, 0.f);
        c[1] = make_float4(i < nc ? s_cyl_hh[i] : 0.f, 0.f, 0.f, 0.f);
      }
      if (threadIdx.x == 0) {
        reinterpret_cast<int4*>(counts)[e] = make_int4(ns, nb, nc, 1);
        ground_z[e] = 0.f;
        float4* bd = reinterpret_cast<float4*>(bounds) + 2 * e;
        bd[0] = f4(F.lo, 0.f);
        bd[1] = f4(F.hi, 0.f);
        float4* sg = reinterpret_cast<float4*>(spawn_goal) + 2 * e;
        sg[0] = f4(F.spawn, 0.f);
        sg[1] = f4(F.goal, 0.f);
      }
    }
  }
  if (!feasible && threadIdx.x == 0) report_err(err, QS_ERR_GENERATION, (int)e);
}

}  // namespace

extern "C" int qs_gen_obstacle_course(const qs_gen_cfg* cfg, int32_t n_envs, float* bounds,
                                      float* spawn_goal, float* spheres, float* boxes,
                                      float* cylinders, int32_t* counts, float* ground_z,
                                      int32_t* err, void* stream) {
  if (n_envs <= 0) return QS_OK;
  // host mirror of make_frame for the bitmap size and capacity checks
  float sx = cfg->goal[0] - cfg->spawn[0], sy = cfg->goal[1] - cfg->spawn[1], sz = cfg->goal[2] - cfg->spawn[2];
  float dist = sqrtf(sx * sx + sy * sy + sz * sz);
  if (!(dist > 2.f) || cfg->density < 0.f) return QS_ERR_BAD_ARGUMENT;
  int n_total = (int)rintf(cfg->density * dist * 2.f * cfg->corridor_halfwidth);
  int n_cyl = (int)rintf(0.4f * n_total), n_sph = (int)rintf(0.3f * n_total);
  int n_box = n_total - n_cyl - n_sph + (cfg->indoor ? 5 : 0);
  if (n_sph > 64 || n_cyl > 64 || n_box > 72 || n_sph > cfg->Sm || n_box > cfg->Bm || n_cyl > cfg->Cm)
    return QS_ERR_BAD_ARGUMENT;
  // generous upper bound of the corridor extent for the bitmap
  float ext = dist + 3.f + 2.f * (cfg->corridor_halfwidth + 1.5f);
  long cells = (long)(ceilf(ext / 0.25f) + 1) * (long)(ceilf(ext / 0.25f) + 1) * 17;
  size_t smem = (size_t)3 * ((cells + 31) / 32) * 4;
  if (smem > 200 * 1024) return QS_ERR_BAD_ARGUMENT;
  // the dynamic shared memory opt-in is per device: cache it per device id
  // and check it (a second device launching without it would fail)
  static bool attr[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return QS_ERR_LAUNCH;
  if (!attr[dev]) {
    if (cudaFuncSetAttribute(k_gen, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess)
      return QS_ERR_LAUNCH;
    attr[dev] = true;
  }
  k_gen<<<n_envs, GEN_BLOCK, smem, (cudaStream_t)stream>>>(*cfg, n_envs, bounds, spawn_goal, spheres,
                                                           boxes, cylinders, counts, ground_z, err);
  return cudaGetLastError() == cudaSuccess ? QS_OK : QS_ERR_LAUNCH;
}

// ---------------------------------------------------------------------------
// race tracks (q/world.py:347-379), one thread per env: gate k sits
// spacing_k along the running heading from gate k-1 (from the spawn for
// k = 0), the heading turning by U(-pi/6, pi/6) before every gate but the
// first, at height U(1, 2.5).  One Philox block per gate: (spacing, turn,
// height).  Bounds: the gates' and spawn's extent +-5 m, floor 0, ceiling
// max(top + 5, 4).

namespace {
__global__ void __launch_bounds__(128) k_track(const qs_track_cfg cfg, int n_envs, float* bounds, float* spawn_goal,
                                               float* gates, int32_t* counts, float* ground_z) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_envs) return;
  if (cfg.env_mask && !cfg.env_mask[e]) return;
  const uint32_t episode = cfg.episode ? (uint32_t)cfg.episode[(long)e * cfg.episode_stride] : 0u;
  Rng rng(cfg.seed, (uint64_t)(e + cfg.env_offset), episode, RNG_TRACK);
  const V3 spawn = v3(0.f, 0.f, 1.5f);
  V3 pos = spawn, lo = spawn, hi = spawn;
  float heading = 0.f;
  const int G = cfg.n_gates;
  for (int k = 0; k < G; ++k) {
    const float4 u = rng.uniform4();
    const float spacing = 4.f + (cfg.spread - 4.f) * u.x;
    if (k) heading += (u.y * 2.f - 1.f) * 0.52359877559829887f;
    float s, c;
    sincosf(heading, &s, &c);
    const V3 d = v3(c, s, 0.f);
    pos = pos + d * spacing;
    const V3 ctr = v3(pos.x, pos.y, 1.f + 1.5f * u.z);
    float* g = gates + ((long)e * G + k) * 8;
    reinterpret_cast<float4*>(g)[0] = make_float4(ctr.x, ctr.y, ctr.z, 0.8f);
    reinterpret_cast<float4*>(g)[1] = make_float4(d.x, d.y, d.z, 0.3f);
    lo = v3(fminf(lo.x, ctr.x), fminf(lo.y, ctr.y), fminf(lo.z, ctr.z));
    hi = v3(fmaxf(hi.x, ctr.x), fmaxf(hi.y, ctr.y), fmaxf(hi.z, ctr.z));
    if (k == G - 1) reinterpret_cast<float4*>(spawn_goal)[2 * e + 1] = make_float4(ctr.x, ctr.y, ctr.z, 0.f);
  }
  reinterpret_cast<float4*>(spawn_goal)[2 * e] = make_float4(spawn.x, spawn.y, spawn.z, 0.f);
  reinterpret_cast<float4*>(bounds)[2 * e] = make_float4(lo.x - 5.f, lo.y - 5.f, 0.f, 0.f);
  reinterpret_cast<float4*>(bounds)[2 * e + 1] = make_float4(hi.x + 5.f, hi.y + 5.f, fmaxf(hi.z + 5.f, 4.f), 0.f);
  reinterpret_cast<int4*>(counts)[e] = make_int4(0, 0, 0, 1);
  ground_z[e] = 0.f;
}
}  // namespace

extern "C" int qs_gen_race_track(const qs_track_cfg* cfg, int32_t n_envs, float* bounds, float* spawn_goal,
                                 float* gates, int32_t* counts, float* ground_z, void* stream) {
  if (!cfg || n_envs < 0 || cfg->n_gates < 1 || cfg->n_gates > QS_MAX_GATES || !(cfg->spread >= 4.f))
    return QS_ERR_BAD_ARGUMENT;
  if (n_envs == 0) return QS_OK;
  if (!bounds || !spawn_goal || !gates || !counts || !ground_z) return QS_ERR_BAD_ARGUMENT;
  k_track<<<(n_envs + 127) / 128, 128, 0, (cudaStream_t)stream>>>(*cfg, n_envs, bounds, spawn_goal, gates, counts,
                                                                 ground_z);
  return cudaGetLastError() == cudaSuccess ? QS_OK : QS_ERR_LAUNCH;
}
