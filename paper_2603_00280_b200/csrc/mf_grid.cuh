// mf_grid.cuh -- heterogeneous GP field (BASELINE config 5, not in the
// reference): trilinear SDF grid for the mean, trilinear per-voxel sigma,
// spatially varying roughness alpha = sqrt2 sigma / l, and free flight by
// delta / ratio tracking against a coarse majorant grid traversed with a 3D
// DDA (exponential sampling per cell, memoryless restarts).
//
// Region rules follow transport.py:161-166 with sigma = sigma(p): collision
// walks live on f in [-6 sigma, 3 sigma]; a tentative collision that lands
// below -6 sigma(p) absorbs the path (the reference tests the depth cap at
// every walker step; here it is tested at tentative collisions -- the
// transmittance of the -3..-6 sigma slab is ~1e-6, transport.py:12-15);
// shadow walks integrate |f| <= 3 sigma only.
#pragma once

#include "mf_math.cuh"

namespace mf {

struct GridDev {
  const float* sdf;
  const float* sig;
  const float* maj;
  int n_sdf, n_sig, n_maj;
  V3 bmin, bmax;
  V3 inv_h_sdf;   // (n-1) / extent, per axis
  V3 inv_h_sig;
  V3 inv_h_maj;   // n_maj / extent
  V3 h_maj;       // cell size
  float k_xy, k_z;  // alpha = k * sigma, k = sqrt2 / l
};

MF_HD float ldg(const float* p) {
#if defined(__CUDA_ARCH__)
  return __ldg(p);
#else
  return *p;
#endif
}

// host-only walk statistics (tools/grid_walk_stats.py builds the host shim
// with -DMF_GRID_STATS): DDA iterations, tentative collisions, skips, walks
#if defined(MF_GRID_STATS) && !defined(__CUDA_ARCH__)
extern long long g_grid_stats[8];
#define MF_GSTAT(i) (++g_grid_stats[i])
#else
#define MF_GSTAT(i) ((void)0)
#endif

MF_HD int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

struct TriSample {
  float v;
  V3 grad;
};

// trilinear value (and optionally the gradient of the interpolant) of an
// n^3 vertex grid at grid coordinates g
template <bool kGrad>
MF_HD TriSample trilinear(const float* a, int n, V3 g, V3 inv_h) {
  float gx = fminf(fmaxf(g.x, 0.0f), (float)(n - 1));
  float gy = fminf(fmaxf(g.y, 0.0f), (float)(n - 1));
  float gz = fminf(fmaxf(g.z, 0.0f), (float)(n - 1));
  int ix = clampi((int)gx, 0, n - 2), iy = clampi((int)gy, 0, n - 2), iz = clampi((int)gz, 0, n - 2);
  float tx = gx - (float)ix, ty = gy - (float)iy, tz = gz - (float)iz;
  const float* p = a + ((size_t)ix * n + iy) * n + iz;
  size_t sy = (size_t)n, sx = (size_t)n * n;
  float c000 = ldg(p), c001 = ldg(p + 1), c010 = ldg(p + sy), c011 = ldg(p + sy + 1);
  float c100 = ldg(p + sx), c101 = ldg(p + sx + 1), c110 = ldg(p + sx + sy),
        c111 = ldg(p + sx + sy + 1);
  float c00 = fmaf(tz, c001 - c000, c000), c01 = fmaf(tz, c011 - c010, c010);
  float c10 = fmaf(tz, c101 - c100, c100), c11 = fmaf(tz, c111 - c110, c110);
  float c0 = fmaf(ty, c01 - c00, c00), c1 = fmaf(ty, c11 - c10, c10);
  TriSample s;
  s.v = fmaf(tx, c1 - c0, c0);
  if (kGrad) {
    float gxv = c1 - c0;
    float gyv = fmaf(tx, c11 - c10, (1.0f - tx) * (c01 - c00));
    float d00 = c001 - c000, d01 = c011 - c010, d10 = c101 - c100, d11 = c111 - c110;
    float d0 = fmaf(ty, d01 - d00, d00), d1 = fmaf(ty, d11 - d10, d10);
    float gzv = fmaf(tx, d1 - d0, d0);
    s.grad = v3(gxv * inv_h.x, gyv * inv_h.y, gzv * inv_h.z);
  } else {
    s.grad = v3(0.0f, 0.0f, 0.0f);
  }
  return s;
}

MF_HD V3 grid_coord(const GridDev& g, V3 p, V3 inv_h) {
  return v3((p.x - g.bmin.x) * inv_h.x, (p.y - g.bmin.y) * inv_h.y, (p.z - g.bmin.z) * inv_h.z);
}

MF_HD float grid_f(const GridDev& g, V3 p) {
  return trilinear<false>(g.sdf, g.n_sdf, grid_coord(g, p, g.inv_h_sdf), g.inv_h_sdf).v;
}

MF_HD float grid_sigma(const GridDev& g, V3 p) {
  return trilinear<false>(g.sig, g.n_sig, grid_coord(g, p, g.inv_h_sig), g.inv_h_sig).v;
}

// Local medium at sigma: generalized kind, alpha = k sigma; `base` supplies
// the mixture ratio, Fresnel / albedo and the slope table.
MF_HD MediumK grid_medium(const MediumK& base, float sigma, float k_xy, float k_z) {
  MediumK m = base;
  m.kind = kGeneralized;
  m.sigma = sigma;
  m.inv_sigma = frcp(sigma);
  float ax = k_xy * sigma, az = k_z * sigma;
  m.ax = ax;
  m.ay = ax;
  m.az = az;
  m.inv_ax = frcp(ax);
  m.inv_ay = m.inv_ax;
  m.inv_az2 = frcp(az * az);
  m.exp_neg_c = expf(-m.inv_az2);
  m.beck_norm = kInvSqrtPi * kInvSqrtPi * m.inv_ax * m.inv_ax;            // 1/(pi ax^2)
  m.d_norm = m.beck_norm * kInvSqrtPi * frcp(az);                         // 1/(pi^1.5 ax^2 az)
  return m;
}

#ifndef MF_GRID_ISO_AREA
#define MF_GRID_ISO_AREA 1
#endif

// extinction at p along dir; 0 outside the region [lo_mult sigma, 3 sigma].
// Also reports f and sigma (for the absorption rule).
MF_HD float grid_extinction(const GridDev& g, const MediumK& base, V3 p, V3 dir, float lo_mult,
                            float* f_out, float* s_out) {
  TriSample fs = trilinear<true>(g.sdf, g.n_sdf, grid_coord(g, p, g.inv_h_sdf), g.inv_h_sdf);
  float sg = fmaxf(grid_sigma(g, p), 1e-6f);
  *f_out = fs.v;
  *s_out = sg;
  if (fs.v < lo_mult * sg || fs.v > 3.0f * sg) return 0.0f;
  float gn2 = dot3(fs.grad, fs.grad);
  float ax = g.k_xy * sg, az = g.k_z * sg;
#if MF_GRID_ISO_AREA
  // alpha_x = alpha_y: sigma(w) depends on the local w.z = <n, dir> alone,
  // so the local frame is not needed -- sigma at (sqrt(1 - c^2), 0, c)
  float c = gn2 > 0.0f ? dot3(fs.grad, dir) * frsqrt(gn2) : dir.z;
  c = fminf(fmaxf(c, -1.0f), 1.0f);
  float area = proj_area_erf<true>(v3(fsqrt(fmaxf(1.0f - c * c, 0.0f)), 0.0f, c), ax, ax, az);
#else
  V3 n = gn2 > 0.0f ? mul3(fs.grad, frsqrt(gn2)) : v3(0.0f, 0.0f, 1.0f);
  Frame fr = frame_about(n);
  V3 wl = to_local(fr, dir);
  float area = proj_area_erf<true>(wl, ax, ax, az);   // render walks: MUFU exp2
#endif
  (void)base;
  return mills<true>(fs.v * frcp(sg)) * frcp(sg) * area;
}

constexpr int kGridIterCap = 1000000;
// empty cells at Chebyshev distance >= this jump (a jump re-locates the
// cell from the position, ~3 plain DDA steps of work)
#ifndef MF_GRID_SKIP_MIN
#define MF_GRID_SKIP_MIN 2
#endif

struct GridWalk {
  int outcome;   // kEscaped / kAbsorbed / kCollided (values of mf_transport.cuh)
  V3 pos;
  float weight;
  int steps;
  int violations;
};

// Slab test against the grid bounds; returns false on a miss.
MF_HD bool grid_box(const GridDev& g, V3 o, V3 d, float* t0, float* t1) {
  float ta = 0.0f, tb = INFINITY;
  float os[3] = {o.x, o.y, o.z}, ds[3] = {d.x, d.y, d.z};
  float lo[3] = {g.bmin.x, g.bmin.y, g.bmin.z}, hi[3] = {g.bmax.x, g.bmax.y, g.bmax.z};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    float inv = 1.0f / ds[a];
    float u = (lo[a] - os[a]) * inv, v = (hi[a] - os[a]) * inv;
    if (ds[a] == 0.0f) {
      if (os[a] < lo[a] || os[a] > hi[a]) return false;
      continue;
    }
    ta = fmaxf(ta, fminf(u, v));
    tb = fminf(tb, fmaxf(u, v));
  }
  *t0 = ta;
  *t1 = tb;
  return ta <= tb;
}

// Delta (ratio == false) or ratio tracking through the majorant grid, as a
// resumable walker: dda() advances the 3D DDA over the majorant cells until
// the next tentative collision (or the end of the walk), tentative()
// evaluates the extinction there and takes the tracking decision.  The
// per-lane arithmetic and random-number consumption are those of one
// sequential loop, whichever driver runs the two halves, and the walk can
// be parked between any two calls: (t, tau, weight, cell, steps) is its
// whole state (park() / resume()); everything else is a function of the
// ray.  The wall distances are therefore computed from the cell index
// (c * wa + wb per axis), never accumulated.
// Random draws: block (segment, call0) of the path's Philox stream gives the
// first optical depth; block (segment, call0 + k) serves the k-th tentative
// collision (x: acceptance / roulette uniform, y: the next optical depth).
struct GridPark {
  float t, tau, weight;
  uint32_t cell;   // cx | cy << 10 | cz << 20 (n_maj <= 1024)
  int steps;
};

template <typename RngBlock>
struct GridWalker {
  RngBlock rng_block;
  GridWalk w;
  V3 pos, dir;
  float t, t1, tau, lo_mult, rr_min;
  float tx, ty, tz, wax, way, waz, wbx, wby, wbz, dt_min, mu;
  int cx, cy, cz, sx, sy, sz;
  bool ratio;
  uint32_t call0;

  MF_HDM GridWalker(RngBlock rb) : rng_block(rb) {}

  // wall distance of cell c on one axis is c * wa + wb (INFINITY for a ray
  // parallel to the walls)
  MF_HDM static void wall_coef(int s, float bmin, float h, float o, float d, float* wa, float* wb) {
    if (!(fabsf(d) > 1e-30f)) {
      *wa = 0.0f;
      *wb = INFINITY;
    } else {
      float id = 1.0f / d;
      *wa = h * id;
      *wb = (bmin + (s > 0 ? h : 0.0f) - o) * id;
    }
  }

  // walls of one axis (spacing h / |d|, the next one at tk) reached by tn
  MF_HDM static int crossed(float tn, float tk, float d, float inv_h) {
    return tn >= tk ? (int)((tn - tk) * (fabsf(d) * inv_h)) + 1 : 0;
  }

  MF_HDM void walls() {
    tx = fmaf((float)cx, wax, wbx);
    ty = fmaf((float)cy, way, wby);
    tz = fmaf((float)cz, waz, wbz);
  }

  MF_HDM void locate(const GridDev& g) {
    V3 q = grid_coord(g, fma3(dir, t, pos), g.inv_h_maj);
    int n = g.n_maj;
    cx = clampi((int)q.x, 0, n - 1);
    cy = clampi((int)q.y, 0, n - 1);
    cz = clampi((int)q.z, 0, n - 1);
    walls();
  }

  // the ray's constants; false: the ray misses the grid.  t0 = entry distance
  MF_HDM bool setup(const GridDev& g, uint32_t call0_, V3 p0, V3 d, bool ratio_walk, float t_max,
                   float rr, float* t0) {
    w.outcome = 0;
    w.pos = p0;
    w.weight = 1.0f;
    w.steps = 0;
    w.violations = 0;
    pos = p0;
    dir = d;
    ratio = ratio_walk;
    rr_min = rr;
    lo_mult = ratio ? -3.0f : -6.0f;
    call0 = call0_;
    if (!grid_box(g, pos, dir, t0, &t1)) return false;
    t1 = fminf(t1, t_max);
    sx = dir.x > 0.0f ? 1 : -1;
    sy = dir.y > 0.0f ? 1 : -1;
    sz = dir.z > 0.0f ? 1 : -1;
    wall_coef(sx, g.bmin.x, g.h_maj.x, pos.x, dir.x, &wax, &wbx);
    wall_coef(sy, g.bmin.y, g.h_maj.y, pos.y, dir.y, &way, &wby);
    wall_coef(sz, g.bmin.z, g.h_maj.z, pos.z, dir.z, &waz, &wbz);
    // parametric length of one cell on the axis the ray crosses fastest
    dt_min = fminf(fminf(wax != 0.0f ? fabsf(wax) : INFINITY, way != 0.0f ? fabsf(way) : INFINITY),
                   waz != 0.0f ? fabsf(waz) : INFINITY);
    return true;
  }

  // false: the ray misses the grid (escaped at once)
  MF_HDM bool begin(const GridDev& g, uint32_t call0_, V3 p0, V3 d, bool ratio_walk, float t_max,
                   float rr) {
    float t0;
    if (!setup(g, call0_, p0, d, ratio_walk, t_max, rr, &t0)) return false;
    t = t0;
    locate(g);
    // optical depth left to the next tentative collision: sampled once per
    // tentative and used up cell by cell (tau -= mu dt), instead of a fresh
    // exponential (a uniform and a log) in every cell the ray crosses -- the
    // same process (the majorant is piecewise constant along the ray), a
    // fraction of the random numbers and logs
    tau = -flog(u01(rng_block(call0).x));
    MF_GSTAT(3);
    return true;
  }

  MF_HDM GridPark park() const {
    return GridPark{t, tau, w.weight, (uint32_t)cx | ((uint32_t)cy << 10) | ((uint32_t)cz << 20),
                    w.steps};
  }

  // continue a parked walk of the same ray (same arguments as begin())
  MF_HDM void resume(const GridDev& g, uint32_t call0_, V3 p0, V3 d, bool ratio_walk, float t_max,
                    float rr, const GridPark& k) {
    float t0;
    setup(g, call0_, p0, d, ratio_walk, t_max, rr, &t0);
    t = k.t;
    tau = k.tau;
    w.weight = k.weight;
    w.steps = k.steps;
    cx = (int)(k.cell & 1023u);
    cy = (int)((k.cell >> 10) & 1023u);
    cz = (int)(k.cell >> 20);
    walls();
  }

  MF_HDM void end_at(float te) { w.pos = fma3(dir, te, pos); }

  // One loop iteration of the DDA.  Returns 1 when a tentative collision
  // lies in the current cell (t is advanced to it; call tentative()), 2 when
  // the walk has left the grid or reached t1 (t is the end parameter; the
  // driver calls end_at(t) once), 0 otherwise.  Apart from the three exits
  // (collision, end, empty-space jump) the step is branch-free, so the
  // lanes of a warp that step together stay converged.
  MF_HDM int dda(const GridDev& g) {
    MF_GSTAT(0);
    int n = g.n_maj;
    float t_exit = fminf(fminf(tx, ty), fminf(tz, t1));
    mu = ldg(g.maj + (unsigned)((cx * n + cy) * n + cz));
    float need = mu * (t_exit - t);
    bool med = mu > 0.0f;
    if (med && tau < need) {
      t = fmaf(tau, frcp(mu), t);
      return 1;
    }
    if (med) MF_GSTAT(4);
    tau = med ? tau - need : tau;   // a select: medium and empty cells stay converged
    // leave the cell.  Empty space (mu = -D): jump (D - 1) cells in every
    // axis, then restart the DDA from the cell at the landing point
    float tj = t + (-mu - 1.0f) * dt_min;
    bool skip = mu <= -(float)MF_GRID_SKIP_MIN && tj > t_exit;
    float tn = skip ? tj : t_exit;
    if (tn >= t1) {
      t = t1;
      return 2;   // escaped the grid (or reached the light)
    }
    t = tn;
    if (skip) MF_GSTAT(2);
    // cell walls crossed on each axis up to tn: one on the exit axis for a
    // plain step (tn is that wall), up to D - 1 per axis for a jump -- one
    // code path for both, so stepping and jumping lanes stay converged
    cx += sx * crossed(tn, tx, dir.x, g.inv_h_maj.x);
    cy += sy * crossed(tn, ty, dir.y, g.inv_h_maj.y);
    cz += sz * crossed(tn, tz, dir.z, g.inv_h_maj.z);
    walls();
    return ((unsigned)cx >= (unsigned)n || (unsigned)cy >= (unsigned)n ||
            (unsigned)cz >= (unsigned)n) ? 2 : 0;
  }

  // The tentative collision at t (majorant mu): true when the walk ends.
  MF_HDM bool tentative(const GridDev& g, const MediumK& base) {
    V3 p = fma3(dir, t, pos);
    if (w.steps >= kGridIterCap) {
      // iteration cap (transport.py:297 raises): a distinct result, counted
      // by the callers as capped, never taken for an escape
      w.pos = p;
      w.outcome = 1;
      w.weight = 0.0f;
      w.steps = -1;
      return true;
    }
    w.steps++;
    MF_GSTAT(1);
    float f, sg;
    float st = grid_extinction(g, base, p, dir, lo_mult, &f, &sg);
    U4 b = rng_block(call0 + (uint32_t)w.steps);
    if (st > mu * 1.00001f) w.violations++;
    if (ratio) {
      w.weight *= fmaxf(1.0f - st / mu, 0.0f);
      if (w.weight < rr_min && w.weight > 0.0f) {
        // Russian roulette on the weight (see walk() in mf_transport.cuh)
        w.weight = u01(b.x) * rr_min < w.weight ? rr_min : 0.0f;
      }
      if (!(w.weight > 0.0f)) {
        w.pos = p;
        return true;
      }
    } else {
      if (f < -6.0f * sg) {
        w.outcome = 1;   // absorbed below the depth cap
        w.pos = p;
        return true;
      }
      if (u01(b.x) * mu < st) {
        w.outcome = 2;
        w.pos = p;
        return true;
      }
    }
    tau = -flog(u01(b.y));
    return false;
  }
};

// The driver: one lane walks on its own.  (A warp-batched driver -- lanes
// step their DDAs and evaluate the tentative collisions together once half
// of the walking lanes have one pending -- gave bit-identical images but
// was slower on config 5: 4.6 - 6.6 ms for batch fractions 0.3 - 1 against
// 3.56 ms.)
template <typename RngBlock>
MF_HD GridWalk grid_walk(const GridDev& g, const MediumK& base, RngBlock rng_block,
                         uint32_t call0, V3 pos, V3 dir, bool ratio, float t_max,
                         float rr_min = 0.0f) {
  GridWalker<RngBlock> W(rng_block);
  if (!W.begin(g, call0, pos, dir, ratio, t_max, rr_min)) return W.w;
  while (true) {
    int r = W.dda(g);
    if (r == 2) {
      W.end_at(W.t);
      break;
    }
    if (r == 1 && W.tentative(g, base)) break;
  }
  return W.w;
}


// ---------------------------------------------------------------------------
// empty-space distances (second pass of mf_grid_majorant)
//
// A cell whose majorant is 0 holds no medium.  Such cells store -D instead,
// D = the Chebyshev distance (in cells) to the nearest cell with medium,
// capped at kSkipMax + 1: from any point of the cell the ray can advance
// (D - 1) cells in every axis without meeting medium, so grid_walk jumps
// over empty space instead of stepping through it cell by cell (no random
// numbers are drawn in empty cells, so the process is unchanged).
constexpr int kSkipMax = 15;

MF_HD float grid_cell_skip(const float* maj, int n, int cx, int cy, int cz) {
  if (maj[((size_t)cx * n + cy) * n + cz] > 0.0f) return maj[((size_t)cx * n + cy) * n + cz];
  for (int k = 1; k <= kSkipMax; ++k) {
    // the shell of the (2k+1)^3 cube around the cell
    for (int i = cx - k; i <= cx + k; ++i) {
      if (i < 0 || i >= n) continue;
      bool face_i = i == cx - k || i == cx + k;
      for (int j = cy - k; j <= cy + k; ++j) {
        if (j < 0 || j >= n) continue;
        bool face_j = face_i || j == cy - k || j == cy + k;
        int step = face_j ? 1 : 2 * k;
        for (int l = cz - k; l <= cz + k; l += step) {
          if (l < 0 || l >= n) continue;
          if (maj[((size_t)i * n + j) * n + l] > 0.0f) return -(float)k;
        }
      }
    }
  }
  return -(float)(kSkipMax + 1);
}

// ---------------------------------------------------------------------------
// majorant of one cell (host-checked formula; run by mf_grid_majorant)

MF_HD float area_max_iso(float a_xy, float a_z) {
  // max over directions of sigma(w) for ax = ay = a_xy: 1D scan in theta
  float best = 0.0f;
  for (int i = 0; i <= 96; ++i) {
    float th = kPi * (float)i / 96.0f;
    V3 w = v3(sinf(th), 0.0f, cosf(th));
    best = fmaxf(best, proj_area_erf(w, a_xy, a_xy, a_z));
  }
  return best * 1.03f;
}

MF_HD float grid_cell_majorant(const GridDev& g, int cx, int cy, int cz) {
  // world extent of the cell
  V3 lo = v3(g.bmin.x + g.h_maj.x * cx, g.bmin.y + g.h_maj.y * cy, g.bmin.z + g.h_maj.z * cz);
  V3 hi = add3(lo, g.h_maj);
  // exact bounds of the trilinear interpolants: min / max over covering vertices
  V3 a = grid_coord(g, lo, g.inv_h_sdf), b = grid_coord(g, hi, g.inv_h_sdf);
  int x0 = clampi((int)floorf(a.x), 0, g.n_sdf - 1), x1 = clampi((int)ceilf(b.x), 0, g.n_sdf - 1);
  int y0 = clampi((int)floorf(a.y), 0, g.n_sdf - 1), y1 = clampi((int)ceilf(b.y), 0, g.n_sdf - 1);
  int z0 = clampi((int)floorf(a.z), 0, g.n_sdf - 1), z1 = clampi((int)ceilf(b.z), 0, g.n_sdf - 1);
  float fmin = INFINITY;
  for (int i = x0; i <= x1; ++i)
    for (int j = y0; j <= y1; ++j)
      for (int k = z0; k <= z1; ++k)
        fmin = fminf(fmin, ldg(g.sdf + ((size_t)i * g.n_sdf + j) * g.n_sdf + k));
  V3 c = grid_coord(g, lo, g.inv_h_sig), d = grid_coord(g, hi, g.inv_h_sig);
  x0 = clampi((int)floorf(c.x), 0, g.n_sig - 1); x1 = clampi((int)ceilf(d.x), 0, g.n_sig - 1);
  y0 = clampi((int)floorf(c.y), 0, g.n_sig - 1); y1 = clampi((int)ceilf(d.y), 0, g.n_sig - 1);
  z0 = clampi((int)floorf(c.z), 0, g.n_sig - 1); z1 = clampi((int)ceilf(d.z), 0, g.n_sig - 1);
  float smin = INFINITY, smax = 0.0f;
  for (int i = x0; i <= x1; ++i)
    for (int j = y0; j <= y1; ++j)
      for (int k = z0; k <= z1; ++k) {
        float v = ldg(g.sig + ((size_t)i * g.n_sig + j) * g.n_sig + k);
        smin = fminf(smin, v);
        smax = fmaxf(smax, v);
      }
  smin = fmaxf(smin, 1e-6f);
  smax = fmaxf(smax, smin);
  if (fmin > 3.0f * smax) return 0.0f;   // entirely above every shell: vacuum
  // sup over sigma in [smin, smax] of rho(max(fmin, -6 sigma), sigma) * max_w sigma(w)
  float best = 0.0f;
  const int K = 12;
  for (int i = 0; i <= K; ++i) {
    float s = smin + (smax - smin) * (float)i / (float)K;
    float f = fmaxf(fmin, -6.0f * s);
    if (f > 3.0f * s) continue;
    float rho = mills(f / s) / s;
    best = fmaxf(best, rho * area_max_iso(g.k_xy * s, g.k_z * s));
  }
  // rho * area varies by < 5 % between the sigma samples of one cell
  return best * 1.15f;
}

}  // namespace mf
