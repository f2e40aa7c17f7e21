// mf_transport.cuh -- device scene, free flight, NEE transmittance.
//
// Reference (float64, wavefront numpy) -> here (fp32, per-path in registers):
//   walk(mode="collision")     transport.py:144-297
//       single plane : analytic free flight, inverting the closed-form
//                      transmittance (medium.py:98-124) in log-Phi space
//                      -- same distribution of collision heights, no
//                      stepping
//       otherwise    : delta tracking with the moving Lipschitz band
//                      majorant rho(f - s/2) * sigma_max, step <= s/2,
//                      sigma_max the exact max_w sigma(w) (tighter than
//                      ndf.py:189-194's direction-free bound)
//   walk(mode="ratio")         transport.py:269-270: closed form for a single
//                      plane, ratio tracking otherwise
//   region rules               transport.py:161-166: collision walks live on
//                      f in [-6s, 3s] and absorb below; shadow walks
//                      integrate |f| <= 3s only
#pragma once

#include "mf_math.cuh"
#include "mf_query.cuh"
#include "mf_grid.cuh"

namespace mf {

constexpr int kMaxPrims = 8;

// (out of line measured slower for the grid walker: 3.45 vs 3.19 ms)
#ifndef MF_WALK_OUTLINE_GRID
#define MF_WALK_OUTLINE_GRID 0
#endif

struct PrimDev {
  int shape;   // 0 plane, 1 sphere, 3 box (MF_SHAPE_*)
  int medium;
  float z0;
  V3 c;
  float radius;
  V3 half;     // box half extents
};

constexpr int kShapePlane = 0, kShapeSphere = 1, kShapeBox = 3;

// Tracking-step length inside a band, in units of the medium's sigma.  The
// per-step majorant is exact over [0, step] whatever the length; shorter
// steps tighten it (fewer null collisions) but cost more majorant
// evaluations.  Measured on config 3 (B200): 0.5 -> 16.0 ms, 1 -> 12.9,
// 2 -> 11.9, 3 -> 12.2, 4.5 -> 13.2 ms.
#ifndef MF_STEP_FRAC
#define MF_STEP_FRAC 2.0f
#endif

struct MediumExtra {
  float sig_max;       // max_w sigma(w), majorant factor for curved shells
  int area_monotone;   // sigma(w) depends on cos(theta) only and decreases with it
  float lphi_hi;       // log Phi(3)   (collision / ratio upper edge)
  float lphi_lo_col;   // log Phi(-6)  (collision absorption edge)
  float lphi_lo_rat;   // log Phi(-3)  (ratio lower edge)
};

struct SceneDev {
  int n_prims;
  int single_plane;    // 1: analytic planar transport
  int mono;            // 1: every radiance / weight factor is grey (pool_kernel<*, true>)
  PrimDev prims[kMaxPrims];
  MediumK media[kMaxPrims];
  MediumExtra mx[kMaxPrims];
  // camera (scene.py:30-51 basis; ortho extension)
  int ortho, width, height;
  V3 cam_pos, cam_fwd, cam_right, cam_up;
  float half_w, half_h;
  V3 env;
  // lat-long environment map (scene.py:61-84): (env_h, env_w, 3) float32,
  // theta down the rows; nullptr = the constant env
  const float* env_map;
  int env_w, env_h;
  int has_sun;
  V3 sun_to;           // unit direction towards the sun (= -DirectionalLight.direction)
  V3 sun_L;
  float sun_sig;       // sigma(sun_to) in the plane frame (single-plane scenes)
  // single plane, closed-form sun transmittance from a collision's log Phi l:
  // Tr = 2^{sun_k2 |sun_lb - clamp(l)|}, sun_k2 = -sigma(sun) / |cos| log2(e)
  float sun_k2, sun_lb;
  int sun_graze;       // |cos| < 1e-6: Tr = 0 unless the band is not crossed
  int has_point;
  V3 point_pos;
  V3 point_I;
  float min_skip;      // 1e-7 * min sigma (transport.py:167)
  int has_grid;        // 1: the single primitive is the grid field below
  GridDev grid;
  int generic_walk;    // single sphere: step with walk<true> instead of sphere_walk
};

// Environment radiance of an escaping direction d (scene.py:61-84): the
// constant, or the lat-long map bilinear in (phi, theta) with phi wrapped
// and theta clamped, texel centres at half-integers -- the reference's
// formula in float32.
// lat-long map lookup, out of line: one copy, off the instruction stream of
// the hot render loops (constant environments never call it)
MF_COLD V3 env_map_radiance(const SceneDev& sc, V3 d) {
  const float kPi = 3.14159265358979f;
  float th = acosf(fminf(fmaxf(d.z, -1.0f), 1.0f));
  float ph = atan2f(d.y, d.x);
  if (ph < 0.0f) ph += 2.0f * kPi;
  int w = sc.env_w, h = sc.env_h;
  float fx = ph / (2.0f * kPi) * (float)w - 0.5f;
  float fy = th / kPi * (float)h - 0.5f;
  float x0f = floorf(fx), y0f = floorf(fy);
  float tx = fx - x0f, ty = fy - y0f;
  int x0 = (int)x0f, y0 = (int)y0f;
  int x0m = ((x0 % w) + w) % w, x1m = (((x0 + 1) % w) + w) % w;
  int y0m = clampi(y0, 0, h - 1), y1m = clampi(y0 + 1, 0, h - 1);
  const float* m = sc.env_map;
  float w00 = (1.0f - tx) * (1.0f - ty), w01 = tx * (1.0f - ty), w10 = (1.0f - tx) * ty,
        w11 = tx * ty;
  float c[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    c[k] = ldg(m + ((size_t)y0m * w + x0m) * 3 + k) * w00 +
           ldg(m + ((size_t)y0m * w + x1m) * 3 + k) * w01 +
           ldg(m + ((size_t)y1m * w + x0m) * 3 + k) * w10 +
           ldg(m + ((size_t)y1m * w + x1m) * 3 + k) * w11;
  }
  return v3(c[0], c[1], c[2]);
}

MF_HD V3 env_radiance(const SceneDev& sc, V3 d) {
  return sc.env_map ? env_map_radiance(sc, d) : sc.env;
}

// ---------------------------------------------------------------------------
// counter-based random stream of one path: key = seed, counter =
// (pixel, sample, segment, call)

struct PathRng {
  uint32_t k0, k1;
  uint32_t pixel, sample;
};

MF_HD U4 rng_block(const PathRng& r, uint32_t segment, uint32_t call) {
  return philox4x32_10(U4{r.pixel, r.sample, segment, call}, r.k0, r.k1);
}

// segment id used for the camera jitter draw
constexpr uint32_t kSegCamera = 0xFFFFFFFFu;
// call ids >= this index the shadow-ray (ratio tracking) stream of a segment
constexpr uint32_t kCallShadow = 0x80000000u;

// ---------------------------------------------------------------------------
// fields

// kSphere: the primitive is known to be a sphere (single-sphere walker)
// box SDF and gradient (sdf.py:55-84): exact distance outside, max of the
// per-axis distances inside; inside, the gradient is the axis of the
// nearest face (first on ties, as numpy's argmax)
MF_HD float box_field(const PrimDev& p, V3 x) {
  float qx = fabsf(x.x - p.c.x) - p.half.x, qy = fabsf(x.y - p.c.y) - p.half.y,
        qz = fabsf(x.z - p.c.z) - p.half.z;
  float ox = fmaxf(qx, 0.0f), oy = fmaxf(qy, 0.0f), oz = fmaxf(qz, 0.0f);
  return fsqrt(ox * ox + oy * oy + oz * oz) + fminf(fmaxf(qx, fmaxf(qy, qz)), 0.0f);
}

MF_HD V3 box_normal(const PrimDev& p, V3 x) {
  V3 d = sub3(x, p.c);
  float qx = fabsf(d.x) - p.half.x, qy = fabsf(d.y) - p.half.y, qz = fabsf(d.z) - p.half.z;
  float ox = fmaxf(qx, 0.0f), oy = fmaxf(qy, 0.0f), oz = fmaxf(qz, 0.0f);
  float on2 = ox * ox + oy * oy + oz * oz;
  if (on2 > 0.0f) {
    float inv = frsqrt(on2);
    return v3(copysignf(ox * inv, d.x), copysignf(oy * inv, d.y), copysignf(oz * inv, d.z));
  }
  if (qx >= qy && qx >= qz) return v3(d.x >= 0.0f ? 1.0f : -1.0f, 0.0f, 0.0f);
  if (qy >= qz) return v3(0.0f, d.y >= 0.0f ? 1.0f : -1.0f, 0.0f);
  return v3(0.0f, 0.0f, d.z >= 0.0f ? 1.0f : -1.0f);
}

template <bool kSphere = false>
MF_HD float prim_field(const PrimDev& p, V3 x) {
  if (!kSphere && p.shape == kShapePlane) return x.z - p.z0;
  if (!kSphere && p.shape == kShapeBox) return box_field(p, x);
  V3 d = sub3(x, p.c);
  return fsqrt(dot3(d, d)) - p.radius;
}

template <bool kSphere = false>
MF_HD V3 prim_normal(const PrimDev& p, V3 x) {
  if (!kSphere && p.shape == kShapePlane) return v3(0.0f, 0.0f, 1.0f);
  if (!kSphere && p.shape == kShapeBox) return box_normal(p, x);
  V3 d = sub3(x, p.c);
  float r2 = dot3(d, d);
  return r2 > 0.0f ? mul3(d, frsqrt(r2)) : v3(0.0f, 0.0f, 1.0f);
}

// distance along the ray to the level set f = level (transport.py:70-92);
// +inf when never reached.  For spheres the side is decided by the sign of
// c = |p - c|^2 - R^2 (outside: first root, which may round to ~0 on the
// surface itself; inside: second root), not by a threshold on the first
// root -- in float32 a ray sitting on the level set must not be sent to the
// far side.
template <bool kSphere = false>
MF_HD float level_distance(const PrimDev& p, V3 pos, V3 dir, float level) {
  if (!kSphere && p.shape == kShapePlane) {
    float t = (level - (pos.z - p.z0)) / dir.z;
    return (t >= 0.0f && t < INFINITY) ? t : INFINITY;
  }
  if (!kSphere && p.shape == kShapeBox) {
    // 1-Lipschitz lower bound |f - level| (transport.py:93), and the recede
    // test (transport.py:105-108): above the level and moving along the
    // gradient, the convex exterior never brings the level back
    float f = box_field(p, pos);
    if (f > level && dot3(box_normal(p, pos), dir) >= 0.0f) return INFINITY;
    return fabsf(f - level);
  }
  float rad = p.radius + level;
  if (!(rad > 0.0f)) return INFINITY;
  V3 oc = sub3(pos, p.c);
  float b = dot3(oc, dir);
  float cc = dot3(oc, oc) - rad * rad;
  float disc = b * b - cc;
  if (cc > 0.0f) {
    // outside the level sphere: reachable only when moving towards it
    if (b >= 0.0f || disc < 0.0f) return INFINITY;
    return fmaxf(-b - fsqrt(disc), 0.0f);
  }
  // inside (or on) the level sphere: leave through the second root
  return fmaxf(-b + fsqrt(fmaxf(disc, 0.0f)), 0.0f);
}

// ---------------------------------------------------------------------------
// analytic planar free flight (single plane)

enum FlightOutcome : int { kEscaped = 0, kAbsorbed = 1, kCollided = 2, kNullCollision = 3 };

struct Flight {
  int outcome;
  V3 pos;
  float lphi;   // log Phi(f / sigma) at pos after a collision, NaN otherwise
};

// log Phi of a start height inside the band (rare on the render path: paths
// enter from above and carry log Phi after each collision); out of line
MF_COLD float log_ndtr_cold(float u) { return log_ndtr(u); }

// position of a collision at log Phi l1 (only read by a point light); out of
// line -- one copy, so every kernel computes it with the same instructions
MF_COLD V3 planar_collision_pos(const PrimDev& pr, const MediumK& m, V3 pos, V3 dir, float h,
                                float c, float l1) {
  float h1 = m.sigma * inv_log_ndtr(l1);
  // keep the root on the travelled side of h despite rounding
  h1 = c > 0.0f ? fmaxf(h1, h) : fminf(h1, h);
  V3 p = fma3(dir, (h1 - h) / c, pos);
  p.z = pr.z0 + h1;
  return p;
}

// grazing flight (|cos theta| < 1e-6): f stays put, so this branch needs the
// true height (from l0 when the height was not tracked); out of line
MF_COLD Flight planar_flight_grazing(const PrimDev& pr, const MediumK& m, V3 pos, V3 dir,
                                    float sig, float tau, float l0, float h, bool from_l0) {
  Flight fl;
  fl.lphi = NAN;
  fl.pos = pos;
  float hg = from_l0 ? m.sigma * inv_log_ndtr(l0) : h;
  float st = mills(hg * m.inv_sigma) * m.inv_sigma * sig;
  if (!(st > 0.0f)) {
    fl.outcome = kEscaped;
    return fl;
  }
  fl.outcome = kCollided;
  pos.z = pr.z0 + hg;
  fl.pos = fma3(dir, tau / st, pos);
  return fl;
}

// One collision-mode flight from pos along dir through the shell of a
// single plane, given u in (0,1).  sig = sigma(dir) in the plane frame.
// The flight is sampled in log-Phi space: lphi = log Phi(f / sigma) at pos
// when known (the previous collision's l1), NaN otherwise (first flight,
// after a grazing one).  A collision returns its l1, which the next flight
// and the shadow ray use instead of re-deriving it from the height; the
// height h1 = sigma Phi^-1(e^l1) (and so the position) is then needed only
// when something reads positions (a point light): need_pos.  Without it
// fl.pos is left stale -- nothing in a single-plane scene depends on x, y,
// and every decision on z is taken on l.
MF_HD Flight planar_flight(const PrimDev& pr, const MediumK& m, const MediumExtra& mx, V3 pos,
                           V3 dir, float sig, float u, float lphi, bool need_pos) {
  Flight fl;
  fl.lphi = NAN;
  fl.pos = pos;
  float s3 = 3.0f * m.sigma;
  float c = dir.z;
  bool known = lphi == lphi;
  float h = pos.z - pr.z0;     // valid unless (known && !need_pos)
  float l0 = lphi;
  if (!known) {
    if (h > s3) {
      if (!(c < 0.0f)) {
        fl.outcome = kEscaped;
        return fl;
      }
      pos = fma3(dir, (s3 - h) / c, pos);
      fl.pos = pos;
      h = s3;
      l0 = mx.lphi_hi;
    } else {
      if (h < -6.0f * m.sigma) {
        fl.outcome = kAbsorbed;
        return fl;
      }
      l0 = log_ndtr_cold(h * m.inv_sigma);
    }
  }
  float tau = -flog(u);
  if (fabsf(c) < 1e-6f) return planar_flight_grazing(pr, m, pos, dir, sig, tau, l0, h,
                                                    known && !need_pos);
  float dl = tau * fabsf(c) / sig;          // change of log Phi along the flight
  float l1;
  if (c > 0.0f) {
    l1 = l0 + dl;
    if (!(l1 < mx.lphi_hi)) {
      fl.outcome = kEscaped;
      return fl;
    }
  } else {
    l1 = l0 - dl;
    if (!(l1 >= mx.lphi_lo_col)) {
      fl.outcome = kAbsorbed;
      return fl;
    }
  }
  fl.outcome = kCollided;
  fl.lphi = l1;
  if (need_pos) fl.pos = planar_collision_pos(pr, m, pos, dir, h, c, l1);
  return fl;
}

// closed-form shadow transmittance of a single plane over |f| <= 3 sigma
// between field values h (start) and h_end (light; +/-inf for the sun);
// lphi = log Phi(h / sigma) when known (NaN otherwise; h is then not read)
MF_HD float planar_shadow_tr(const MediumK& m, const MediumExtra& mx, float h, float h_end,
                             float c, float sig, float lphi) {
  float s3 = 3.0f * m.sigma;
  float ea = fminf(fmaxf(h, -s3), s3);
  float eb = fminf(fmaxf(h_end, -s3), s3);
  // clamping f to the band is clamping log Phi to [log Phi(-3), log Phi(3)]
  float la = lphi == lphi ? fminf(fmaxf(lphi, mx.lphi_lo_rat), mx.lphi_hi)
                          : (ea >= s3 ? mx.lphi_hi : (ea <= -s3 ? mx.lphi_lo_rat : NAN));
  float lb = eb >= s3 ? mx.lphi_hi : (eb <= -s3 ? mx.lphi_lo_rat : NAN);
  // the ends still unknown through one copy of log_ndtr (I-cache)
#pragma unroll 1
  for (int i = 0; i < 2; ++i) {
    float cur = i == 0 ? la : lb;
    if (!(cur == cur)) {
      float l = log_ndtr((i == 0 ? ea : eb) * m.inv_sigma);
      la = i == 0 ? l : la;
      lb = i == 0 ? lb : l;
    }
  }
  if (la == lb) return 1.0f;
  if (fabsf(c) < 1e-6f) return 0.0f;
  return expf(-sig / fabsf(c) * fabsf(lb - la));
}

// Grid-field walk of a path's random stream (segment, calls call0...).
#if MF_WALK_OUTLINE_GRID && defined(__CUDACC__)
#define MF_GRID_WALK_FN __host__ __device__ __noinline__
#else
#define MF_GRID_WALK_FN MF_HD
#endif
MF_GRID_WALK_FN GridWalk grid_walk_path(const GridDev& g, const MediumK& base, PathRng r,
                                        uint32_t seg, uint32_t call0, V3 pos, V3 dir, bool ratio,
                                        float t_max, float rr_min) {
  return grid_walk(g, base, [&](uint32_t call) { return rng_block(r, seg, call); }, call0, pos,
                   dir, ratio, t_max, rr_min);
}

// ---------------------------------------------------------------------------
// general walker (delta / ratio tracking), any number of plane / sphere shells

// sigma(w) for the walker, out of line: three call sites in the tracking
// loop share one copy in the instruction stream (config 3: 11.07 -> 10.56 ms).
// Walks are render / transmittance-estimate work: MUFU exp2 (kFast).
MF_COLD float proj_area_outlined(int kind, float ax, float ay, float az, V3 w) {
  return kind == kGGX ? proj_area_ggx(w, ax, ay) : proj_area_erf<true>(w, ax, ay, az);
}

struct WalkResult {
  int outcome;
  int prim;
  V3 pos;
  float weight;   // ratio tracking transmittance
  int steps;
  int violations;
  float travel;   // distance walked
};

// Extinction of prim j at x along dir (local frame), 0 outside its region.
template <bool kSphere = false>
MF_HD float prim_extinction(const SceneDev& sc, int j, V3 x, V3 dir, float lo_mult) {
  const PrimDev& p = sc.prims[j];
  const MediumK& m = sc.media[j];
  float f = prim_field<kSphere>(p, x);
  if (f < lo_mult * m.sigma || f > 3.0f * m.sigma) return 0.0f;
  Frame fr = frame_about(prim_normal<kSphere>(p, x));
  float sg = proj_area_outlined(m.kind, m.ax, m.ay, m.az, to_local(fr, dir));
  return mills<true>(f * m.inv_sigma) * m.inv_sigma * sg;
}

// ratio == false: delta tracking (collision mode); ratio == true: ratio
// tracking of the transmittance up to distance t_max (shadow rays).
// Random draws: Philox blocks (segment, call0 + k), 4 uniforms each.
// rr_min > 0 (ratio mode): Russian roulette on the ratio-tracking weight --
// below rr_min it survives with probability weight / rr_min at weight rr_min
// (unbiased: the expectation of every sample is unchanged), so a shadow ray
// through an optically thick shell stops once it can no longer contribute
// instead of tracking the whole shell.
#ifndef MF_WALK_OUTLINE
#define MF_WALK_OUTLINE 1
#endif
#if MF_WALK_OUTLINE && defined(__CUDACC__)
#define MF_WALK_FN __host__ __device__ __noinline__
#else
#define MF_WALK_FN MF_HD
#endif
// Out of line on the device: the flight and the shadow walks share one copy
// of the tracking loop in the instruction stream.
// Resumable walker state: walk_begin + walk_step (one iteration of the
// tracking loop) let a kernel interleave the steps of many walks; walk()
// runs one walk to the end.
struct WalkState {
  V3 p;          // current position
  V3 dir;
  float travel, t_max, weight, rr_min, lo_mult;
  uint32_t call;
  U4 bits;
  int avail;
  int steps, violations;
  int outcome, prim;
  V3 pos;        // final position
  bool ratio;
  bool tentative;   // stop at the first tentative collision (sample_collision)
};

MF_HD void walk_begin(WalkState& w, V3 pos, V3 dir, bool ratio, float t_max, uint32_t call0,
                      float rr_min, bool tentative = false) {
  w.p = pos;
  w.dir = dir;
  w.travel = 0.0f;
  w.t_max = t_max;
  w.weight = 1.0f;
  w.rr_min = rr_min;
  w.lo_mult = ratio ? -3.0f : -6.0f;
  w.call = call0;
  w.bits = U4{0, 0, 0, 0};
  w.avail = 0;
  w.steps = 0;
  w.violations = 0;
  w.outcome = kEscaped;
  w.prim = -1;
  w.pos = pos;
  w.ratio = ratio;
  w.tentative = tentative;
}

// One iteration of the delta / ratio tracking loop (transport.py:196-297);
// returns true when the walk has ended (w.outcome, w.pos, w.prim, w.weight).
// kOne: the scene is one sphere (BASELINE config 3) -- the primitive loops
// run once with their arrays in registers and the plane branches fold away;
// the arithmetic is the general walker's, so the results are identical.
template <bool kOne = false>
MF_HD bool walk_step(const SceneDev& sc, const PathRng& rng, uint32_t segment, WalkState& w) {
  const int n_prims = kOne ? 1 : sc.n_prims;
  // fields, band membership, gaps (transport.py:197-212)
  bool any_band = false;
  float gap_min = INFINITY;
  bool all_done = true;
  float maj = 0.0f;
  float cap = INFINITY;
  float fs[kMaxPrims];
  for (int j = 0; j < n_prims; ++j) {
    const PrimDev& p = sc.prims[j];
    const MediumK& m = sc.media[j];
    float f = prim_field<kOne>(p, w.p);
    fs[j] = f;
    float lo = w.lo_mult * m.sigma, hi = 3.0f * m.sigma;
    if (!w.ratio && f < lo) {
      w.outcome = kAbsorbed;
      w.pos = w.p;
      return true;
    }
    if (f >= lo && f <= hi) {
      any_band = true;
      // boxes bound f only by its Lipschitz constant: the reference's
      // sigma / 2 steps (transport.py:163) keep that band majorant tight
      cap = fminf(cap, (!kOne && p.shape == kShapeBox ? 0.5f : MF_STEP_FRAC) * m.sigma);
    } else {
      float g = level_distance<kOne>(p, w.p, w.dir, f > hi ? hi : lo);
      gap_min = fminf(gap_min, g);
      if (g < INFINITY) all_done = false;
      cap = fminf(cap, fmaxf(g, sc.min_skip));
    }
  }
  // majorant over the step [0, cap] (transport.py:226-231 with exact
  // geometry): min of f along the step (planes: linear; spheres: closest
  // approach) and, for media whose sigma(w) decreases with cos(theta), the
  // direction factor at the step start (cos(theta) grows along a chord)
  for (int j = 0; j < n_prims; ++j) {
    const PrimDev& p = sc.prims[j];
    const MediumK& m = sc.media[j];
    float f = fs[j];
    float lo = w.lo_mult * m.sigma, hi = 3.0f * m.sigma;
    if (!(f >= lo && f <= hi)) continue;
    float fmin, dirf;
    if (!kOne && p.shape == kShapePlane) {
      fmin = f + cap * fminf(w.dir.z, 0.0f);
      dirf = proj_area_outlined(m.kind, m.ax, m.ay, m.az, w.dir);
    } else if (!kOne && p.shape == kShapeBox) {
      // 1-Lipschitz field, curved frame: the moving band (transport.py:
      // 226-231) with the exact direction maximum
      fmin = f - cap;
      dirf = sc.mx[j].sig_max;
    } else {
      V3 oc = sub3(w.p, p.c);
      float b = dot3(oc, w.dir);
      float r2 = dot3(oc, oc);
      float ts = fminf(fmaxf(-b, 0.0f), cap);
      fmin = fsqrt(fmaxf(fmaf(ts, ts + 2.0f * b, r2), 0.0f)) - p.radius;
      if (sc.mx[j].area_monotone) {
        float c = b * frsqrt(fmaxf(r2, 1e-30f));
        c = fminf(fmaxf(c, -1.0f), 1.0f);
        dirf = proj_area_outlined(m.kind, m.ax, m.ay, m.az,
                                  v3(fsqrt(fmaxf(1.0f - c * c, 0.0f)), 0.0f, c)) * 1.0001f;
      } else {
        dirf = sc.mx[j].sig_max;
      }
    }
    float fb = fmaxf(fmin - 1e-6f * (1.0f + fabsf(f)), lo);
    maj += mills<true>(fb * m.inv_sigma) * m.inv_sigma * dirf;
  }
  if (!any_band) {
    if (all_done || w.travel + gap_min >= w.t_max) {
      w.outcome = kEscaped;
      w.pos = w.p;
      return true;
    }
    // float32: step past the level set by a few ulps of |w.p| so the next
    // iteration lands inside the band (transport.py:221 uses min_skip)
    float ulp = 4.8e-7f * (1.0f + fmaxf(fabsf(w.p.x), fmaxf(fabsf(w.p.y), fabsf(w.p.z))));
    float skip = fmaxf(gap_min, sc.min_skip) + ulp;
    w.p = fma3(w.dir, skip, w.p);
    w.travel += skip;
    return false;
  }
  if (w.avail == 0) {
    w.bits = rng_block(rng, segment, w.call++);
    w.avail = 4;
  }
  float u1 = u01(w.bits.x);
  w.bits.x = w.bits.y; w.bits.y = w.bits.z; w.bits.z = w.bits.w;
  --w.avail;
  float dt = maj > 0.0f ? -flog(u1) / maj : INFINITY;
  w.steps++;
  if (dt > cap) {
    w.p = fma3(w.dir, cap, w.p);
    w.travel += cap;
    if (w.ratio && w.travel >= w.t_max) {
      w.outcome = kEscaped;
      w.pos = w.p;
      return true;
    }
    return false;
  }
  w.p = fma3(w.dir, dt, w.p);
  w.travel += dt;
  if (w.ratio && w.travel >= w.t_max) {
    w.outcome = kEscaped;
    w.pos = w.p;
    return true;
  }
  float parts[kMaxPrims];
  float st = 0.0f;
  for (int j = 0; j < n_prims; ++j) {
    parts[j] = prim_extinction<kOne>(sc, j, w.p, w.dir, w.lo_mult);
    st += parts[j];
  }
  if (st > maj * 1.00001f) w.violations++;
  if (w.ratio) {
    w.weight *= fmaxf(1.0f - st / maj, 0.0f);
    if (w.weight < w.rr_min && w.weight > 0.0f) {
      if (w.avail == 0) {
        w.bits = rng_block(rng, segment, w.call++);
        w.avail = 4;
      }
      float ur = u01(w.bits.x);
      w.bits.x = w.bits.y; w.bits.y = w.bits.z; w.bits.z = w.bits.w;
      --w.avail;
      w.weight = ur * w.rr_min < w.weight ? w.rr_min : 0.0f;
    }
    if (!(w.weight > 0.0f)) {
      w.outcome = kEscaped;
      w.pos = w.p;
      return true;
    }
  } else {
    if (w.avail == 0) {
      w.bits = rng_block(rng, segment, w.call++);
      w.avail = 4;
    }
    float u2 = u01(w.bits.x);
    w.bits.x = w.bits.y; w.bits.y = w.bits.z; w.bits.z = w.bits.w;
    --w.avail;
    float pick = u2 * maj;
    if (pick < st) {
      // u2 * majorant doubles as the primitive selector (transport.py:276-279)
      float acc = 0.0f;
      int k = n_prims - 1;
      for (int j = 0; j < n_prims; ++j) {
        acc += parts[j];
        if (pick < acc) {
          k = j;
          break;
        }
      }
      w.outcome = kCollided;
      w.prim = k;
      w.pos = w.p;
      return true;
    }
    if (w.tentative) {
      // a null collision ends a sample_collision walk (transport.py:
      // 397-415): the primitive of the largest extinction part
      int k = 0;
      for (int j = 1; j < n_prims; ++j)
        if (parts[j] > parts[k]) k = j;
      w.outcome = kNullCollision;
      w.prim = k;
      w.pos = w.p;
      return true;
    }
  }
  return false;   // null collision: the walk goes on
}

template <bool kOne = false>
MF_WALK_FN WalkResult walk(const SceneDev& sc, PathRng rng, uint32_t segment,
                           uint32_t call0, V3 pos, V3 dir, bool ratio, float t_max,
                           float rr_min = 0.0f, bool tentative = false) {
  WalkState s;
  walk_begin(s, pos, dir, ratio, t_max, call0, rr_min, tentative);
  WalkResult w;
  for (int iter = 0; iter < 1000000; ++iter) {
    if (walk_step<kOne>(sc, rng, segment, s)) {
      w.outcome = s.outcome;
      w.prim = s.prim;
      w.pos = s.pos;
      w.weight = s.weight;
      w.steps = s.steps;
      w.violations = s.violations;
      w.travel = s.travel;
      return w;
    }
  }
  w.outcome = kAbsorbed;  // iteration cap: treated as lost (counted by the caller)
  w.prim = -1;
  w.pos = s.p;
  w.weight = s.weight;
  w.steps = -1;
  w.violations = s.violations;
  w.travel = s.travel;
  return w;
}

// ---------------------------------------------------------------------------
// single-sphere walker (BASELINE config 3): tracking against the tangent-line
// majorant.
//
// Along a ray, f(t) = |p + t d - c| - R is convex, so it lies above its
// tangent at the current point: f(t) >= f0 + g0 t, g0 = df/dt = cos of the
// ray against the radial direction.  The density rho(f) = mills(f/s)/s
// decreases in f, and for media whose sigma(w) depends on cos(theta) only and
// decreases with it (area_monotone; every isotropic-roughness medium) sigma
// along a chord is largest at its start, because cos(theta) = g grows along
// any straight line.  Hence for every t >= 0
//     mu(t) <= mubar(t) = Sigma(g0) rho(f0 + g0 t),
// and mubar has a closed-form optical depth,
//     int_0^t mubar = Sigma(g0) / g0 [log Phi((f0 + g0 t)/s) - log Phi(f0/s)],
// so the next tentative collision is sampled EXACTLY by inverting log Phi
// (the planar flight's math) instead of stepping a piecewise-constant
// majorant through the band.  The acceptance mu / mubar is ~1 (the chord
// hugs its tangent over the distance to a collision), so a flight or a
// shadow ray is one or two iterations instead of ~6 bounded steps; each
// iteration re-linearises at the null-collision point.  Where the tangent
// leaves the region before the sampled optical depth is reached, the walk
// moves to that edge and re-linearises (memorylessness).  Region rules as in
// walk(): collision walks live on [-6s, 3s] and absorb below; ratio walks
// integrate |f| <= 3s and cross the core below -3s as vacuum
// (transport.py:161-166).  The process is the reference's delta / ratio
// tracking (transport.py:226-285) with a tighter, non-constant majorant.
//
// Grazing tangents (|g0| < 1e-3, where (f1 - f0) / g0 cancels) fall back to
// a constant majorant over a sigma-long window.
constexpr float kSphereGmin = 1e-3f;

template <bool kFast = true, int kSpec = kSpecRuntime>
MF_HD float sphere_sigma_dir(const MediumK& m, float g) {
  // Sigma(cos theta): sigma(w) of a local direction with w.z = g
  if (kFast && m.area_q) return area_q_eval(m.area_q, g, m.ax, m.az);
  float sn = fsqrt(fmaxf(1.0f - g * g, 0.0f));
  if (kFast && spec_gen(kSpec)) return proj_area_erf_cold(v3(sn, 0.0f, g), m.ax, m.ay, m.az);
  return kSpec == kSpecRuntime && m.kind == kGGX ? proj_area_ggx(v3(sn, 0.0f, g), m.ax, m.ay)
                        : proj_area_erf<kFast>(v3(sn, 0.0f, g), m.ax, m.ay, m.az);
}

// The walker as a resumable object: step() runs one iteration of the loop
// (a vacuum skip, an edge move or a tentative collision) and returns true
// when the walk has ended (w is final).  Between two steps the whole state
// is (p, w.travel, w.weight, w.steps, the position in the random stream),
// so a walk can be parked and resumed (park_rng() / resume()): the path
// pool's W visits advance 32 walks together and park the unfinished ones.
// kSpec (see proj_area): the medium's NDF kind known at compile time
template <int kSpec = kSpecRuntime>
struct SphereWalker {
  const SceneDev& sc;
  PathRng rng;
  uint32_t segment;
  V3 p, dir;
  bool ratio;
  float t_max, rr_min;
  WalkResult w;
  uint32_t call;
  U4 bits;
  int avail;

  MF_HDM SphereWalker(const SceneDev& scene) : sc(scene) {}

  MF_HDM void begin(PathRng r, uint32_t seg, uint32_t call0, V3 pos, V3 d, bool ratio_walk,
                   float tmax, float rr) {
    rng = r;
    segment = seg;
    p = pos;
    dir = d;
    ratio = ratio_walk;
    t_max = tmax;
    rr_min = rr;
    w.outcome = kEscaped;
    w.prim = -1;
    w.pos = pos;
    w.weight = 1.0f;
    w.steps = 0;
    w.violations = 0;
    w.travel = 0.0f;
    call = call0;
    bits = U4{0, 0, 0, 0};
    avail = 0;
  }

  // the position in the random stream as one word (the calls of a walk are
  // consecutive from call0; a walk draws far fewer than 2^29 blocks)
  MF_HDM uint32_t park_rng(uint32_t call0) const { return ((call - call0) << 2) | (uint32_t)avail; }

  // continue a parked walk: begin()'s arguments plus the parked state
  MF_HDM void resume(PathRng r, uint32_t seg, uint32_t call0, V3 d, bool ratio_walk, float tmax,
                    float rr, V3 p_now, float travel, float weight, int steps, uint32_t rs) {
    begin(r, seg, call0, p_now, d, ratio_walk, tmax, rr);
    w.travel = travel;
    w.weight = weight;
    w.steps = steps;
    call = call0 + (rs >> 2);
    avail = (int)(rs & 3u);
    if (avail) {
      // the unread words of the block drawn last
      bits = rng_block(rng, segment, call - 1u);
      for (int k = avail; k < 4; ++k) {
        bits.x = bits.y;
        bits.y = bits.z;
        bits.z = bits.w;
      }
    }
  }

  MF_HDM float draw() {
    if (avail == 0) {
      bits = rng_block(rng, segment, call++);
      avail = 4;
    }
    float u = u01(bits.x);
    bits.x = bits.y;
    bits.y = bits.z;
    bits.z = bits.w;
    --avail;
    return u;
  }

  MF_HDM bool end(int outcome, V3 at) {
    w.outcome = outcome;
    w.pos = at;
    return true;
  }

  // one iteration; true when the walk has ended
  MF_HDM bool step() {
    const PrimDev& pr = sc.prims[0];
    const MediumK& m = sc.media[0];
    const MediumExtra& mx = sc.mx[0];
    const float s = m.sigma, is = m.inv_sigma;
    const float lo = ratio ? -3.0f * s : -6.0f * s, hi = 3.0f * s;
    const float l_lo = ratio ? mx.lphi_lo_rat : mx.lphi_lo_col, l_hi = mx.lphi_hi;
    // the tight bound, x 1.0001 for the float rounding of f and g along radial
    // chords.  Ratio walks use it too: a looser majorant keeps more weight per
    // tentative collision, but measured on config 3 (128^2 x 256 spp, 16
    // renders) the shadow estimator's variance is invisible in the image
    // (per-pixel variance 8.46e-5 at scale 1.0001, 1.5 and 2) while each
    // doubling of the scale doubles the iterations (5.4 / 9.4 / 12.5 per path,
    // 2.72 / 3.63 / 4.26 ms); the stepping walker: 12.4, 3.52 ms, 1.06e-4
    const float mscale = 1.0001f;
    V3 oc = sub3(p, pr.c);
    float r2 = dot3(oc, oc);
    float ir = frsqrt(fmaxf(r2, 1e-30f));
    float f = r2 * ir - pr.radius;
    float g = fminf(fmaxf(dot3(oc, dir) * ir, -1.0f), 1.0f);
    if (!ratio && f < lo)                // below the depth cap (transport.py:199-205)
      return end(kAbsorbed, p);
    if (f < lo || f > hi) {
      // vacuum: above the shell, or (ratio) the core; skip to the band
      float gd = level_distance<true>(pr, p, dir, f > hi ? hi : lo);
      if (!(gd < INFINITY) || w.travel + gd >= t_max) return end(kEscaped, p);
      float ulp = 4.8e-7f * (1.0f + fmaxf(fabsf(p.x), fmaxf(fabsf(p.y), fabsf(p.z))));
      float skip = fmaxf(gd, sc.min_skip) + ulp;
      p = fma3(dir, skip, p);
      w.travel += skip;
      return false;
    }
    // majorant of the chord from here: Sigma at its start times rho of the
    // tangent line (the 1.0001 absorbs float rounding of f, g along radial
    // chords, where the bound is tight)
    float sig0 = (mx.area_monotone ? sphere_sigma_dir<true, kSpec>(m, g) : mx.sig_max) * mscale;
    float tau = -flog(draw());
    w.steps++;
    float t1, mubar1;
    bool edge = false;
    if (fabsf(g) >= kSphereGmin) {
      float v0 = f * is;
      float l0 = log_ndtr(v0);
      float l1 = fmaf(g * tau, frcp(sig0), l0);
      if (g > 0.0f && !(l1 < l_hi)) {
        // the tangent leaves the band first; f grows from here on (past the
        // closest approach), so the ray leaves the shell for good
        return end(kEscaped, p);
      }
      if (g < 0.0f && !(l1 >= l_lo)) {
        // the tangent reaches the region's lower edge first: go there and
        // re-linearise (the true f there is >= the edge); a few ulps past it
        // so a ray sitting on the edge moves on into the core
        float ulp = 4.8e-7f * (1.0f + fmaxf(fabsf(p.x), fmaxf(fabsf(p.y), fabsf(p.z))));
        t1 = fmaxf((lo - f) / g, 0.0f) + ulp;
        edge = true;
        mubar1 = 0.0f;
      } else {
        float v1 = inv_log_ndtr(l1);
        t1 = fmaxf(s * (v1 - v0) / g, 0.0f);
        // rho at the tangent point: phi(v1) / Phi(v1), Phi(v1) = e^{l1}
        mubar1 = sig0 * is * kInvSqrt2Pi * exp_t<true>(fmaf(-0.5f * v1, v1, -l1));
      }
    } else {
      // grazing: constant majorant over a window of length s
      float fb = fmaxf(f + fminf(g, 0.0f) * s - 1e-6f * (1.0f + fabsf(f)), lo);
      float mub = sig0 * mills<true>(fb * is) * is;
      float dt = tau / mub;
      if (dt > s) {
        t1 = s;
        edge = true;
        mubar1 = 0.0f;
      } else {
        t1 = dt;
        mubar1 = mub;
      }
    }
    if (w.travel + t1 >= t_max) {         // reached the light (ratio walks)
      V3 at = fma3(dir, t_max - w.travel, p);
      w.travel = t_max;
      return end(kEscaped, at);
    }
    p = fma3(dir, t1, p);
    w.travel += t1;
    if (edge) return false;
    // the true extinction at the tentative point
    V3 oc1 = sub3(p, pr.c);
    float r21 = dot3(oc1, oc1);
    float ir1 = frsqrt(fmaxf(r21, 1e-30f));
    float f1 = r21 * ir1 - pr.radius;
    float g1 = fminf(fmaxf(dot3(oc1, dir) * ir1, -1.0f), 1.0f);
    float mu = 0.0f;
    if (f1 >= lo && f1 <= hi) {
      float sg = mx.area_monotone ? sphere_sigma_dir<true, kSpec>(m, g1)
                                  : proj_area_outlined(m.kind, m.ax, m.ay, m.az,
                                                       to_local(frame_about(mul3(oc1, ir1)), dir));
      mu = mills<true>(f1 * is) * is * sg;
    }
    if (mu > mubar1 * 1.00001f) w.violations++;
    if (ratio) {
      w.weight *= fmaxf(1.0f - mu / mubar1, 0.0f);
      if (w.weight < rr_min && w.weight > 0.0f) {
        float ur = draw();
        w.weight = ur * rr_min < w.weight ? rr_min : 0.0f;
      }
      if (!(w.weight > 0.0f)) return end(kEscaped, p);
    } else if (draw() * mubar1 < mu) {
      w.prim = 0;
      return end(kCollided, p);
    }
    return false;
  }

  // iteration cap reached (counted by the caller)
  MF_HDM void cap() {
    w.outcome = kAbsorbed;
    w.pos = p;
    w.steps = -1;
  }
};

template <int kSpec = kSpecRuntime>
MF_WALK_FN WalkResult sphere_walk(const SceneDev& sc, PathRng rng, uint32_t segment,
                                  uint32_t call0, V3 pos, V3 dir, bool ratio, float t_max,
                                  float rr_min = 0.0f) {
  SphereWalker<kSpec> W(sc);
  W.begin(rng, segment, call0, pos, dir, ratio, t_max, rr_min);
  for (int iter = 0; iter < 1000000; ++iter) {
    if (W.step()) return W.w;
  }
  W.cap();
  return W.w;
}

}  // namespace mf
