// mf_scene_build.h -- host-side flattening of mf_scene into the device
// SceneDev (shared by the CUDA library and the host test shim).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "mf_prepare.h"
#include "mf_transport.cuh"

namespace mf {

inline double log_ndtr_host(double u) { return std::log(0.5 * std::erfc(-u / std::sqrt(2.0))); }

// max over directions of sigma(w) in the local frame (exact majorant
// factor; replaces the direction-free bound of ndf.py:189-194)
// sigma(w) depends on cos(theta) only (ax == ay) and is non-increasing in
// it: then the direction factor of a chord majorant is its start value
inline int area_monotone_host(const MediumK& m) {
  if (m.ax != m.ay) return 0;
  float prev = INFINITY;
  for (int i = 0; i <= 4096; ++i) {
    float c = -1.0f + 2.0f * (float)i / 4096.0f;
    float v = proj_area(m, v3(std::sqrt(std::max(0.0f, 1.0f - c * c)), 0.0f, c));
    if (v > prev * (1.0f + 1e-6f)) return 0;
    prev = v;
  }
  return 1;
}

inline double sigma_max_host(const MediumK& m) {
  double best = 0.0;
  const int nt = 2048, np = 16;
  for (int i = 0; i <= nt; ++i) {
    double th = M_PI * i / nt;
    for (int j = 0; j <= np; ++j) {
      double ph = 0.5 * M_PI * j / np;
      V3 w = v3((float)(std::sin(th) * std::cos(ph)), (float)(std::sin(th) * std::sin(ph)),
                (float)std::cos(th));
      best = std::max(best, (double)proj_area(m, w));
    }
  }
  // the grid max of a smooth function under-estimates by O(h^2); pad
  // generously (a majorant only needs to be an upper bound)
  return best * 1.01 + 1e-6;
}

// (sig_max, area_monotone) of a roughness triple, memoised: the dense
// direction scans above cost milliseconds and scenes are rebuilt per call
inline void direction_factors(const MediumK& m, float* sig_max, int* monotone) {
  static std::mutex mu;
  static std::map<std::tuple<int, float, float, float>, std::pair<float, int>> memo;
  auto key = std::make_tuple(m.kind, m.ax, m.ay, m.az);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = memo.find(key);
    if (it != memo.end()) {
      *sig_max = it->second.first;
      *monotone = it->second.second;
      return;
    }
  }
  float sm = (float)sigma_max_host(m);
  int mono = area_monotone_host(m);
  std::lock_guard<std::mutex> lk(mu);
  if (memo.size() > 4096) memo.clear();
  memo[key] = std::make_pair(sm, mono);
  *sig_max = sm;
  *monotone = mono;
}

// sigma(w) (ndf.py:156-164) in float64 of an azimuthally symmetric erf-family
// medium at w.z = z: sigma = s/2 e^{-a^2} ierfcx(|a|) (+ |z| for z < 0),
// s^2 = ax^2 (1 - z^2) + az^2 z^2, a = z / s, ierfcx(x) = 1/sqrt(pi) -
// x erfcx(x); erfcx from erfc in float64 (|a| <= 26 keeps e^{a^2} erfc(a)
// finite; beyond, the asymptotic series)
inline double proj_area_iso_f64(double z, double ax, double az) {
  double s = std::sqrt(std::max(ax * ax * (1.0 - z * z) + az * az * z * z, 0.0));
  if (!(s > 0.0)) return std::max(-z, 0.0);
  double a = z / s, x = std::fabs(a);
  double ex;
  if (x < 26.0) {
    ex = std::exp(x * x) * std::erfc(x);
  } else {
    double r = 1.0 / (2.0 * x * x);
    ex = (1.0 - r * (1.0 - 3.0 * r * (1.0 - 5.0 * r))) / (x * 1.7724538509055160273);
  }
  double v = 0.5 * s * std::exp(-x * x) * (0.56418958354775628695 - x * ex);
  return a >= 0.0 ? v : v - z;
}

// The render kernels' table of sigma(w) for an azimuthally symmetric
// GENERALIZED medium (ax == ay, az > 0: sigma depends on z = w.z alone):
// per piece i of kAreaQN over z in [-1, 1], the cubic through
// R(z) = log2 sigma(z) + [z > 0] a(z)^2 log2(e) at t = 0, 1/3, 2/3, 1 of the
// piece.  Dividing out the Gaussian factor e^{-a^2} of the upper
// hemisphere (which area_q_eval puts back exactly) leaves a smooth R; the
// table is kept only when area_q_eval reproduces the float64 sigma to
// 1e-6 + 1.2e-7 (a^2 + |d ln sigma / dz|) relative -- the fp32 rounding of
// the exponent (the formula's MUFU exp2 path has it as well) and of z
// itself -- at eight further points per piece, else false (the kernels
// use the formula).
inline bool area_q_build(const MediumK& m, float4* q) {
  if (m.kind != kGeneralized || m.ax != m.ay || !(m.az > 0.0f)) return false;
  const double ax = m.ax, az = m.az;
  auto a2 = [&](double z) {
    double s2 = ax * ax * (1.0 - z * z) + az * az * z * z;
    return z * z / s2;
  };
  auto R = [&](double z) {
    double v = proj_area_iso_f64(z, ax, az);
    return (v > 0.0 && std::isfinite(v)) ? std::log2(v) + (z > 0.0 ? a2(z) * 1.4426950408889634 : 0.0)
                                         : NAN;
  };
  const double h = 2.0 / kAreaQN;
  for (int i = 0; i < kAreaQN; ++i) {
    double z0 = -1.0 + h * i;
    double l[4];
    for (int k = 0; k < 4; ++k) {
      l[k] = R(k == 3 ? -1.0 + h * (i + 1) : z0 + h * k / 3.0);
      if (!std::isfinite(l[k])) return false;
    }
    // monomial coefficients of the cubic through (0, l0) (1/3, l1) (2/3, l2) (1, l3)
    double c0 = l[0];
    double c1 = (-11.0 * l[0] + 18.0 * l[1] - 9.0 * l[2] + 2.0 * l[3]) / 2.0;
    double c2 = (18.0 * l[0] - 45.0 * l[1] + 36.0 * l[2] - 9.0 * l[3]) / 2.0;
    double c3 = (-9.0 * l[0] + 27.0 * l[1] - 27.0 * l[2] + 9.0 * l[3]) / 2.0;
    q[i] = float4{(float)c0, (float)c1, (float)c2, (float)c3};
  }
  // check the device evaluation (host build of area_q_eval) at 8 points per piece
  for (int i = 0; i < kAreaQN; ++i) {
    for (int k = 1; k <= 8; ++k) {
      float z = (float)(-1.0 + h * (i + (k - 0.5) / 8.0));
      double ex = proj_area_iso_f64(z, ax, az);
      double got = area_q_eval(q, z, m.ax, m.az);
      // + the conditioning: sigma's response to a rounding of z itself
      double dz = 1e-6;
      double dl = std::fabs(std::log(proj_area_iso_f64(std::min(1.0, z + dz), ax, az) /
                                     proj_area_iso_f64(std::max(-1.0, z - dz), ax, az))) / (2.0 * dz);
      double tol = 1e-6 + 1.2e-7 * (z > 0.0f ? a2(z) : 0.0) + 1.2e-7 * dl;
      if (!(std::fabs(got / ex - 1.0) <= tol)) return false;
    }
  }
  return true;
}

inline int build_scene(const mf_scene& in, SceneDev* out, std::string* err) {
  if (in.n_prims < 0 || in.n_prims > MF_MAX_PRIMS)
    return (*err = std::string("n_prims out of range"), MF_ERR_PARAM);
  if (in.n_media < 0 || in.n_media > MF_MAX_MEDIA)
    return (*err = std::string("n_media out of range"), MF_ERR_PARAM);
  SceneDev sc;
  std::memset(&sc, 0, sizeof(sc));
  sc.n_prims = in.n_prims;
  double min_sigma = INFINITY;
  for (int j = 0; j < in.n_prims; ++j) {
    PrimK pk;
    int rc = prepare_primitive(in.prims[j], in.n_media, &pk, err);
    if (rc) return rc;
    MediumK mk;
    rc = prepare_medium(in.media[pk.medium], &mk, err);
    if (rc) return rc;
    sc.prims[j].shape = pk.shape;
    sc.prims[j].medium = j;
    sc.prims[j].z0 = pk.z0;
    sc.prims[j].c = v3(pk.cx, pk.cy, pk.cz);
    sc.prims[j].radius = pk.radius;
    sc.prims[j].half = v3(pk.hx, pk.hy, pk.hz);
    sc.media[j] = mk;
    double s = in.media[pk.medium].sigma;
    min_sigma = std::min(min_sigma, s);
    // exact majorant factor, needed only by the tracking walker (curved shells)
    bool planar_only = in.n_prims == 1 && in.prims[0].shape == MF_SHAPE_PLANE;
    if (planar_only) {
      sc.mx[j].sig_max = mk.sig_bound;
      sc.mx[j].area_monotone = 0;
    } else {
      direction_factors(mk, &sc.mx[j].sig_max, &sc.mx[j].area_monotone);
    }
    sc.mx[j].lphi_hi = (float)log_ndtr_host(3.0);
    sc.mx[j].lphi_lo_col = (float)log_ndtr_host(-6.0);
    sc.mx[j].lphi_lo_rat = (float)log_ndtr_host(-3.0);
  }
  sc.min_skip = std::isfinite(min_sigma) ? (float)(1e-7 * min_sigma) : 1e-7f;
  sc.single_plane = (in.n_prims == 1 && in.prims[0].shape == MF_SHAPE_PLANE) ? 1 : 0;
  sc.has_grid = 0;
  // grid field (BASELINE config 5): exactly one MF_SHAPE_GRID primitive
  int n_grid = 0;
  for (int j = 0; j < in.n_prims; ++j) n_grid += in.prims[j].shape == MF_SHAPE_GRID;
  if (n_grid || in.has_grid) {
    if (!in.has_grid || n_grid != 1 || in.n_prims != 1)
      return (*err = std::string("a grid field must be the scene's only primitive"), MF_ERR_UNSUPPORTED);
    const mf_grid_field& g = in.grid;
    if (!g.d_sdf || !g.d_sigma || !g.d_majorant || g.n_sdf < 2 || g.n_sigma < 2 || g.n_maj < 1)
      return (*err = std::string("grid field arrays / sizes invalid"), MF_ERR_PARAM);
    if (!(g.l_xy > 0.0) || !(g.l_z > 0.0))
      return (*err = std::string("grid correlation lengths must be > 0"), MF_ERR_PARAM);
    GridDev gd;
    gd.sdf = g.d_sdf;
    gd.sig = g.d_sigma;
    gd.maj = g.d_majorant;
    gd.n_sdf = g.n_sdf;
    gd.n_sig = g.n_sigma;
    gd.n_maj = g.n_maj;
    gd.bmin = v3((float)g.bmin[0], (float)g.bmin[1], (float)g.bmin[2]);
    gd.bmax = v3((float)g.bmax[0], (float)g.bmax[1], (float)g.bmax[2]);
    double ext[3];
    for (int a = 0; a < 3; ++a) {
      ext[a] = g.bmax[a] - g.bmin[a];
      if (!(ext[a] > 0.0)) return (*err = std::string("grid bounds are empty"), MF_ERR_PARAM);
    }
    gd.inv_h_sdf = v3((float)((g.n_sdf - 1) / ext[0]), (float)((g.n_sdf - 1) / ext[1]),
                      (float)((g.n_sdf - 1) / ext[2]));
    gd.inv_h_sig = v3((float)((g.n_sigma - 1) / ext[0]), (float)((g.n_sigma - 1) / ext[1]),
                      (float)((g.n_sigma - 1) / ext[2]));
    gd.inv_h_maj = v3((float)(g.n_maj / ext[0]), (float)(g.n_maj / ext[1]),
                      (float)(g.n_maj / ext[2]));
    gd.h_maj = v3((float)(ext[0] / g.n_maj), (float)(ext[1] / g.n_maj), (float)(ext[2] / g.n_maj));
    gd.k_xy = (float)(std::sqrt(2.0) / g.l_xy);
    gd.k_z = (float)(std::sqrt(2.0) / g.l_z);
    sc.has_grid = 1;
    sc.grid = gd;
    sc.single_plane = 0;
    sc.min_skip = 1e-8f;
  }

  // camera basis (scene.py:30-41), in double
  const mf_camera& cam = in.camera;
  if (cam.width < 1 || cam.height < 1) return (*err = std::string("camera size must be >= 1"), MF_ERR_PARAM);
  double f[3] = {cam.look_at[0] - cam.position[0], cam.look_at[1] - cam.position[1],
                 cam.look_at[2] - cam.position[2]};
  double fn = std::sqrt(f[0] * f[0] + f[1] * f[1] + f[2] * f[2]);
  if (!(fn > 0.0)) return (*err = std::string("camera look_at equals position"), MF_ERR_PARAM);
  for (double& v : f) v /= fn;
  double up[3] = {0.0, 0.0, 1.0};
  if (std::fabs(f[2]) > 0.999) {
    up[1] = 1.0;
    up[2] = 0.0;
  }
  double r[3] = {f[1] * up[2] - f[2] * up[1], f[2] * up[0] - f[0] * up[2],
                 f[0] * up[1] - f[1] * up[0]};
  double rn = std::sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  for (double& v : r) v /= rn;
  double tu[3] = {r[1] * f[2] - r[2] * f[1], r[2] * f[0] - r[0] * f[2], r[0] * f[1] - r[1] * f[0]};
  sc.ortho = cam.ortho;
  sc.width = cam.width;
  sc.height = cam.height;
  sc.cam_pos = v3((float)cam.position[0], (float)cam.position[1], (float)cam.position[2]);
  sc.cam_fwd = v3((float)f[0], (float)f[1], (float)f[2]);
  sc.cam_right = v3((float)r[0], (float)r[1], (float)r[2]);
  sc.cam_up = v3((float)tu[0], (float)tu[1], (float)tu[2]);
  double hh = cam.ortho ? 0.5 * cam.film_height : std::tan(0.5 * cam.fov_deg * M_PI / 180.0);
  sc.half_h = (float)hh;
  sc.half_w = (float)(hh * cam.width / cam.height);
  sc.env = v3((float)in.env[0], (float)in.env[1], (float)in.env[2]);
  sc.env_map = in.d_env_map;
  sc.env_w = in.env_width;
  sc.env_h = in.env_height;
  if (sc.env_map && (sc.env_w < 1 || sc.env_h < 1))
    return (*err = std::string("environment map size must be >= 1 x 1"), MF_ERR_PARAM);
  sc.has_sun = in.has_sun;
  if (in.has_sun) {
    double d[3] = {in.sun_dir[0], in.sun_dir[1], in.sun_dir[2]};
    double dn = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    if (!(dn > 0.0)) return (*err = std::string("sun direction must be nonzero"), MF_ERR_PARAM);
    sc.sun_to = v3((float)(-d[0] / dn), (float)(-d[1] / dn), (float)(-d[2] / dn));
    sc.sun_L = v3((float)in.sun_radiance[0], (float)in.sun_radiance[1], (float)in.sun_radiance[2]);
    if (sc.n_prims > 0) sc.sun_sig = proj_area(sc.media[0], sc.sun_to);
    if (sc.n_prims > 0) {
      double c = std::fabs((double)sc.sun_to.z);
      sc.sun_graze = c < 1e-6 ? 1 : 0;
      sc.sun_k2 = sc.sun_graze ? 0.0f : (float)(-(double)sc.sun_sig / c * 1.4426950408889634);
      sc.sun_lb = sc.sun_to.z > 0.0f ? sc.mx[0].lphi_hi : sc.mx[0].lphi_lo_rat;
    }
  }
  sc.has_point = in.has_point;
  if (in.has_point) {
    sc.point_pos = v3((float)in.point_pos[0], (float)in.point_pos[1], (float)in.point_pos[2]);
    sc.point_I = v3((float)in.point_intensity[0], (float)in.point_intensity[1],
                    (float)in.point_intensity[2]);
    // the light must sit outside every shell (its shadow walk is not clipped
    // at shells containing it)
    for (int j = 0; j < in.n_prims; ++j) {
      const PrimDev& p = sc.prims[j];
      V3 lp = sc.point_pos;
      float fv = prim_field(p, lp);
      if (!(fv > 3.0f * sc.media[j].sigma))
        return (*err = std::string("point light inside a shell is not supported"), MF_ERR_UNSUPPORTED);
    }
  }
  // grey scene: Fresnel one or a grey albedo, and grey lights / environment;
  // then all three colour channels of a path carry the same value
  auto grey = [](V3 v) { return v.x == v.y && v.y == v.z; };
  sc.mono = 1;
  for (int j = 0; j < sc.n_prims; ++j) {
    const MediumK& m = sc.media[j];
    bool g = m.fresnel == kOne ||
             (m.fresnel == kAlbedo && m.albedo[0] == m.albedo[1] && m.albedo[1] == m.albedo[2]);
    if (!g) sc.mono = 0;
  }
  if (!grey(sc.env) || (sc.has_sun && !grey(sc.sun_L)) || (sc.has_point && !grey(sc.point_I)) ||
      sc.env_map)
    sc.mono = 0;
  *out = sc;
  return MF_OK;
}


}  // namespace mf
