// mf_prepare.h -- host-side validation of the C-ABI scene structs and
// derivation (in double) of the per-medium constants the kernels use.
// Validation mirrors the reference constructors:
//   MacrofacetMedium.__post_init__  medium.py:53-63
//   RoughnessTriple.__post_init__   ndf.py:60-66
//   Sphere.__post_init__            sdf.py:41-44
#pragma once

#include <cmath>
#include <string>

#include "../../include/macrofacet_b200.h"
#include "mf_math.cuh"

namespace mf {

// Direction-free projected-area bound (ndf.py:189-194).
inline double reference_sigma_bound(int kind, double ax, double ay, double az) {
  if (kind == MF_KIND_GGX) return 0.5 * (std::fmax(1.0, std::fmax(ax, ay)) + 1.0);
  double zz = kind == MF_KIND_GENERALIZED ? az : 0.0;
  return std::sqrt(ax * ax + ay * ay + zz * zz) / (2.0 * 1.7724538509055160273) + 1.0;
}

inline bool finite_pos(double v) { return std::isfinite(v) && v > 0.0; }

// Returns MF_OK or MF_ERR_PARAM with *err set.
inline int prepare_medium(const mf_medium& in, MediumK* out, std::string* err) {
  if (!finite_pos(in.sigma)) {
    *err = "sigma must be finite and > 0, got " + std::to_string(in.sigma);
    return MF_ERR_PARAM;
  }
  if (!(in.mix_ratio >= 0.0 && in.mix_ratio <= 1.0)) {
    *err = "mix_ratio must lie in [0, 1], got " + std::to_string(in.mix_ratio);
    return MF_ERR_PARAM;
  }
  if (!finite_pos(in.ax) || !finite_pos(in.ay)) {
    *err = "ax and ay must be finite and > 0";
    return MF_ERR_PARAM;
  }
  if (in.kind != MF_KIND_BECKMANN && in.kind != MF_KIND_GGX && in.kind != MF_KIND_GENERALIZED) {
    *err = "unknown NDF kind " + std::to_string(in.kind);
    return MF_ERR_PARAM;
  }
  double az = in.kind == MF_KIND_GENERALIZED ? in.az : 0.0;
  if (in.kind == MF_KIND_GENERALIZED && !finite_pos(az)) {
    *err = "GENERALIZED medium requires az > 0";
    return MF_ERR_PARAM;
  }
  if (in.fresnel != MF_FRESNEL_CONDUCTOR && in.fresnel != MF_FRESNEL_ONE &&
      in.fresnel != MF_FRESNEL_ALBEDO) {
    *err = "unknown fresnel mode " + std::to_string(in.fresnel);
    return MF_ERR_PARAM;
  }
  MediumK m{};
  m.kind = in.kind;
  m.fresnel = in.fresnel;
  m.ax = (float)in.ax;
  m.ay = (float)in.ay;
  m.az = (float)az;
  m.sigma = (float)in.sigma;
  m.inv_sigma = (float)(1.0 / in.sigma);
  m.mix = (float)in.mix_ratio;
  m.inv_mix = in.mix_ratio > 0.0 ? (float)(1.0 / in.mix_ratio) : 0.0f;
  m.inv_1m_mix = in.mix_ratio < 1.0 ? (float)(1.0 / (1.0 - in.mix_ratio)) : 0.0f;
  {
    auto pow2 = [](double x) {   // x > 0 an exact power of two in float32
      int e;
      float f = (float)x;
      return x > 0.0 && (double)f == x && std::frexp(f, &e) == 0.5f;
    };
    m.remap_exact = (pow2(in.mix_ratio) || in.mix_ratio == 0.0) &&
                    (pow2(1.0 - in.mix_ratio) || in.mix_ratio == 1.0);
  }
  m.inv_ax = (float)(1.0 / in.ax);
  m.inv_ay = (float)(1.0 / in.ay);
  const double pi = 3.14159265358979323846;
  if (in.kind == MF_KIND_GENERALIZED) {
    double c = 1.0 / (az * az);
    m.inv_az2 = (float)c;
    m.exp_neg_c = (float)std::exp(-c);
    m.d_norm = (float)(1.0 / (std::pow(pi, 1.5) * in.ax * in.ay * az));
  }
  m.beck_norm = (float)(1.0 / (pi * in.ax * in.ay));
  m.sig_bound = (float)reference_sigma_bound(in.kind, in.ax, in.ay, az);
  for (int c = 0; c < 3; ++c) {
    m.eta[c] = (float)in.eta[c];
    m.k[c] = (float)in.k[c];
    m.albedo[c] = (float)in.albedo[c];
  }
  *out = m;
  return MF_OK;
}

// Geometry of one primitive in the form the kernels read.
struct PrimK {
  int shape;
  int medium;
  float z0;
  float cx, cy, cz, radius;
  float hx, hy, hz;
};

inline int prepare_primitive(const mf_primitive& in, int n_media, PrimK* out, std::string* err) {
  if (in.shape != MF_SHAPE_PLANE && in.shape != MF_SHAPE_SPHERE && in.shape != MF_SHAPE_GRID &&
      in.shape != MF_SHAPE_BOX) {
    *err = "unsupported primitive shape " + std::to_string(in.shape);
    return MF_ERR_UNSUPPORTED;
  }
  if (in.medium < 0 || in.medium >= n_media) {
    *err = "primitive medium index out of range";
    return MF_ERR_PARAM;
  }
  if (in.shape == MF_SHAPE_SPHERE && !finite_pos(in.radius)) {
    *err = "sphere radius must be > 0, got " + std::to_string(in.radius);
    return MF_ERR_PARAM;
  }
  if (in.shape == MF_SHAPE_BOX &&
      !(finite_pos(in.half_extents[0]) && finite_pos(in.half_extents[1]) &&
        finite_pos(in.half_extents[2]))) {
    *err = "box half extents must be > 0";   // sdf.py:61-62
    return MF_ERR_PARAM;
  }
  PrimK p{};
  p.shape = in.shape;
  p.hx = (float)in.half_extents[0];
  p.hy = (float)in.half_extents[1];
  p.hz = (float)in.half_extents[2];
  p.medium = in.medium;
  p.z0 = (float)in.z0;
  p.cx = (float)in.center[0];
  p.cy = (float)in.center[1];
  p.cz = (float)in.center[2];
  p.radius = (float)in.radius;
  *out = p;
  return MF_OK;
}

}  // namespace mf
