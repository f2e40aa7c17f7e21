// mf_query.cuh -- one coefficient query (BASELINE config 1), shared by the
// CUDA kernel and the host test shim so both run the identical code.
//
// Per query (reference, all float64):
//   sigma_t = extinction(wo, f, medium, frame)          medium.py:91-95
//   phase   = phase_eval(wo, wi, medium, frame)         medium.py:158-178
//   pdf     = density of wi under _phase_sample_u       ndf.py:397-405, medium.py:186-189
//   (ws, pdf_s, w_s) = _phase_sample_u(wo_l, m, u)      medium.py:181-193
// Two uniforms per query feed the three-uniform sampler as
// (u1, u1', u2), u1' = u1/R or (u1-R)/(1-R).
#pragma once

#include "mf_math.cuh"

namespace mf {

struct FieldPoint {
  float f;
  V3 n;
};

// f and the frame normal of a plane (z = z0) or sphere field at p
// (sdf.py:18-52; the gradient of a sphere at its centre is taken as +z)
MF_HD FieldPoint field_at(int shape, float z0, V3 c, float radius, V3 p) {
  FieldPoint o;
  if (shape == 0) {
    o.f = p.z - z0;
    o.n = v3(0.0f, 0.0f, 1.0f);
  } else {
    V3 d = sub3(p, c);
    float r2 = dot3(d, d);
    if (r2 > 0.0f) {
      float ir = frsqrt(r2);
      o.f = r2 * ir - radius;
      o.n = mul3(d, ir);
    } else {
      o.f = -radius;
      o.n = v3(0.0f, 0.0f, 1.0f);
    }
  }
  return o;
}

MF_HD float div_rn(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fdiv_rn(a, b);
#else
  return a / b;
#endif
}

// the remap on the render path, by the reciprocals prepared on the host
// (identical to the correctly rounded quotients when R and 1 - R are powers
// of two, e.g. R = 1/2)
MF_HD float remap_branch_uniform_render(float u1, const MediumK& m) {
  return u1 < m.mix ? u1 * m.inv_mix : (u1 - m.mix) * m.inv_1m_mix;
}

// u1' of the two-uniform convention, correctly rounded so the host test can
// reproduce it bit-for-bit in numpy float32: the reciprocal products when
// they are exact (m.remap_exact), else IEEE divisions
MF_HD float remap_branch_uniform(float u1, const MediumK& m) {
  if (m.remap_exact) return remap_branch_uniform_render(u1, m);
  return u1 < m.mix ? div_rn(u1, m.mix) : div_rn(u1 - m.mix, 1.0f - m.mix);
}

struct QueryResult {
  float sigma_t;
  V3 phase;
  float pdf;
  V3 ws;
  float pdf_s;
  V3 w;
  int flags;
  int iters;
};

MF_HD QueryResult query_local(const MediumK& m, float f, const Frame& fr, V3 wo, V3 wi, float u1,
                              float u2, unsigned mask = 0xffffffffu);

MF_HD QueryResult query_point(const MediumK& m, int shape, float z0, V3 c, float radius, V3 p,
                              V3 wo, V3 wi, float u1, float u2) {
  FieldPoint fp = field_at(shape, z0, c, radius, p);
  return query_local(m, fp.f, frame_about(fp.n), wo, wi, u1, u2);
}

MF_HD QueryResult query_local(const MediumK& m, float f, const Frame& fr, V3 wo, V3 wi, float u1,
                              float u2, unsigned mask) {
  QueryResult q;
  // caller uniforms are clamped into the open interval: u = 0 or 1 (e.g. a
  // float64 draw rounded to float32) make the inverse CDFs infinite, also in
  // the reference (ndf.py:353 erfinv(+-1))
  u1 = fminf(fmaxf(u1, 5.9604644775390625e-08f), 0.99999994f);
  u2 = fminf(fmaxf(u2, 5.9604644775390625e-08f), 0.99999994f);
  V3 wol = to_local(fr, wo);
  V3 wil = to_local(fr, wi);
  float sig_o = proj_area(m, wol);
  q.sigma_t = mills(f * m.inv_sigma) * m.inv_sigma * sig_o;
  float sig_b = proj_area_erf(wol, m.ax, m.ay, 0.0f);
  q.flags = 0;
  q.iters = 0;
  // the reference raises DegenerateVisibilityError where sigma(wo) < 1e-12
  // (ndf.py:312-313): flagged, outputs zero.  Evaluated branch-free so the
  // sampler's warp mask stays the full set of lanes that entered.
  bool degenerate = !(sig_o >= 1e-12f);
  float sig_safe = degenerate ? 1.0f : sig_o;
  q.phase = phase_eval(m, wol, wil, sig_safe);
  q.pdf = phase_pdf(m, wol, wil, sig_b);
  float uu = remap_branch_uniform(u1, m);
  PhaseSample s = phase_sample<true>(m, wol, sig_safe, sig_b, u1, uu, u2, mask);
  q.ws = to_world(fr, s.wi);
  q.pdf_s = s.pdf;
  q.w = s.weight;
  q.iters = s.iters;
  if (degenerate) {
    q.flags = 1;
    q.phase = v3(0.0f, 0.0f, 0.0f);
    q.pdf = 0.0f;
    q.ws = wo;
    q.pdf_s = 0.0f;
    q.w = v3(0.0f, 0.0f, 0.0f);
  }
  return q;
}

}  // namespace mf
