// mf_kernels.cu -- sm_100a kernels of the macrofacet hot path and the
// extern "C" boundary declared in include/macrofacet_b200.h.
//
// Kernels
//   query_kernel      config-1 coefficient queries (medium.py:91-207), SoA
//   path_kernel       persistent megakernel: raygen + free flight + NEE +
//                     phase sampling + RR for every path of a pass; warps
//                     refill dead lanes from a global work counter each
//                     segment (warp-level compaction / path regeneration),
//                     so path state never leaves registers
//                     (render.py:32-108, transport.py:144-297)
//   finalize_kernel   per-pixel 64-bit fixed-point sums (accumulated by the
//                     render kernels themselves, accumulate_fx) -> the
//                     caller's fp32 buffer (render.py:150,165-166)
//   pool_kernel       shared-memory path pool for single-plane scenes (configs
//                     2, 4): R / B / H visits over per-warp slot rings, every
//                     visit at full warp width
//   curved_pool_kernel the same pool for one sphere (config 3; grid fields with two lights)
//   grid_pool_kernel  the pool with pooled walks for a grid field (config 5): W visits
//                     batch DDA steps and tentative collisions, walks park and resume
//   ratio_kernel      ratio-tracking transmittance samples (transport.py:300-313)
//   walk_kernel       walk / sample_collision of caller rays (transport.py:144-416)
//   curve_kernel      closed-form curves of one medium (cli.py:132-175)
//   slope_table_kernel, grid_majorant_kernel, grid_skip_kernel, env_max_kernel
//                     per-device / per-grid / per-render set-up
//   gp::*             the GP-realisation oracle (mf_gp.cuh)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/macrofacet_b200.h"
#include "mf_prepare.h"
#include "mf_scene_build.h"
#include "mf_transport.cuh"
#include "mf_gp.cuh"

using namespace mf;

namespace {

thread_local std::string g_err;
thread_local uint64_t g_launches = 0;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define MF_CUDA(call)                                                                 \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return fail(MF_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr int kBlock = 128;
// resident blocks per SM the path kernel is compiled for (register cap
// 65536 / (kBlock * kMinBlocks))
#ifndef MF_MIN_BLOCKS
#define MF_MIN_BLOCKS 6
#endif
constexpr int kMinBlocks = MF_MIN_BLOCKS;
// the same for the path pool (its smem pools allow up to 7 blocks per SM)
#ifndef MF_POOL_MIN_BLOCKS
#define MF_POOL_MIN_BLOCKS 8
#endif
constexpr int kPoolMinBlocks = MF_POOL_MIN_BLOCKS;

enum StatIdx {
  kStPaths = 0,
  kStSegments,
  kStScatters,
  kStNee,
  kStSlopeIters,
  kStTrackSteps,
  kStEscaped,
  kStAbsorbed,
  kStViolations,
  kStDegenerate,
  kStNonfinite,
  kStCapped,
  kStCount
};

// ---------------------------------------------------------------------------
// closed-form curves (mf_curve)

struct CurveArgs {
  MediumK m;
  int kind;
  const float *x, *y, *z;
  int64_t n;
  V3 wo;
  float z0;
  float sig_wo;   // sigma(wo) (VNDF) or Lambda(wo) (transmittance)
  float* out;
};

__global__ void __launch_bounds__(256) curve_kernel(const __grid_constant__ CurveArgs a) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float r;
    if (a.kind == MF_CURVE_TRANSMITTANCE) {
      // planar_transmittance (medium.py:98-124): exp(-Lambda * dlog Phi)
      float h1 = __ldg(a.x + i);
      float dl = log_ndtr(h1 * a.m.inv_sigma) - log_ndtr(a.z0 * a.m.inv_sigma);
      r = expf(-a.sig_wo * dl);
    } else if (a.kind == MF_CURVE_DENSITY) {
      r = mills(__ldg(a.x + i) * a.m.inv_sigma) * a.m.inv_sigma;
    } else if (a.kind == MF_CURVE_FRESNEL) {
      r = fresnel_conductor(__ldg(a.x + i), a.m.eta[0], a.m.k[0]);
    } else if (a.kind == MF_CURVE_GDF) {
      // Gaussian gradient density conditioned on a crossing (ndf.py:232-239)
      float gx = __ldg(a.x + i) * a.m.inv_ax, gy = __ldg(a.y + i) * a.m.inv_ay;
      float gz = (__ldg(a.z + i) - 1.0f) * (1.0f / a.m.az);
      r = expf(-fmaf(gx, gx, fmaf(gy, gy, gz * gz))) * a.m.d_norm;
    } else {
      V3 w = v3(__ldg(a.x + i), __ldg(a.y + i), __ldg(a.z + i));
      if (a.kind == MF_CURVE_LAMBDA) r = proj_area(a.m, w) / w.z;
      else if (a.kind == MF_CURVE_PROJECTED_AREA) r = proj_area(a.m, w);
      else if (a.kind == MF_CURVE_NDF) r = ndf(a.m, w);
      else r = vndf_eval(a.m, w, a.wo, a.sig_wo);
    }
    a.out[i] = r;
  }
}

// ---------------------------------------------------------------------------
// config-1 query kernel

struct QueryArgs {
  MediumK m;
  int shape;
  float z0;
  V3 c;
  float radius;
  mf_query_in in;
  mf_query_out out;
  int64_t n;
};

// Config-1 queries, binned by mixture branch, per warp.  Phase A (one query
// per lane): inputs, local frame, sigma_t, phase value, pdf, and the whole
// sample of queries taking the cheap hemisphere branch (or degenerate);
// queries taking the Beckmann branch (half of them) are queued in the warp's
// shared-memory ring.  Phase B, whenever 32 are queued (and once more at the
// end): the visible-slope solver -- most of a query's work -- on a full warp
// instead of on the ~half of each warp's lanes whose branch chose it.  No
// block barriers: each warp owns its ring.  Every query runs query_local's
// arithmetic (medium.py:91-207, ndf.py:383-427).
constexpr int kQBlock = 256;
constexpr int kQRing = 64;           // power of two >= 2 x 32
struct QueryRing {
  uint32_t idx_lo[kQRing], idx_hi[kQRing];   // query index
  float wo[3][kQRing];                       // local wo
  float fr[9][kQRing];                       // local frame (t, b, n)
  float uu[kQRing], u2[kQRing], sig_o[kQRing], sig_b[kQRing];
};

__device__ __forceinline__ void query_write_sample(const mf_query_out& o, int64_t i, V3 ws,
                                                   float pdf_s, V3 w) {
  if (o.wsx) o.wsx[i] = ws.x;
  if (o.wsy) o.wsy[i] = ws.y;
  if (o.wsz) o.wsz[i] = ws.z;
  if (o.pdf_s) o.pdf_s[i] = pdf_s;
  if (o.w_r) o.w_r[i] = w.x;
  if (o.w_g) o.w_g[i] = w.y;
  if (o.w_b) o.w_b[i] = w.z;
}

// the visible normal of the sample and its mixture density (vndf_sample);
// out of the config-1 path unless requested (uniform test on the pointer)
template <bool kNormal>
__device__ __forceinline__ void query_write_normal(const mf_query_out& o, int64_t i,
                                                   const Frame& fr, const PhaseSample& smp) {
  if (kNormal) {
    V3 wm = to_world(fr, smp.wm);
    if (o.wmx) o.wmx[i] = wm.x;
    if (o.wmy) o.wmy[i] = wm.y;
    if (o.wmz) o.wmz[i] = wm.z;
    if (o.pdf_m) o.pdf_m[i] = smp.pdf_m;
  }
}

// Beckmann branch and tail of ring entry k
template <bool kNormal>
__device__ __forceinline__ void query_beckmann(const QueryArgs& a, const QueryRing& R, int k) {
  const MediumK& m = a.m;
  int64_t j = (int64_t)(((uint64_t)R.idx_hi[k] << 32) | R.idx_lo[k]);
  V3 wol = v3(R.wo[0][k], R.wo[1][k], R.wo[2][k]);
  Frame fr;
  fr.t = v3(R.fr[0][k], R.fr[1][k], R.fr[2][k]);
  fr.b = v3(R.fr[3][k], R.fr[4][k], R.fr[5][k]);
  fr.n = v3(R.fr[6][k], R.fr[7][k], R.fr[8][k]);
  V3 v = neg3(wol);
  int iters = 0;
  V3 wm = beckmann_visible_normal<true>(m, v, R.uu[k], R.u2[k], &iters);
  PhaseSample smp = phase_sample_tail(m, v, wm, dot3(v, wm), R.sig_o[k], R.sig_b[k], true);
  query_write_sample(a.out, j, to_world(fr, smp.wi), smp.pdf, smp.weight);
  query_write_normal<kNormal>(a.out, j, fr, smp);
}

// kNormal: the caller asked for the sampled visible normal / its density
// (vndf_sample); the config-1 build carries neither
template <bool kNormal>
__global__ void __launch_bounds__(kQBlock) query_kernel(const __grid_constant__ QueryArgs a) {
  __shared__ QueryRing rings[kQBlock / 32];
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  QueryRing& R = rings[threadIdx.x >> 5];
  const MediumK& m = a.m;
  const mf_query_out& o = a.out;
  unsigned head = 0, tail = 0;   // warp-uniform ring positions
  int64_t warp_id = ((int64_t)blockIdx.x * kQBlock + threadIdx.x) >> 5;
  int64_t n_warps = ((int64_t)gridDim.x * kQBlock) >> 5;
  for (int64_t c0 = warp_id * 32; c0 < a.n; c0 += n_warps * 32) {
    int64_t i = c0 + lane;
    bool queue = false;
    V3 wol = v3(0.0f, 0.0f, 0.0f);
    Frame fr;
    float uu = 0.0f, u2 = 0.0f, sig_safe = 1.0f, sig_b = 0.0f;
    if (i < a.n) {
      V3 p = v3(__ldg(a.in.px + i), __ldg(a.in.py + i), __ldg(a.in.pz + i));
      V3 wo = v3(__ldg(a.in.wox + i), __ldg(a.in.woy + i), __ldg(a.in.woz + i));
      V3 wi = v3(__ldg(a.in.wix + i), __ldg(a.in.wiy + i), __ldg(a.in.wiz + i));
      float u1 = __ldg(a.in.u1 + i);
      u2 = __ldg(a.in.u2 + i);
      FieldPoint fp = field_at(a.shape, a.z0, a.c, a.radius, p);
      if (a.in.f) fp.f = __ldg(a.in.f + i);
      if (a.in.frame) {
        const float* F = a.in.frame;
        fr.t = v3(__ldg(F + i), __ldg(F + a.n + i), __ldg(F + 2 * a.n + i));
        fr.b = v3(__ldg(F + 3 * a.n + i), __ldg(F + 4 * a.n + i), __ldg(F + 5 * a.n + i));
        fr.n = v3(__ldg(F + 6 * a.n + i), __ldg(F + 7 * a.n + i), __ldg(F + 8 * a.n + i));
      } else {
        fr = frame_about(fp.n);
      }
      // query_local up to the sampler (mf_query.cuh)
      u1 = fminf(fmaxf(u1, 5.9604644775390625e-08f), 0.99999994f);
      u2 = fminf(fmaxf(u2, 5.9604644775390625e-08f), 0.99999994f);
      wol = to_local(fr, wo);
      V3 wil = to_local(fr, wi);
      float sig_o = proj_area(m, wol);
      float sigma_t = mills(fp.f * m.inv_sigma) * m.inv_sigma * sig_o;
      sig_b = proj_area_erf(wol, m.ax, m.ay, 0.0f);
      bool degenerate = !(sig_o >= 1e-12f);
      sig_safe = degenerate ? 1.0f : sig_o;
      V3 phase = phase_eval(m, wol, wil, sig_safe);
      float pdf = phase_pdf(m, wol, wil, sig_b);
      uu = remap_branch_uniform(u1, m);
      bool guided = sig_b > 1e-12f;
      if (degenerate) {
        phase = v3(0.0f, 0.0f, 0.0f);
        pdf = 0.0f;
      }
      if (o.sigma_t) o.sigma_t[i] = sigma_t;
      if (o.phase_r) o.phase_r[i] = phase.x;
      if (o.phase_g) o.phase_g[i] = phase.y;
      if (o.phase_b) o.phase_b[i] = phase.z;
      if (o.pdf) o.pdf[i] = pdf;
      if (o.flags) o.flags[i] = degenerate ? 1 : 0;
      if (degenerate) {
        query_write_sample(o, i, wo, 0.0f, v3(0.0f, 0.0f, 0.0f));
        if (kNormal) {
          if (o.wmx) o.wmx[i] = 0.0f;
          if (o.wmy) o.wmy[i] = 0.0f;
          if (o.wmz) o.wmz[i] = 0.0f;
          if (o.pdf_m) o.pdf_m[i] = 0.0f;
        }
      } else if (guided && u1 < m.mix) {
        queue = true;
      } else {
        // hemisphere branch of the mixture (ndf.py:375-380) and the tail
        V3 v = neg3(wol);
        V3 wm = hemisphere_about(v, uu, u2);
        PhaseSample smp = phase_sample_tail(m, v, wm, uu, sig_safe, sig_b, guided);
        query_write_sample(o, i, to_world(fr, smp.wi), smp.pdf, smp.weight);
        query_write_normal<kNormal>(o, i, fr, smp);
      }
    }
    // enqueue the Beckmann-branch queries of this chunk
    unsigned qm = __ballot_sync(full, queue);
    if (queue) {
      int k = (int)((tail + (unsigned)__popc(qm & lt)) & (kQRing - 1));
      R.idx_lo[k] = (uint32_t)i;
      R.idx_hi[k] = (uint32_t)((uint64_t)i >> 32);
      R.wo[0][k] = wol.x; R.wo[1][k] = wol.y; R.wo[2][k] = wol.z;
      R.fr[0][k] = fr.t.x; R.fr[1][k] = fr.t.y; R.fr[2][k] = fr.t.z;
      R.fr[3][k] = fr.b.x; R.fr[4][k] = fr.b.y; R.fr[5][k] = fr.b.z;
      R.fr[6][k] = fr.n.x; R.fr[7][k] = fr.n.y; R.fr[8][k] = fr.n.z;
      R.uu[k] = uu; R.u2[k] = u2; R.sig_o[k] = sig_safe; R.sig_b[k] = sig_b;
    }
    tail += (unsigned)__popc(qm);
    __syncwarp();
    if (tail - head >= 32) {
      query_beckmann<kNormal>(a, R, (int)((head + (unsigned)lane) & (kQRing - 1)));
      head += 32;
      __syncwarp();
    }
  }
  // drain
  int left = (int)(tail - head);
  if (lane < left) query_beckmann<kNormal>(a, R, (int)((head + (unsigned)lane) & (kQRing - 1)));
}

// ---------------------------------------------------------------------------
// path megakernel

// Division by a runtime constant d: q = floor(n * ceil(2^64 / d) / 2^64),
// exact for every 32-bit n and d (the error n (ceil - 2^64/d) / 2^64 < 2^-32
// never carries past the next multiple of 1/d); d = 1 is special-cased.
// Three integer instructions instead of the ~20 of a 32-bit IDIV sequence
// (raygen maps a path index to (sample, tile, pixel) with four of them).
struct FastDiv {
  unsigned long long m;   // ceil(2^64 / d), 0 for d == 1
  uint32_t d;
};

inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  f.m = d > 1 ? (~0ull / d) + 1ull : 0ull;
  return f;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return f.m ? (uint32_t)__umul64hi((unsigned long long)n, f.m) : n;
}

struct PassDev {
  uint32_t k0, k1;
  // Philox round keys (k0 + r W0, k1 + r W1), so the unrolled rounds of the
  // render kernels' own draws read them as constant-bank operands
  uint32_t rk[20];
  int max_bounces;
  uint32_t n_paths;      // paths in this pass
  uint32_t S;            // samples per local pixel in this pass
  uint32_t sample_begin; // global sample index of the pass's first sample
  uint32_t n_local;      // local pixels of this rank (render mode)
  int shard, rank, nranks, tile, tiles_x;
  FastDiv div_local, div_t2, div_tiles_x, div_tile, div_width, div_S;
  int pixel_major;       // path order: 1 all samples of a pixel together, 0 sample-major
  int mono;              // grey scene: the accumulator holds channel 0 only
  // render mode: per-pixel fixed-point sums (accumulate_fx), channel-major
  // per local pixel: fx[lp * (mono ? 1 : 3) + c] += rint(L_c * fx_scale)
  unsigned long long* fx;
  float fx_scale;        // 2^k (host-chosen, mf_render)
  float fx_limit;        // per-path bound of L * fx_scale: the sums cannot overflow
  float* rad;            // caller-ray mode (trace_paths): SoA [3][n_paths]
  unsigned int* counter;
  unsigned long long* stats;
  // caller-ray mode (trace_paths)
  const float* org;      // SoA [3][n]
  const float* dir;
  const uint32_t* pix;
  const uint32_t* smp;
};

// local pixel index -> global pixel index (and its x, y), or -1 (tile
// padding)
__device__ __forceinline__ int local_to_pixel(const SceneDev& sc, const PassDev& ps, uint32_t lp,
                                              uint32_t* px = nullptr, uint32_t* py = nullptr) {
  uint32_t x, y;
  if (ps.shard == MF_SHARD_SAMPLES) {
    y = fdiv(lp, ps.div_width);
    x = lp - y * (uint32_t)sc.width;
  } else {
    uint32_t k = fdiv(lp, ps.div_t2);
    uint32_t j = lp - k * ps.div_t2.d;
    uint32_t t = (uint32_t)ps.rank + k * (uint32_t)ps.nranks;
    uint32_t ty = fdiv(t, ps.div_tiles_x), tx = t - ty * (uint32_t)ps.tiles_x;
    uint32_t jy = fdiv(j, ps.div_tile), jx = j - jy * (uint32_t)ps.tile;
    x = tx * ps.tile + jx;
    y = ty * ps.tile + jy;
    if (x >= (uint32_t)sc.width || y >= (uint32_t)sc.height) return -1;
  }
  if (px) {
    *px = x;
    *py = y;
  }
  return (int)(y * (uint32_t)sc.width + x);
}

// inverse of local_to_pixel: this rank's local index of an image pixel, or
// -1 when another rank owns its tile
__device__ __forceinline__ int64_t pixel_to_local(const SceneDev& sc, const PassDev& ps,
                                                  uint32_t pixel) {
  if (ps.shard == MF_SHARD_SAMPLES) return pixel;
  uint32_t y = fdiv(pixel, ps.div_width), x = pixel - y * (uint32_t)sc.width;
  uint32_t ty = fdiv(y, ps.div_tile), tx = fdiv(x, ps.div_tile);
  uint32_t t = ty * (uint32_t)ps.tiles_x + tx;
  uint32_t k = t / (uint32_t)ps.nranks;
  if (t - k * (uint32_t)ps.nranks != (uint32_t)ps.rank) return -1;
  uint32_t jy = y - ty * (uint32_t)ps.tile, jx = x - tx * (uint32_t)ps.tile;
  return (int64_t)k * ps.div_t2.d + jy * (uint32_t)ps.tile + jx;
}

struct PathState {
  V3 pos, dir, T, L;
  V3 cpos;               // pending collision (flight -> scatter stage)
  int ck;                // primitive of the pending collision
  float csig;            // sigma(dir) when known in the collision frame, else -1
  float u_br, u_s2, u_rr;  // the segment's branch / slope / RR uniforms
  float lphi;            // single plane: log Phi(f / sigma) at pos, NaN when unknown
  int bounce;
  bool pre;              // raygen drew segment 0's block: u_rr holds u_flight
  uint32_t pid;          // result slot: caller-ray index, or the local pixel (render)
  PathRng rng;
};

struct Counters {
  uint32_t v[kStCount];
};

__device__ __forceinline__ void camera_ray(const SceneDev& sc, uint32_t px, uint32_t py, float jx,
                                           float jy, V3* o, V3* d) {
  float nx = ((float)px + jx) / (float)sc.width * 2.0f - 1.0f;
  float ny = 1.0f - ((float)py + jy) / (float)sc.height * 2.0f;
  if (sc.ortho) {
    *o = fma3(sc.cam_up, ny * sc.half_h, fma3(sc.cam_right, nx * sc.half_w, sc.cam_pos));
    *d = sc.cam_fwd;
  } else {
    *o = sc.cam_pos;
    *d = normalize3(fma3(sc.cam_up, ny * sc.half_h, fma3(sc.cam_right, nx * sc.half_w, sc.cam_fwd)));
  }
}

// Russian-roulette threshold of the renderer's shadow-ray weights (walk());
// the transmittance_estimate API (ratio_kernel) keeps plain ratio tracking.
// At 1 a weight below 1 survives as 1 with probability equal to itself, i.e.
// the shadow ray is delta-tracked (a binary visibility estimate).  Measured
// per-pixel variance (eight seeds, tools/shadow_rr_eff.py) does not move
// with the threshold -- path sampling dominates it -- while the walks get
// shorter: config 5 5.71 / 5.10 / 4.79 / 4.51 ms and config 3 1.636 / 1.522 /
// 1.483 / 1.464 ms at 0.05 / 0.35 / 0.7 / 1, variance 1.84e-2 / 1.85e-2 /
// 1.89e-2 / 1.81e-2 and 4.41e-4 / 4.41e-4 / 4.41e-4 / 4.42e-4.
#ifndef MF_SHADOW_RR
#define MF_SHADOW_RR 1.0f
#endif
constexpr float kShadowRR = MF_SHADOW_RR;

// shadow transmittance from pos towards unit direction wl over distance t_max
// kSpec: the medium's kind / Fresnel known at compile time (proj_area);
// kPool: the path-pool kernels, which never run the general walker for a
// single sphere (MF_GENERIC_WALK selects the megakernel)
template <int kMode, int kSpec = kSpecRuntime, bool kPool = false>
__device__ __forceinline__ float shadow_tr(const SceneDev& sc, const PathState& st, V3 pos, V3 wl,
                                           float t_max, float h_end, Counters& cn,
                                           float sig_known = -1.0f) {
  if constexpr (kMode == 0) {
    const MediumK& m = sc.media[0];
    float sig = sig_known >= 0.0f ? sig_known : proj_area<kSpecRuntime, true>(m, wl);
    return planar_shadow_tr(m, sc.mx[0], pos.z - sc.prims[0].z0, h_end, wl.z, sig, st.lphi);
  } else if constexpr (kMode == 2) {
    GridWalk w = grid_walk_path(sc.grid, sc.media[0], st.rng, (uint32_t)st.bounce, kCallShadow,
                                pos, wl, true, t_max, kShadowRR);
    cn.v[kStTrackSteps] += (uint32_t)max(w.steps, 0);
    cn.v[kStViolations] += (uint32_t)w.violations;
    if (w.steps < 0) cn.v[kStCapped]++;   // iteration cap: raised by the host
    return w.steps < 0 ? 0.0f : w.weight;
  } else {
    WalkResult w = kMode == 3 && (kPool || !sc.generic_walk)
                       ? sphere_walk<kSpec>(sc, st.rng, (uint32_t)st.bounce, kCallShadow, pos, wl,
                                            true, t_max, kShadowRR)
                       : walk<kMode == 3>(sc, st.rng, (uint32_t)st.bounce, kCallShadow, pos, wl,
                                          true, t_max, kShadowRR);
    cn.v[kStTrackSteps] += (uint32_t)max(w.steps, 0);
    cn.v[kStViolations] += (uint32_t)w.violations;
    if (w.steps < 0) cn.v[kStCapped]++;
    return w.steps < 0 ? 0.0f : w.weight;
  }
}

// shadow transmittance towards the sun from a single-plane collision whose
// log Phi is unknown (after a grazing flight): the general closed form, out
// of line (one copy in the instruction stream, rarely executed)
__device__ __noinline__ float planar_sun_tr_cold(const SceneDev& sc, float h, float lphi) {
  return planar_shadow_tr(sc.media[0], sc.mx[0], h, sc.sun_to.z > 0.0f ? INFINITY : -INFINITY,
                          sc.sun_to.z, sc.sun_sig, lphi);
}

// point-light NEE at a single-plane collision: the radiance increment
// T phase I Tr / r^2 (the plane frame is the identity).  Out of line: point
// lights are not on the benchmark path, and one copy gives the pool and the
// megakernel the same instructions (their images must match bit for bit).
__device__ __noinline__ V3 planar_point_nee(const SceneDev& sc, const PathState& st, V3 wo,
                                            float sig_o, V3 pos, int* nee) {
  const MediumK& m = sc.media[0];
  V3 d = sub3(sc.point_pos, pos);
  float r2 = dot3(d, d);
  float ir = frsqrt(r2);
  V3 wl = mul3(d, ir);
  V3 ph = phase_eval<kSpecRuntime, true>(m, wo, wl, sig_o);
  if (!(ph.x > 0.0f || ph.y > 0.0f || ph.z > 0.0f)) return v3(0.0f, 0.0f, 0.0f);
  *nee = 1;
  float sig = proj_area<kSpecRuntime, true>(m, wl);
  float tr = planar_shadow_tr(m, sc.mx[0], pos.z - sc.prims[0].z0,
                              sc.point_pos.z - sc.prims[0].z0, wl.z, sig, st.lphi);
  float s = tr * frcp(r2);
  return v3(st.T.x * ph.x * sc.point_I.x * s, st.T.y * ph.y * sc.point_I.y * s,
            st.T.z * ph.z * sc.point_I.z * s);
}

// sun transmittance from a single-plane collision (both render kernels):
// with the collision's log Phi known, the closed form (planar_shadow_tr)
// reduces to clamping it to the band and one MUFU exp2 -- the sun end is a
// band edge fixed per render (sun_lb, sun_k2 prepared on the host)
__device__ __forceinline__ float planar_sun_tr(const SceneDev& sc, float lphi, V3 pos) {
  if (!(lphi == lphi)) return planar_sun_tr_cold(sc, pos.z - sc.prims[0].z0, lphi);
  const MediumExtra& mx = sc.mx[0];
  float la = fminf(fmaxf(lphi, mx.lphi_lo_rat), mx.lphi_hi);
  if (la == sc.sun_lb) return 1.0f;
  if (sc.sun_graze) return 0.0f;
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(sc.sun_k2 * fabsf(sc.sun_lb - la)));
  return r;
}

template <int kMode>
__device__ __forceinline__ bool scatter_stages(const SceneDev& sc, const PassDev& ps,
                                               PathState& st, Counters& cn, unsigned amask,
                                               const MediumK& m, const Frame& fr, V3 pos,
                                               float sig_known, bool done, float u_br,
                                               float u_s2, float u_rr);

// Russian roulette on small NEE contributions of grid fields (kMode 2), whose
// shadow rays are long walks (config 3's sphere walks are 2 - 3 iterations:
// there the roulette's own block costs what it saves, 3192 -> 3123 Mpaths/s,
// so spheres and general shells walk every shadow ray): when the brightest channel of c = T phase E
// is below kNeeRR x the brightest channel of the light's E, the shadow ray
// is walked with probability p = cmax / (kNeeRR Emax) and c is scaled by 1/p,
// else skipped -- unbiased, and the added per-sample variance is at most
// c x kNeeRR Emax.  The uniform is word x of block (segment, call) of the
// path's stream, call = kCallNeeRR (sun) or kCallNeeRR + 1 (point light).
// Returns false when the shadow ray is skipped.  Measured over eight seeds
// (tools/shadow_rr_eff.py; kNeeRR 0 / 0.02 / 0.05 / 0.1 / 0.2 / 0.5): config 5
// 4.60 / 3.96 / 3.79 / 3.63 / 3.47 / 3.27 ms with per-pixel variance 1.8120e-2 /
// 1.8122e-2 / 1.8144e-2 / 1.824e-2 / 1.861e-2 / 2.025e-2; config 3 1.482 /
// 1.496 / 1.484 / 1.445 / 1.407 / 1.352 ms, variance 4.423e-4 ... 4.501e-4.
// 0.05 costs 0.1 % of variance.
#ifndef MF_NEE_RR
#define MF_NEE_RR 0.05f
#endif
constexpr float kNeeRR = MF_NEE_RR;
constexpr uint32_t kCallNeeRR = 0x7FFFFFF0u;
__device__ __forceinline__ bool nee_roulette(V3& c, V3 E, uint32_t bits_x) {
  if (!(kNeeRR > 0.0f)) return true;
  float cmax = fmaxf(c.x, fmaxf(c.y, c.z));
  float thr = kNeeRR * fmaxf(E.x, fmaxf(E.y, E.z));
  if (cmax >= thr) return true;
  float p = cmax / thr;
  if (!(u01(bits_x) < p)) return false;
  c = mul3(c, 1.0f / p);
  return true;
}

// next-event estimation at a collision on a curved shell / grid field (sun
// and point light, shadow rays walked in ratio mode): the megakernel's
// stage 2 and the sphere pool's visits run this one copy, so their images
// agree bit for bit
template <int kMode, int kSpec = kSpecRuntime, bool kPool = false>
__device__ __forceinline__ void curved_nee(const SceneDev& sc, PathState& st, Counters& cn,
                                           const MediumK& m, const Frame& fr, V3 wo, float sig_o,
                                           V3 pos) {
  if (sc.has_sun) {
    V3 wl = to_local(fr, sc.sun_to);
    V3 ph = phase_eval<kSpec, true>(m, wo, wl, sig_o);
    if (ph.x > 0.0f || ph.y > 0.0f || ph.z > 0.0f) {
      cn.v[kStNee]++;
      V3 c = v3(st.T.x * ph.x * sc.sun_L.x, st.T.y * ph.y * sc.sun_L.y, st.T.z * ph.z * sc.sun_L.z);
      if (kMode != 2 || kNeeRR <= 0.0f ||
          nee_roulette(c, sc.sun_L, kMode == 2 && kNeeRR > 0.0f ? rng_block(st.rng, (uint32_t)st.bounce, kCallNeeRR).x : 0u)) {
        float tr = shadow_tr<kMode, kSpec, kPool>(sc, st, pos, sc.sun_to, INFINITY,
                                    sc.sun_to.z > 0.0f ? INFINITY : -INFINITY, cn, sc.sun_sig);
        st.L = add3(st.L, v3(c.x * tr, c.y * tr, c.z * tr));
      }
    }
  }
  if (sc.has_point) {
    V3 d = sub3(sc.point_pos, pos);
    float r2 = dot3(d, d);
    float ir = frsqrt(r2);
    V3 wlw = mul3(d, ir);
    V3 wl = to_local(fr, wlw);
    V3 ph = phase_eval<kSpec, true>(m, wo, wl, sig_o);
    if (ph.x > 0.0f || ph.y > 0.0f || ph.z > 0.0f) {
      cn.v[kStNee]++;
      V3 c = v3(st.T.x * ph.x * sc.point_I.x, st.T.y * ph.y * sc.point_I.y,
                st.T.z * ph.z * sc.point_I.z);
      if (kMode != 2 || kNeeRR <= 0.0f ||
          nee_roulette(c, sc.point_I,
                       kMode == 2 && kNeeRR > 0.0f ? rng_block(st.rng, (uint32_t)st.bounce, kCallNeeRR + 1u).x : 0u)) {
        float tr = shadow_tr<kMode, kSpec, kPool>(sc, st, pos, wlw, r2 * ir,
                                                  sc.point_pos.z - sc.prims[0].z0, cn);
        float s = tr * frcp(r2);
        st.L = add3(st.L, v3(c.x * s, c.y * s, c.z * s));
      }
    }
  }
}

// Stage 1 of a segment: draw the segment's uniforms and fly to the next real
// collision (transport.py:144-297).  Returns true on a collision (state kept
// in st.cpos / st.ck / st.csig for the scatter stage); on escape / absorption
// the environment term is added and false is returned (path finished).
// kMode: 0 single plane (analytic), 1 general shells (tracking), 2 grid field
// kNeedPos (single plane): 1 / 0 when the caller knows at compile time
// whether a point light reads positions, -1 to ask the scene
template <int kMode, int kSpec = kSpecRuntime, int kNeedPos = -1, bool kPool = false>
__device__ __forceinline__ bool flight_stage(const SceneDev& sc, const PassDev& ps, PathState& st,
                                             Counters& cn) {
  cn.v[kStSegments]++;
  float u_fl;
  if (st.pre) {
    // segment 0 of a render path: its block was drawn at raygen (the camera
    // jitter took its spare bits); the RR uniform of segment 0 is never read
    // (Russian roulette starts after bounce 8)
    u_fl = st.u_rr;
    st.pre = false;
  } else {
    U4 b = philox_rk(U4{st.rng.pixel, st.rng.sample, (uint32_t)st.bounce, 0u}, ps.rk);
    u_fl = u01(b.x);
    st.u_br = u01(b.y);
    st.u_s2 = u01(b.z);
    st.u_rr = u01(b.w);
  }
  st.ck = 0;
  st.csig = -1.0f;
  int outcome;
  if constexpr (kMode == 2) {
    GridWalk w = grid_walk_path(sc.grid, sc.media[0], st.rng, (uint32_t)st.bounce, 1u, st.pos,
                                st.dir, false, INFINITY, 0.0f);
    cn.v[kStTrackSteps] += (uint32_t)max(w.steps, 0);
    cn.v[kStViolations] += (uint32_t)w.violations;
    st.cpos = w.pos;
    outcome = w.steps < 0 ? -1 : w.outcome;
  } else if constexpr (kMode == 0) {
    const MediumK& m = sc.media[0];
    float sig = proj_area<kSpec, true>(m, st.dir);
    st.csig = sig;   // sigma(dir) is sigma(wo) in the (identity) plane frame
    // positions matter only to a point light
    Flight fl = planar_flight(sc.prims[0], m, sc.mx[0], st.pos, st.dir, sig, u_fl, st.lphi,
                              kNeedPos < 0 ? sc.has_point != 0 : kNeedPos == 1);
    st.cpos = fl.pos;
    st.lphi = fl.lphi;
    outcome = fl.outcome;
  } else {
    WalkResult w = kMode == 3 && (kPool || !sc.generic_walk)
                       ? sphere_walk<kSpec>(sc, st.rng, (uint32_t)st.bounce, 1u, st.pos, st.dir,
                                            false, INFINITY)
                       : walk<kMode == 3>(sc, st.rng, (uint32_t)st.bounce, 1u, st.pos, st.dir,
                                          false, INFINITY);
    cn.v[kStTrackSteps] += (uint32_t)max(w.steps, 0);
    cn.v[kStViolations] += (uint32_t)w.violations;
    st.cpos = w.pos;
    st.ck = max(w.prim, 0);
    outcome = w.steps < 0 ? -1 : w.outcome;
  }
  if (outcome == kEscaped) {
    V3 e = env_radiance(sc, st.dir);   // render.py:54-57
    st.L = add3(st.L, v3(st.T.x * e.x, st.T.y * e.y, st.T.z * e.z));
    cn.v[kStEscaped]++;
    return false;
  }
  if (outcome == kAbsorbed) {
    cn.v[kStAbsorbed]++;
    return false;
  }
  if (outcome < 0) {
    cn.v[kStCapped]++;
    return false;
  }
  return true;
}

// Stages 2-3 at the collision found by flight_stage: local medium / frame,
// then NEE, phase sampling, depth cap, RR.  Returns true when the path ends.
//
// SIMT structure: single exits and explicit warp re-convergence
// (__syncwarp over the participating lanes) between stages.  Without it the
// lanes that escape / take the other mixture branch are not re-joined until
// the function ends and every later stage runs once per lane group
// (measured: 5.6 active lanes per warp instruction).
template <int kMode>
__device__ __forceinline__ bool scatter_stage(const SceneDev& sc, const PassDev& ps,
                                              PathState& st, Counters& cn, unsigned amask) {
  V3 pos = st.cpos;
  if constexpr (kMode == 2) {
    TriSample fs = trilinear<true>(sc.grid.sdf, sc.grid.n_sdf,
                                   grid_coord(sc.grid, pos, sc.grid.inv_h_sdf),
                                   sc.grid.inv_h_sdf);
    float sg = fmaxf(grid_sigma(sc.grid, pos), 1e-6f);
    MediumK mg = grid_medium(sc.media[0], sg, sc.grid.k_xy, sc.grid.k_z);
    float gn2 = dot3(fs.grad, fs.grad);
    V3 nrm = gn2 > 0.0f ? mul3(fs.grad, frsqrt(gn2)) : v3(0.0f, 0.0f, 1.0f);
    return scatter_stages<kMode>(sc, ps, st, cn, amask, mg, frame_about(nrm), pos, -1.0f, false,
                                 st.u_br, st.u_s2, st.u_rr);
  } else {
    V3 nrm = kMode == 0 ? v3(0.0f, 0.0f, 1.0f) : prim_normal<kMode == 3>(sc.prims[st.ck], pos);
    return scatter_stages<kMode>(sc, ps, st, cn, amask, sc.media[st.ck], frame_about(nrm), pos,
                                 kMode == 0 ? st.csig : -1.0f, false, st.u_br, st.u_s2,
                                 st.u_rr);
  }
}

// Stages 2-3 of a segment at a real collision (NEE, phase sampling, depth
// cap, RR) for medium m and local frame fr; sig_known >= 0 is sigma(dir).
template <int kMode>
__device__ __forceinline__ bool scatter_stages(const SceneDev& sc, const PassDev& ps,
                                               PathState& st, Counters& cn, unsigned amask,
                                               const MediumK& m, const Frame& fr, V3 pos,
                                               float sig_known, bool done, float u_br,
                                               float u_s2, float u_rr) {
  V3 wo = to_local(fr, st.dir);
  float sig_o = sig_known >= 0.0f ? sig_known : proj_area<kSpecRuntime, true>(m, wo);
  if (!done) {
    cn.v[kStScatters]++;
    if (!(sig_o >= 1e-12f)) {
      cn.v[kStDegenerate]++;
      done = true;
    }
  }
  // ---- stage 2: next-event estimation (render.py:71-82; point light:
  //      BASELINE extension)
  if (kMode == 0) {
    if (!done && sc.has_sun) {
      V3 wl = to_local(fr, sc.sun_to);
      V3 ph = phase_eval<kSpecRuntime, true>(m, wo, wl, sig_o);
      if (ph.x > 0.0f || ph.y > 0.0f || ph.z > 0.0f) {
        cn.v[kStNee]++;
        float tr = planar_sun_tr(sc, st.lphi, pos);
        st.L = add3(st.L, v3(st.T.x * ph.x * sc.sun_L.x * tr, st.T.y * ph.y * sc.sun_L.y * tr,
                             st.T.z * ph.z * sc.sun_L.z * tr));
      }
    }
    if (!done && sc.has_point) {
      int nee = 0;
      st.L = add3(st.L, planar_point_nee(sc, st, wo, sig_o, pos, &nee));
      cn.v[kStNee] += (uint32_t)nee;
    }
  } else if (!done) {
    curved_nee<kMode>(sc, st, cn, m, fr, wo, sig_o, pos);
  }
  __syncwarp(amask);
  // ---- stage 3: phase sampling (render.py:84-90), two-uniform convention
  unsigned smask = __ballot_sync(amask, !done);
  if (!done) {
    float sig_b = m.kind == kBeckmann ? sig_o : proj_area_erf<true>(wo, m.ax, m.ay, 0.0f);
    float uu = remap_branch_uniform_render(u_br, m);
    PhaseSample smp = phase_sample<false, true>(m, wo, sig_o, sig_b, u_br, uu, u_s2, smask);
    cn.v[kStSlopeIters] += (uint32_t)smp.iters;
    st.dir = to_world(fr, smp.wi);
    st.T = v3(st.T.x * smp.weight.x, st.T.y * smp.weight.y, st.T.z * smp.weight.z);
    st.pos = pos;
    st.bounce++;
    if (st.bounce >= ps.max_bounces) {             // render.py:92-94
      done = true;
    } else if (st.bounce > 8) {                    // render.py:96-105
      float q = fminf(fmaxf(st.T.x, fmaxf(st.T.y, st.T.z)), 1.0f);
      if (u_rr >= q) {
        done = true;
      } else {
        st.T = mul3(st.T, 1.0f / q);
      }
    }
  }
  __syncwarp(amask);
  return done;
}

// Start the path with index `my` in lane state st (raygen, render.py:149-160
// keying); returns false for tile padding (no path).
template <bool kCallerRays>
__device__ __forceinline__ bool start_path(const SceneDev& sc, const PassDev& ps, PathState& st,
                                           uint32_t my) {
  st.pid = my;
  st.rng.k0 = ps.k0;
  st.rng.k1 = ps.k1;
  st.T = v3(1.0f, 1.0f, 1.0f);
  st.L = v3(0.0f, 0.0f, 0.0f);
  st.lphi = NAN;
  st.bounce = 0;
  st.pre = false;
  if (kCallerRays) {
    st.rng.pixel = ps.pix[my];
    st.rng.sample = ps.smp[my];
    st.pos = v3(ps.org[my], ps.org[ps.n_paths + my], ps.org[2u * ps.n_paths + my]);
    st.dir = v3(ps.dir[my], ps.dir[ps.n_paths + my], ps.dir[2u * ps.n_paths + my]);
    return true;
  }
  // path order.  Sample-major (the path pool): the 32 paths a warp starts
  // together belong to 32 consecutive pixels, so the fixed-point adds of
  // paths finishing together hit distinct (adjacent) accumulator words
  // instead of one.  Pixel-major (the tracking megakernels, whose paths are
  // long and whose adds rarely collide): a warp's paths share their camera
  // ray up to the jitter, so their first walks stay coherent.
  uint32_t s, lp;
  if (ps.pixel_major) {
    lp = fdiv(my, ps.div_S);
    s = my - lp * ps.S;
  } else {
    s = fdiv(my, ps.div_local);
    lp = my - s * ps.n_local;
  }
  st.pid = lp;   // the path's radiance goes to its local pixel's sums
  uint32_t px, py;
  int pixel = local_to_pixel(sc, ps, lp, &px, &py);
  if (pixel < 0) return false;   // tile padding
  st.rng.pixel = (uint32_t)pixel;
  st.rng.sample = ps.sample_begin + s;
  // one block serves the camera jitter and segment 0: (u_flight, u_branch,
  // u_slope) from words x, y, z as in every segment, the jitter from word w
  // and from the 23 low bits of x, y, z that u01 leaves unused
  U4 b = philox_rk(U4{st.rng.pixel, st.rng.sample, 0u, 0u}, ps.rk);
  uint32_t low = (b.x & 0x1FFu) | ((b.y & 0x1FFu) << 9) | ((b.z & 0x1Fu) << 18);
  camera_ray(sc, px, py, u01(b.w), u01(low << 9), &st.pos, &st.dir);
  st.u_rr = u01(b.x);   // u_flight of segment 0 (see flight_stage)
  st.u_br = u01(b.y);
  st.u_s2 = u01(b.z);
  st.pre = true;
  return true;
}

// Per-pixel accumulation fused into the render kernels (render.py:150,
// 165-166): a finished path adds rint(L * 2^k) to its pixel's 64-bit
// fixed-point sum with one fire-and-forget atomic (RED.ADD.64) per channel.
// Integer addition is associative, so the sums -- and the image -- do not
// depend on the order in which paths finish (any launch geometry, pool
// schedule or tile / rank split), and no per-path radiance ever goes to HBM.
// L * 2^k is exact in fp32 (a power-of-two scale), so every value >= 2^(24-k)
// enters the sum with its full fp32 mantissa and the sum itself is exact;
// fx_limit keeps spp such values below 2^63.  A path whose radiance is
// non-finite, negative or beyond the limit is counted (the host raises
// NumericFailureError, RadianceImage.validate, image.py:38-42) and adds 0.
__device__ __forceinline__ void accumulate_fx(const PassDev& ps, uint32_t slot, float v,
                                              Counters& cn) {
  float q = v * ps.fx_scale;
  if (!(q >= 0.0f && q < ps.fx_limit)) {   // also catches NaN
    cn.v[kStNonfinite]++;
    return;
  }
  unsigned long long iq = __float2ull_rn(q);
  if (iq) atomicAdd(ps.fx + slot, iq);
}

template <bool kCallerRays>
__device__ __forceinline__ void finish_path(const PassDev& ps, const PathState& st, Counters& cn) {
  float r = st.L.x, g = st.L.y, bl = st.L.z;
  if constexpr (kCallerRays) {
    if (!(isfinite(r) && isfinite(g) && isfinite(bl)) || r < 0.0f || g < 0.0f || bl < 0.0f) {
      cn.v[kStNonfinite]++;
    }
    ps.rad[st.pid] = r;
    ps.rad[ps.n_paths + st.pid] = g;
    ps.rad[2u * ps.n_paths + st.pid] = bl;
  } else if (ps.mono) {
    // grey scene: the three channels are equal by construction
    accumulate_fx(ps, st.pid, r, cn);
  } else {
    accumulate_fx(ps, st.pid * 3u, r, cn);
    accumulate_fx(ps, st.pid * 3u + 1u, g, cn);
    accumulate_fx(ps, st.pid * 3u + 2u, bl, cn);
  }
}

// Warp-level regeneration: the dead lanes of the warp take popc(dead) path
// indices with one atomicAdd and start them.  Every lane must call this.
template <bool kCallerRays>
__device__ __forceinline__ void refill(const SceneDev& sc, const PassDev& ps, PathState& st,
                                       bool& active, bool& exhausted, Counters& cn) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  unsigned need = __ballot_sync(full, !active && !exhausted);
  if (!need) return;
  int leader = __ffs(need) - 1;
  unsigned base = 0;
  if (lane == leader) base = atomicAdd(ps.counter, (unsigned)__popc(need));
  base = __shfl_sync(full, base, leader);
  if (!active && !exhausted) {
    uint32_t my = base + (uint32_t)__popc(need & ((1u << lane) - 1u));
    if (my < ps.n_paths) {
      active = start_path<kCallerRays>(sc, ps, st, my);
      if (active) cn.v[kStPaths]++;
    } else {
      exhausted = true;
    }
  }
}

template <int kMode, bool kCallerRays>
__global__ void __launch_bounds__(kBlock, kMinBlocks) path_kernel(const __grid_constant__ SceneDev sc,
                                                       const __grid_constant__ PassDev ps) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  Counters cn;
#pragma unroll
  for (int i = 0; i < kStCount; ++i) cn.v[i] = 0;
  PathState st;
  bool active = false, exhausted = false;
  while (true) {
    refill<kCallerRays>(sc, ps, st, active, exhausted, cn);
    if (__ballot_sync(full, active) == 0) {
      if (__ballot_sync(full, !exhausted) == 0) break;
      continue;
    }
    bool coll = false;
    if (active) {
      coll = flight_stage<kMode>(sc, ps, st, cn);
      if (!coll) {
        finish_path<kCallerRays>(ps, st, cn);
        active = false;
      }
    }
    // (a "second chance" refill + flight of lanes whose path just ended was
    // measured slower: 1.78 vs 1.72 ms on config 2, 16.8 vs 13.5 on config 3)
    unsigned smask = __ballot_sync(full, active && coll);
    if (active && coll) {
      if (scatter_stage<kMode>(sc, ps, st, cn, smask)) {
        finish_path<kCallerRays>(ps, st, cn);
        active = false;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kStCount; ++i) {
    unsigned v = __reduce_add_sync(full, cn.v[i]);
    if (lane == 0 && v) atomicAdd(ps.stats + i, (unsigned long long)v);
  }
}

// ---------------------------------------------------------------------------
// Path pool (single-plane renders): decouple paths from lanes.
//
// The megakernel above binds one path to one lane, so a warp pays for every
// stage any of its lanes needs: the costly Beckmann visible-normal sampler
// runs with the ~half of the lanes whose mixture branch chose it (10 of 32
// active on config 2, ncu), and raygen with the few lanes whose path just
// ended (9 of 32).  Here every warp owns kPool path slots in shared memory
// (SoA) and one ring of slot indices per visit kind; each iteration pops up
// to 32 slots of one ring and runs that visit on them:
//   R  raygen into empty slots, then the first flight;
//   B  (a collision whose mixture branch is Beckmann) NEE, the Beckmann
//      visible normal, the phase tail (pdf, weight, new direction), depth
//      cap / RR, then the next flight;
//   H  the same with the hemisphere branch's normal;
// where "flight" = free flight and the mixture branch choice, which parks
// the collided path on the B or H ring.  Every slot is empty or waits for B
// or H, so with 96 slots one of the three always has a full warp of 32 until
// the path indices run out, and every costly stage (NEE, either sampler, the
// tail) runs at full warp width.  Each path executes exactly the
// megakernel's arithmetic on the same Philox stream, so the image is
// bit-identical to path_kernel<0> (tests/test_gpu_render.py); only the order
// in which paths advance changes.

#ifndef MF_POOL
#define MF_POOL 96
#endif
// render kernels: evaluate each upper slope-residual form only when some
// lane of the warp needs it (rare with kSlopeUpperRender)
#ifndef MF_RENDER_SLOPE_GUARD
#define MF_RENDER_SLOPE_GUARD 1
#endif
constexpr bool kRenderSlopeGuard = MF_RENDER_SLOPE_GUARD;
constexpr int kPool = MF_POOL;
static_assert(kPool % 32 == 0 && kPool <= 128, "pool size: whole warps of slots");
constexpr int kPoolWords = kPool / 32;
constexpr int kRing = 128;   // power of two >= kPool
constexpr int kWarpsPerBlock = kBlock / 32;

enum PoolStage : int { kStageRaygen = 0, kStageBeck = 1, kStageHemi = 2 };
constexpr uint8_t kTagEmpty = 0, kTagBeck = 1, kTagHemi = 2;

// float fields of a slot: dir3 T3 L3 sig_o u_rr lphi u_br u_s2, then
// pos.z (read by the flight after a grazing one, whose log Phi is unknown)
// and pos.x, pos.y when a point light reads positions (grey scenes, kMono:
// T and L are one channel each and the slot is 4 words shorter)
template <bool kMono>
struct PoolF {
  static constexpr int kC = kMono ? 1 : 3;
  static constexpr int kDir = 0, kT = 3, kL = 3 + kC, kSigO = 3 + 2 * kC, kUrr = kSigO + 1,
                       kLphi = kSigO + 2, kU = kSigO + 3, kPz = kSigO + 5, kPxy = kSigO + 6;
};
template <bool kPoint, bool kMono>
struct PoolSlots {
  float f[PoolF<kMono>::kPxy + (kPoint ? 2 : 0)][kPool];
  uint32_t u[4][kPool];   // pid pixel sample bounce
  // one ring of slot indices per tag (empty / waiting for B / for H): a
  // visit pops up to 32 slots of its ring, and every processed slot is
  // pushed onto the ring of its new tag
  uint8_t ring[3][kRing];
};

template <bool kPoint, bool kMono>
__device__ __forceinline__ void pool_store(PoolSlots<kPoint, kMono>& P, int s, const PathState& st,
                                           float sig_o) {
  using F = PoolF<kMono>;
  P.f[F::kDir][s] = st.dir.x; P.f[F::kDir + 1][s] = st.dir.y; P.f[F::kDir + 2][s] = st.dir.z;
  P.f[F::kT][s] = st.T.x;
  P.f[F::kL][s] = st.L.x;
  if constexpr (!kMono) {
    P.f[F::kT + 1][s] = st.T.y; P.f[F::kT + 2][s] = st.T.z;
    P.f[F::kL + 1][s] = st.L.y; P.f[F::kL + 2][s] = st.L.z;
  }
  P.f[F::kSigO][s] = sig_o;
  P.f[F::kUrr][s] = st.u_rr; P.f[F::kLphi][s] = st.lphi;
  P.f[F::kU][s] = st.u_br;  P.f[F::kU + 1][s] = st.u_s2;
  P.f[F::kPz][s] = st.pos.z;
  if constexpr (kPoint) {
    P.f[F::kPxy][s] = st.pos.x; P.f[F::kPxy + 1][s] = st.pos.y;
  }
  P.u[0][s] = st.pid;   P.u[1][s] = st.rng.pixel; P.u[2][s] = st.rng.sample;
  P.u[3][s] = (uint32_t)st.bounce;
}

// kMono: the three channels of T and L are set to the one stored value; only
// channel x is stored back and written out, so the y / z arithmetic is dead
// code the compiler removes
template <bool kPoint, bool kMono>
__device__ __forceinline__ void pool_load(const PoolSlots<kPoint, kMono>& P, int s,
                                          const PassDev& ps, PathState& st, float& sig_o) {
  using F = PoolF<kMono>;
  st.dir = v3(P.f[F::kDir][s], P.f[F::kDir + 1][s], P.f[F::kDir + 2][s]);
  if constexpr (kMono) {
    float t = P.f[F::kT][s], l = P.f[F::kL][s];
    st.T = v3(t, t, t);
    st.L = v3(l, l, l);
  } else {
    st.T = v3(P.f[F::kT][s], P.f[F::kT + 1][s], P.f[F::kT + 2][s]);
    st.L = v3(P.f[F::kL][s], P.f[F::kL + 1][s], P.f[F::kL + 2][s]);
  }
  sig_o = P.f[F::kSigO][s];
  st.u_rr = P.f[F::kUrr][s];
  st.lphi = P.f[F::kLphi][s];
  st.u_br = P.f[F::kU][s];
  st.u_s2 = P.f[F::kU + 1][s];
  // x, y are never read without a point light (a single plane is
  // translation invariant)
  if constexpr (kPoint) st.pos = v3(P.f[F::kPxy][s], P.f[F::kPxy + 1][s], P.f[F::kPz][s]);
  else st.pos = v3(0.0f, 0.0f, P.f[F::kPz][s]);
  st.pid = P.u[0][s];
  st.rng.k0 = ps.k0;
  st.rng.k1 = ps.k1;
  st.rng.pixel = P.u[1][s];
  st.rng.sample = P.u[2][s];
  st.bounce = (int)P.u[3][s];
  st.pre = false;
}

// next-event estimation at a collision of the single plane (the stage-2
// block of scatter_stages<0>, same arithmetic); kPoint: the scene has a point
// light (its code is compiled out otherwise).  The plane frame is the
// identity (frame_about(0,0,1) = (1,0,0),(0,1,0),(0,0,1)), so directions are
// used as they are.  With the collision's log Phi known, the sun's closed-form
// transmittance (planar_shadow_tr) reduces to clamping it to the band and one
// exponential: the sun end is a band edge fixed per render.
template <bool kPoint, int kSpec, bool kMono = false>
__device__ __forceinline__ void planar_nee(const SceneDev& sc, PathState& st, Counters& cn,
                                           V3 wo, float sig_o, V3 pos) {
  const MediumK& m = sc.media[0];
  if (sc.has_sun) {
    V3 ph = phase_eval<kSpec, true>(m, wo, sc.sun_to, sig_o);
    // grey: the three channels are equal, x decides
    if (kMono ? ph.x > 0.0f : (ph.x > 0.0f || ph.y > 0.0f || ph.z > 0.0f)) {
      cn.v[kStNee]++;
      float tr = planar_sun_tr(sc, st.lphi, pos);
      st.L = add3(st.L, v3(st.T.x * ph.x * sc.sun_L.x * tr, st.T.y * ph.y * sc.sun_L.y * tr,
                           st.T.z * ph.z * sc.sun_L.z * tr));
    }
  }
  if (kPoint && sc.has_point) {
    int nee = 0;
    st.L = add3(st.L, planar_point_nee(sc, st, wo, sig_o, pos, &nee));
    cn.v[kStNee] += (uint32_t)nee;
  }
}

template <bool kPoint, bool kMono, int kSpec>
__global__ void __launch_bounds__(kBlock, kPoolMinBlocks) pool_kernel(const __grid_constant__ SceneDev sc,
                                                                  const __grid_constant__ PassDev ps) {
  __shared__ PoolSlots<kPoint, kMono> pools[kWarpsPerBlock];
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  PoolSlots<kPoint, kMono>& P = pools[threadIdx.x >> 5];
  const MediumK& m = sc.media[0];
  Counters cn;
#pragma unroll
  for (int i = 0; i < kStCount; ++i) cn.v[i] = 0;
  auto finish = [&](const PathState& q) {
    // grey scenes (kMono): channel x only, ps.mono is set
    if constexpr (kMono) accumulate_fx(ps, q.pid, q.L.x, cn);
    else finish_path<false>(ps, q, cn);
  };
#pragma unroll
  for (int w = 0; w < kPoolWords; ++w) P.ring[kTagEmpty][w * 32 + lane] = (uint8_t)(w * 32 + lane);
  __syncwarp();
  // ring heads / tails (warp-uniform): every slot starts empty
  unsigned he = 0, hb = 0, hh = 0, te = kPool, tb = 0, th = 0;
  bool exhausted = false;    // warp-uniform
  while (true) {
    int ne = exhausted ? 0 : (int)(te - he), nb = (int)(tb - hb), nh = (int)(th - hh);
    // a full warp of one visit kind if any; else the largest partial one
    int stage;
    if (nb >= 32) stage = kStageBeck;
    else if (nh >= 32) stage = kStageHemi;
    else if (ne >= 32) stage = kStageRaygen;
    else if (nb > 0 && nb >= nh) stage = kStageBeck;
    else if (nh > 0) stage = kStageHemi;
    else if (ne > 0) stage = kStageRaygen;
    else break;
    // pop up to 32 slots of the visit's ring, the i-th to lane i
    int cnt = stage == kStageBeck ? nb : (stage == kStageHemi ? nh : ne);
    unsigned head = stage == kStageBeck ? hb : (stage == kStageHemi ? hh : he);
    int n = cnt < 32 ? cnt : 32;
    int slot = lane < n ? (int)P.ring[stage][(head + (unsigned)lane) & (kRing - 1)] : -1;
    if (stage == kStageBeck) hb += (unsigned)n;
    else if (stage == kStageHemi) hh += (unsigned)n;
    else he += (unsigned)n;

    uint8_t tag = kTagEmpty;
    PathState st;
    float sig_o = 0.0f, sig_b = 0.0f;
    bool fly = false;
    if (stage == kStageRaygen) {
      // raygen, full width: path indices with one atomicAdd
      unsigned need = __ballot_sync(full, slot >= 0);
      unsigned base = 0;
      if (lane == 0) base = atomicAdd(ps.counter, (unsigned)__popc(need));
      base = __shfl_sync(full, base, 0);
      if (base + (unsigned)__popc(need) >= ps.n_paths) exhausted = true;
      uint32_t my = base + (uint32_t)lane;
      if (slot >= 0 && my < ps.n_paths && start_path<false>(sc, ps, st, my)) {
        cn.v[kStPaths]++;
        fly = true;
      }
    } else if (slot >= 0) {
      pool_load<kPoint, kMono>(P, slot, ps, st, sig_o);
      V3 v = neg3(st.dir);   // the plane frame is the identity
      // next-event estimation of the collision (scatter_stages<0> stage 2)
      planar_nee<kPoint, kSpec, kMono>(sc, st, cn, st.dir, sig_o, st.pos);
      // the visible normal of the visit's mixture branch (phase_sample,
      // two-uniform convention; ndf.py:358-380)
      float uu = remap_branch_uniform_render(st.u_br, m);
      // Beckmann guide area of wo (the mixture pdf's sigma_b), here at full
      // width; a B slot without a guide (sigma_b <= 1e-12) takes the
      // hemisphere branch, as phase_sample does
      sig_b = (kSpec == kSpecBeckAlbedo || (kSpec == kSpecRuntime && m.kind == kBeckmann))
                  ? sig_o : proj_area_erf<true>(st.dir, m.ax, m.ay, 0.0f);
      V3 wm;
      float vm;
      if (stage == kStageBeck && sig_b > 1e-12f) {
        int iters = 0;
        wm = beckmann_visible_normal<kRenderSlopeGuard, true>(m, v, uu, st.u_s2, &iters);
        vm = dot3(v, wm);
        cn.v[kStSlopeIters] += (uint32_t)iters;
      } else {
        wm = hemisphere_about(v, uu, st.u_s2);
        vm = uu;   // z of wm in v's frame, exactly
      }
      // stage 3 of scatter_stages<0>: phase tail, depth cap, RR
      PhaseSample smp = phase_sample_tail<kSpec, true>(m, v, wm, vm, sig_o, sig_b, sig_b > 1e-12f);
      st.dir = smp.wi;
      st.T = v3(st.T.x * smp.weight.x, st.T.y * smp.weight.y, st.T.z * smp.weight.z);
      st.bounce++;
      bool done = false;
      if (st.bounce >= ps.max_bounces) {             // render.py:92-94
        done = true;
      } else if (st.bounce > 8) {                    // render.py:96-105
        float q = kMono ? fminf(st.T.x, 1.0f) : fminf(fmaxf(st.T.x, fmaxf(st.T.y, st.T.z)), 1.0f);
        if (st.u_rr >= q) {
          done = true;
        } else {
          st.T = mul3(st.T, 1.0f / q);
        }
      }
      if (done) finish(st);
      else fly = true;
    }
    __syncwarp();
    if (fly) {
      // flight and the mixture branch (scatter_stages<0> up to the branch;
      // the NEE runs in the next visit)
      if (!flight_stage<0, kSpec, kPoint ? 1 : 0>(sc, ps, st, cn)) {
        finish(st);
      } else {
        sig_o = st.csig;
        st.pos = st.cpos;
        cn.v[kStScatters]++;
        if (!(sig_o >= 1e-12f)) {
          cn.v[kStDegenerate]++;
          finish(st);
        } else {
          tag = st.u_br < m.mix ? kTagBeck : kTagHemi;
        }
      }
    }
    if (slot >= 0 && tag != kTagEmpty) pool_store<kPoint, kMono>(P, slot, st, sig_o);
    // push every processed slot onto the ring of its new tag
    {
      unsigned me = __ballot_sync(full, slot >= 0 && tag == kTagEmpty);
      unsigned mb = __ballot_sync(full, slot >= 0 && tag == kTagBeck);
      unsigned mh = __ballot_sync(full, slot >= 0 && tag == kTagHemi);
      if (slot >= 0) {
        unsigned mine = tag == kTagEmpty ? me : (tag == kTagBeck ? mb : mh);
        unsigned tail = tag == kTagEmpty ? te : (tag == kTagBeck ? tb : th);
        P.ring[tag][(tail + (unsigned)__popc(mine & lt)) & (kRing - 1)] = (uint8_t)slot;
      }
      te += (unsigned)__popc(me);
      tb += (unsigned)__popc(mb);
      th += (unsigned)__popc(mh);
    }
    __syncwarp();
  }
#pragma unroll
  for (int i = 0; i < kStCount; ++i) {
    unsigned v = __reduce_add_sync(full, cn.v[i]);
    if (lane == 0 && v) atomicAdd(ps.stats + i, (unsigned long long)v);
  }
}

// Path pool for one sphere (config 3) or a grid field (config 5, kMode 2):
// pool_kernel's slot rings and visit
// kinds (R raygen + flight; B / H: NEE, the Beckmann / hemisphere visible
// normal, the phase tail, depth cap / RR, the next flight) with the curved
// shell's pieces: the local frame about the collision point's normal, NEE
// with ratio-tracked shadow rays (curved_nee, sphere_walk) and the
// tangent-majorant flight (flight_stage<3>) or the grid walker.  Every path
// runs the megakernel's arithmetic on the same random stream and makes the
// same decisions (identical event counts); the sphere image is
// bit-identical to path_kernel<3> (MF_MEGAKERNEL=1), the grid image agrees
// to float rounding (~1e-5 relative in a few percent of pixels: the
// compiler contracts a few multiply-adds differently in the two inlining
// contexts).  The slot layout is pool_kernel's with a
// point light (positions stored).
#ifndef MF_SPHERE_POOL_MIN_BLOCKS
#define MF_SPHERE_POOL_MIN_BLOCKS 7
#endif
#ifndef MF_GRID_POOL_MIN_BLOCKS
#define MF_GRID_POOL_MIN_BLOCKS 6   // config 5: 3.60 -> 3.48 ms against 7
#endif
// The medium and local frame at a collision point: the sphere's medium and
// the frame about its normal (kMode 3), or the grid field's medium from
// sigma(p) and the frame about the trilinear SDF gradient (kMode 2) -- the
// same operations as scatter_stage<kMode>
template <int kMode>
struct CollisionLocal;

template <>
struct CollisionLocal<3> {
  const MediumK& m;
  Frame fr;
  __device__ __forceinline__ CollisionLocal(const SceneDev& sc, V3 pos)
      : m(sc.media[0]), fr(frame_about(prim_normal<true>(sc.prims[0], pos))) {}
};

template <>
struct CollisionLocal<2> {
  MediumK m;
  Frame fr;
  __device__ __forceinline__ CollisionLocal(const SceneDev& sc, V3 pos) {
    TriSample fs = trilinear<true>(sc.grid.sdf, sc.grid.n_sdf,
                                   grid_coord(sc.grid, pos, sc.grid.inv_h_sdf), sc.grid.inv_h_sdf);
    float sg = fmaxf(grid_sigma(sc.grid, pos), 1e-6f);
    m = grid_medium(sc.media[0], sg, sc.grid.k_xy, sc.grid.k_z);
    float gn2 = dot3(fs.grad, fs.grad);
    V3 nrm = gn2 > 0.0f ? mul3(fs.grad, frsqrt(gn2)) : v3(0.0f, 0.0f, 1.0f);
    fr = frame_about(nrm);
  }
};

template <int kMode, bool kMono, int kSpec>
__global__ void __launch_bounds__(kBlock, kMode == 2 ? MF_GRID_POOL_MIN_BLOCKS
                                                     : MF_SPHERE_POOL_MIN_BLOCKS) curved_pool_kernel(
    const __grid_constant__ SceneDev sc, const __grid_constant__ PassDev ps) {
  __shared__ PoolSlots<true, kMono> pools[kWarpsPerBlock];
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  PoolSlots<true, kMono>& P = pools[threadIdx.x >> 5];
  Counters cn;
#pragma unroll
  for (int i = 0; i < kStCount; ++i) cn.v[i] = 0;
  auto finish = [&](const PathState& q) {
    if constexpr (kMono) accumulate_fx(ps, q.pid, q.L.x, cn);
    else finish_path<false>(ps, q, cn);
  };
#pragma unroll
  for (int w = 0; w < kPoolWords; ++w) P.ring[kTagEmpty][w * 32 + lane] = (uint8_t)(w * 32 + lane);
  __syncwarp();
  unsigned he = 0, hb = 0, hh = 0, te = kPool, tb = 0, th = 0;
  bool exhausted = false;
  while (true) {
    int ne = exhausted ? 0 : (int)(te - he), nb = (int)(tb - hb), nh = (int)(th - hh);
    int stage;
    if (nb >= 32) stage = kStageBeck;
    else if (nh >= 32) stage = kStageHemi;
    else if (ne >= 32) stage = kStageRaygen;
    else if (nb > 0 && nb >= nh) stage = kStageBeck;
    else if (nh > 0) stage = kStageHemi;
    else if (ne > 0) stage = kStageRaygen;
    else break;
    int cnt = stage == kStageBeck ? nb : (stage == kStageHemi ? nh : ne);
    unsigned head = stage == kStageBeck ? hb : (stage == kStageHemi ? hh : he);
    int n = cnt < 32 ? cnt : 32;
    int slot = lane < n ? (int)P.ring[stage][(head + (unsigned)lane) & (kRing - 1)] : -1;
    if (stage == kStageBeck) hb += (unsigned)n;
    else if (stage == kStageHemi) hh += (unsigned)n;
    else he += (unsigned)n;

    uint8_t tag = kTagEmpty;
    PathState st;
    float sig_o = 0.0f;
    bool fly = false;
    if (stage == kStageRaygen) {
      unsigned need = __ballot_sync(full, slot >= 0);
      unsigned base = 0;
      if (lane == 0) base = atomicAdd(ps.counter, (unsigned)__popc(need));
      base = __shfl_sync(full, base, 0);
      if (base + (unsigned)__popc(need) >= ps.n_paths) exhausted = true;
      uint32_t my = base + (uint32_t)lane;
      if (slot >= 0 && my < ps.n_paths && start_path<false>(sc, ps, st, my)) {
        cn.v[kStPaths]++;
        fly = true;
      }
    } else if (slot >= 0) {
      pool_load<true, kMono>(P, slot, ps, st, sig_o);
      // scatter_stages<kMode> at the stored collision: frame, NEE, phase sample
      CollisionLocal<kMode> loc(sc, st.pos);
      const MediumK& m = loc.m;
      const Frame& fr = loc.fr;
      V3 wo = to_local(fr, st.dir);
      curved_nee<kMode, kSpec, true>(sc, st, cn, m, fr, wo, sig_o, st.pos);
      V3 v = neg3(wo);
      float uu = remap_branch_uniform_render(st.u_br, m);
      float sig_b = (kSpec == kSpecBeckAlbedo || (kSpec == kSpecRuntime && m.kind == kBeckmann))
                        ? sig_o : proj_area_erf<true>(wo, m.ax, m.ay, 0.0f);
      V3 wm;
      float vm;
      if (stage == kStageBeck && sig_b > 1e-12f) {
        int iters = 0;
        wm = beckmann_visible_normal<kRenderSlopeGuard, true>(m, v, uu, st.u_s2, &iters);
        vm = dot3(v, wm);
        cn.v[kStSlopeIters] += (uint32_t)iters;
      } else {
        wm = hemisphere_about(v, uu, st.u_s2);
        vm = uu;
      }
      PhaseSample smp = phase_sample_tail<kSpec, true>(m, v, wm, vm, sig_o, sig_b,
                                                              sig_b > 1e-12f);
      st.dir = to_world(fr, smp.wi);
      st.T = v3(st.T.x * smp.weight.x, st.T.y * smp.weight.y, st.T.z * smp.weight.z);
      st.bounce++;
      bool done = false;
      if (st.bounce >= ps.max_bounces) {             // render.py:92-94
        done = true;
      } else if (st.bounce > 8) {                    // render.py:96-105
        float q = kMono ? fminf(st.T.x, 1.0f) : fminf(fmaxf(st.T.x, fmaxf(st.T.y, st.T.z)), 1.0f);
        if (st.u_rr >= q) {
          done = true;
        } else {
          st.T = mul3(st.T, 1.0f / q);
        }
      }
      if (done) finish(st);
      else fly = true;
    }
    __syncwarp();
    if (fly) {
      if (!flight_stage<kMode, kSpec, -1, true>(sc, ps, st, cn)) {
        finish(st);
      } else {
        // the collision's medium, frame and sigma(wo), as scatter_stages
        st.pos = st.cpos;
        CollisionLocal<kMode> loc(sc, st.pos);
        sig_o = proj_area<kSpec, true>(loc.m, to_local(loc.fr, st.dir));
        cn.v[kStScatters]++;
        if (!(sig_o >= 1e-12f)) {
          cn.v[kStDegenerate]++;
          finish(st);
        } else {
          tag = st.u_br < loc.m.mix ? kTagBeck : kTagHemi;
        }
      }
    }
    if (slot >= 0 && tag != kTagEmpty) pool_store<true, kMono>(P, slot, st, sig_o);
    {
      unsigned me = __ballot_sync(full, slot >= 0 && tag == kTagEmpty);
      unsigned mb = __ballot_sync(full, slot >= 0 && tag == kTagBeck);
      unsigned mh = __ballot_sync(full, slot >= 0 && tag == kTagHemi);
      if (slot >= 0) {
        unsigned mine = tag == kTagEmpty ? me : (tag == kTagBeck ? mb : mh);
        unsigned tail = tag == kTagEmpty ? te : (tag == kTagBeck ? tb : th);
        P.ring[tag][(tail + (unsigned)__popc(mine & lt)) & (kRing - 1)] = (uint8_t)slot;
      }
      te += (unsigned)__popc(me);
      tb += (unsigned)__popc(mb);
      th += (unsigned)__popc(mh);
    }
    __syncwarp();
  }
#pragma unroll
  for (int i = 0; i < kStCount; ++i) {
    unsigned v = __reduce_add_sync(full, cn.v[i]);
    if (lane == 0 && v) atomicAdd(ps.stats + i, (unsigned long long)v);
  }
}

// ---------------------------------------------------------------------------
// Grid-field path pool with pooled walks (config 5; sun / environment
// lighting).  In curved_pool_kernel<2> a lane runs a whole flight or shadow
// walk inside its visit: ncu showed the tentative collisions (two trilinear
// fetches, Mills ratio, projected area: 2/3 of the issue slots) at 4 active
// lanes and the DDA at 8, because the lanes of a warp reach their tentative
// collisions at different cells and finish their walks at different
// lengths.  Here a walk is a pool citizen of its own: a fourth ring (W)
// holds slots whose path waits on a walk -- the shadow ray of its last
// collision, then the flight of its next segment -- and a W visit advances
// up to 32 of them together, alternating two re-converged phases: DDA
// steps for the lanes that have no tentative collision pending, until most
// have one; then the tentative collisions of all pending lanes at once.
// When fewer than a fraction of the visit's walks remain, the unfinished
// ones are parked (GridPark: t, tau, weight, cell, steps -- five words; the
// walker recomputes everything else from the ray) and rejoin the ring, so
// the next W visit starts full again.  B / H visits do the collision's
// local medium / frame, sigma(wo), the NEE phase value, the normal and the
// phase sample, depth cap / RR and the next segment's uniforms, and queue
// the shadow walk; the walk's end adds contribution x transmittance and
// queues the flight.  Per path the arithmetic and the random stream are
// those of path_kernel<2> / curved_pool_kernel<2> (same GridWalker calls on
// the same Philox blocks), so images agree to float rounding
// (test_grid_walk_pool_matches_curved_pool).
#ifndef MF_GRID_WALK_POOL_MIN_BLOCKS
#define MF_GRID_WALK_POOL_MIN_BLOCKS 6
#endif
// leave the DDA phase when stepping lanes * kGwNum <= pending lanes * kGwDen
#ifndef MF_GW_NUM
#define MF_GW_NUM 1
#endif
#ifndef MF_GW_DEN
#define MF_GW_DEN 1
#endif
// park the visit's unfinished walks when fewer than kGwExit / 8 of them remain
#ifndef MF_GW_EXIT
#define MF_GW_EXIT 4
#endif
// slots per warp of the grid pool
#ifndef MF_GRID_POOL
#define MF_GRID_POOL 96
#endif
constexpr int kGPool = MF_GRID_POOL;
static_assert(kGPool % 32 == 0 && kGPool <= kRing, "grid pool size: whole warps of slots");
constexpr int kStageWalk = 3;
constexpr uint8_t kTagWalk = 3;
constexpr uint32_t kGwShadow = 1u << 16, kGwDone = 1u << 17, kGwFresh = 1u << 18;

template <bool kMono>
struct GridPoolF {
  static constexpr int kC = kMono ? 1 : 3;
  static constexpr int kDir = 0, kPos = 3, kT = 6, kL = 6 + kC, kNee = 6 + 2 * kC,
                       kUrr = 6 + 3 * kC, kUbr = kUrr + 1, kUs2 = kUrr + 2, kWt = kUrr + 3,
                       kWtau = kUrr + 4, kWw = kUrr + 5, kCount = kUrr + 6;
};
template <bool kMono>
struct GridPoolSlots {
  float f[GridPoolF<kMono>::kCount][kGPool];
  uint32_t u[6][kGPool];   // pid pixel sample bounce|flags cell steps
  uint8_t ring[4][kRing];
};

template <bool kMono, int kSpec>
__global__ void __launch_bounds__(kBlock, MF_GRID_WALK_POOL_MIN_BLOCKS) grid_pool_kernel(
    const __grid_constant__ SceneDev sc, const __grid_constant__ PassDev ps) {
  using F = GridPoolF<kMono>;
  __shared__ GridPoolSlots<kMono> pools[kWarpsPerBlock];
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  GridPoolSlots<kMono>& P = pools[threadIdx.x >> 5];
  Counters cn;
#pragma unroll
  for (int i = 0; i < kStCount; ++i) cn.v[i] = 0;
  auto load3 = [&](int f0, int s) { return v3(P.f[f0][s], P.f[f0 + 1][s], P.f[f0 + 2][s]); };
  auto store3 = [&](int f0, int s, V3 v) {
    P.f[f0][s] = v.x; P.f[f0 + 1][s] = v.y; P.f[f0 + 2][s] = v.z;
  };
  auto loadc = [&](int f0, int s) {
    if constexpr (kMono) {
      float t = P.f[f0][s];
      return v3(t, t, t);
    } else {
      return load3(f0, s);
    }
  };
  auto storec = [&](int f0, int s, V3 v) {
    P.f[f0][s] = v.x;
    if constexpr (!kMono) { P.f[f0 + 1][s] = v.y; P.f[f0 + 2][s] = v.z; }
  };
  auto finish = [&](uint32_t pid, V3 L) {
    if constexpr (kMono) {
      accumulate_fx(ps, pid, L.x, cn);
    } else {
      accumulate_fx(ps, pid * 3u, L.x, cn);
      accumulate_fx(ps, pid * 3u + 1u, L.y, cn);
      accumulate_fx(ps, pid * 3u + 2u, L.z, cn);
    }
  };
#pragma unroll
  for (int w = 0; w < kGPool / 32; ++w) P.ring[kTagEmpty][w * 32 + lane] = (uint8_t)(w * 32 + lane);
  __syncwarp();
  unsigned head[4] = {0, 0, 0, 0}, tail[4] = {kGPool, 0, 0, 0};
  bool exhausted = false;
  while (true) {
    int ne = exhausted ? 0 : (int)(tail[0] - head[0]);
    int nb = (int)(tail[1] - head[1]), nh = (int)(tail[2] - head[2]), nw = (int)(tail[3] - head[3]);
    int stage;
    if (nw >= 32) stage = kStageWalk;
    else if (nb >= 32) stage = kStageBeck;
    else if (nh >= 32) stage = kStageHemi;
    else if (ne >= 32) stage = kStageRaygen;
    else {
      int best = nw;
      stage = kStageWalk;
      if (nb > best) { best = nb; stage = kStageBeck; }
      if (nh > best) { best = nh; stage = kStageHemi; }
      if (ne > best) { best = ne; stage = kStageRaygen; }
      if (best == 0) break;
    }
    int cnt = stage == kStageWalk ? nw : (stage == kStageBeck ? nb : (stage == kStageHemi ? nh : ne));
    unsigned hd = stage == kStageWalk ? head[3]
                                      : (stage == kStageBeck ? head[1]
                                                             : (stage == kStageHemi ? head[2] : head[0]));
    int n = cnt < 32 ? cnt : 32;
    int slot = lane < n ? (int)P.ring[stage][(hd + (unsigned)lane) & (kRing - 1)] : -1;
    if (stage == kStageWalk) head[3] += (unsigned)n;
    else if (stage == kStageBeck) head[1] += (unsigned)n;
    else if (stage == kStageHemi) head[2] += (unsigned)n;
    else head[0] += (unsigned)n;

    uint8_t tag = kTagEmpty;
    if (stage == kStageRaygen) {
      unsigned need = __ballot_sync(full, slot >= 0);
      unsigned base = 0;
      if (lane == 0) base = atomicAdd(ps.counter, (unsigned)__popc(need));
      base = __shfl_sync(full, base, 0);
      if (base + (unsigned)__popc(need) >= ps.n_paths) exhausted = true;
      uint32_t my = base + (uint32_t)lane;
      PathState st;
      if (slot >= 0 && my < ps.n_paths && start_path<false>(sc, ps, st, my)) {
        cn.v[kStPaths]++;
        cn.v[kStSegments]++;
        store3(F::kDir, slot, st.dir);
        store3(F::kPos, slot, st.pos);
        storec(F::kT, slot, st.T);
        storec(F::kL, slot, st.L);
        P.f[F::kUrr][slot] = st.u_rr;
        P.f[F::kUbr][slot] = st.u_br;
        P.f[F::kUs2][slot] = st.u_s2;
        P.u[0][slot] = st.pid;
        P.u[1][slot] = st.rng.pixel;
        P.u[2][slot] = st.rng.sample;
        P.u[3][slot] = kGwFresh;   // bounce 0, flight
        tag = kTagWalk;
      }
    } else if (stage == kStageWalk) {
      // ---- W visit: advance up to 32 walks ----
      uint32_t pix = 0, smp = 0, seg = 0, bfl = 0;
      auto rb = [&](uint32_t call) { return philox_rk(U4{pix, smp, seg, call}, ps.rk); };
      GridWalker<decltype(rb)> W(rb);
      // lane state: 0 stepping (DDA), 1 a tentative collision pending, 2 the
      // DDA ended the walk, 4 a tentative collision ended it, 3 no walk
      int ls = 3;
      bool shadow = false;
      if (slot >= 0) {
        bfl = P.u[3][slot];
        pix = P.u[1][slot];
        smp = P.u[2][slot];
        shadow = (bfl & kGwShadow) != 0;
        uint32_t bounce = bfl & 0xFFFFu;
        V3 o = load3(F::kPos, slot);
        V3 d = shadow ? sc.sun_to : load3(F::kDir, slot);
        // the shadow ray belongs to the segment that ended in the collision
        seg = shadow ? bounce - 1u : bounce;
        uint32_t call0 = shadow ? kCallShadow : 1u;
        float rr = shadow ? kShadowRR : 0.0f;
        ls = 0;
        if (bfl & kGwFresh) {
          if (!W.begin(sc.grid, call0, o, d, shadow, INFINITY, rr)) ls = 4;   // missed the grid
        } else {
          GridPark pk{P.f[F::kWt][slot], P.f[F::kWtau][slot], P.f[F::kWw][slot], P.u[4][slot],
                      (int)P.u[5][slot]};
          W.resume(sc.grid, call0, o, d, shadow, INFINITY, rr, pk);
        }
      }
      const int n0 = __popc(__ballot_sync(full, ls == 0));
      int nact = n0;
      while (true) {
        // DDA phase: lanes without a pending tentative collision step on,
        // until kGwNum / (kGwNum + kGwDen) of the phase's lanes have one (or
        // have ended)
        const int stop = nact * MF_GW_DEN;
        while (true) {
          if (ls == 0) ls = W.dda(sc.grid);
          if (__popc(__ballot_sync(full, ls == 0)) * (MF_GW_NUM + MF_GW_DEN) <= stop) break;
        }
        // tentative collisions of every pending lane
        if (ls == 1) ls = W.tentative(sc.grid, sc.media[0]) ? 4 : 0;
        nact = __popc(__ballot_sync(full, ls == 0));
        if (nact * 8 < n0 * MF_GW_EXIT || nact == 0) break;
      }
      if (ls == 2) W.end_at(W.t);
      const bool active = ls == 0, ended = ls == 2 || ls == 4;
      if (active) {
        // park the unfinished walk
        GridPark pk = W.park();
        cn.v[kStViolations] += (uint32_t)W.w.violations;
        P.f[F::kWt][slot] = pk.t;
        P.f[F::kWtau][slot] = pk.tau;
        P.f[F::kWw][slot] = pk.weight;
        P.u[4][slot] = pk.cell;
        P.u[5][slot] = (uint32_t)pk.steps;
        P.u[3][slot] = bfl & ~kGwFresh;
        tag = kTagWalk;
      } else if (ended) {
        const GridWalk& w = W.w;
        cn.v[kStTrackSteps] += (uint32_t)max(w.steps, 0);
        cn.v[kStViolations] += (uint32_t)w.violations;
        if (shadow) {
          if (w.steps < 0) cn.v[kStCapped]++;   // iteration cap: raised by the host
          float tr = w.steps < 0 ? 0.0f : w.weight;
          V3 c = loadc(F::kNee, slot), L = loadc(F::kL, slot);
          L = add3(L, v3(c.x * tr, c.y * tr, c.z * tr));
          if (bfl & kGwDone) {
            finish(P.u[0][slot], L);
          } else {
            storec(F::kL, slot, L);
            P.u[3][slot] = (bfl & 0xFFFFu) | kGwFresh;   // the next segment's flight
            cn.v[kStSegments]++;
            tag = kTagWalk;
          }
        } else {
          int outcome = w.steps < 0 ? -1 : w.outcome;
          if (outcome == kCollided) {
            store3(F::kPos, slot, w.pos);
            tag = P.f[F::kUbr][slot] < sc.media[0].mix ? kTagBeck : kTagHemi;
          } else {
            V3 L = loadc(F::kL, slot);
            if (outcome == kEscaped) {
              V3 T = loadc(F::kT, slot);
              V3 e = env_radiance(sc, W.dir);   // render.py:54-57
              L = add3(L, v3(T.x * e.x, T.y * e.y, T.z * e.z));
              cn.v[kStEscaped]++;
            } else if (outcome == kAbsorbed) {
              cn.v[kStAbsorbed]++;
            } else {
              cn.v[kStCapped]++;
            }
            finish(P.u[0][slot], L);
          }
        }
      }
    } else if (slot >= 0) {
      // ---- B / H visit: the collision's scatter stages up to the walks ----
      PathState st;
      st.dir = load3(F::kDir, slot);
      st.pos = load3(F::kPos, slot);
      st.T = loadc(F::kT, slot);
      st.L = loadc(F::kL, slot);
      st.u_rr = P.f[F::kUrr][slot];
      st.u_br = P.f[F::kUbr][slot];
      st.u_s2 = P.f[F::kUs2][slot];
      uint32_t pid = P.u[0][slot], pix = P.u[1][slot], smp = P.u[2][slot];
      st.bounce = (int)(P.u[3][slot] & 0xFFFFu);
      CollisionLocal<2> loc(sc, st.pos);
      const MediumK& m = loc.m;
      const Frame& fr = loc.fr;
      V3 wo = to_local(fr, st.dir);
      float sig_o = proj_area<kSpec, true>(m, wo);
      cn.v[kStScatters]++;
      if (!(sig_o >= 1e-12f)) {
        cn.v[kStDegenerate]++;
        finish(pid, st.L);
      } else {
        // NEE towards the sun: the phase value now, the transmittance by the
        // queued shadow walk
        bool want_shadow = false;
        V3 nee = v3(0.0f, 0.0f, 0.0f);
        if (sc.has_sun) {
          V3 wl = to_local(fr, sc.sun_to);
          V3 ph = phase_eval<kSpec, true>(m, wo, wl, sig_o);
          if (ph.x > 0.0f || ph.y > 0.0f || ph.z > 0.0f) {
            cn.v[kStNee]++;
            nee = v3(st.T.x * ph.x * sc.sun_L.x, st.T.y * ph.y * sc.sun_L.y,
                     st.T.z * ph.z * sc.sun_L.z);
            // curved_nee's roulette on a small contribution (same block)
            want_shadow = kNeeRR <= 0.0f ||
                          nee_roulette(nee, sc.sun_L,
                                       kNeeRR > 0.0f
                                           ? philox_rk(U4{pix, smp, (uint32_t)st.bounce, kCallNeeRR},
                                                       ps.rk).x
                                           : 0u);
          }
        }
        V3 v = neg3(wo);
        float uu = remap_branch_uniform_render(st.u_br, m);
        float sig_b = (kSpec == kSpecBeckAlbedo || (kSpec == kSpecRuntime && m.kind == kBeckmann))
                          ? sig_o : proj_area_erf<true>(wo, m.ax, m.ay, 0.0f);
        V3 wm;
        float vm;
        if (stage == kStageBeck && sig_b > 1e-12f) {
          int iters = 0;
          wm = beckmann_visible_normal<kRenderSlopeGuard, true>(m, v, uu, st.u_s2, &iters);
          vm = dot3(v, wm);
          cn.v[kStSlopeIters] += (uint32_t)iters;
        } else {
          wm = hemisphere_about(v, uu, st.u_s2);
          vm = uu;
        }
        PhaseSample smpl = phase_sample_tail<kSpec, true>(m, v, wm, vm, sig_o, sig_b,
                                                         sig_b > 1e-12f);
        st.dir = to_world(fr, smpl.wi);
        st.T = v3(st.T.x * smpl.weight.x, st.T.y * smpl.weight.y, st.T.z * smpl.weight.z);
        st.bounce++;
        bool done = false;
        if (st.bounce >= ps.max_bounces) {             // render.py:92-94
          done = true;
        } else if (st.bounce > 8) {                    // render.py:96-105
          float q = kMono ? fminf(st.T.x, 1.0f) : fminf(fmaxf(st.T.x, fmaxf(st.T.y, st.T.z)), 1.0f);
          if (st.u_rr >= q) {
            done = true;
          } else {
            st.T = mul3(st.T, 1.0f / q);
          }
        }
        if (done && !want_shadow) {
          finish(pid, st.L);
        } else {
          uint32_t fl = (uint32_t)st.bounce;
          if (!done) {
            // the next segment's uniforms (flight_stage's block)
            U4 b = philox_rk(U4{pix, smp, (uint32_t)st.bounce, 0u}, ps.rk);
            P.f[F::kUbr][slot] = u01(b.y);
            P.f[F::kUs2][slot] = u01(b.z);
            P.f[F::kUrr][slot] = u01(b.w);
            store3(F::kDir, slot, st.dir);
            storec(F::kT, slot, st.T);
          } else {
            fl |= kGwDone;
          }
          if (want_shadow) {
            storec(F::kNee, slot, nee);
            fl |= kGwShadow;
          } else {
            cn.v[kStSegments]++;
          }
          P.u[3][slot] = fl | kGwFresh;
          tag = kTagWalk;
        }
      }
    }
    __syncwarp();
    {
      unsigned m0 = __ballot_sync(full, slot >= 0 && tag == kTagEmpty);
      unsigned m1 = __ballot_sync(full, slot >= 0 && tag == kTagBeck);
      unsigned m2 = __ballot_sync(full, slot >= 0 && tag == kTagHemi);
      unsigned m3 = __ballot_sync(full, slot >= 0 && tag == kTagWalk);
      if (slot >= 0) {
        unsigned mine = tag == kTagEmpty ? m0 : (tag == kTagBeck ? m1 : (tag == kTagHemi ? m2 : m3));
        unsigned tl = tag == kTagEmpty ? tail[0]
                                       : (tag == kTagBeck ? tail[1] : (tag == kTagHemi ? tail[2] : tail[3]));
        P.ring[tag][(tl + (unsigned)__popc(mine & lt)) & (kRing - 1)] = (uint8_t)slot;
      }
      tail[0] += (unsigned)__popc(m0);
      tail[1] += (unsigned)__popc(m1);
      tail[2] += (unsigned)__popc(m2);
      tail[3] += (unsigned)__popc(m3);
    }
    __syncwarp();
  }
#pragma unroll
  for (int i = 0; i < kStCount; ++i) {
    unsigned v = __reduce_add_sync(full, cn.v[i]);
    if (lane == 0 && v) atomicAdd(ps.stats + i, (unsigned long long)v);
  }
}

// fixed-point pixel sums -> the caller's fp32 image (render.py:165-166):
// one thread per local pixel, sum * 2^-k / spp in double, added to (or
// written into) accum[pixel][c]
__global__ void __launch_bounds__(256) finalize_kernel(const __grid_constant__ SceneDev sc,
                                                        const __grid_constant__ PassDev ps,
                                                        uint32_t n_pix, double inv_scale_spp,
                                                        int add, float* accum) {
  uint32_t pixel = blockIdx.x * blockDim.x + threadIdx.x;
  if (pixel >= n_pix) return;
  float* a = accum + (size_t)pixel * 3;
  int64_t lp = pixel_to_local(sc, ps, pixel);
  if (lp < 0) {                     // another rank's tile
    if (!add) a[0] = a[1] = a[2] = 0.0f;
    return;
  }
  float t[3];
  if (ps.mono) {
    t[0] = t[1] = t[2] = (float)((double)ps.fx[lp] * inv_scale_spp);
  } else {
#pragma unroll
    for (int c = 0; c < 3; ++c) t[c] = (float)((double)ps.fx[(size_t)lp * 3 + c] * inv_scale_spp);
  }
  float v0 = t[0], v1 = t[1], v2 = t[2];
  if (add) {
    v0 += a[0];
    v1 += a[1];
    v2 += a[2];
  }
  a[0] = v0;
  a[1] = v1;
  a[2] = v2;
  // RadianceImage.validate (image.py:38-42) of the stored value (an added
  // caller value may be anything)
  if (!(isfinite(v0) && isfinite(v1) && isfinite(v2)) || v0 < 0.0f || v1 < 0.0f || v2 < 0.0f)
    atomicAdd(ps.stats + kStNonfinite, 1ull);
}

// ratio-tracking transmittance samples (transport.py:300-313)
__global__ void __launch_bounds__(kBlock) ratio_kernel(const __grid_constant__ SceneDev sc,
                                                        uint32_t k0, uint32_t k1, uint32_t stream_lo,
                                                        V3 org, V3 dir, uint32_t n, float* w_out,
                                                        unsigned long long* stats) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t steps = 0, viol = 0, capped = 0;
  if (i < n) {
    PathRng rng{k0, k1, stream_lo, i};
    if (sc.has_grid) {
      GridWalk w = grid_walk(sc.grid, sc.media[0],
                             [&](uint32_t call) { return rng_block(rng, 0u, call); },
                             kCallShadow, org, dir, true, INFINITY);
      w_out[i] = w.weight;
      steps = (uint32_t)max(w.steps, 0);
      viol = (uint32_t)w.violations;
      capped = w.steps < 0 ? 1u : 0u;
    } else {
      WalkResult w = walk(sc, rng, 0u, kCallShadow, org, dir, true, INFINITY);
      w_out[i] = w.weight;
      steps = (uint32_t)max(w.steps, 0);
      viol = (uint32_t)w.violations;
      capped = w.steps < 0 ? 1u : 0u;
    }
  }
  unsigned a = __reduce_add_sync(0xffffffffu, steps);
  unsigned b = __reduce_add_sync(0xffffffffu, viol);
  unsigned c = __reduce_add_sync(0xffffffffu, capped);
  if ((threadIdx.x & 31) == 0) {
    if (a) atomicAdd(stats + kStTrackSteps, (unsigned long long)a);
    if (b) atomicAdd(stats + kStViolations, (unsigned long long)b);
    if (c) atomicAdd(stats + kStCapped, (unsigned long long)c);
  }
}

// walk() / sample_collision() for caller-given rays (transport.py:144-297,
// 316-416): one thread per ray, the tracking walker (grid walker for grid
// fields) on the ray's own Philox stream
struct WalkArgs {
  const float *org, *dir;
  const uint32_t *pix, *smp;
  uint32_t k0, k1, segment;
  int mode;
  uint32_t n;
  int8_t* state;
  float *pos, *travel, *weight;
  int32_t* prim;
  unsigned long long* stats;
};

__global__ void __launch_bounds__(kBlock) walk_kernel(const __grid_constant__ SceneDev sc,
                                                       const __grid_constant__ WalkArgs a) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t steps = 0, viol = 0, capped = 0;
  if (i < a.n) {
    PathRng rng{a.k0, a.k1, a.pix[i], a.smp[i]};
    V3 o = v3(a.org[i], a.org[a.n + i], a.org[2u * a.n + i]);
    V3 d = v3(a.dir[i], a.dir[a.n + i], a.dir[2u * a.n + i]);
    bool ratio = a.mode == MF_WALK_RATIO;
    uint32_t call0 = ratio ? kCallShadow : 1u;
    int outcome, prim = -1;
    V3 pos;
    float weight, travel;
    if (sc.has_grid) {
      GridWalk w = grid_walk_path(sc.grid, sc.media[0], rng, a.segment, call0, o, d, ratio,
                                  INFINITY, 0.0f);
      outcome = w.steps < 0 ? kAbsorbed : w.outcome;
      prim = outcome == kCollided ? 0 : -1;
      pos = w.pos;
      weight = w.weight;
      travel = dot3(sub3(w.pos, o), d);
      steps = (uint32_t)max(w.steps, 0);
      viol = (uint32_t)w.violations;
      capped = w.steps < 0 ? 1u : 0u;
    } else {
      // a single sphere uses the renderer's tangent-majorant walker
      bool one_sphere = sc.n_prims == 1 && sc.prims[0].shape == kShapeSphere &&
                        a.mode != MF_WALK_TENTATIVE;
      WalkResult w = one_sphere ? sphere_walk(sc, rng, a.segment, call0, o, d, ratio, INFINITY)
                                : walk(sc, rng, a.segment, call0, o, d, ratio, INFINITY, 0.0f,
                                       a.mode == MF_WALK_TENTATIVE);
      outcome = w.outcome;
      prim = (outcome == kCollided || outcome == kNullCollision) ? w.prim : -1;
      pos = w.pos;
      weight = w.weight;
      travel = w.travel;
      steps = (uint32_t)max(w.steps, 0);
      viol = (uint32_t)w.violations;
      capped = w.steps < 0 ? 1u : 0u;
    }
    if (a.state) a.state[i] = (int8_t)outcome;
    if (a.pos) {
      a.pos[i] = pos.x;
      a.pos[a.n + i] = pos.y;
      a.pos[2u * a.n + i] = pos.z;
    }
    if (a.travel) a.travel[i] = travel;
    if (a.weight) a.weight[i] = weight;
    if (a.prim) a.prim[i] = prim;
  }
  unsigned s0 = __reduce_add_sync(0xffffffffu, steps);
  unsigned s1 = __reduce_add_sync(0xffffffffu, viol);
  unsigned s2 = __reduce_add_sync(0xffffffffu, capped);
  unsigned s3 = __reduce_add_sync(0xffffffffu, i < a.n ? 1u : 0u);
  if ((threadIdx.x & 31) == 0) {
    if (s0) atomicAdd(a.stats + kStTrackSteps, (unsigned long long)s0);
    if (s1) atomicAdd(a.stats + kStViolations, (unsigned long long)s1);
    if (s2) atomicAdd(a.stats + kStCapped, (unsigned long long)s2);
    if (s3) atomicAdd(a.stats + kStPaths, (unsigned long long)s3);
  }
}

// largest value of a lat-long environment map (the fixed-point scale of a
// render must cover it); non-negative floats order like their bit patterns
__global__ void __launch_bounds__(256) env_max_kernel(const float* m, size_t n, unsigned* out) {
  float v = 0.0f;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    float x = __ldg(m + i);
    v = (x == x) ? fmaxf(v, fabsf(x)) : INFINITY;
  }
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 16));
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 8));
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 4));
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(v));
}

// ---------------------------------------------------------------------------
// visible-slope guess table (built once per device by the solver itself)

__global__ void __launch_bounds__(128) slope_table_kernel(float* tab) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < kTabNT * kTabNU) tab[k] = slope_table_node(k / kTabNU, k % kTabNU);
}

// ---------------------------------------------------------------------------
// grid-field majorant (one thread per cell)

__global__ void __launch_bounds__(128) grid_majorant_kernel(const __grid_constant__ GridDev g,
                                                             float* out) {
  int n = g.n_maj;
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n * n * n) return;
  int cx = c / (n * n), cy = (c / n) % n, cz = c % n;
  out[c] = grid_cell_majorant(g, cx, cy, cz);
}

// second pass: empty cells store -(distance to medium) (grid_cell_skip);
// in place is safe -- only the sign of a neighbour is read
__global__ void __launch_bounds__(128) grid_skip_kernel(float* maj, int n) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n * n * n) return;
  maj[c] = grid_cell_skip(maj, n, c / (n * n), (c / n) % n, c % n);
}

// ---------------------------------------------------------------------------
// roofline microbenchmarks: 8 independent FFMA chains / 4 MUFU.EX2 chains

// erf / erfc / exp(-x) in float64 (CUDA's correctly-rounded-to-a-few-ulp
// double functions; erf(-x) = -erf(x) exactly as the reference's)
__global__ void __launch_bounds__(256) special_f64_kernel(int which, const double* x, int64_t n,
                                                          double* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = x[i];
  out[i] = which == 0 ? copysign(erf(fabs(v)), v) : (which == 1 ? erfc(v) : exp(-v));
}

// one piece of the radial gradient-distribution quadrature per block, one
// Gauss-Legendre node per lane (float64), warp-reduced in node order
struct GdfRadial {
  double a, b, c, shift, half;
  int n_sub;
  double x[32], w[32];
};

__global__ void __launch_bounds__(32) gdf_radial_kernel(const __grid_constant__ GdfRadial g,
                                                        double* piece) {
  int p = blockIdx.x, k = threadIdx.x;
  double mid = (2.0 * p + 1.0) * g.half;
  double t = mid + g.half * g.x[k];
  double f = t * t * t * exp(-(g.a * t * t - 2.0 * g.b * t + g.c) - g.shift) * g.w[k];
  for (int o = 16; o > 0; o >>= 1) f += __shfl_down_sync(0xffffffffu, f, o);
  if (k == 0) piece[p] = f;
}

__global__ void __launch_bounds__(256) peak_ffma_kernel(float* out, int iters, float a, float b) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  float x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  float s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 123.456f) out[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) peak_mufu_kernel(float* out, int iters) {
  float x0 = threadIdx.x * -1e-6f, x1 = x0 - 0.1f, x2 = x0 - 0.2f, x3 = x0 - 0.3f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x0));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x1));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x2));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x3));
    }
  }
  float s = x0 + x1 + x2 + x3;
  if (s == 123.456f) out[threadIdx.x] = s;
}

// ---------------------------------------------------------------------------
// host side

// device pointer of this device's slope table (built on first use)
int slope_table(const float** out, cudaStream_t st) {
  static std::mutex mu;
  static float* tabs[64] = {nullptr};
  int dev = 0;
  MF_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (dev >= 64) return fail(MF_ERR_CUDA, "device index out of range");
  if (!tabs[dev]) {
    float* t = nullptr;
    MF_CUDA(cudaMalloc((void**)&t, (size_t)kTabNT * kTabNU * sizeof(float)));
    slope_table_kernel<<<(kTabNT * kTabNU + 127) / 128, 128, 0, st>>>(t);
    g_launches++;
    MF_CUDA(cudaGetLastError());
    MF_CUDA(cudaStreamSynchronize(st));
    tabs[dev] = t;
  }
  *out = tabs[dev];
  return MF_OK;
}

// The render kernels' sigma(w) tables (area_q_build), one per distinct
// roughness triple and device, uploaded once and kept for the process.
int area_table(const MediumK& m, const float4** out) {
  static std::mutex mu;
  static std::map<std::tuple<int, float, float, float, int>, const float4*> cache;
  int dev = 0;
  MF_CUDA(cudaGetDevice(&dev));
  auto key = std::make_tuple(m.kind, m.ax, m.ay, m.az, dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it == cache.end()) {
    std::vector<float4> q(kAreaQN);
    float4* d = nullptr;
    if (area_q_build(m, q.data())) {
      MF_CUDA(cudaMalloc((void**)&d, kAreaQN * sizeof(float4)));
      MF_CUDA(cudaMemcpy(d, q.data(), kAreaQN * sizeof(float4), cudaMemcpyHostToDevice));
    }
    it = cache.emplace(key, d).first;
  }
  *out = it->second;
  return MF_OK;
}

int attach_slope_table(SceneDev* sc, cudaStream_t st) {
  const float* tab = nullptr;
  int rc = slope_table(&tab, st);
  if (rc) return rc;
  for (int j = 0; j < kMaxPrims; ++j) sc->media[j].slope_tab = tab;
  // sigma(w) tables for the render kernels (not for grid fields, whose
  // roughness follows sigma(p))
  const char* e = std::getenv("MF_AREA_TABLE");   // =0: the formula (A/B test hook)
  if (!sc->has_grid && !(e && e[0] == '0')) {
    for (int j = 0; j < sc->n_prims && j < kMaxPrims; ++j) {
      rc = area_table(sc->media[j], &sc->media[j].area_q);
      if (rc) return rc;
    }
  }
  return MF_OK;
}

struct Occupancy {
  int sms = 0;
  int blocks[32] = {};
};

template <bool kPoint, bool kMono, int kSpec>
cudaError_t occ_pool(int* blocks) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, pool_kernel<kPoint, kMono, kSpec>,
                                                       kBlock, 0);
}

template <bool kPoint, bool kMono, int kSpec>
void launch_pool(int grid, const SceneDev& sc, const PassDev& ps, cudaStream_t st) {
  pool_kernel<kPoint, kMono, kSpec><<<grid, kBlock, 0, st>>>(sc, ps);
}

// the curved pools' GENERALIZED + albedo build.  (With the NDF out of line
// the kernel is 4 % smaller, but its time moves by +-5 % with where ptxas
// places the callee -- the kernel sits at the instruction-cache limit --
// so the inline build is kept.)
constexpr int kCurvedSpec = kSpecGenAlbedo;

template <int kMode, bool kMono, int kSpec>
cudaError_t occ_curved(int* blocks) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks,
                                                       curved_pool_kernel<kMode, kMono, kSpec>,
                                                       kBlock, 0);
}

// the curved pool (one sphere: kMode 3, grid field: kMode 2) for the scene:
// kSpec 1 when the medium is GENERALIZED with albedo Fresnel (the grid
// field's local media always are GENERALIZED), which folds the NDF /
// projected-area / Fresnel dispatch away
void launch_curved_pool(int mode, const SceneDev& sc, const PassDev& ps, const Occupancy& occ,
                        int64_t need, cudaStream_t st) {
  bool gen = mode == 2 || sc.media[0].kind == kGeneralized;
  int spec = gen && sc.media[0].fresnel == kAlbedo ? 1 : 0;
  int pk = 20 + (mode == 2 ? 2 : 0) + (sc.mono ? 1 : 0) + 4 * spec;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)occ.sms * occ.blocks[pk], need));
  using K = void (*)(SceneDev, PassDev);
  static const K ks[8] = {curved_pool_kernel<3, false, 0>, curved_pool_kernel<3, true, 0>,
                          curved_pool_kernel<2, false, 0>, curved_pool_kernel<2, true, 0>,
                          curved_pool_kernel<3, false, kCurvedSpec>,
                          curved_pool_kernel<3, true, kCurvedSpec>,
                          curved_pool_kernel<2, false, kCurvedSpec>,
                          curved_pool_kernel<2, true, kCurvedSpec>};
  ks[pk - 20]<<<grid, kBlock, 0, st>>>(sc, ps);
}

int device_occupancy(Occupancy* occ) {
  static std::mutex mu;
  static Occupancy cache[64];
  static bool have[64] = {false};
  int dev = 0;
  MF_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && have[dev]) {
    *occ = cache[dev];
    return MF_OK;
  }
  Occupancy o;
  MF_CUDA(cudaDeviceGetAttribute(&o.sms, cudaDevAttrMultiProcessorCount, dev));
  MF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.blocks[0], path_kernel<0, false>,
                                                        kBlock, 0));
  MF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.blocks[1], path_kernel<1, false>,
                                                        kBlock, 0));
  MF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.blocks[2], path_kernel<2, false>,
                                                        kBlock, 0));
  MF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.blocks[3], path_kernel<0, true>,
                                                        kBlock, 0));
  MF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.blocks[4], path_kernel<1, true>,
                                                        kBlock, 0));
  MF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.blocks[5], path_kernel<2, true>,
                                                        kBlock, 0));
  // single-sphere megakernel (mode 3): blocks[14] / [15] (caller rays)
  MF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.blocks[14], path_kernel<3, false>,
                                                        kBlock, 0));
  MF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.blocks[15], path_kernel<3, true>,
                                                        kBlock, 0));
  // pool kernels: blocks[6 + point + 2 mono + 4 spec]; spec 2 at [16..19]
  MF_CUDA((occ_pool<false, false, 0>(&o.blocks[6])));
  MF_CUDA((occ_pool<true, false, 0>(&o.blocks[7])));
  MF_CUDA((occ_pool<false, true, 0>(&o.blocks[8])));
  MF_CUDA((occ_pool<true, true, 0>(&o.blocks[9])));
  MF_CUDA((occ_pool<false, false, 1>(&o.blocks[10])));
  MF_CUDA((occ_pool<true, false, 1>(&o.blocks[11])));
  MF_CUDA((occ_pool<false, true, 1>(&o.blocks[12])));
  MF_CUDA((occ_pool<true, true, 1>(&o.blocks[13])));
  // curved pools: blocks[20 + 2 (mode == 2) + mono + 4 spec]
  MF_CUDA((occ_curved<3, false, 0>(&o.blocks[20])));
  MF_CUDA((occ_curved<3, true, 0>(&o.blocks[21])));
  MF_CUDA((occ_curved<2, false, 0>(&o.blocks[22])));
  MF_CUDA((occ_curved<2, true, 0>(&o.blocks[23])));
  MF_CUDA((occ_curved<3, false, kCurvedSpec>(&o.blocks[24])));
  MF_CUDA((occ_curved<3, true, kCurvedSpec>(&o.blocks[25])));
  MF_CUDA((occ_curved<2, false, kCurvedSpec>(&o.blocks[26])));
  MF_CUDA((occ_curved<2, true, kCurvedSpec>(&o.blocks[27])));
  // grid path pool with pooled walks: blocks[28 + mono + 2 spec]
  MF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.blocks[28], grid_pool_kernel<false, 0>, kBlock, 0));
  MF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.blocks[29], grid_pool_kernel<true, 0>, kBlock, 0));
  MF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.blocks[30], grid_pool_kernel<false, kCurvedSpec>, kBlock, 0));
  MF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.blocks[31], grid_pool_kernel<true, kCurvedSpec>, kBlock, 0));
  MF_CUDA((occ_pool<false, false, 2>(&o.blocks[16])));
  MF_CUDA((occ_pool<true, false, 2>(&o.blocks[17])));
  MF_CUDA((occ_pool<false, true, 2>(&o.blocks[18])));
  MF_CUDA((occ_pool<true, true, 2>(&o.blocks[19])));
  for (int& b : o.blocks) b = std::max(b, 1);
  if (dev < 64) {
    cache[dev] = o;
    have[dev] = true;
  }
  *occ = o;
  return MF_OK;
}

void fill_stats(const unsigned long long* h, mf_stats* s) {
  s->path_kernel_ms = 0.0;
  s->paths = h[kStPaths];
  s->segments = h[kStSegments];
  s->scatters = h[kStScatters];
  s->nee = h[kStNee];
  s->slope_iters = h[kStSlopeIters];
  s->track_steps = h[kStTrackSteps];
  s->escaped = h[kStEscaped];
  s->absorbed = h[kStAbsorbed];
  s->majorant_violations = h[kStViolations];
  s->degenerate = h[kStDegenerate];
  s->nonfinite = h[kStNonfinite];
  s->capped = h[kStCapped];
}

int check_stats(const mf_stats& s) {
  if (s.majorant_violations)
    return fail(MF_ERR_MAJORANT, "extinction exceeded its majorant (" +
                                     std::to_string(s.majorant_violations) + " events)");
  if (s.capped) return fail(MF_ERR_CAP, "walker exceeded its iteration cap");
  if (s.nonfinite)
    return fail(MF_ERR_NUMERIC, "non-finite, negative or out-of-range (above 2^20 x the "
                                "brightest emitter) radiance in " +
                                    std::to_string(s.nonfinite) + " paths / pixels");
  return MF_OK;
}

// scratch: per-pixel fixed-point sums, work counter, stats
struct Scratch {
  unsigned long long* fx = nullptr;
  unsigned int* counter = nullptr;
  unsigned long long* stats = nullptr;
};

// The device's default stream-ordered pool releases freed memory back to the
// driver at every synchronisation unless told otherwise; re-mapping the
// ~50 MB of per-path scratch then costs milliseconds per render.  Keep it.
int retain_pool_memory() {
  static std::mutex mu;
  static bool done[64] = {false};
  int dev = 0;
  MF_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && done[dev]) return MF_OK;
  cudaMemPool_t pool;
  MF_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t keep = UINT64_MAX;
  MF_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  if (dev < 64) done[dev] = true;
  return MF_OK;
}

// one stream-ordered block, zeroed with one memset: stats (kStCount u64,
// padded to 256 B), the work counters (64 u32) and the pixel sums
int scratch_alloc(Scratch* s, size_t n_fx, cudaStream_t st) {
  int rc = retain_pool_memory();
  if (rc) return rc;
  static_assert(kStCount * sizeof(unsigned long long) <= 256, "stats block");
  size_t bytes = 512 + n_fx * sizeof(unsigned long long);
  char* base = nullptr;
  MF_CUDA(cudaMallocAsync((void**)&base, bytes, st));
  MF_CUDA(cudaMemsetAsync(base, 0, bytes, st));
  s->stats = (unsigned long long*)base;
  s->counter = (unsigned int*)(base + 256);
  s->fx = n_fx ? (unsigned long long*)(base + 512) : nullptr;
  return MF_OK;
}

int scratch_free(Scratch* s, cudaStream_t st) {
  if (s->stats) MF_CUDA(cudaFreeAsync(s->stats, st));
  *s = Scratch();
  return MF_OK;
}

bool megakernel_requested() {
  const char* e = std::getenv("MF_MEGAKERNEL");
  return e && e[0] == '1';
}

int launch_paths(const SceneDev& sc_in, const PassDev& ps, bool caller_rays, cudaStream_t st) {
  Occupancy occ;
  int rc = device_occupancy(&occ);
  if (rc) return rc;
  SceneDev sc = sc_in;
  // modes: 0 single plane, 1 general shells, 2 grid field, 3 one sphere
  // MF_GENERIC_WALK=1: the general tracking walker for a single sphere
  // (mode 1), =2: the single-sphere instantiation of that walker (mode 3 with
  // sc.generic_walk) instead of the tangent-majorant sphere_walk
  const char* gw = std::getenv("MF_GENERIC_WALK");
  bool generic = gw && gw[0] == '1';
  sc.generic_walk = gw && gw[0] == '2';
  int mode = sc.has_grid ? 2
                         : (sc.single_plane ? 0
                                            : (sc.n_prims == 1 && sc.prims[0].shape == kShapeSphere &&
                                                       !generic
                                                   ? 3
                                                   : 1));
  int grid = occ.sms * (mode == 3 ? occ.blocks[caller_rays ? 15 : 14]
                                  : occ.blocks[mode + (caller_rays ? 3 : 0)]);
  int64_t need = ((int64_t)ps.n_paths + kBlock - 1) / kBlock;
  grid = (int)std::max<int64_t>(1, std::min<int64_t>(grid, need));
  if (mode == 0) {
    if (caller_rays) path_kernel<0, true><<<grid, kBlock, 0, st>>>(sc, ps);
#ifndef MF_NO_POOL
    // MF_MEGAKERNEL=1 selects the lane-per-path megakernel instead (the
    // pool's bit-exactness test compares the two)
    else if (megakernel_requested()) path_kernel<0, false><<<grid, kBlock, 0, st>>>(sc, ps);
    else {
      int spec = sc.media[0].fresnel != kAlbedo ? 0
                 : (sc.media[0].kind == kGeneralized ? 1 : (sc.media[0].kind == kBeckmann ? 2 : 0));
      int v = (sc.has_point ? 1 : 0) + (sc.mono ? 2 : 0);
      int pk = spec == 2 ? 16 + v : 6 + v + (spec ? 4 : 0);
      grid = (int)std::max<int64_t>(1, std::min<int64_t>(occ.sms * occ.blocks[pk], need));
      using L = void (*)(int, const SceneDev&, const PassDev&, cudaStream_t);
      static const L pools[12] = {launch_pool<false, false, 0>, launch_pool<true, false, 0>,
                                  launch_pool<false, true, 0>,  launch_pool<true, true, 0>,
                                  launch_pool<false, false, 1>, launch_pool<true, false, 1>,
                                  launch_pool<false, true, 1>,  launch_pool<true, true, 1>,
                                  launch_pool<false, false, 2>, launch_pool<true, false, 2>,
                                  launch_pool<false, true, 2>,  launch_pool<true, true, 2>};
      pools[spec * 4 + v](grid, sc, ps, st);
    }
#else
    else path_kernel<0, false><<<grid, kBlock, 0, st>>>(sc, ps);
#endif
  } else if (mode == 1) {
    if (caller_rays) path_kernel<1, true><<<grid, kBlock, 0, st>>>(sc, ps);
    else path_kernel<1, false><<<grid, kBlock, 0, st>>>(sc, ps);
  } else if (mode == 3) {
    if (caller_rays) path_kernel<3, true><<<grid, kBlock, 0, st>>>(sc, ps);
    else if (megakernel_requested() || sc.generic_walk) path_kernel<3, false><<<grid, kBlock, 0, st>>>(sc, ps);
    else {
      // the sphere path pool (MF_MEGAKERNEL=1: the megakernel, for the
      // bit-exactness test)
      launch_curved_pool(3, sc, ps, occ, need, st);
    }
  } else {
    if (caller_rays) path_kernel<2, true><<<grid, kBlock, 0, st>>>(sc, ps);
    else if (megakernel_requested()) path_kernel<2, false><<<grid, kBlock, 0, st>>>(sc, ps);
    else {
      // the grid-field path pools (MF_MEGAKERNEL=1: the megakernel): pooled
      // walks unless a point light needs per-path shadow directions
      // (MF_GRID_WALK_POOL=0: walks inside the visits, for the comparison test)
      const char* gp = std::getenv("MF_GRID_WALK_POOL");
      if (sc.has_point || ps.max_bounces > 0xFFFF || sc.grid.n_maj > 1024 || (gp && gp[0] == '0')) {
        launch_curved_pool(2, sc, ps, occ, need, st);
      } else {
        int spec = sc.media[0].fresnel == kAlbedo ? 1 : 0;
        int pk = 28 + (sc.mono ? 1 : 0) + 2 * spec;
        int g2 = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)occ.sms * occ.blocks[pk], need));
        using K = void (*)(SceneDev, PassDev);
        static const K ks[4] = {grid_pool_kernel<false, 0>, grid_pool_kernel<true, 0>,
                                grid_pool_kernel<false, kCurvedSpec>,
                                grid_pool_kernel<true, kCurvedSpec>};
        ks[pk - 28]<<<g2, kBlock, 0, st>>>(sc, ps);
      }
    }
  }
  g_launches++;
  MF_CUDA(cudaGetLastError());
  return MF_OK;
}

// paths per launch: path indices are 32-bit (one launch covers a whole
// render unless it exceeds this; the fixed-point sums carry across launches)
constexpr size_t kMaxPassPaths = size_t(1) << 31;

// Fixed-point scale 2^k of the pixel sums (accumulate_fx) for a render of
// `spp` samples per pixel whose brightest emitter (environment, sun, point
// light channel) is e_max: each path may carry up to 2^20 e_max of radiance
// and the sum of spp of them stays below 2^63.  Returns k and the per-path
// limit of L * 2^k.
void fx_scale(double e_max, uint64_t spp, float* scale, float* limit, int* k_out) {
  int lg_s = 0;
  while (lg_s < 62 && (uint64_t(1) << lg_s) < spp) ++lg_s;
  int lg_e = (int)std::ceil(std::log2(std::max(e_max, 1e-30)));
  int k = 63 - lg_s - 20 - lg_e;
  k = std::max(-100, std::min(100, k));
  *scale = std::ldexp(1.0f, k);
  *limit = std::ldexp(1.0f, 63 - lg_s);
  *k_out = k;
}

double scene_emax(const SceneDev& sc) {
  double e = std::max({(double)sc.env.x, (double)sc.env.y, (double)sc.env.z});
  if (sc.has_sun) e = std::max({e, (double)sc.sun_L.x, (double)sc.sun_L.y, (double)sc.sun_L.z});
  if (sc.has_point)
    e = std::max({e, (double)sc.point_I.x, (double)sc.point_I.y, (double)sc.point_I.z});
  return e;
}

}  // namespace

// A queued render (mf_render_async): its read-back block of event
// counters (pinned host memory, recycled), the completion event and the
// path-kernel timing events.
struct mf_render_ticket {
  bool empty = true;
  unsigned long long* h_stats = nullptr;
  cudaEvent_t done = nullptr;
  std::vector<cudaEvent_t> ev;
};

namespace {
std::mutex g_pinned_mu;
std::vector<unsigned long long*> g_pinned_free;

unsigned long long* pinned_stats_get() {
  {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    if (!g_pinned_free.empty()) {
      unsigned long long* p = g_pinned_free.back();
      g_pinned_free.pop_back();
      return p;
    }
  }
  void* p = nullptr;
  if (cudaHostAlloc(&p, 32 * sizeof(unsigned long long), cudaHostAllocDefault) != cudaSuccess)
    return nullptr;
  return (unsigned long long*)p;
}

void pinned_stats_put(unsigned long long* p) {
  std::lock_guard<std::mutex> lk(g_pinned_mu);
  g_pinned_free.push_back(p);
}
}  // namespace

extern "C" {

const char* mf_last_error(void) { return g_err.c_str(); }

int mf_grid_majorant(const mf_grid_field* grid, float* d_majorant_out, void* stream) {
  if (!grid || !d_majorant_out) return fail(MF_ERR_PARAM, "null argument");
  // reuse the scene builder's validation: a one-primitive grid scene
  mf_scene tmp;
  std::memset(&tmp, 0, sizeof(tmp));
  tmp.n_prims = 1;
  tmp.n_media = 1;
  tmp.prims[0].shape = MF_SHAPE_GRID;
  tmp.media[0].kind = MF_KIND_GENERALIZED;
  tmp.media[0].fresnel = MF_FRESNEL_ONE;
  tmp.media[0].ax = tmp.media[0].ay = tmp.media[0].az = 1.0;
  tmp.media[0].sigma = 1.0;
  tmp.media[0].mix_ratio = 0.5;
  tmp.camera.width = tmp.camera.height = 1;
  tmp.camera.look_at[2] = -1.0;
  tmp.has_grid = 1;
  tmp.grid = *grid;
  tmp.grid.d_majorant = d_majorant_out;
  SceneDev sc;
  std::string berr;
  int rc = build_scene(tmp, &sc, &berr);
  if (rc) return fail(rc, berr);
  int cells = grid->n_maj * grid->n_maj * grid->n_maj;
  grid_majorant_kernel<<<(cells + 127) / 128, 128, 0, (cudaStream_t)stream>>>(sc.grid,
                                                                              d_majorant_out);
  g_launches++;
  MF_CUDA(cudaGetLastError());
  grid_skip_kernel<<<(cells + 127) / 128, 128, 0, (cudaStream_t)stream>>>(d_majorant_out,
                                                                          grid->n_maj);
  g_launches++;
  MF_CUDA(cudaGetLastError());
  return MF_OK;
}

int mf_gp_camera_rays(const double pos[3], const double fwd[3], const double right[3],
                      const double up[3], double half_w, double half_h, int32_t width,
                      int32_t height, const uint64_t* d_bases, int32_t rounds, double* d_o,
                      double* d_d, void* stream) {
  if (!pos || !fwd || !right || !up || !d_bases || !d_o || !d_d || width < 1 || height < 1 ||
      rounds < 0)
    return fail(MF_ERR_PARAM, "bad gp_camera_rays arguments");
  mf::gp::CamRays c;
  for (int k = 0; k < 3; ++k) {
    c.pos[k] = pos[k];
    c.fwd[k] = fwd[k];
    c.right[k] = right[k];
    c.up[k] = up[k];
  }
  c.half_w = half_w;
  c.half_h = half_h;
  c.w = width;
  c.h = height;
  int64_t n = (int64_t)width * height * rounds;
  if (!n) return MF_OK;
  mf::gp::camera_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      c, d_bases, rounds, d_o, d_d);
  g_launches++;
  MF_CUDA(cudaGetLastError());
  return MF_OK;
}

int mf_gp_round_sum(const double* d_rad, int32_t width, int32_t height, int32_t rounds,
                    int32_t accumulate, double* d_img, void* stream) {
  if (!d_rad || !d_img || width < 1 || height < 1 || rounds < 1)
    return fail(MF_ERR_PARAM, "bad gp_round_sum arguments");
  int64_t hw = (int64_t)width * height;
  mf::gp::round_sum_kernel<<<(unsigned)((hw * 3 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      d_rad, hw, rounds, accumulate ? 1 : 0, d_img);
  g_launches++;
  MF_CUDA(cudaGetLastError());
  return MF_OK;
}

int mf_special_f64(int which, const double* d_x, int64_t n, double* d_out, void* stream) {
  if (which < 0 || which > 2) return fail(MF_ERR_PARAM, "unknown special function");
  if (n < 0 || (n > 0 && (!d_x || !d_out))) return fail(MF_ERR_PARAM, "bad special_f64 arguments");
  if (!n) return MF_OK;
  special_f64_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(which, d_x, n,
                                                                                   d_out);
  g_launches++;
  MF_CUDA(cudaGetLastError());
  return MF_OK;
}

int mf_gdf_radial(double a, double b, double c, double shift, double t_max, int32_t n_sub,
                  const double nodes[32], const double weights[32], double* total, void* stream) {
  if (!nodes || !weights || !total || n_sub < 1 || n_sub > 4096 || !(t_max > 0.0))
    return fail(MF_ERR_PARAM, "bad gdf_radial arguments");
  cudaStream_t st = (cudaStream_t)stream;
  GdfRadial g;
  g.a = a; g.b = b; g.c = c; g.shift = shift;
  g.half = 0.5 * t_max / n_sub;
  g.n_sub = n_sub;
  for (int k = 0; k < 32; ++k) {
    g.x[k] = nodes[k];
    g.w[k] = weights[k];
  }
  double* d = nullptr;
  MF_CUDA(cudaMallocAsync((void**)&d, (size_t)n_sub * sizeof(double), st));
  gdf_radial_kernel<<<n_sub, 32, 0, st>>>(g, d);
  g_launches++;
  MF_CUDA(cudaGetLastError());
  std::vector<double> h(n_sub);
  MF_CUDA(cudaMemcpyAsync(h.data(), d, (size_t)n_sub * sizeof(double), cudaMemcpyDeviceToHost, st));
  MF_CUDA(cudaStreamSynchronize(st));
  MF_CUDA(cudaFreeAsync(d, st));
  double s = 0.0;
  for (double v : h) s += v;   // pieces summed in order on the host
  *total = s * g.half;
  return MF_OK;
}

int mf_measure_peak_fp64(double* dfma_ginst_s, void* stream) {
  if (!dfma_ginst_s) return fail(MF_ERR_PARAM, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 0;
  MF_CUDA(cudaGetDevice(&dev));
  MF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* dummy = nullptr;
  MF_CUDA(cudaMallocAsync((void**)&dummy, 256 * sizeof(double), st));
  cudaEvent_t e0, e1;
  MF_CUDA(cudaEventCreate(&e0));
  MF_CUDA(cudaEventCreate(&e1));
  const int blocks = sms * 8, threads = 256, it = 2048;
  double best = 0.0;
  for (int rep = 0; rep < 3; ++rep) {
    MF_CUDA(cudaEventRecord(e0, st));
    mf::gp::peak_dfma_kernel<<<blocks, threads, 0, st>>>(dummy, it, 0.9999, 1e-4);
    MF_CUDA(cudaEventRecord(e1, st));
    MF_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    MF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    double nops = (double)blocks * threads * it * 8;
    if (rep) best = std::max(best, nops / (ms * 1e-3) / 1e9);
    g_launches++;
  }
  MF_CUDA(cudaGetLastError());
  MF_CUDA(cudaFreeAsync(dummy, st));
  MF_CUDA(cudaEventDestroy(e0));
  MF_CUDA(cudaEventDestroy(e1));
  *dfma_ginst_s = best;
  return MF_OK;
}

int mf_measure_peaks(double* fp32_ginst_s, double* sfu_ginst_s, void* stream) {
  if (!fp32_ginst_s || !sfu_ginst_s) return fail(MF_ERR_PARAM, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 0;
  MF_CUDA(cudaGetDevice(&dev));
  MF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  float* dummy = nullptr;
  MF_CUDA(cudaMallocAsync((void**)&dummy, 256 * sizeof(float), st));
  cudaEvent_t e0, e1;
  MF_CUDA(cudaEventCreate(&e0));
  MF_CUDA(cudaEventCreate(&e1));
  const int blocks = sms * 8, threads = 256;
  double best_f = 0.0, best_s = 0.0;
  for (int rep = 0; rep < 3; ++rep) {
    const int it_f = 4096;
    MF_CUDA(cudaEventRecord(e0, st));
    peak_ffma_kernel<<<blocks, threads, 0, st>>>(dummy, it_f, 0.9999f, 1e-4f);
    MF_CUDA(cudaEventRecord(e1, st));
    MF_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    MF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    double n = (double)blocks * threads * it_f * 16 * 8;
    if (rep) best_f = std::max(best_f, n / (ms * 1e-3) / 1e9);
    const int it_s = 1024;
    MF_CUDA(cudaEventRecord(e0, st));
    peak_mufu_kernel<<<blocks, threads, 0, st>>>(dummy, it_s);
    MF_CUDA(cudaEventRecord(e1, st));
    MF_CUDA(cudaEventSynchronize(e1));
    MF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    n = (double)blocks * threads * it_s * 16 * 4;
    if (rep) best_s = std::max(best_s, n / (ms * 1e-3) / 1e9);
    g_launches += 2;
  }
  MF_CUDA(cudaGetLastError());
  MF_CUDA(cudaFreeAsync(dummy, st));
  MF_CUDA(cudaEventDestroy(e0));
  MF_CUDA(cudaEventDestroy(e1));
  *fp32_ginst_s = best_f;
  *sfu_ginst_s = best_s;
  return MF_OK;
}
int mf_abi_version(void) { return MF_ABI_VERSION; }
uint64_t mf_launch_count(void) { return g_launches; }

int mf_query_batch(const mf_medium* medium, const mf_primitive* field, const mf_query_in* d_in,
                   const mf_query_out* d_out, int64_t n, void* stream) {
  if (!medium || !field || !d_in || !d_out) return fail(MF_ERR_PARAM, "null argument");
  if (n < 0) return fail(MF_ERR_PARAM, "n must be >= 0");
  QueryArgs a;
  std::memset(&a, 0, sizeof(a));
  std::string err;
  int rc = prepare_medium(*medium, &a.m, &err);
  if (rc) return fail(rc, err);
  PrimK pk;
  mf_primitive f = *field;
  f.medium = 0;
  rc = prepare_primitive(f, 1, &pk, &err);
  if (rc) return fail(rc, err);
  a.shape = pk.shape;
  a.z0 = pk.z0;
  a.c = v3(pk.cx, pk.cy, pk.cz);
  a.radius = pk.radius;
  a.in = *d_in;
  a.out = *d_out;
  a.n = n;
  if (n == 0) return MF_OK;
  {
    const float* tab = nullptr;
    rc = slope_table(&tab, (cudaStream_t)stream);
    if (rc) return rc;
    a.m.slope_tab = tab;
  }
  const float* req[] = {a.in.px, a.in.py, a.in.pz, a.in.wox, a.in.woy, a.in.woz,
                        a.in.wix, a.in.wiy, a.in.wiz, a.in.u1, a.in.u2};
  for (const float* p : req)
    if (!p) return fail(MF_ERR_PARAM, "query input array is null");
  int dev = 0, sms = 148;
  MF_CUDA(cudaGetDevice(&dev));
  MF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // two resident waves: every warp loops over many 32-query chunks, so its
  // Beckmann ring fills to full warps
  int per_sm = 1;
  bool normal = a.out.wmx || a.out.wmy || a.out.wmz || a.out.pdf_m;
  MF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &per_sm, normal ? query_kernel<true> : query_kernel<false>, kQBlock, 0));
  int64_t blocks = (n + kQBlock - 1) / kQBlock;
  int grid = (int)std::min<int64_t>(blocks, (int64_t)sms * std::max(per_sm, 1) * 2);
  if (normal) query_kernel<true><<<grid, kQBlock, 0, (cudaStream_t)stream>>>(a);
  else query_kernel<false><<<grid, kQBlock, 0, (cudaStream_t)stream>>>(a);
  g_launches++;
  MF_CUDA(cudaGetLastError());
  return MF_OK;
}

int mf_curve(const mf_medium* medium, int kind, const float* d_x, const float* d_y,
             const float* d_z, int64_t n, const double params[4], float* d_out, void* stream) {
  if (!medium || !params || (n > 0 && (!d_x || !d_out))) return fail(MF_ERR_PARAM, "null argument");
  if (kind < MF_CURVE_LAMBDA || kind > MF_CURVE_GDF)
    return fail(MF_ERR_PARAM, "unknown curve kind " + std::to_string(kind));
  bool scalar = kind == MF_CURVE_TRANSMITTANCE || kind == MF_CURVE_DENSITY || kind == MF_CURVE_FRESNEL;
  if (!scalar && n > 0 && (!d_y || !d_z))
    return fail(MF_ERR_PARAM, "direction arrays are null");
  if (n < 0) return fail(MF_ERR_PARAM, "n must be >= 0");
  CurveArgs a;
  std::memset(&a, 0, sizeof(a));
  std::string err;
  int rc = prepare_medium(*medium, &a.m, &err);
  if (rc) return fail(rc, err);
  a.kind = kind;
  a.x = d_x;
  a.y = d_y;
  a.z = d_z;
  a.n = n;
  a.out = d_out;
  double wx = params[0], wy = params[1], wz = params[2];
  double wn = std::sqrt(wx * wx + wy * wy + wz * wz);
  if (kind == MF_CURVE_VNDF || kind == MF_CURVE_TRANSMITTANCE) {
    if (!(wn > 0.0) || !std::isfinite(wn)) return fail(MF_ERR_PARAM, "wo must be a finite non-zero vector");
    wx /= wn;
    wy /= wn;
    wz /= wn;
  }
  a.wo = v3((float)wx, (float)wy, (float)wz);
  a.z0 = (float)params[3];
  if (kind == MF_CURVE_VNDF) {
    a.sig_wo = proj_area(a.m, a.wo);
    if (!(a.sig_wo >= 1e-12f))
      return fail(MF_ERR_DEGENERATE, "sigma(wo) < 1e-12: visible normals undefined");
  }
  if (kind == MF_CURVE_GDF && medium->kind != MF_KIND_GENERALIZED)
    return fail(MF_ERR_PARAM, "gdf_pdf requires az > 0");
  if (kind == MF_CURVE_TRANSMITTANCE) {
    if (std::fabs(wz) < 1e-12)
      return fail(MF_ERR_UNSUPPORTED, "planar transmittance is undefined at cos(theta) = 0");
    if (a.m.kind == kGGX)
      return fail(MF_ERR_UNSUPPORTED, "closed-form transmittance covers the erf-family lambda only");
    a.sig_wo = proj_area(a.m, a.wo) / a.wo.z;
  }
  if (n == 0) return MF_OK;
  int dev = 0, sms = 148;
  MF_CUDA(cudaGetDevice(&dev));
  MF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8);
  curve_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(a);
  g_launches++;
  MF_CUDA(cudaGetLastError());
  return MF_OK;
}

int mf_render_async(const mf_scene* scene, const mf_render_params* params, float* d_accum,
                    mf_render_ticket** ticket, void* stream) {
  if (!ticket) return fail(MF_ERR_PARAM, "null ticket");
  *ticket = nullptr;
  if (!scene || !params || !d_accum) return fail(MF_ERR_PARAM, "null argument");
  const mf_render_params& p = *params;
  if (p.spp < 1) return fail(MF_ERR_PARAM, "spp must be >= 1, got " + std::to_string(p.spp));
  if (p.max_bounces < 1)
    return fail(MF_ERR_PARAM, "max_bounces must be >= 1, got " + std::to_string(p.max_bounces));
  if (p.nranks < 1 || p.rank < 0 || p.rank >= p.nranks)
    return fail(MF_ERR_PARAM, "bad rank / nranks");
  if (p.shard != MF_SHARD_TILES && p.shard != MF_SHARD_SAMPLES)
    return fail(MF_ERR_PARAM, "unknown shard mode");
  if (p.shard == MF_SHARD_TILES && (p.tile < 1 || p.tile > 65535))
    return fail(MF_ERR_PARAM, "tile must lie in [1, 65535]");
  SceneDev sc;
  std::string berr;
  int rc = build_scene(*scene, &sc, &berr);
  if (rc) return fail(rc, berr);
  rc = attach_slope_table(&sc, (cudaStream_t)stream);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  size_t npix = (size_t)sc.width * sc.height;

  PassDev ps;
  std::memset(&ps, 0, sizeof(ps));
  ps.k0 = (uint32_t)(p.seed & 0xffffffffu);
  ps.k1 = (uint32_t)(p.seed >> 32);
  philox_round_keys(ps.k0, ps.k1, ps.rk);
  ps.max_bounces = p.max_bounces;
  ps.shard = p.shard;
  ps.rank = p.rank;
  ps.nranks = p.nranks;
  ps.tile = p.tile;
  ps.div_width = make_fastdiv((uint32_t)sc.width);
  ps.div_tile = make_fastdiv((uint32_t)std::max(p.tile, 1));
  ps.div_t2 = make_fastdiv((uint32_t)std::max(p.tile, 1) * (uint32_t)std::max(p.tile, 1));
  // local pixels and this rank's sample range
  size_t n_local;
  uint32_t s_begin = 0, s_count = (uint32_t)p.spp;
  if (p.shard == MF_SHARD_TILES) {
    int tx = (sc.width + p.tile - 1) / p.tile, ty = (sc.height + p.tile - 1) / p.tile;
    ps.tiles_x = tx;
    ps.div_tiles_x = make_fastdiv((uint32_t)tx);
    int n_tiles = tx * ty;
    int mine = n_tiles > p.rank ? (n_tiles - p.rank + p.nranks - 1) / p.nranks : 0;
    n_local = (size_t)mine * p.tile * p.tile;
  } else {
    n_local = npix;
    uint64_t a = (uint64_t)p.spp * p.rank / p.nranks, b = (uint64_t)p.spp * (p.rank + 1) / p.nranks;
    s_begin = (uint32_t)a;
    s_count = (uint32_t)(b - a);
  }
  if (n_local == 0 || s_count == 0) {
    *ticket = new mf_render_ticket();   // nothing to render: an empty ticket
    return MF_OK;
  }
  size_t max_pass = kMaxPassPaths;
  if (const char* e = std::getenv("MF_MAX_PASS_PATHS")) {   // test hook: force several launches
    long long v = std::atoll(e);
    if (v > 0) max_pass = std::min<size_t>(max_pass, (size_t)v);
  }
  uint32_t S_pass = (uint32_t)std::max<size_t>(1, std::min<size_t>(s_count, max_pass / n_local));
  if (n_local * S_pass > 0xffffffffull) return fail(MF_ERR_PARAM, "image too large for one pass");
  // grey scenes keep one channel per pixel (all kernels; channels are equal)
  ps.mono = sc.mono;
  ps.pixel_major = sc.single_plane ? 0 : 1;
  if (const char* e = std::getenv("MF_PATH_ORDER")) ps.pixel_major = e[0] == 'p' ? 1 : 0;
  size_t n_fx = n_local * (ps.mono ? 1 : 3);
  Scratch scr;
  rc = scratch_alloc(&scr, n_fx, st);
  if (rc) return rc;
  ps.fx = scr.fx;
  ps.counter = scr.counter;
  ps.stats = scr.stats;
  int k = 0;
  double emax = scene_emax(sc);
  if (sc.env_map) {
    size_t nm = (size_t)sc.env_w * sc.env_h * 3;
    MF_CUDA(cudaMemsetAsync(scr.counter + 32, 0, sizeof(unsigned), st));
    env_max_kernel<<<(unsigned)std::min<size_t>((nm + 255) / 256, 1024), 256, 0, st>>>(
        sc.env_map, nm, scr.counter + 32);
    g_launches++;
    MF_CUDA(cudaGetLastError());
    unsigned bits = 0;
    MF_CUDA(cudaMemcpyAsync(&bits, scr.counter + 32, sizeof(bits), cudaMemcpyDeviceToHost, st));
    MF_CUDA(cudaStreamSynchronize(st));
    float mx;
    std::memcpy(&mx, &bits, sizeof(mx));
    if (!std::isfinite(mx)) {
      scratch_free(&scr, st);
      return fail(MF_ERR_PARAM, "environment map holds non-finite values");
    }
    emax = std::max(emax, (double)mx);
  }
  fx_scale(emax, s_count, &ps.fx_scale, &ps.fx_limit, &k);
  // path-kernel timing: one event pair per launch, read after the final sync
  std::vector<cudaEvent_t> ev;
  for (uint32_t s0 = 0; s0 < s_count; s0 += S_pass) {
    uint32_t S = std::min(S_pass, s_count - s0);
    ps.S = S;
    ps.sample_begin = s_begin + s0;
    ps.n_paths = (uint32_t)(n_local * S);
    ps.n_local = (uint32_t)n_local;
    ps.div_local = make_fastdiv((uint32_t)n_local);
    ps.div_S = make_fastdiv(S);
    if (s0 > 0) MF_CUDA(cudaMemsetAsync(scr.counter, 0, sizeof(unsigned int), st));
    ev.resize(ev.size() + 2, nullptr);
    MF_CUDA(cudaEventCreate(&ev[ev.size() - 2]));
    MF_CUDA(cudaEventCreate(&ev[ev.size() - 1]));
    MF_CUDA(cudaEventRecord(ev[ev.size() - 2], st));
    rc = launch_paths(sc, ps, false, st);
    if (!rc) MF_CUDA(cudaEventRecord(ev[ev.size() - 1], st));
    if (rc) {
      for (cudaEvent_t e : ev) cudaEventDestroy(e);
      scratch_free(&scr, st);
      return rc;
    }
  }
  ps.n_local = (uint32_t)n_local;
  // over every image pixel: owned ones get sum / spp, the others +0.0 in
  // overwrite mode (no separate clearing of the caller's buffer)
  finalize_kernel<<<(uint32_t)((npix + 255) / 256), 256, 0, st>>>(
      sc, ps, (uint32_t)npix, std::ldexp(1.0, -k) / (double)p.spp, p.accumulate ? 1 : 0, d_accum);
  g_launches++;
  MF_CUDA(cudaGetLastError());
  // the event counters always come back (mf_render_finish validates them:
  // majorant violations, iteration caps and invalid radiance raise, as the
  // reference's render() always validates -- transport.py:264-268,297;
  // image.py:38-42)
  mf_render_ticket* t = new mf_render_ticket();
  t->h_stats = pinned_stats_get();
  if (!t->h_stats) {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    scratch_free(&scr, st);
    delete t;
    return fail(MF_ERR_CUDA, "cannot allocate pinned host memory");
  }
  MF_CUDA(cudaMemcpyAsync(t->h_stats, scr.stats, kStCount * sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost, st));
  MF_CUDA(cudaEventCreateWithFlags(&t->done, cudaEventDisableTiming));
  MF_CUDA(cudaEventRecord(t->done, st));
  t->ev.swap(ev);
  t->empty = false;
  *ticket = t;
  return scratch_free(&scr, st);   // stream-ordered: after the read-back
}

int mf_render_finish(mf_render_ticket* t, mf_stats* stats) {
  if (!t) return fail(MF_ERR_PARAM, "null ticket");
  if (t->empty) {
    if (stats) std::memset(stats, 0, sizeof(*stats));
    delete t;
    return MF_OK;
  }
  cudaError_t e = cudaEventSynchronize(t->done);
  mf_stats local;
  mf_stats& out_st = stats ? *stats : local;
  int out = MF_OK;
  if (e != cudaSuccess) {
    out = fail(MF_ERR_CUDA, std::string("render: ") + cudaGetErrorString(e));
  } else {
    fill_stats(t->h_stats, &out_st);
    double kernel_ms = 0.0;
    for (size_t i = 0; i + 1 < t->ev.size(); i += 2) {
      float ms = 0.0f;
      if (cudaEventElapsedTime(&ms, t->ev[i], t->ev[i + 1]) == cudaSuccess) kernel_ms += ms;
    }
    out_st.path_kernel_ms = kernel_ms;
    out = check_stats(out_st);
  }
  for (cudaEvent_t ev : t->ev) cudaEventDestroy(ev);
  cudaEventDestroy(t->done);
  pinned_stats_put(t->h_stats);
  delete t;
  return out;
}

int mf_render(const mf_scene* scene, const mf_render_params* params, float* d_accum,
              mf_stats* stats, void* stream) {
  mf_render_ticket* t = nullptr;
  int rc = mf_render_async(scene, params, d_accum, &t, stream);
  if (rc) return rc;
  return mf_render_finish(t, stats);
}

int mf_trace_paths(const mf_scene* scene, const float* d_org, const float* d_dir,
                   const uint32_t* d_pixel, const uint32_t* d_sample, uint64_t seed,
                   int32_t max_bounces, int64_t n, float* d_radiance, mf_stats* stats,
                   void* stream) {
  if (!scene || !d_org || !d_dir || !d_pixel || !d_sample || !d_radiance)
    return fail(MF_ERR_PARAM, "null argument");
  if (max_bounces < 1)
    return fail(MF_ERR_PARAM, "max_bounces must be >= 1, got " + std::to_string(max_bounces));
  if (n < 0 || n > 0xffffffffll) return fail(MF_ERR_PARAM, "n out of range");
  SceneDev sc;
  std::string berr;
  int rc = build_scene(*scene, &sc, &berr);
  if (rc) return fail(rc, berr);
  rc = attach_slope_table(&sc, (cudaStream_t)stream);
  if (rc) return rc;
  if (n == 0) {
    if (stats) std::memset(stats, 0, sizeof(*stats));
    return MF_OK;
  }
  cudaStream_t st = (cudaStream_t)stream;
  Scratch scr;
  rc = scratch_alloc(&scr, 0, st);
  if (rc) return rc;
  PassDev ps;
  std::memset(&ps, 0, sizeof(ps));
  ps.k0 = (uint32_t)(seed & 0xffffffffu);
  ps.k1 = (uint32_t)(seed >> 32);
  philox_round_keys(ps.k0, ps.k1, ps.rk);
  ps.max_bounces = max_bounces;
  ps.n_paths = (uint32_t)n;
  ps.S = 1;
  ps.rad = d_radiance;
  ps.counter = scr.counter;
  ps.stats = scr.stats;
  ps.org = d_org;
  ps.dir = d_dir;
  ps.pix = d_pixel;
  ps.smp = d_sample;
  MF_CUDA(cudaMemsetAsync(scr.counter, 0, sizeof(unsigned int), st));
  rc = launch_paths(sc, ps, true, st);
  int out = rc;
  if (!rc) {
    // always validated, as render()
    unsigned long long h[kStCount];
    MF_CUDA(cudaMemcpyAsync(h, scr.stats, sizeof(h), cudaMemcpyDeviceToHost, st));
    MF_CUDA(cudaStreamSynchronize(st));
    mf_stats local;
    mf_stats& o = stats ? *stats : local;
    fill_stats(h, &o);
    out = check_stats(o);
  }
  int rc2 = scratch_free(&scr, st);
  return out ? out : rc2;
}

int mf_walk(const mf_scene* scene, const float* d_org, const float* d_dir,
            const uint32_t* d_pixel, const uint32_t* d_sample, uint64_t seed, uint32_t segment,
            int32_t mode, int64_t n, int8_t* d_state, float* d_pos, float* d_travel,
            float* d_weight, int32_t* d_prim, mf_stats* stats, void* stream) {
  if (!scene || (n > 0 && (!d_org || !d_dir || !d_pixel || !d_sample)))
    return fail(MF_ERR_PARAM, "null argument");
  if (mode != MF_WALK_COLLISION && mode != MF_WALK_RATIO && mode != MF_WALK_TENTATIVE)
    return fail(MF_ERR_PARAM, "mode must be collision, ratio or tentative");
  if (n < 0 || n > 0x7fffffffll) return fail(MF_ERR_PARAM, "n out of range");
  SceneDev sc;
  std::string berr;
  int rc = build_scene(*scene, &sc, &berr);
  if (rc) return fail(rc, berr);
  if (mode == MF_WALK_TENTATIVE && sc.has_grid)
    return fail(MF_ERR_UNSUPPORTED, "sample_collision is not available for grid fields");
  if (stats) std::memset(stats, 0, sizeof(*stats));
  if (n == 0) return MF_OK;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* stt = nullptr;
  MF_CUDA(cudaMallocAsync((void**)&stt, kStCount * sizeof(unsigned long long), st));
  MF_CUDA(cudaMemsetAsync(stt, 0, kStCount * sizeof(unsigned long long), st));
  WalkArgs a;
  std::memset(&a, 0, sizeof(a));
  a.org = d_org;
  a.dir = d_dir;
  a.pix = d_pixel;
  a.smp = d_sample;
  a.k0 = (uint32_t)(seed & 0xffffffffu);
  a.k1 = (uint32_t)(seed >> 32);
  a.segment = segment;
  a.mode = mode;
  a.n = (uint32_t)n;
  a.state = d_state;
  a.pos = d_pos;
  a.travel = d_travel;
  a.weight = d_weight;
  a.prim = d_prim;
  a.stats = stt;
  walk_kernel<<<(uint32_t)((n + kBlock - 1) / kBlock), kBlock, 0, st>>>(sc, a);
  g_launches++;
  MF_CUDA(cudaGetLastError());
  unsigned long long h[kStCount];
  MF_CUDA(cudaMemcpyAsync(h, stt, sizeof(h), cudaMemcpyDeviceToHost, st));
  MF_CUDA(cudaFreeAsync(stt, st));
  MF_CUDA(cudaStreamSynchronize(st));
  mf_stats local;
  mf_stats& o = stats ? *stats : local;
  fill_stats(h, &o);
  if (o.majorant_violations)
    return fail(MF_ERR_MAJORANT, "extinction exceeded its majorant (" +
                                     std::to_string(o.majorant_violations) + " events)");
  if (o.capped) return fail(MF_ERR_CAP, "walker exceeded its iteration cap");
  return MF_OK;
}

int mf_transmittance(const mf_scene* scene, const double origin[3], const double direction[3],
                     int64_t n, uint64_t seed, uint64_t stream_id, double* mean, double* se,
                     void* stream) {
  if (!scene || !origin || !direction || !mean || !se) return fail(MF_ERR_PARAM, "null argument");
  if (n < 1 || n > 0x7fffffffll) return fail(MF_ERR_PARAM, "n_samples out of range");
  SceneDev sc;
  std::string berr;
  int rc = build_scene(*scene, &sc, &berr);
  if (rc) return fail(rc, berr);
  rc = attach_slope_table(&sc, (cudaStream_t)stream);
  if (rc) return rc;
  double dn = std::sqrt(direction[0] * direction[0] + direction[1] * direction[1] +
                        direction[2] * direction[2]);
  if (!(dn > 0.0)) return fail(MF_ERR_PARAM, "direction must be nonzero");
  cudaStream_t st = (cudaStream_t)stream;
  float* w = nullptr;
  unsigned long long* stt = nullptr;
  MF_CUDA(cudaMallocAsync((void**)&w, (size_t)n * sizeof(float), st));
  MF_CUDA(cudaMallocAsync((void**)&stt, kStCount * sizeof(unsigned long long), st));
  MF_CUDA(cudaMemsetAsync(stt, 0, kStCount * sizeof(unsigned long long), st));
  V3 o = v3((float)origin[0], (float)origin[1], (float)origin[2]);
  V3 d = v3((float)(direction[0] / dn), (float)(direction[1] / dn), (float)(direction[2] / dn));
  uint32_t nb = (uint32_t)((n + kBlock - 1) / kBlock);
  ratio_kernel<<<nb, kBlock, 0, st>>>(sc, (uint32_t)seed, (uint32_t)(seed >> 32),
                                      (uint32_t)stream_id, o, d, (uint32_t)n, w, stt);
  g_launches++;
  MF_CUDA(cudaGetLastError());
  std::vector<float> hw((size_t)n);
  unsigned long long hs[kStCount];
  MF_CUDA(cudaMemcpyAsync(hw.data(), w, (size_t)n * sizeof(float), cudaMemcpyDeviceToHost, st));
  MF_CUDA(cudaMemcpyAsync(hs, stt, sizeof(hs), cudaMemcpyDeviceToHost, st));
  MF_CUDA(cudaFreeAsync(w, st));
  MF_CUDA(cudaFreeAsync(stt, st));
  MF_CUDA(cudaStreamSynchronize(st));
  if (hs[kStViolations])
    return fail(MF_ERR_MAJORANT, "extinction exceeded its majorant in ratio tracking");
  if (hs[kStCapped])
    return fail(MF_ERR_CAP, "ratio tracking exceeded its iteration cap in " +
                                std::to_string(hs[kStCapped]) + " samples");
  // mean and standard error in double, fixed order (transport.py:310-313)
  double s = 0.0;
  for (float v : hw) s += v;
  double m = s / (double)n;
  double ss = 0.0;
  for (float v : hw) ss += ((double)v - m) * ((double)v - m);
  *mean = m;
  *se = n > 1 ? std::sqrt(ss / (double)(n - 1)) / std::sqrt((double)n) : 0.0;
  return MF_OK;
}


// --- Gaussian-random-field oracle (mf_gp.cuh) ---------------------------

static mf::gp::Grid gp_grid(const mf_gp_grid& g) {
  mf::gp::Grid G;
  G.g = g.d_grid;
  G.n = g.n;
  G.h = g.spacing;
  G.origin = g.origin;
  G.planar = g.planar;
  G.bound = g.d_bound;
  return G;
}

static int gp_check(const mf_gp_grid* g) {
  if (!g || !g->d_grid || g->n < 2 || !(g->spacing > 0.0))
    return fail(MF_ERR_PARAM, "gp grid: null array, n < 2 or spacing <= 0");
  return MF_OK;
}

static unsigned gp_blocks(int64_t n) { return (unsigned)((n + 255) / 256); }

int mf_gp_noise(const uint64_t* d_bases, int32_t n_streams, uint64_t counter0, int64_t n,
                double* d_out, void* stream) {
  if (!d_bases || !d_out || n_streams < 0 || n < 0) return fail(MF_ERR_PARAM, "bad gp_noise arguments");
  if (!n || !n_streams) return MF_OK;
  mf::gp::noise_kernel<<<gp_blocks(n * n_streams), 256, 0, (cudaStream_t)stream>>>(
      d_bases, n_streams, counter0, n, d_out);
  g_launches++;
  MF_CUDA(cudaGetLastError());
  return MF_OK;
}

int mf_gp_uniform(const uint64_t* d_bases, int32_t n_streams, uint64_t counter0, int64_t n,
                  double* d_out, void* stream) {
  if (!d_bases || !d_out || n_streams < 0 || n < 0)
    return fail(MF_ERR_PARAM, "bad gp_uniform arguments");
  if (!n || !n_streams) return MF_OK;
  mf::gp::uniform_kernel<<<gp_blocks(n * n_streams), 256, 0, (cudaStream_t)stream>>>(
      d_bases, n_streams, counter0, n, d_out);
  g_launches++;
  MF_CUDA(cudaGetLastError());
  return MF_OK;
}

int mf_gp_eval(const mf_gp_grid* grid, const double* d_p, const int32_t* d_real, int64_t n,
               double* d_f, double* d_grad, void* stream) {
  int rc = gp_check(grid);
  if (rc) return rc;
  if (!d_p || n < 0) return fail(MF_ERR_PARAM, "bad gp_eval arguments");
  if (!n || (!d_f && !d_grad)) return MF_OK;
  mf::gp::eval_kernel<<<gp_blocks(n), 256, 0, (cudaStream_t)stream>>>(gp_grid(*grid), n, d_p,
                                                                       d_real, d_f, d_grad);
  g_launches++;
  MF_CUDA(cudaGetLastError());
  return MF_OK;
}

int mf_gp_first_hit(const mf_gp_grid* grid, const double* d_org, const double* d_dir,
                    const int32_t* d_real, int64_t n, double step, const double* d_tmax_real,
                    double t_max, uint8_t* d_hit, double* d_pos, double* d_normal,
                    double* d_travel, void* stream) {
  int rc = gp_check(grid);
  if (rc) return rc;
  if (!d_org || !d_dir || !d_hit || !d_pos || !d_normal || !d_travel || n < 0 || !(step > 0.0))
    return fail(MF_ERR_PARAM, "bad gp_first_hit arguments");
  if (!n) return MF_OK;
  mf::gp::first_hit_kernel<<<gp_blocks(n), 256, 0, (cudaStream_t)stream>>>(
      gp_grid(*grid), n, d_org, d_dir, d_real, step, d_tmax_real, t_max, d_hit, d_pos, d_normal,
      d_travel);
  g_launches++;
  MF_CUDA(cudaGetLastError());
  return MF_OK;
}

int mf_gp_reflect_paths(const mf_gp_grid* grid, double* d_o, double* d_d, double* d_thr,
                        double* d_rad, const int32_t* d_real, int64_t n, int32_t n_real,
                        double sigma, double env, double eps, double step, int32_t max_bounces,
                        const double* eta, const double* k, uint64_t* d_evals, void* stream) {
  int rc = gp_check(grid);
  if (rc) return rc;
  if (!d_o || !d_d || !d_thr || !d_rad || !d_real || n < 0 || n_real < 1 || !(step > 0.0))
    return fail(MF_ERR_PARAM, "bad gp_reflect_paths arguments");
  if (!n || max_bounces < 1) return MF_OK;
  cudaStream_t st = (cudaStream_t)stream;
  mf::gp::Paths P;
  P.o = d_o; P.d = d_d; P.thr = d_thr; P.rad = d_rad; P.real = d_real; P.n = n;
  P.sigma = sigma; P.env = env; P.eps = eps; P.step = step;
  P.fresnel = (eta && k) ? 1 : 0;
  P.evals = (unsigned long long*)d_evals;
  for (int c = 0; c < 3; ++c) {
    P.eta[c] = P.fresnel ? eta[c] : 0.0;
    P.k[c] = P.fresnel ? k[c] : 0.0;
  }
  // scratch: alive flags, per-realisation march length, live count
  size_t bytes = (size_t)n + 8 * (size_t)n_real + 64;
  char* base = nullptr;
  MF_CUDA(cudaMallocAsync((void**)&base, bytes, st));
  P.tcap = (unsigned long long*)base;
  P.live = (unsigned int*)(base + 8 * (size_t)n_real);
  P.alive = (uint8_t*)(base + 8 * (size_t)n_real + 64);
  MF_CUDA(cudaMemsetAsync(P.alive, 1, (size_t)n, st));
  mf::gp::Grid G = gp_grid(*grid);
  unsigned live = 0;
  for (int b = 0; b < max_bounces; ++b) {
    MF_CUDA(cudaMemsetAsync(base, 0, 8 * (size_t)n_real + 64, st));
    mf::gp::escape_kernel<<<gp_blocks(n), 256, 0, st>>>(G, P);
    g_launches++;
    MF_CUDA(cudaGetLastError());
    MF_CUDA(cudaMemcpyAsync(&live, P.live, sizeof(live), cudaMemcpyDeviceToHost, st));
    MF_CUDA(cudaStreamSynchronize(st));
    if (!live) break;
    mf::gp::reflect_kernel<<<gp_blocks(n), 256, 0, st>>>(G, P);
    g_launches++;
    MF_CUDA(cudaGetLastError());
  }
  MF_CUDA(cudaFreeAsync(base, st));
  return MF_OK;
}

}  // extern "C"

#include "mf_comm.cuh"
