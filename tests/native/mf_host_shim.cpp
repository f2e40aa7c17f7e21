// Host (CPU) build of the device math, for tests only: lets the CPU test
// suite check every fp32 formula of csrc/mf_math.cuh / mf_query.cuh
// against the float64 oracle without a GPU.  Not part of the product (the
// package never loads this library; there is no CPU fallback).
#include <cstdint>
#include <cstring>
#include <string>

#include "../../paper_2603_00280_b200/csrc/mf_prepare.h"
#include "../../paper_2603_00280_b200/csrc/mf_query.cuh"

using namespace mf;

#include <vector>

// host copy of the device slope table (built on first use, same code)
static const float* host_slope_table() {
  static std::vector<float> tab;
  if (tab.empty()) {
    tab.resize((size_t)kTabNT * kTabNU);
    for (int i = 0; i < kTabNT; ++i)
      for (int j = 0; j < kTabNU; ++j) tab[(size_t)i * kTabNU + j] = slope_table_node(i, j);
  }
  return tab.data();
}

extern "C" {

// which: 0 erfcx, 1 ierfcx, 2 bterm, 3 erfc, 4 ndtri, 5 mills, 6 log_ndtr,
//        7 inv_log_ndtr, 8 erfinv(2x-1)
int mfh_special(int which, const float* x, float* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    float v = x[i], r = 0.0f;
    switch (which) {
      case 0: r = erfcx_pos(v); break;
      case 1: r = ierfcx_pos(v); break;
      case 2: r = bterm_pos(v); break;
      case 3: r = erfc_f(v); break;
      case 4: r = ndtri(v); break;
      case 5: r = mills(v); break;
      case 6: r = log_ndtr(v); break;
      case 7: r = inv_log_ndtr(v); break;
      case 8: r = erfinv_2u_minus_1(v); break;
      default: return 1;
    }
    out[i] = r;
  }
  return 0;
}

int mfh_slope(const float* nu, const float* u1, float* x, int32_t* iters, int64_t n) {
  const float* tab = host_slope_table();
  for (int64_t i = 0; i < n; ++i) {
    int it = 0;
    x[i] = visible_slope_x(nu[i], u1[i], &it, tab, atan2f(1.0f, nu[i]));
    iters[i] = it;
  }
  return 0;
}

// in: 11 SoA float arrays (px py pz wox woy woz wix wiy wiz u1 u2)
// out: 16 SoA float arrays (sigma_t, phase rgb, pdf, ws xyz, pdf_s, w rgb,
//      flags, iters, proj_area(wo local), ndf(wi local as normal))
int mfh_query(const mf_medium* med, const mf_primitive* field, const float* const* in,
              float* const* out, int64_t n) {
  MediumK m;
  std::string err;
  if (prepare_medium(*med, &m, &err) != MF_OK) return 1;
  m.slope_tab = host_slope_table();
  V3 c = v3((float)field->center[0], (float)field->center[1], (float)field->center[2]);
  for (int64_t i = 0; i < n; ++i) {
    V3 p = v3(in[0][i], in[1][i], in[2][i]);
    V3 wo = v3(in[3][i], in[4][i], in[5][i]);
    V3 wi = v3(in[6][i], in[7][i], in[8][i]);
    QueryResult q = query_point(m, field->shape, (float)field->z0, c, (float)field->radius, p,
                                wo, wi, in[9][i], in[10][i]);
    out[0][i] = q.sigma_t;
    out[1][i] = q.phase.x;
    out[2][i] = q.phase.y;
    out[3][i] = q.phase.z;
    out[4][i] = q.pdf;
    out[5][i] = q.ws.x;
    out[6][i] = q.ws.y;
    out[7][i] = q.ws.z;
    out[8][i] = q.pdf_s;
    out[9][i] = q.w.x;
    out[10][i] = q.w.y;
    out[11][i] = q.w.z;
    out[12][i] = (float)q.flags;
    out[13][i] = (float)q.iters;
    out[14][i] = proj_area(m, wo);
    out[15][i] = ndf(m, wi);
  }
  return 0;
}

}  // extern "C"

#include "../../paper_2603_00280_b200/csrc/mf_scene_build.h"

extern "C" {

// Host run of the device walker (csrc/mf_transport.cuh walk) for n rays:
// org/dir SoA [3][n]; path i keyed (pixel = i, sample = 0, segment 0).
// out: state[n] (0 escaped, 1 absorbed, 2 collided), pos SoA [3][n], weight[n]
// rr_min: Russian-roulette threshold of ratio weights (0: plain ratio tracking)
static int g_sphere_walk = 0;
static int32_t* steps = nullptr;

// select the walker of mfh_walk: 0 the general tracking walker, 1 the
// single-sphere tangent-majorant walker (sphere_walk); optional per-ray
// iteration counts
void mfh_set_walker(int sphere, int32_t* steps_out) {
  g_sphere_walk = sphere;
  steps = steps_out;
}

int mfh_walk(const mf_scene* scene, const float* org, const float* dir, int64_t n, uint64_t seed,
             int ratio, int32_t* state, float* pos, float* weight, float majorant_scale,
             int64_t* violations, float rr_min) {
  SceneDev sc;
  std::string err;
  if (build_scene(*scene, &sc, &err) != MF_OK) return 1;
  for (int j = 0; j < kMaxPrims; ++j) sc.media[j].slope_tab = host_slope_table();
  for (int j = 0; j < sc.n_prims; ++j) sc.mx[j].sig_max *= majorant_scale;
  *violations = 0;
  for (int64_t i = 0; i < n; ++i) {
    PathRng r{(uint32_t)seed, (uint32_t)(seed >> 32), (uint32_t)i, 0u};
    V3 o = v3(org[i], org[n + i], org[2 * n + i]);
    V3 d = v3(dir[i], dir[n + i], dir[2 * n + i]);
    if (sc.has_grid) {
      GridWalk w = grid_walk(sc.grid, sc.media[0],
                             [&](uint32_t call) { return rng_block(r, 0u, call); },
                             ratio ? kCallShadow : 1u, o, d, ratio != 0, INFINITY, rr_min);
      state[i] = w.outcome;
      pos[i] = w.pos.x;
      pos[n + i] = w.pos.y;
      pos[2 * n + i] = w.pos.z;
      weight[i] = w.weight;
      *violations += w.violations;
      continue;
    }
    WalkResult w = g_sphere_walk ? sphere_walk(sc, r, 0u, ratio ? kCallShadow : 1u, o, d,
                                               ratio != 0, INFINITY, rr_min)
                                 : walk(sc, r, 0u, ratio ? kCallShadow : 1u, o, d, ratio != 0,
                                        INFINITY, rr_min);
    if (steps) steps[i] = w.steps;
    state[i] = w.outcome;
    pos[i] = w.pos.x;
    pos[n + i] = w.pos.y;
    pos[2 * n + i] = w.pos.z;
    weight[i] = w.weight;
    *violations += w.violations;
  }
  return 0;
}

}  // extern "C"

extern "C" {

// host build of the majorant grid (same per-cell code as the device)
int mfh_grid_majorant(const mf_grid_field* grid, float* out) {
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
  tmp.grid.d_majorant = out;
  SceneDev sc;
  std::string err;
  if (build_scene(tmp, &sc, &err) != MF_OK) return 1;
  int n = grid->n_maj;
  for (int c = 0; c < n * n * n; ++c) out[c] = grid_cell_majorant(sc.grid, c / (n * n), (c / n) % n, c % n);
  for (int c = 0; c < n * n * n; ++c) out[c] = grid_cell_skip(out, n, c / (n * n), (c / n) % n, c % n);
  return 0;
}

}  // extern "C"

extern "C" {
// grid field probes (f, sigma, extinction along dir) at points, host build
int mfh_grid_probe(const mf_scene* scene, const float* p, const float* dir, int64_t n,
                   float* out) {
  SceneDev sc;
  std::string err;
  if (build_scene(*scene, &sc, &err) != MF_OK) return 1;
  for (int64_t i = 0; i < n; ++i) {
    V3 x = v3(p[3 * i], p[3 * i + 1], p[3 * i + 2]);
    V3 d = v3(dir[3 * i], dir[3 * i + 1], dir[3 * i + 2]);
    float f, s;
    float e = grid_extinction(sc.grid, sc.media[0], x, d, -6.0f, &f, &s);
    out[3 * i] = f;
    out[3 * i + 1] = s;
    out[3 * i + 2] = e;
  }
  return 0;
}
}  // extern "C"

extern "C" {
float mfh_u01(uint32_t bits) { return u01(bits); }
}

#ifdef MF_GRID_STATS
// walk statistics of the grid walker (tools/grid_walk_stats.py only)
namespace mf {
long long g_grid_stats[8];
}
extern "C" long long* mfh_grid_stats() { return mf::g_grid_stats; }
#endif
