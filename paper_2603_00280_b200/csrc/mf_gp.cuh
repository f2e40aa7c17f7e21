// mf_gp.cuh -- the brute-force Gaussian-random-field oracle on the device
// (reference gp.py): periodic stationary field
// realisations and first zero crossings of their trilinear interpolant, in
// float64 like the reference.
//
//   gp::noise_kernel     the white noise of RandomStream.normal (rng.py:46-97:
//                        SplitMix64 over a Weyl sequence, Box-Muller over
//                        the two halves of the counter range), bit for bit
//   gp::eval_kernel      field_at / gradient_at (gp.py:80-131)
//   gp::first_hit_kernel first_hit (gp.py:148-197): the fixed-step march
//                        (min(l)/8) to the first sign change, 30 bisections,
//                        the normalised central-difference gradient
//   gp::escape_kernel,   the bounce loop of ensemble_radiance (gp.py:340-398):
//   gp::reflect_kernel   escape test + per-realisation march length, then
//                        the march and the specular bounce
//
// One thread per ray; rays carry the index of their realisation, so a launch
// covers a whole batch of realisations (the FFT filtering of the noise runs
// in cuFFT, batched, from the Python side).  Every floating-point operation
// is written with round-to-nearest intrinsics in the reference's order (no
// FMA contraction), so sign tests and hit distances follow numpy's.
#pragma once

#include <cstdint>

namespace mf {
namespace gp {

// float64 arithmetic in numpy's rounding (separate multiply and add)
__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dd(double a, double b) { return __ddiv_rn(a, b); }

struct Grid {
  const double* g;    // realisation r at g + r * n^3, x-major (ix * n + iy) * n + iz
  int n;
  double h;           // spacing
  double origin;      // -extent / 2 on every axis
  int planar;         // mean mu = z (else zero)
  const double* bound;  // per realisation max |stationary value|, or null
};

// SplitMix64 output of the Weyl sequence from base (rng.py raw_u64)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double uniform_from(uint64_t base, uint64_t ctr) {
  return (double)(mix64(base + ctr * 0x9E3779B97F4A7C15ull) >> 11) * (1.0 / 9007199254740992.0);
}

// trilinear periodic interpolant of realisation r (gp.py:86-105)
__device__ __forceinline__ double stationary_at(const Grid& G, int r, double px, double py,
                                                double pz) {
  const int n = G.n;
  const double* g = G.g + (size_t)r * n * n * n;
  double ux = dd(ds(px, G.origin), G.h), uy = dd(ds(py, G.origin), G.h),
         uz = dd(ds(pz, G.origin), G.h);
  double fx = floor(ux), fy = floor(uy), fz = floor(uz);
  long long ix = (long long)fx, iy = (long long)fy, iz = (long long)fz;
  double tx = ds(ux, (double)ix), ty = ds(uy, (double)iy), tz = ds(uz, (double)iz);
  double acc = 0.0;
#pragma unroll
  for (int o = 0; o < 8; ++o) {
    int ox = (o >> 2) & 1, oy = (o >> 1) & 1, oz = o & 1;
    long long jx = ((ix + ox) % n + n) % n, jy = ((iy + oy) % n + n) % n,
              jz = ((iz + oz) % n + n) % n;
    double w = dm(dm(ox ? tx : ds(1.0, tx), oy ? ty : ds(1.0, ty)), oz ? tz : ds(1.0, tz));
    acc = da(acc, dm(w, g[(jx * n + jy) * n + jz]));
  }
  return acc;
}

__device__ __forceinline__ double field_at(const Grid& G, int r, double px, double py, double pz) {
  double b = stationary_at(G, r, px, py, pz);
  return G.planar ? da(b, pz) : b;
}

// central differences of the interpolant, step one cell (gp.py:114-127)
__device__ __forceinline__ void gradient_at(const Grid& G, int r, double px, double py, double pz,
                                            double* gx, double* gy, double* gz) {
  const double h = G.h, h2 = dm(2.0, G.h);
  *gx = dd(ds(stationary_at(G, r, da(px, h), py, pz), stationary_at(G, r, ds(px, h), py, pz)), h2);
  *gy = dd(ds(stationary_at(G, r, px, da(py, h), pz), stationary_at(G, r, px, ds(py, h), pz)), h2);
  *gz = dd(ds(stationary_at(G, r, px, py, da(pz, h)), stationary_at(G, r, px, py, ds(pz, h))), h2);
  if (G.planar) *gz = da(*gz, 1.0);
}

struct Hit {
  bool hit;
  double px, py, pz, nx, ny, nz, travel;
  int evals;   // interpolant evaluations (march + bisection + gradient)
};

constexpr int kHitBisections = 30;


// first_hit (gp.py:148-197) of one ray in realisation r: the march visits
// t = step, 2 step (by repeated addition, as the reference's shared loop
// variable), ... while t <= t_max + step
__device__ __forceinline__ Hit first_hit(const Grid& G, int r, double ox, double oy, double oz,
                                         double dx, double dy, double dz, double step,
                                         double t_max) {
  double f_prev = field_at(G, r, ox, oy, oz);
  double t_prev = 0.0, lo = 0.0, hi = 0.0;
  bool found = false;
  int evals = 1;
  const double t_end = da(t_max, step);
  // planar mean: f = z + g with |g| <= B, so once the ray's height is past
  // +-B on the side it is heading to and the last value has that sign, no
  // later march point can change sign -- stop (the same "no hit" the full
  // march reaches, bit for bit)
  const double B = (G.planar && G.bound) ? G.bound[r] : INFINITY;
  for (double t = step; t <= t_end; t = da(t, step)) {
    double zt = da(oz, dm(t, dz));
    if ((dz >= 0.0 && zt > B && f_prev > 0.0) || (dz <= 0.0 && zt < -B && f_prev < 0.0)) break;
    double f = field_at(G, r, da(ox, dm(t, dx)), da(oy, dm(t, dy)), zt);
    ++evals;
    if (signbit(f) != signbit(f_prev)) {
      lo = t_prev;
      hi = t;
      found = true;
      break;
    }
    f_prev = f;
    t_prev = t;
  }
  Hit h;
  h.hit = found;
  if (found) {
    double f_lo = field_at(G, r, da(ox, dm(lo, dx)), da(oy, dm(lo, dy)), da(oz, dm(lo, dz)));
    for (int k = 0; k < kHitBisections; ++k) {
      double mid = dm(0.5, da(lo, hi));
      double fm = field_at(G, r, da(ox, dm(mid, dx)), da(oy, dm(mid, dy)), da(oz, dm(mid, dz)));
      bool same = signbit(fm) == signbit(f_lo);
      if (same) {
        lo = mid;
        f_lo = fm;
      } else {
        hi = mid;
      }
    }
    h.travel = dm(0.5, da(lo, hi));
    evals += 1 + kHitBisections;
  } else {
    h.travel = INFINITY;
  }
  double tt = found ? h.travel : 0.0;
  h.px = da(ox, dm(tt, dx));
  h.py = da(oy, dm(tt, dy));
  h.pz = da(oz, dm(tt, dz));
  double gx, gy, gz;
  gradient_at(G, r, h.px, h.py, h.pz, &gx, &gy, &gz);
  double nr = __dsqrt_rn(da(da(dm(gx, gx), dm(gy, gy)), dm(gz, gz)));
  double den = nr > 0.0 ? nr : 1.0;
  h.nx = dd(gx, den);
  h.ny = dd(gy, den);
  h.nz = dd(gz, den);
  h.evals = evals + 6;
  return h;
}

// unpolarised conductor Fresnel, one channel (medium.py:127-147), float64
__device__ __forceinline__ double fresnel_conductor(double cos_i, double eta, double k) {
  double c = fmin(fmax(cos_i, 0.0), 1.0);
  double c2 = dm(c, c);
  double s2 = ds(1.0, c2);
  double t0 = ds(ds(dm(eta, eta), dm(k, k)), s2);
  double a2b2 = __dsqrt_rn(fmax(da(dm(t0, t0), dm(dm(dm(dm(4.0, eta), eta), k), k)), 0.0));
  double t1 = da(a2b2, c2);
  double a = __dsqrt_rn(fmax(dm(0.5, da(a2b2, t0)), 0.0));
  double t2 = dm(dm(2.0, a), c);
  double denom = da(t1, t2);
  double rs = denom > 0.0 ? dd(ds(t1, t2), denom) : 0.0;
  double t3 = da(dm(c2, a2b2), dm(s2, s2));
  double t4 = dm(t2, s2);
  double d34 = da(t3, t4);
  double rp = dd(dm(rs, ds(t3, t4)), d34 > 0.0 ? d34 : 1.0);
  return dm(0.5, da(rs, rp));
}

// ---------------------------------------------------------------------------
// kernels

// RandomStream.normal of n values per stream, streams bases[0..n_streams):
// uniforms u1 = counters [c0, c0 + m), u2 = [c0 + m, c0 + 2m), m = ceil(n/2);
// z[i] = r_i cos(2 pi u2_i) for i < m, r_{i-m} sin(2 pi u2_{i-m}) above
__global__ void noise_kernel(const uint64_t* bases, int n_streams, uint64_t c0, int64_t n,
                             double* out) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n * n_streams) return;
  int s = (int)(k / n);
  int64_t i = k - (int64_t)s * n;
  int64_t m = (n + 1) / 2;
  int64_t j = i < m ? i : i - m;
  uint64_t b = bases[s];
  double u1 = uniform_from(b, c0 + (uint64_t)j);
  double u2 = uniform_from(b, c0 + (uint64_t)(m + j));
  double r = __dsqrt_rn(dm(-2.0, log1p(-u1)));
  double a = dm(6.283185307179586, u2);
  out[k] = dm(r, i < m ? cos(a) : sin(a));
}

// uniforms of one stream per realisation (RandomStream.uniform), n each
__global__ void uniform_kernel(const uint64_t* bases, int n_streams, uint64_t c0, int64_t n,
                               double* out) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n * n_streams) return;
  int s = (int)(k / n);
  out[k] = uniform_from(bases[s], c0 + (uint64_t)(k - (int64_t)s * n));
}

// field_at / gradient_at at n points (SoA [3][n]) of realisations real[i]
__global__ void eval_kernel(const __grid_constant__ Grid G, int64_t n, const double* p,
                            const int32_t* real, double* f, double* grad) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int r = real ? real[i] : 0;
  double x = p[i], y = p[n + i], z = p[2 * n + i];
  if (f) f[i] = field_at(G, r, x, y, z);
  if (grad) gradient_at(G, r, x, y, z, grad + i, grad + n + i, grad + 2 * n + i);
}

// first_hit of n rays (SoA [3][n]); t_max per realisation (t_max_r) or one
// value for all
__global__ void first_hit_kernel(const __grid_constant__ Grid G, int64_t n, const double* o,
                                 const double* d, const int32_t* real, double step,
                                 const double* t_max_r, double t_max, uint8_t* hit, double* pos,
                                 double* nrm, double* travel) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int r = real ? real[i] : 0;
  Hit h = first_hit(G, r, o[i], o[n + i], o[2 * n + i], d[i], d[n + i], d[2 * n + i], step,
                    t_max_r ? t_max_r[r] : t_max);
  hit[i] = h.hit ? 1 : 0;
  pos[i] = h.px; pos[n + i] = h.py; pos[2 * n + i] = h.pz;
  nrm[i] = h.nx; nrm[n + i] = h.ny; nrm[2 * n + i] = h.nz;
  travel[i] = h.travel;
}

// the state of ensemble_radiance's specular paths (gp.py:361-397), SoA
struct Paths {
  double *o, *d, *thr, *rad;   // [3][n]
  uint8_t* alive;
  const int32_t* real;
  int64_t n;
  double sigma, env, eps, step;
  int fresnel;
  double eta[3], k[3];
  unsigned long long* tcap;    // per realisation: max march length (ordered bits)
  unsigned int* live;          // live rays after the escape test
  unsigned long long* evals;   // interpolant evaluations (work counter), or null
};

// escape upward above the shell (gp.py:366-372), then the march length of
// the survivors (gp.py:376): the max over a realisation's live rays
__global__ void escape_kernel(const __grid_constant__ Grid G, const __grid_constant__ Paths P) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n || !P.alive[i]) return;
  const int64_t n = P.n;
  int r = P.real[i];
  double ox = P.o[i], oy = P.o[n + i], oz = P.o[2 * n + i], dz = P.d[2 * n + i];
  bool up = dz > 0.0;
  bool abv = field_at(G, r, ox, oy, oz) > dm(4.0, P.sigma);
  if (up && abv) {
    for (int c = 0; c < 3; ++c) P.rad[c * n + i] = da(P.rad[c * n + i], dm(P.thr[c * n + i], P.env));
    P.alive[i] = 0;
    return;
  }
  double cap = dd(da(dm(6.0, P.sigma), fabs(oz)), fmax(fabs(dz), 0.05));
  atomicMax(P.tcap + r, (unsigned long long)__double_as_longlong(cap));   // cap > 0
  atomicAdd(P.live, 1u);
}

// march, then gather the environment on a miss or reflect specularly
// (gp.py:377-397)
__global__ void reflect_kernel(const __grid_constant__ Grid G, const __grid_constant__ Paths P) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n || !P.alive[i]) return;
  const int64_t n = P.n;
  int r = P.real[i];
  double t_max = __longlong_as_double((long long)P.tcap[r]);
  double dx = P.d[i], dy = P.d[n + i], dz = P.d[2 * n + i];
  Hit h = first_hit(G, r, P.o[i], P.o[n + i], P.o[2 * n + i], dx, dy, dz, P.step, t_max);
  if (P.evals) atomicAdd(P.evals, (unsigned long long)h.evals);
  if (!h.hit) {
    for (int c = 0; c < 3; ++c) P.rad[c * n + i] = da(P.rad[c * n + i], dm(P.thr[c * n + i], P.env));
    P.alive[i] = 0;
    return;
  }
  // v = -d_in; cos_i = |<v, n>|; d = reflect(v, n) = 2 <v, n> n - v
  double vx = -dx, vy = -dy, vz = -dz;
  double vn = da(da(dm(vx, h.nx), dm(vy, h.ny)), dm(vz, h.nz));
  if (P.fresnel) {
    double ci = fabs(vn);
    for (int c = 0; c < 3; ++c)
      P.thr[c * n + i] = dm(P.thr[c * n + i], fresnel_conductor(ci, P.eta[c], P.k[c]));
  }
  double nd[3] = {ds(dm(dm(2.0, vn), h.nx), vx), ds(dm(dm(2.0, vn), h.ny), vy),
                  ds(dm(dm(2.0, vn), h.nz), vz)};
  double p[3] = {h.px, h.py, h.pz};
  for (int c = 0; c < 3; ++c) {
    P.d[c * n + i] = nd[c];
    P.o[c * n + i] = da(p[c], dm(P.eps, nd[c]));
  }
}

// Camera rays of ensemble_radiance's rounds (scene.py:30-51 on the round's
// jitter uniforms, gp.py:352-357), float64 in numpy's operation order:
// round r, pixel (py, px): jitter x = uniform(bases[r], py w + px), jitter y
// = uniform(bases[r], h w + py w + px); origins at the camera
struct CamRays {
  double pos[3], fwd[3], right[3], up[3];
  double half_w, half_h;
  int w, h;
};

__global__ void camera_kernel(const __grid_constant__ CamRays c, const uint64_t* bases, int rounds,
                              double* o, double* d) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t hw = (int64_t)c.w * c.h, n = hw * rounds;
  if (i >= n) return;
  int r = (int)(i / hw);
  int64_t q = i - (int64_t)r * hw;
  int py = (int)(q / c.w), px = (int)(q - (int64_t)py * c.w);
  double jx = uniform_from(bases[r], (uint64_t)q), jy = uniform_from(bases[r], (uint64_t)(hw + q));
  double nx = ds(dm(dd(da((double)px, jx), (double)c.w), 2.0), 1.0);
  double ny = ds(1.0, dm(dd(da((double)py, jy), (double)c.h), 2.0));
  double ax = dm(nx, c.half_w), ay = dm(ny, c.half_h);
  double v[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) v[k] = da(da(c.fwd[k], dm(ax, c.right[k])), dm(ay, c.up[k]));
  double nrm = __dsqrt_rn(da(da(dm(v[0], v[0]), dm(v[1], v[1])), dm(v[2], v[2])));
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    d[k * n + i] = dd(v[k], nrm);
    o[k * n + i] = c.pos[k];
  }
}

// the ensemble image: per pixel and channel the rounds' radiance summed in
// round order (the reference's img += rad per round), divided by the count
__global__ void round_sum_kernel(const double* rad, int64_t hw, int rounds, int add, double* img) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= hw * 3) return;
  int c = (int)(i / hw);
  int64_t q = i - (int64_t)c * hw;
  const int64_t n = hw * rounds;
  double s = add ? img[q * 3 + c] : 0.0;   // continue an earlier batch's sum
  for (int r = 0; r < rounds; ++r) s = da(s, rad[c * n + (int64_t)r * hw + q]);
  img[q * 3 + c] = s;
}

// DFMA issue-rate microbenchmark (the FP64 roofline of these kernels)
__global__ void __launch_bounds__(256) peak_dfma_kernel(double* out, int iters, double a,
                                                        double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 123.456) out[threadIdx.x] = s;
}

}  // namespace gp
}  // namespace mf
