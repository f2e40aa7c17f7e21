/* macrofacet_b200.h -- C ABI of the B200-native macrofacet hot path.
 *
 * Plain C types only (no torch, no CUDA types in signatures: streams are
 * passed as `void*` holding a cudaStream_t, 0 = legacy default stream).
 * Device pointers are marked d_*; everything else is host memory.
 *
 * Each entry point replaces one reference Python call on the hot path of
 * /root/reference/pkg/src/macrofacet (file:line below); the Python mirror
 * in paper_2603_00280_b200/ keeps the reference signatures on top of it
 * (see INTEGRATION.md for the ctypes binding).
 *
 * Status codes map onto the reference exception tree (errors.py:4-41):
 *   MF_ERR_PARAM        -> ParameterDomainError (ValueError)
 *   MF_ERR_DEGENERATE   -> DegenerateVisibilityError   (ndf.py:312-313)
 *   MF_ERR_MAJORANT     -> InternalConsistencyError    (transport.py:264-268)
 *   MF_ERR_CAP          -> InternalConsistencyError    (transport.py:297)
 *   MF_ERR_NUMERIC      -> NumericFailureError
 *   MF_ERR_UNSUPPORTED  -> UnsupportedGeometryError    (medium.py:108-112)
 *   MF_ERR_CUDA         -> MacrofacetError
 * The message of the last failure on the calling thread: mf_last_error().
 */
#ifndef MACROFACET_B200_H
#define MACROFACET_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MF_ABI_VERSION 4

enum mf_status {
  MF_OK = 0,
  MF_ERR_PARAM = 1,
  MF_ERR_DEGENERATE = 2,
  MF_ERR_MAJORANT = 3,
  MF_ERR_CAP = 4,
  MF_ERR_NUMERIC = 5,
  MF_ERR_UNSUPPORTED = 6,
  MF_ERR_CUDA = 7
};

/* NdfKind (ndf.py:69-72) */
enum mf_kind { MF_KIND_BECKMANN = 0, MF_KIND_GGX = 1, MF_KIND_GENERALIZED = 2 };
/* Fresnel term: conductor (medium.py:127-147), F == 1 (fresnel_one,
 * medium.py:150-152) or a constant per-channel albedo (BASELINE configs 2-5;
 * not in the reference, SURVEY.md 8(a) "Albedo") */
enum mf_fresnel { MF_FRESNEL_CONDUCTOR = 0, MF_FRESNEL_ONE = 1, MF_FRESNEL_ALBEDO = 2 };

/* MacrofacetMedium (medium.py:35-67).  For BECKMANN/GGX, az is ignored (0). */
typedef struct mf_medium {
  int32_t kind;
  int32_t fresnel;
  double ax, ay, az;
  double sigma;
  double mix_ratio;
  double eta[3];
  double k[3];
  double albedo[3];
} mf_medium;

/* SDF primitives (sdf.py:18-84); MF_SHAPE_GRID is the BASELINE config-5
 * extension: the scene's mf_grid_field (trilinear SDF + per-voxel sigma) */
enum mf_shape { MF_SHAPE_PLANE = 0, MF_SHAPE_SPHERE = 1, MF_SHAPE_GRID = 2, MF_SHAPE_BOX = 3 };

/* ShellPrimitive (scene.py:99-101): one shape bound to media[medium] */
typedef struct mf_primitive {
  int32_t shape;
  int32_t medium;
  double z0;              /* plane z = z0, outside above */
  double center[3];       /* sphere, box */
  double radius;          /* sphere */
  double half_extents[3]; /* box (sdf.py:55-84) */
} mf_primitive;

/* Camera (scene.py:19-51); ortho != 0 selects the orthographic extension:
 * a film film_height world units tall centred on `position`, rays parallel
 * to look_at - position. */
typedef struct mf_camera {
  int32_t ortho;
  int32_t width, height;
  double position[3];
  double look_at[3];
  double fov_deg;
  double film_height;
} mf_camera;

#define MF_MAX_PRIMS 8
#define MF_MAX_MEDIA 8

/* Heterogeneous GP field (BASELINE config 5; not in the reference): mean =
 * trilinear SDF grid, per-point sigma = trilinear sigma grid, roughness
 * alpha_xy = sqrt2 sigma / l_xy, alpha_z = sqrt2 sigma / l_z.  Grids are
 * device float32, vertex-centred over [bmin, bmax], index (ix*n + iy)*n + iz.
 * d_majorant: n_maj^3 cell bounds of the extinction built by
 * mf_grid_majorant. */
typedef struct mf_grid_field {
  const float* d_sdf;
  const float* d_sigma;
  const float* d_majorant;
  int32_t n_sdf, n_sigma, n_maj;
  double bmin[3], bmax[3];
  double l_xy, l_z;
} mf_grid_field;

/* ShellScene (scene.py:104-129) + lights.  sun_dir is the direction the
 * light travels (DirectionalLight, scene.py:87-96); the point light
 * (position, intensity, NEE weight I/r^2) is a BASELINE-config extension. */
typedef struct mf_scene {
  int32_t n_prims;
  int32_t n_media;
  mf_primitive prims[MF_MAX_PRIMS];
  mf_medium media[MF_MAX_MEDIA];
  mf_camera camera;
  double env[3]; /* constant environment radiance (scene.py:54-84) */
  /* lat-long environment map (Environment.latlong, scene.py:61-84): device
   * float32 (env_height, env_width, 3), theta down the rows, bilinear with
   * wrapped phi; NULL = the constant env above */
  const float* d_env_map;
  int32_t env_width, env_height;
  int32_t has_sun;
  double sun_dir[3];
  double sun_radiance[3];
  int32_t has_point;
  double point_pos[3];
  double point_intensity[3];
  int32_t has_grid;   /* the single MF_SHAPE_GRID primitive uses `grid` */
  mf_grid_field grid;
} mf_scene;

/* Sharding of one render across ranks. */
enum mf_shard { MF_SHARD_TILES = 0, MF_SHARD_SAMPLES = 1 };

/* render(scene, spp, seed, max_bounces, tile) (render.py:127-180) */
typedef struct mf_render_params {
  uint64_t seed;
  int32_t spp;          /* samples per pixel of the whole (all-rank) render */
  int32_t max_bounces;  /* >= 1 (render.py:34-35) */
  int32_t tile;         /* tile edge in pixels for MF_SHARD_TILES */
  int32_t shard;        /* enum mf_shard */
  int32_t rank, nranks;
  int32_t accumulate;   /* 0: overwrite d_accum, 1: add into it */
} mf_render_params;

/* device-side event counters, summed over the call */
typedef struct mf_stats {
  uint64_t paths;
  uint64_t segments;      /* free-flight segments (one per scatter + final) */
  uint64_t scatters;      /* real collisions */
  uint64_t nee;           /* next-event connections */
  uint64_t slope_iters;   /* Newton iterations of the visible-slope sampler */
  uint64_t track_steps;   /* delta/ratio-tracking tentative steps */
  uint64_t escaped;
  uint64_t absorbed;
  uint64_t majorant_violations;
  uint64_t degenerate;    /* sigma(wo) < 1e-12 at a scatter (returns 0) */
  uint64_t nonfinite;     /* paths / pixels with non-finite or negative radiance */
  uint64_t capped;        /* paths cut by the segment cap */
  double path_kernel_ms;  /* CUDA-event time of the path megakernel launches */
} mf_stats;

/* ---------------------------------------------------------------------
 * Coefficient queries (BASELINE config 1).  Replaces, per query i:
 *   extinction(wo, f, medium, frame)           medium.py:91-95
 *   phase_eval(wo, wi, medium, frame)          medium.py:158-178
 *   phase pdf of wi (restated)                 ndf.py:397-405 + medium.py:186-189
 *   _phase_sample_u(wo_local, medium, u)       medium.py:181-193
 * with f and the frame taken from `field` at point p (plane: f = p.z - z0,
 * normal +z; sphere: f = |p - c| - r, normal (p - c)/|p - c|), and the
 * two-uniform convention u = (u1, u1', u2) of SURVEY.md 8(a).
 * All arrays are device SoA float32 of length n; any output may be NULL.
 * Directions are world-space unit vectors; the sampled direction is
 * returned in world space.
 */
typedef struct mf_query_in {
  const float *px, *py, *pz;
  const float *wox, *woy, *woz;
  const float *wix, *wiy, *wiz;
  const float *u1, *u2;
  /* optional overrides (NULL = derive from `field` at p):
   * f     [n]     field value (extinction(wo, f, ...) style calls)
   * frame [9][n]  tangent xyz, bitangent xyz, normal xyz (core.py:132-153) */
  const float* f;
  const float* frame;
} mf_query_in;

typedef struct mf_query_out {
  float* sigma_t;
  float *phase_r, *phase_g, *phase_b;
  float* pdf;
  float *wsx, *wsy, *wsz;
  float* pdf_s;
  float *w_r, *w_g, *w_b;
  int32_t* flags; /* bit0 degenerate view (sigma(wo) < 1e-12) */
  float *wmx, *wmy, *wmz; /* the sampled visible normal (vndf_sample, ndf.py:409-427) */
  float* pdf_m;           /* its mixture density (ndf.py:397-405) */
} mf_query_out;

int mf_query_batch(const mf_medium* medium, const mf_primitive* field, const mf_query_in* d_in,
                   const mf_query_out* d_out, int64_t n, void* stream);

/* ---------------------------------------------------------------------
 * Whole render into the caller's device accumulation buffer d_accum
 * (H * W * 3 float32, row-major (y, x, rgb) like RadianceImage.pixels),
 * holding radiance / spp for this rank's share (render.py:127-180).
 * Non-owned pixels (tile sharding) are left untouched (overwrite mode
 * writes +0.0 there), so a sum-reduce over ranks is exact.
 * The render kernels sum each pixel's paths in 64-bit fixed point (order
 * independent: the image is bit-identical for any launch geometry or tile
 * split).  The call synchronises the stream once at the end and always
 * validates: majorant violations, walker caps and non-finite / negative /
 * out-of-range radiance turn into error statuses (render() validates,
 * image.py:38-42).  stats (may be NULL) receives the event counters and
 * the path kernels' CUDA-event time.
 */
int mf_render(const mf_scene* scene, const mf_render_params* params, float* d_accum,
              mf_stats* stats, void* stream);

/* The same render in two halves, for callers that queue several renders
 * (panels, steps) on one stream without a host synchronisation between
 * them: mf_render_async validates the arguments, queues the whole render
 * and its event-counter read-back on `stream` and returns a ticket;
 * mf_render_finish waits for that ticket's work, fills stats (may be NULL)
 * and returns the status mf_render would have returned (the same
 * validation).  Every ticket must be finished exactly once; tickets of one
 * stream may be finished in any order.  mf_render == async + finish. */
typedef struct mf_render_ticket mf_render_ticket;
int mf_render_async(const mf_scene* scene, const mf_render_params* params, float* d_accum,
                    mf_render_ticket** ticket, void* stream);
int mf_render_finish(mf_render_ticket* ticket, mf_stats* stats);

/* trace_paths(origins, directions, scene, max_bounces, brng) (render.py:32-108)
 * for caller-given rays: d_org / d_dir are SoA float32 [3][n], path i is
 * keyed by (d_pixel[i], d_sample[i]) under `seed`; d_radiance SoA [3][n]. */
int mf_trace_paths(const mf_scene* scene, const float* d_org, const float* d_dir,
                   const uint32_t* d_pixel, const uint32_t* d_sample, uint64_t seed,
                   int32_t max_bounces, int64_t n, float* d_radiance, mf_stats* stats,
                   void* stream);

/* walk(scene, pos, direction, rng, mode, active) (transport.py:144-297) and
 * sample_collision(ray, scene, rng) (transport.py:316-416) for caller-given
 * rays: d_org / d_dir SoA float32 [3][n]; ray i draws from Philox keyed by
 * `seed` with counter (d_pixel[i], d_sample[i], segment, call).
 *   mode MF_WALK_COLLISION  delta tracking to a real collision, escape, or
 *                           absorption below -6 sigma
 *   mode MF_WALK_RATIO      ratio tracking of the transmittance (|f| <= 3 sigma)
 *   mode MF_WALK_TENTATIVE  stop at the first tentative collision
 * Outputs (any may be NULL): d_state int8 (0 escaped, 1 absorbed, 2 real
 * collision, 3 null collision), d_pos SoA [3][n], d_travel, d_weight,
 * d_prim (int32, -1 when none).  Majorant violations / iteration caps
 * raise (transport.py:264-268,297). */
enum mf_walk_mode { MF_WALK_COLLISION = 0, MF_WALK_RATIO = 1, MF_WALK_TENTATIVE = 2 };
int mf_walk(const mf_scene* scene, const float* d_org, const float* d_dir,
            const uint32_t* d_pixel, const uint32_t* d_sample, uint64_t seed, uint32_t segment,
            int32_t mode, int64_t n, int8_t* d_state, float* d_pos, float* d_travel,
            float* d_weight, int32_t* d_prim, mf_stats* stats, void* stream);

/* transmittance_estimate(ray, scene, n, rng) (transport.py:300-313):
 * ratio-tracking mean and standard error over n samples (host results). */
int mf_transmittance(const mf_scene* scene, const double origin[3], const double direction[3],
                     int64_t n, uint64_t seed, uint64_t stream_id, double* mean, double* se,
                     void* stream);

/* ---------------------------------------------------------------------
 * Closed-form curves of one medium on the device (the `curves` CLI command,
 * cli.py:132-175, and the device validation suites, validate.py:57-209).
 * Directions are SoA float32 device arrays d_x, d_y, d_z (unit vectors,
 * local frame); params (host doubles) = {wo_x, wo_y, wo_z, z0}.
 *   MF_CURVE_LAMBDA          Lambda(w) = sigma(w) / w_z   generalized_lambda, ndf.py:120-144
 *   MF_CURVE_PROJECTED_AREA  sigma(w)                     projected_area_dir, ndf.py:174-186
 *   MF_CURVE_NDF             D(w)                         generalized_ndf_dir / beckmann / ggx
 *   MF_CURVE_VNDF            D_wo(w), wo = params[0..2]   vndf_eval, ndf.py:299-315
 *   MF_CURVE_TRANSMITTANCE   closed-form planar Tr along wo from field value
 *                            h0 = params[3] to h1 = d_x[i]
 *                            (planar_transmittance, medium.py:98-124; d_y/d_z unused)
 * Transmittance raises MF_ERR_UNSUPPORTED for GGX or |wo_z| < 1e-12, as the
 * reference does. */
enum mf_curve_kind {
  MF_CURVE_LAMBDA = 0,
  MF_CURVE_PROJECTED_AREA = 1,
  MF_CURVE_NDF = 2,
  MF_CURVE_VNDF = 3,
  MF_CURVE_TRANSMITTANCE = 4,
  MF_CURVE_DENSITY = 5,    /* rho(f) = phi(f/s) / (s Phi(f/s)), f = d_x[i]   density, medium.py:70-88 */
  MF_CURVE_FRESNEL = 6,    /* conductor F(cos_i = d_x[i]) of channel 0 (eta[0], k[0]),
                              fresnel_conductor, medium.py:127-147 */
  MF_CURVE_GDF = 7         /* gradient density at g = (d_x, d_y, d_z), gdf_pdf, ndf.py:232-239
                              (GENERALIZED media only) */
};
int mf_curve(const mf_medium* medium, int kind, const float* d_x, const float* d_y,
             const float* d_z, int64_t n, const double params[4], float* d_out, void* stream);

/* Build the majorant grid of a grid field: for every one of the n_maj^3
 * cells an upper bound of the extinction over the cell and over all
 * directions (exact min/max of the trilinear SDF and sigma over the cell's
 * vertices; max over sigma samples and directions of rho * sigma_proj).
 * Cells without medium store -D instead, D >= 1 the Chebyshev distance in
 * cells to the nearest cell with medium (capped at 16): the walker's
 * empty-space jumps.  Writes d_majorant_out (n_maj^3 floats). */
int mf_grid_majorant(const mf_grid_field* grid, float* d_majorant_out, void* stream);

/* ---------------------------------------------------------------------
 * Multi-GPU exchange: the one collective of a sharded
 * render, the sum of the per-rank accumulation buffers onto `root`.  The
 * reference has no multi-process path (its render() joins a thread pool,
 * render.py:168-176); these calls replace that join across GPUs.
 *
 * `comm` is an ncclComm_t.  A caller that owns one passes it directly; the
 * helpers below create one from a unique id that the caller distributes
 * (any out-of-band channel, e.g. a torch.distributed broadcast).  NCCL is
 * loaded at run time (the process's already-loaded libnccl.so.2 when there
 * is one), so the library itself has no link-time NCCL dependency.
 *
 * mode MF_REDUCE_NCCL    : one in-place ncclReduce(sum, fp32) -- exact and
 *                          order-free under tile sharding (disjoint pixels)
 * mode MF_REDUCE_ORDERED : root receives every rank's buffer (grouped
 *                          ncclSend/ncclRecv into a stream-ordered scratch)
 *                          and sums them in rank order 0..n-1 in one
 *                          kernel -- bit-reproducible for a fixed rank
 *                          count under sample sharding too
 * All calls are stream-ordered on `stream`; d_buf on root holds the sum. */
enum mf_reduce_mode { MF_REDUCE_NCCL = 0, MF_REDUCE_ORDERED = 1 };
#define MF_COMM_ID_BYTES 128
int mf_comm_unique_id(unsigned char id_out[MF_COMM_ID_BYTES]);
int mf_comm_init(const unsigned char id[MF_COMM_ID_BYTES], int nranks, int rank, void** comm_out);
int mf_comm_destroy(void* comm);
int mf_reduce(void* comm, float* d_buf, size_t count, int root, int mode, void* stream);

/* Issue-rate peaks of this device measured by microbenchmark kernels
 * (independent FFMA chains / MUFU.EX2 chains, all SMs), in 1e9 lane
 * instructions per second: the FP32 / SFU roofline denominators. */
/* Camera rays of ensemble_radiance's rounds (scene.py:30-51 with each
 * round's jitter uniforms, gp.py:352-357) into SoA [3][rounds h w] d_o / d_d:
 * pos / fwd / right / up / half_w / half_h are the camera basis computed as
 * Camera.rays does; d_bases[r] the SplitMix64 base of round r's stream.
 * mf_gp_round_sum: d_img (h w 3, row-major) = the rounds' radiance (SoA
 * [3][rounds h w]) summed in round order, continuing d_img's values when
 * accumulate != 0. */
int mf_gp_camera_rays(const double pos[3], const double fwd[3], const double right[3],
                      const double up[3], double half_w, double half_h, int32_t width,
                      int32_t height, const uint64_t* d_bases, int32_t rounds, double* d_o,
                      double* d_d, void* stream);
int mf_gp_round_sum(const double* d_rad, int32_t width, int32_t height, int32_t rounds,
                    int32_t accumulate, double* d_img, void* stream);

/* float64 special functions on the device (the reference's core.py:29-98
 * erf / erfc / the Gaussian pieces): which 0 erf, 1 erfc, 2 exp(-x) */
int mf_special_f64(int which, const double* d_x, int64_t n, double* d_out, void* stream);

/* Radial Gauss-Legendre quadrature of the gradient distribution along wm
 * (ndf_from_gdf_quadrature, ndf.py:254-293): the sum over n_sub equal
 * pieces of [0, t_max] x 32 nodes (host arrays nodes / weights) of
 * t^3 exp(-(a t^2 - 2 b t + c) - shift), times the piece half-width, in
 * float64; *total receives it (host). */
int mf_gdf_radial(double a, double b, double c, double shift, double t_max, int32_t n_sub,
                  const double nodes[32], const double weights[32], double* total, void* stream);

/* DFMA issue-rate microbenchmark: the FP64 roofline of the mf_gp_* kernels */
int mf_measure_peak_fp64(double* dfma_ginst_s, void* stream);
int mf_measure_peaks(double* fp32_ginst_s, double* sfu_ginst_s, void* stream);

/* diagnostics */
const char* mf_last_error(void);
int mf_abi_version(void);
/* number of kernel launches this thread has issued through the library */
uint64_t mf_launch_count(void);

/* ---------------------------------------------------------------------
 * Gaussian-random-field oracle (reference gp.py):
 * periodic field realisations and their first zero crossings, float64.
 * The FFT filtering of the white noise (gp.py:131-141) is the caller's
 * (cuFFT through torch.fft, batched); these entry points draw the noise,
 * evaluate the trilinear interpolant and march rays through it.  A batch
 * holds n_real realisations of n^3 values each; ray / point i belongs to
 * realisation d_real[i] (NULL: all to realisation 0).  Arrays of 3-vectors
 * are SoA [3][count] float64. */
typedef struct mf_gp_grid {
  const double* d_grid; /* realisation r at d_grid + r n^3, index (ix n + iy) n + iz */
  int32_t n;
  double spacing;
  double origin;        /* lower corner on every axis (-extent / 2) */
  int32_t planar;       /* 1: mean mu(p) = p_z; 0: zero mean */
  const double* d_bound; /* per realisation max |stationary value| (planar mean: lets a march
                            stop once no later point can change sign), or NULL */
} mf_gp_grid;

/* RandomStream(seed, stream).normal(n) (rng.py:87-97) of the streams whose
 * SplitMix64 base states are d_bases[0..n_streams) (counters start at
 * counter0): d_out[s * n + i].  mf_gp_uniform: RandomStream.uniform(n). */
int mf_gp_noise(const uint64_t* d_bases, int32_t n_streams, uint64_t counter0, int64_t n,
                double* d_out, void* stream);
int mf_gp_uniform(const uint64_t* d_bases, int32_t n_streams, uint64_t counter0, int64_t n,
                  double* d_out, void* stream);
/* GpRealization.field_at / gradient_at (gp.py:80-127); d_f / d_grad may be NULL */
int mf_gp_eval(const mf_gp_grid* grid, const double* d_p, const int32_t* d_real, int64_t n,
               double* d_f, double* d_grad, void* stream);
/* first_hit (gp.py:148-197): march step `step`, range t_max (or
 * d_tmax_real[realisation] when not NULL) */
int mf_gp_first_hit(const mf_gp_grid* grid, const double* d_org, const double* d_dir,
                    const int32_t* d_real, int64_t n, double step, const double* d_tmax_real,
                    double t_max, uint8_t* d_hit, double* d_pos, double* d_normal,
                    double* d_travel, void* stream);
/* the specular bounce loop of ensemble_radiance (gp.py:361-397) for n paths
 * in place: origins d_o, directions d_d, throughput d_thr, radiance d_rad
 * (SoA [3][n]); eta / k: conductor Fresnel per channel (host arrays of 3),
 * NULL for F = 1; d_evals (may be NULL) accumulates the interpolant
 * evaluations (the oracle's work unit) */
int mf_gp_reflect_paths(const mf_gp_grid* grid, double* d_o, double* d_d, double* d_thr,
                        double* d_rad, const int32_t* d_real, int64_t n, int32_t n_real,
                        double sigma, double env, double eps, double step, int32_t max_bounces,
                        const double* eta, const double* k, uint64_t* d_evals, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MACROFACET_B200_H */
