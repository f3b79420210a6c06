/* libvolcache_b200 — C ABI of the B200 cache-record path.
 *
 * Drop-in boundary for the reference's record-build / lookup / render entry points
 * (reference = /root/reference/pkg/src/volcache, "src/" below).  The reference has no
 * FFI of its own: its boundary is the Python functions, so each entry point cites the
 * Python interface it replaces and the Python mirror in paper_1805_09258_b200/ binds
 * these symbols with ctypes.
 *
 * Conventions
 *  - Plain pointers and sizes; float64 in/out (the reference's dtype); int32 indices.
 *  - Arrays are device pointers unless VC_MEM_HOST is set in `flags`, in which case
 *    every array argument is host memory and the library stages the copies.
 *  - Return 0 on success, a negative VC_E* code on failure; vc_last_error() gives the
 *    thread-local message.  VC_EINVAL / VC_EOUTSIDE mirror the reference's ValueError
 *    cases (src/subdivision.py:155-158); the others are RuntimeErrors.
 *  - Handles are immutable after creation apart from their internal scratch: use one
 *    scene handle per host thread (or serialize calls) — calls on one handle are
 *    stream-ordered on the stream they are given.
 */
#ifndef VOLCACHE_B200_H
#define VOLCACHE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VC_OK 0
#define VC_EINVAL (-1)
#define VC_EOUTSIDE (-2)
#define VC_ECUDA (-3)
#define VC_ETRI (-4)
#define VC_ENOMEM (-5)
#define VC_EHOOK (-6) /* a caller-supplied hook reported failure */

/* flags */
#define VC_MEM_HOST 1     /* all array pointers are host memory */
#define VC_SEED_WORDS 2   /* rng = uint32 SeedSequence entropy words, seed_words per record */
#define VC_MAKE_RECORDS 4 /* also finalize records (make_record) into `records` */
#define VC_ISOTROPIC 8    /* make_record(..., anisotropic=False) */
#define VC_TRACE_BOUNDS 16 /* vc_trace: trace_or_bounds semantics */
#define VC_DEFER_CHECK 32 /* vc_build_records with device arrays: do not wait for the bounds check */

typedef struct vc_scene vc_scene;
typedef struct vc_cache vc_cache;

int vc_version(void);
const char* vc_last_error(void);
/* Kernel launches issued by this library since load (the bench's gpu_launches claim). */
int64_t vc_kernel_launches(void);
/* Per-kernel CUDA-event profile (events recorded on the launching stream while on).
 * vc_profile(1) clears and enables; vc_profile_read fills per-class milliseconds and
 * launch counts for up to max_classes classes, in the order: primary, rings, wave_scan,
 * gather, delaunay, tri_compact, degree, assemble, make_record, seedseq, interpolate,
 * march; returns the number of classes. */
int vc_profile(int on);
int vc_profile_read(double* ms, int64_t* launches, int max_classes);

/* Scene upload + BVH build.  Replaces Scene/_Packed2D/_Packed3D (src/scene.py:124-219).
 * vertices: n_surfaces × dim × dim (segment endpoints or triangle corners), host memory.
 * emission, albedo: n_surfaces × 3; bounds: dim each.  Host memory always. */
int vc_scene_create(int dim, int n_surfaces, const double* vertices, const double* emission,
                    const double* albedo, const double* bounds_min, const double* bounds_max,
                    double sigma_s, double sigma_a, vc_scene** out);
void vc_scene_destroy(vc_scene* scene);
/* Extension (no reference counterpart: the reference has area emitters only, SPEC.md:149;
 * BASELINE.json cfg1/cfg2/cfg4 name point lights, cfg3 a directional light).  Delta lights of
 * the scene, n_lights × 8 doubles in host memory: kind (0 = point, 1 = directional), v[3]
 * (position, or the unit vector pointing toward the light; 2D uses v[0..1]), rgb (radiant
 * intensity, or irradiance on a plane facing the light), 0.  They light reflective surfaces
 * (same cosine and normalisation as direct_lighting, src/transport.py:175-225), every media
 * sample of a record (σs × mean incident radiance, beside mean_surface_gather,
 * src/transport.py:288-310) and the cache point itself (closed-form value, gradient and
 * Hessian with the point visibility held constant).  Call before building records; 0 clears. */
int vc_scene_set_lights(vc_scene* scene, int n_lights, const double* rows);
/* Deferred bounds check.  vc_build_records raises the reference's ValueError for a point outside
 * the medium bounds (src/subdivision.py:155-158); with device arrays that needs one host read of
 * a device flag per call.  With VC_DEFER_CHECK in params->flags the call returns as soon as its
 * work is enqueued (a flagged wave still builds no rings) and the flag is OR-ed into a word
 * that this function reads and clears: VC_EOUTSIDE if any deferred call of this host thread since
 * the last read saw a point outside the bounds.  Synchronises `stream`. */
int vc_check_deferred(void* stream);
/* Scratch budget for one record wave (bytes; default a third of device memory, ≤ 64 GiB). */
int vc_scene_set_budget(vc_scene* scene, int64_t bytes);

typedef struct {
  int n_angular;       /* directions per record (estimate_moments n_angular) */
  double march_step;   /* ring spacing (march_step) */
  int n_inner;         /* gather directions per media sample (n_inner) */
  int n_light_samples; /* emitter quadrature samples (n_light_samples) */
  double epsilon;      /* make_record error budget */
  int flags;           /* VC_* flags */
  int seed_words;      /* entropy words per record when VC_SEED_WORDS */
  int media_bounces;   /* extension: media scattering events per gather path (0/1 = the
                          reference's one-bounce gather; ≤ 8): the multiple-scattering loop of
                          path_trace_radiance continued from each media sample, its draws taken
                          from the record's stream after every draw the reference makes */
  double hg_g;         /* extension: Henyey–Greenstein g of the media (0 = the reference's isotropic
                          medium; 3D): scattering at each media sample toward the cache point weighs
                          its gather paths by 4π·p_g, further media events sample HG directions */
} vc_build_params;

/* Batch estimate_moments (+ make_record for both kinds).
 * Replaces subdivision.estimate_moments (src/subdivision.py:373-393) called once per
 * point from CacheSet.compute (src/renderer.py:246-262), and cache.make_record
 * (src/cache.py:153-189).
 *   x          n_records × dim cache points
 *   rng        n_records × 4 uint64 PCG64 (state_hi, state_lo, inc_hi, inc_lo), the
 *              numpy bit_generator state of default_rng(rng_seed); or, with
 *              VC_SEED_WORDS, n_records × seed_words uint32 SeedSequence entropy
 *   adjacency  NULL (GPU spherical Delaunay) or n_records × (2n−4) × 3 int32 triangles
 *              (3D; e.g. qhull's simplices, src/scene.py:388-399)
 *   moments    n_records × 2 × (3 + 3d + 3d²): [single, multiple] × (L, grad, hess)
 *   stats      n_records × 8 int64: elements_evaluated, elements_dropped, star_vertices,
 *              media samples, rings, triangulation status, evaluated single, multiple
 *   records    NULL or n_records × 2 × (d + 3 + 3d + d² + d): position, value, grad,
 *              axes (row-major, columns = principal axes), radii
 *   stream     cudaStream_t (NULL = legacy default stream) */
int vc_build_records(vc_scene* scene, int n_records, const double* x, const void* rng,
                     const int32_t* adjacency, const vc_build_params* params, double* moments,
                     int64_t* stats, double* records, void* stream);

/* One record with its per-direction internals copied to host (parity inspection).
 * dirs n×d, s n, idx n, counts n, tris (2n−4)×3 (3D) — any may be NULL; media
 * (media_cap × 3 float32) receives min(P, media_cap) samples, *P the count. */
int vc_build_inspect(vc_scene* scene, const double* x, const void* rng, const int32_t* adjacency,
                     const vc_build_params* params, double* dirs, double* s, int32_t* idx,
                     int32_t* counts, int32_t* tris, float* media, int64_t media_cap, int64_t* P,
                     double* moments, int64_t* stats);

/* make_record for n records × {single, multiple} moments (src/cache.py:146-189).
 * moments n × 2 × (3 + 3d + 3d²) → records n × 2 × (d + 3 + 3d + d² + d). */
int vc_make_records(int n, int dim, const double* x, const double* moments, double epsilon,
                    double scene_scale, double max_emission, int flags, double* records, void* stream);

/* Per-element form factors with derivatives: ff_segment_derivs_batch (2D) /
 * ff_triangle_derivs_batch (3D), src/formfactor.py:85-158, :298-343.  Element i has the
 * point x[i] (m × d) and vertices verts[i] (m × d × d, vertex-major); outputs ok (m),
 * value (m), grad (m × d), hess (m × d × d, symmetric); not-ok elements are zeros.
 * precision 0: the float64 device functions of the record build; 1 (3D only): the
 * float32 element path (ok-mask still decided in float64).  VC_MEM_HOST: host arrays. */
int vc_form_factors(int dim, int m, const double* x, const double* verts, int precision, int flags,
                    uint8_t* ok, double* value, double* grad, double* hess, void* stream);

/* Nearest hit per ray: trace (src/scene.py:271-292; misses t = inf, idx = −1) or, with
 * VC_TRACE_BOUNDS, trace_or_bounds (src/scene.py:306-315; misses t = bounds exit).
 * o, d: m × dim float64; t: m float64; idx: m int32 (original surface index). */
int vc_trace(vc_scene* scene, int m, const double* o, const double* d, double* t, int32_t* idx, int flags,
             void* stream);

/* Outgoing surface radiance per hit: surface_radiance_batch(scene, idx, points, dirs,
 * n_light_samples) (src/transport.py:240-254) — emission (two-sided) + albedo · direct
 * lighting by the emitter quadrature with one shadow ray per sample; idx < 0 → 0.
 * points, dirs: m × dim float64; idx: m int32; out: m × 3 float64. */
int vc_surface_radiance(vc_scene* scene, int m, const double* points, const double* dirs, const int32_t* idx,
                        int n_light_samples, double* out, int flags, void* stream);

/* numpy SeedSequence(words) → PCG64 state (host), for n records of nw words each. */
int vc_seed_states(int n, const uint32_t* words, int nw, uint64_t* states);

typedef struct {
  int n_angular;         /* stratified primary directions (baseline_estimate n_angular) */
  int max_media_bounces; /* collisions per path = max_media_bounces − 1 */
  int n_light_samples;
  double alpha;          /* baseline_alpha: scales log_gradient_radius */
  int flags;             /* VC_MEM_HOST, VC_SEED_WORDS */
  int seed_words;
  int64_t* draws;        /* NULL or n: PCG64 doubles each record's stream consumed, as the
                            reference's rng (the collision loop stops at the first bounce
                            without a collision, src/subdivision.py:480-486) */
} vc_baseline_params;

/* Occlusion-unaware baseline for n records: baseline_estimate (src/subdivision.py:416-521)
 * + make_baseline_record (src/cache.py:212-226).  x, rng as vc_build_records.
 *   estimates  NULL or n × 2 × (3 + 3d): [single, multiple] × (value, grad)
 *   records    NULL or n × 2 × (d + 3 + 3d + d² + d): sphere records in the cache row
 *              layout (axes = identity, every radius = log_gradient_radius)
 *   samples    NULL or n × 2 × 2 × n_angular: [kind] × (luminance values, gradient norms) */
int vc_baseline_records(vc_scene* scene, int n_records, const double* x, const void* rng,
                        const vc_baseline_params* params, double* estimates, double* records, double* samples,
                        void* stream);

/* path_trace_radiance (src/transport.py:318-391) at m query points: out m × 2 × 3 =
 * (J_single, J_multiple).  rng per point as vc_build_records (flags VC_SEED_WORDS +
 * seed_words, or PCG64 states); points sharing a stream get common random numbers
 * (fd_derivatives, src/renderer.py:590-643).  VC_MEM_HOST: host arrays. */
int vc_path_trace(vc_scene* scene, int m, const double* x, const void* rng, int64_t n_samples,
                  int max_media_bounces, int n_light_samples, int flags, int seed_words, double* out, void* stream);

/* Record cache + lookup.  Replaces RadianceCache (src/cache.py:262-334) and
 * interpolate (src/cache.py:342-360).  records: n × (d + 3 + 3d + d² + d) float64,
 * host memory. */
int vc_cache_create(int dim, const double* bounds_min, const double* bounds_max, int n_records,
                    const double* records, vc_cache** out);
void vc_cache_destroy(vc_cache* cache);
/* Append n records (rows as vc_cache_create; host memory with VC_MEM_HOST, else device,
 * e.g. rows received over NCCL) and re-index: RadianceCache.insert (src/cache.py:298-315)
 * for a batch, without re-uploading the records already held.  Creation tags are −1. */
int vc_cache_insert(vc_cache* cache, int n_records, const double* records, int flags, void* stream);
/* log_space = 1: the cache holds BaselineRecord spheres and blends with
 * log_space_interpolate (src/cache.py:363-394); 0 (default): ellipsoids, interpolate. */
int vc_cache_set_blend(vc_cache* cache, int log_space);
/* Blended J per query (NaN row when uncovered) and the covering-record count.
 * xq m × d, J m × 3, count m (int32, may be NULL). */
int vc_cache_interpolate(vc_cache* cache, int m, const double* xq, double* J, int32_t* count,
                         int flags, void* stream);

typedef struct {
  double position[3], look_at[3], up[3];
  double fov_degrees;
  int width, height;
  int row0, rows; /* crop: image rows [row0, row0+rows) (rows = 0 → all) */
  int col0, cols; /* crop: columns */
} vc_camera;

typedef struct {
  int spp;
  double march_step;
  int seed;
  int n_angular;
  int n_inner;
  int n_light_samples;
  double epsilon;
  int estimator;         /* VC_EST_* used for direct evaluations at cache misses */
  int max_media_bounces; /* baseline and path estimators */
  int path_samples;      /* path estimator: path_samples_per_point */
  int grow;              /* 1: frozen = False — misses insert their records (full image only) */
  int isotropic;         /* grow + subdivision: mode "ours-iso" */
  double baseline_alpha; /* grow + baseline */
} vc_render_params;

/* Camera render (src/renderer.py:402-484): camera march with cache lookups.  Frozen
 * (grow = 0): steps no cache pair covers are evaluated directly
 * through the record build with seeds (seed, 211, k, i, m).  image: height × width × 3
 * float64 (only the crop is written); stats: cache_hits, direct_evaluations. */
int vc_render(vc_scene* scene, vc_cache* single, vc_cache* multiple, const vc_camera* camera,
              const vc_render_params* params, double* image, int64_t* stats, int flags,
              void* stream);

/* Record rows and creation tags (march-point ordinal, −1 for records given to
 * vc_cache_create) of a cache, in insertion order.  records: n × record size float64,
 * tags: n int64 (either may be NULL); host memory with VC_MEM_HOST, else device. */
int64_t vc_cache_size(const vc_cache* cache);
int vc_cache_records(const vc_cache* cache, double* records, int64_t* tags, int flags, void* stream);

#define VC_EST_SUBDIVISION 0 /* estimate_moments + make_record, ellipsoid records */
#define VC_EST_BASELINE 1    /* baseline_estimate + make_baseline_record, sphere records */
#define VC_EST_PATH 2        /* path_trace_radiance (render mode "path": every point evaluated) */

#define VC_TARGET_FIELD 1  /* FieldGrid: 2D cell centers, scanline order (src/renderer.py:88-131) */
#define VC_TARGET_CAMERA 2 /* Camera: pixel-center rays marched at march_step (src/renderer.py:134-193) */

typedef struct {
  int target;                 /* VC_TARGET_FIELD or VC_TARGET_CAMERA */
  vc_camera camera;           /* camera target (crop fields ignored) */
  int field_nx, field_ny;     /* field target: cells */
  double field_min[2], field_max[2]; /* field target: FieldGrid bounds */
  double march_step;          /* RenderSettings.march_step (camera march and ring spacing) */
  int seed;                   /* RenderSettings.seed: record seeds (seed, 401, i) */
  int n_angular, n_inner, n_light_samples;
  double epsilon;
  int isotropic;              /* mode "ours-iso" */
  int window;                 /* record builds per speculative window (0: 2048, max 2048) */
  int64_t lookahead;          /* initial lookahead in march points (0: 65536) */
  int estimator;              /* VC_EST_SUBDIVISION (ours-*), VC_EST_BASELINE, VC_EST_PATH (render only) */
  int max_media_bounces;      /* baseline and path estimators */
  double baseline_alpha;      /* baseline estimator only: log_gradient_radius scale */
  int path_samples;           /* path estimator: path_samples_per_point */
  /* Multi-GPU populate (subdivision estimator): when set, every speculative build wave is
   * handed to this hook instead of the local record build.  It receives the wave's n points
   * (device n × dim float64) and seed words (device n × seed_words uint32) and must fill
   * rec_out (device n × 2 × record size float64, single then multiple) and stats_out
   * (device n × 8 int64) for all n, in order, on `stream` — e.g. every rank builds a
   * contiguous share and the shares are all-gathered over NCCL, so every rank resolves the
   * same wave (paper_1805_09258_b200.dist.populate_sharded).  Returns 0 or a VC_E* code. */
  int (*build_hook)(void* user, int n, const double* x, const uint32_t* words, int seed_words, double* rec_out,
                    int64_t* stats_out, void* stream);
  void* build_hook_user;
} vc_populate_params;

/* populate_cache (src/renderer.py:302-327) for the cache modes ours-aniso / ours-iso:
 * march the target's points in scanline order and insert a (single, multiple) record
 * pair, per-cache masked, wherever a cache lacks coverage.  The result equals the
 * sequential loop's caches record for record (speculative windows, exact resolution).
 * Returns two new caches; stats (may be NULL) = points_marched, records_single,
 * records_multiple, windows, builds, discarded_builds, early_stops, 0. */
int vc_populate(vc_scene* scene, const vc_populate_params* params, vc_cache** single, vc_cache** multiple,
                int64_t* stats, void* stream);

/* FieldGrid render (src/renderer.py:425-437) for the cache modes: S(x) = full_angle(2) ·
 * (J_single + J_multiple) at the cell centers, image ny × nx × 3 float64.  Cells no cache
 * pair covers are evaluated directly with seeds (seed, 307, iy, ix); with frozen = 0 they
 * also insert their records into the caches in scanline order (sequentially exact, as
 * vc_populate) and read the blended value back.  stats: cache_hits, direct_evaluations. */
int vc_render_field(vc_scene* scene, vc_cache* single, vc_cache* multiple, const vc_populate_params* params,
                    int frozen, double* image, int64_t* stats, int flags, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* VOLCACHE_B200_H */
