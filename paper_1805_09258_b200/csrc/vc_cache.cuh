// Record cache on device: handle type, device view and the support / blend routines
// shared by the lookup, the camera march and the populate engine.
//
// Index: the reference keeps records in an MX-CIF tree whose point query returns
// exactly the records with support > 0 (src/cache.py:262-334, ≡ linear scan).  Here the
// index is a spatial hash over a pyramid of grids on the same padded root cube: level k
// has 2^k cells per axis (k ≤ 16, the reference tree's depth cap), and a record is listed
// in every cell of the deepest level whose cells are at least twice its axis-aligned
// extent (the exact AABB of its support ellipsoid, padded) — ≤ 2^d cells.  Occupied cells
// sit in an open-addressing table (key = level and cell coordinates) mapping to their run
// of entries; each entry carries the record's float32 rejection row inline, so a lookup
// scans contiguous rows.  A query probes one cell per occupied level plus the overflow
// list of records whose box leaves the root cube, and applies the reference's strict
// support test — the covering set is identical to the linear scan.  The index is rebuilt
// on the device (count → scan → stable radix sort by cell → hash insert) after every insert
// batch.
//
// Every record carries a tag (the ordinal of the march point that created it, or −1):
// a query with limit t sees only records with tag < t, which is how the populate
// engine evaluates "the cache as it was when point t was reached" after records of
// later points have been appended speculatively.
#pragma once

#include <climits>
#include <vector>

#include "vc_api_internal.h"
#include "vc_device.cuh"

namespace vc {

constexpr int kMaxLevel = 16;  // finest grid: 2^16 cells per axis

// float32 rejection row of a record: position, M = axes / radii (column j scaled by
// 1/radius_j; for sphere records I / radius) and tol, a bound on |q32 − q| for every point
// whose true q = Σ_j (Δ·axes_j / r_j)² ≤ 1 (i.e. |Δ| ≤ √d·r_max), so q32 > 1 + tol proves
// support ≤ 0 (not covering).  3D: {p.xyz, tol}, {M00 M01 M02 M10}, {M11 M12 M20 M21},
// {M22 0 0 0}; 2D: {p.xy, tol, M00}, {M01 M10 M11 0}.
constexpr int kSide = 4;

// One spatial-hash index over a contiguous range of a cache's records.
struct DevIndex {
  unsigned level_mask;         // bit k: level k lists at least one record
  int hbits;                   // hash table: 2^hbits slots
  int key_shift;               // d · (deepest occupied level): cell keys are k << key_shift | cell
  int n_overflow;
  const unsigned long long* hkey;  // cell key per slot (~0: empty); cell = (z·2^k + y)·2^k + x
  const int2* hrange;          // the cell's entries [start, end)
  const int* items;            // record of each entry (cell order; insertion order within a cell)
  const float4* rows;          // kSide rejection rows per entry (copies of side[items[t]])
  const int* overflow;         // records whose box leaves the root cube (record order)
};

// ix[0] indexes records [0, n_main), ix[1] the records appended since (the populate engine
// re-indexes only those after each window); a query visits, per level, ix[0]'s cell then
// ix[1]'s, then both overflow lists — record for record the order of one index over all.
struct DevCache {
  int dim, n;
  int blend;                   // 0: ellipsoid records, linear blend; 1: sphere records, log-space blend
  double origin[3];
  double size, inv_size;       // root cube
  DevIndex ix[2];
  const double* rec;           // n × record_size(dim), reference layout
  const long long* tag;        // n creation ordinals
  const float4* side;          // n × kSide float32 rejection rows (record_side)
};

__host__ __device__ __forceinline__ unsigned hash_slot(unsigned long long key, int hbits) {
  return (unsigned)((key * 0x9E3779B97F4A7C15ULL) >> (64 - hbits));
}

}  // namespace vc

// Host side of one DevIndex (device arrays grow only).
struct CacheIndex {
  unsigned long long* hkey = nullptr;
  int2* hrange = nullptr;
  int hbits = 10, key_shift = 0;
  size_t hcap = 0;
  int* items = nullptr;
  float4* rows = nullptr;
  size_t items_cap = 0;
  int* overflow = nullptr;
  int n_overflow = 0;
  size_t ovf_cap = 0;
  unsigned level_mask = 0;
  vc::DevIndex dev() const {
    return vc::DevIndex{level_mask, hbits, key_shift, n_overflow, hkey, hrange, items, rows, overflow};
  }
  void clear() {
    level_mask = 0;
    n_overflow = 0;
  }
  ~CacheIndex() {
    cudaFree(hkey);
    cudaFree(hrange);
    cudaFree(items);
    cudaFree(rows);
    cudaFree(overflow);
  }
};

struct vc_cache {
  int dim = 0, n = 0;
  int blend = 0;  // 1: baseline cache (BaselineRecord spheres, log_space_interpolate)
  double origin[3] = {0, 0, 0}, size = 0.0;
  // Level choice: a record's cells are ≥ cell_span × its largest AABB half-extent.  Lookups and
  // marches run at 0.35 (≤ 7 cells per axis: small cells list few records that do not cover the
  // query — cfg5 frame 377 ms at span 2, 224 at 1 on pixel strips; with the tiled march 172.5
  // at 1, 142.0 at 0.5, 134.1 at 0.35, 142.7 at 0.25); the populate engine, which rebuilds
  // after every window, runs with 2 (≤ 2 per axis, fewer entries to sort) and re-indexes at the
  // lookup span when it finishes.
  double cell_span = 0.35;
  // ix[0] covers records [0, n_main); appends up to max(4096, n_main / 4) records are indexed
  // in ix[1] alone, then everything is re-indexed into ix[0] (cache_rebuild)
  CacheIndex ix[2];
  int n_main = 0;
  double* d_rec = nullptr;
  long long* d_tag = nullptr;
  float4* d_side = nullptr;  // kSide float4 per record (rejection rows)
  size_t rec_cap = 0;  // records
  vc::Workspace ws;    // index-build scratch
  vc::DevCache dev() const {
    vc::DevCache c{};
    c.dim = dim;
    c.n = n;
    c.blend = blend;
    for (int a = 0; a < 3; ++a) c.origin[a] = origin[a];
    c.size = size;
    c.inv_size = 1.0 / size;
    c.ix[0] = ix[0].dev();
    c.ix[1] = ix[1].dev();
    c.rec = d_rec;
    c.tag = d_tag;
    c.side = d_side;
    return c;
  }
  ~vc_cache() {
    cudaFree(d_rec);
    cudaFree(d_tag);
    cudaFree(d_side);
  }
};

namespace vc {

// ---------------------------------------------------------------------------
// Camera rays and medium span (src/renderer.py:133-193, :382-394)
// ---------------------------------------------------------------------------

struct DevCamera {
  double pos[3], fwd[3], right[3], up[3];
  double tan_half, aspect;
  int w, h, row0, rows, col0, cols;
};

__device__ inline void camera_ray(const DevCamera& cam, int px, int py, double jx, double jy, double* o, double* d) {
  double u = __ddiv_rn(add((double)px, jx), (double)cam.w);
  double v = __ddiv_rn(add((double)py, jy), (double)cam.h);
  double xn = mul(mul(sub(mul(2.0, u), 1.0), cam.tan_half), cam.aspect);
  double yn = mul(sub(1.0, mul(2.0, v)), cam.tan_half);
  double nn = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    d[a] = add(add(cam.fwd[a], mul(xn, cam.right[a])), mul(yn, cam.up[a]));
    nn = add(nn, mul(d[a], d[a]));
  }
  nn = sqrt(nn);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    d[a] = __ddiv_rn(d[a], nn);
    o[a] = cam.pos[a];
  }
}

__device__ inline void bounds_span(const DevScene& S, const double* o, const double* d, double& t_in,
                                   double& t_out, bool& valid) {
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  double nr = 0.0, fr = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double t1 = __ddiv_rn(sub(S.bmin[a], o[a]), d[a]);
    double t2 = __ddiv_rn(sub(S.bmax[a], o[a]), d[a]);
    double near = np_min(t1, t2), far = np_max(t1, t2);
    near = isnan(near) ? -INFINITY : near;
    far = isnan(far) ? INFINITY : far;
    nr = (a == 0) ? near : np_max(nr, near);
    fr = (a == 0) ? far : np_min(fr, far);
  }
  (void)nan;
  t_in = fmax(nr, 0.0);
  t_out = fr;
  valid = t_out > t_in;
}

// Camera render with insertion: ray prefix over (pass, pixel) and the direct values of
// the points that built records, in ordinal order (vc_populate.cu → vc_render).
struct RenderStream {
  long long* first = nullptr;
  long long* c_ord = nullptr;
  double* c_val = nullptr;
  long long c_n = 0, total = 0;
  ~RenderStream() {
    cudaFree(first);
    cudaFree(c_ord);
    cudaFree(c_val);
  }
};
int populate_run(vc_scene* sc, const vc_populate_params* pp, int seed_kind, vc_cache* cs, vc_cache* cm,
                 int64_t* stats, cudaStream_t st, double* commit_J, int spp, RenderStream* rs);

// Host-side cache management (vc_cache.cu).
int make_dev_camera(const vc_camera& cam, DevCamera* out);
int cache_init(vc_cache* c, int dim, const double* bmin, const double* bmax);
int cache_reserve(vc_cache* c, size_t n_records, cudaStream_t st);
// Append k record rows gathered from src (row j = src + sel[j]·stride doubles) with tags.
int cache_append(vc_cache* c, const double* src, size_t stride, const int* d_sel, const long long* d_tags,
                 int k, cudaStream_t st);
int cache_truncate(vc_cache* c, int n, cudaStream_t st);
int cache_rebuild(vc_cache* c, cudaStream_t st);       // incremental (appended records in ix[1])
int cache_rebuild_full(vc_cache* c, cudaStream_t st);  // every record in ix[0]

// support coordinate 1 − ‖(Δ·A)/r‖ (src/cache.py:112-116)
template <int D>
__device__ __forceinline__ double record_support(const double* R, const double* x, double* dl) {
  const double* pos = R;
  const double* ax = R + D + 3 + 3 * D;
  const double* rad = R + D + 3 + 3 * D + D * D;
#pragma unroll
  for (int a = 0; a < D; ++a) dl[a] = sub(x[a], pos[a]);
  double q = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    double al = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) al = add(al, mul(dl[i], ax[i * D + j]));
    double t = __ddiv_rn(al, rad[j]);
    q = add(q, mul(t, t));
  }
  return sub(1.0, sqrt(q));
}

// sphere record: 1 − ‖Δ‖/radius (src/cache.py:142-145); radius stored in every radii slot
template <int D>
__device__ __forceinline__ double sphere_support(const double* R, const double* x, double* dl) {
  const double* rad = R + D + 3 + 3 * D + D * D;
  double q = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    dl[a] = sub(x[a], R[a]);
    q = add(q, mul(dl[a], dl[a]));
  }
  return sub(1.0, __ddiv_rn(sqrt(q), rad[0]));
}

// Cubic weight of a support coordinate (src/cache.py:49-56).
__device__ __forceinline__ double support_weight(double sup) {
  double d = fmin(fmax(sup, 0.0), 1.0);
  return sub(mul(mul(3.0, d), d), mul(mul(mul(2.0, d), d), d));
}

// support coordinate, first-order estimate, cubic weight (src/cache.py:49-56, :112-121)
template <int D>
__device__ __forceinline__ void blend_record(const double* R, const double* x, double num[3], double& den,
                                             int& hits) {
  const double* val = R + D;
  const double* grd = R + D + 3;
  double dl[D];
  double sup = record_support<D>(R, x, dl);
  if (!(sup > 0.0)) return;
  ++hits;
  double w = support_weight(sup);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double e = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) e = add(e, mul(grd[c * D + i], dl[i]));
    e = add(val[c], e);
    e = fmax(e, 0.0);
    num[c] = add(num[c], mul(w, e));
  }
  den = add(den, w);
}

// float32 rejection of a row (see record_side): true when the record certainly has
// support ≤ 0 at x; x32 is x rounded to float32.  NaN (a zero radius) never rejects.
template <int D>
__device__ __forceinline__ bool row_rejects(const float4* sd, const float* x32) {
  const float4 s0 = __ldg(sd), s1 = __ldg(sd + 1);
  if constexpr (D == 3) {
    const float4 s2 = __ldg(sd + 2), s3 = __ldg(sd + 3);
    const float d0 = x32[0] - s0.x, d1 = x32[1] - s0.y, d2 = x32[2] - s0.z;
    const float a0 = d0 * s1.x + d1 * s1.w + d2 * s2.z;
    const float a1 = d0 * s1.y + d1 * s2.x + d2 * s2.w;
    const float a2 = d0 * s1.z + d1 * s2.y + d2 * s3.x;
    const float q = a0 * a0 + a1 * a1 + a2 * a2;
    return q > 1.0f + s0.w;
  } else {
    const float d0 = x32[0] - s0.x, d1 = x32[1] - s0.y;
    const float a0 = d0 * s0.w + d1 * s1.y;
    const float a1 = d0 * s1.x + d1 * s1.z;
    const float q = a0 * a0 + a1 * a1;
    return q > 1.0f + s0.z;
  }
}

// Visit the records of x that survive the float32 rejection, in index order (coarse level
// first, then the overflow list); f(record_index) returns true to stop early.
template <int D, typename F>
__device__ __forceinline__ bool index_cell(const DevIndex& X, int k, unsigned long long cell, const float* x32, F& f) {
  if (!((X.level_mask >> k) & 1u)) return false;
  const unsigned long long key = (unsigned long long)k << X.key_shift | cell;
  const unsigned hm = (1u << X.hbits) - 1u;
  for (unsigned h = hash_slot(key, X.hbits);; h = (h + 1) & hm) {
    const unsigned long long kk = X.hkey[h];
    if (kk == key) {
      const int2 r = X.hrange[h];
      for (int t = r.x; t < r.y; ++t)
        if (!row_rejects<D>(X.rows + (size_t)t * kSide, x32) && f(X.items[t])) return true;
      return false;
    }
    if (kk == ~0ULL) return false;
  }
}

template <int D, typename F>
__device__ __forceinline__ void cache_visit(const DevCache& C, const double* x, F&& f) {
  float x32[D];
  double u[D];
  bool in = true;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    x32[a] = (float)x[a];
    u[a] = (x[a] - C.origin[a]) * C.inv_size;  // the same map as the registration (k_idx_*)
    in = in && u[a] >= 0.0 && u[a] < 1.0;
  }
  if (in) {
    for (unsigned m = C.ix[0].level_mask | C.ix[1].level_mask; m; m &= m - 1) {
      const int k = __ffs(m) - 1;
      const double s = (double)(1u << k);
      unsigned long long cell = 0;
#pragma unroll
      for (int a = D - 1; a >= 0; --a) cell = (cell << k) | (unsigned long long)min((int)floor(u[a] * s), (1 << k) - 1);
      if (index_cell<D>(C.ix[0], k, cell, x32, f)) return;
      if (index_cell<D>(C.ix[1], k, cell, x32, f)) return;
    }
  }
  for (int p = 0; p < 2; ++p)
    for (int t = 0; t < C.ix[p].n_overflow; ++t) {
      const int r = C.ix[p].overflow[t];
      if (!row_rejects<D>(C.side + (size_t)r * kSide, x32) && f(r)) return;
    }
}

// log-space blend term of one sphere record (src/cache.py:363-394)
template <int D>
__device__ __forceinline__ void log_blend_record(const double* R, const double* x, double num[3], double den[3],
                                                 int& hits) {
  const double* val = R + D;
  const double* grd = R + D + 3;
  double dl[D];
  double sup = sphere_support<D>(R, x, dl);
  if (!(sup > 0.0)) return;
  ++hits;
  const double w = support_weight(sup);
  if (!(w > 0.0)) return;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    if (!(val[c] > 0.0)) continue;
    double gd = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) gd = add(gd, mul(grd[c * D + i], dl[i]));
    const double le = add(log(val[c]), __ddiv_rn(gd, val[c]));
    num[c] = add(num[c], mul(w, le));
    den[c] = add(den[c], w);
  }
}

// Blended J over records with tag < limit; false when the reference returns None
// (interpolate, src/cache.py:342-360; log_space_interpolate, :363-394).
template <int D>
__device__ inline bool cache_interpolate(const DevCache& C, const double* x, double J[3], int* count,
                                         long long limit = LLONG_MAX) {
  double num[3] = {0.0, 0.0, 0.0}, den[3] = {0.0, 0.0, 0.0};
  int hits = 0;
  const int RS = record_size(D);
  if (C.blend == 0) {
    cache_visit<D>(C, x, [&](int r) {
      if (C.tag[r] < limit) blend_record<D>(C.rec + (size_t)r * RS, x, num, den[0], hits);
      return false;
    });
    if (count) *count = hits;
    if (hits == 0 || !(den[0] > 0.0)) return false;
    J[0] = __ddiv_rn(num[0], den[0]);
    J[1] = __ddiv_rn(num[1], den[0]);
    J[2] = __ddiv_rn(num[2], den[0]);
    return true;
  }
  cache_visit<D>(C, x, [&](int r) {
    if (C.tag[r] < limit) log_blend_record<D>(C.rec + (size_t)r * RS, x, num, den, hits);
    return false;
  });
  if (count) *count = hits;
  const bool live = den[0] > 0.0 || den[1] > 0.0 || den[2] > 0.0;
  if (hits == 0 || !live) return false;
#pragma unroll
  for (int c = 0; c < 3; ++c) J[c] = den[c] > 0.0 ? exp(__ddiv_rn(num[c], den[c])) : 0.0;
  return true;
}

// interpolate(cache, x) is not None ⇔ some record with tag < limit has support > 0 and
// a positive weight (the blend denominator is a sum of non-negative weights); for the
// log-space blend the record must also hold a positive channel.
template <int D>
__device__ inline bool cache_covers(const DevCache& C, const double* x, long long limit) {
  const int RS = record_size(D);
  bool hit = false;
  cache_visit<D>(C, x, [&](int r) {
    if (C.tag[r] >= limit) return false;
    const double* R = C.rec + (size_t)r * RS;
    double dl[D];
    if (C.blend == 0) {
      double sup = record_support<D>(R, x, dl);
      hit = sup > 0.0 && support_weight(sup) > 0.0;
    } else {
      double sup = sphere_support<D>(R, x, dl);
      hit = sup > 0.0 && support_weight(sup) > 0.0 && (R[D] > 0.0 || R[D + 1] > 0.0 || R[D + 2] > 0.0);
    }
    return hit;
  });
  return hit;
}

}  // namespace vc
