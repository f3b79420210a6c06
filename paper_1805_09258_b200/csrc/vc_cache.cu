// Record cache on device: index build, interpolation, frozen-cache camera march.
// (Index layout and the tag rule: vc_cache.cuh.)
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "vc_build.h"
#include "vc_cache.cuh"

namespace vc {

// ---------------------------------------------------------------------------
// Index build on the device
// ---------------------------------------------------------------------------

struct IdxGeom {
  int dim;
  double origin[3], size, inv_size;
  double span;  // cells of a record's level are ≥ span × its largest AABB extent
};

// Level and cell range of record R; false → overflow list (box leaves the root cube or is
// not finite).  The box is the AABB of the support ellipsoid {Δ : Σ_j (Δ·A_j / r_j)² ≤ 1}
// with orthonormal axes A_j: half-extent e_a = √(Σ_j A_aj² r_j²) (≤ the reference tree's
// max radius), padded for the float64 support test's rounding and the rounding of pos ± e.
// Cell coordinates use the query's map u = (x − origin)·(1/size), floor(u·2^k): both sides
// apply the same monotone function, so a covered point's cell lies in the record's range.
__device__ inline bool record_cells(const IdxGeom& G, const double* R, int& lv, int clo[3], int chi[3]) {
  const int d = G.dim;
  const double* ax = R + d + 3 + 3 * d;
  const double* rad = ax + d * d;
  double e[3] = {0, 0, 0}, emax = 0.0;
  bool fits = true;
  for (int a = 0; a < d; ++a) {
    double q = 0.0;
    for (int j = 0; j < d; ++j) {
      const double t = ax[a * d + j] * rad[j];
      q += t * t;
    }
    e[a] = sqrt(q) * (1.0 + 1e-9) + 1e-12 * G.size + 1e-14 * (fabs(R[a]) + G.size);
    fits = fits && isfinite(e[a]);
    emax = fmax(emax, e[a]);
  }
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  for (int a = 0; a < d && fits; ++a) {
    lo[a] = (R[a] - e[a] - G.origin[a]) * G.inv_size;
    hi[a] = (R[a] + e[a] - G.origin[a]) * G.inv_size;
    if (!(lo[a] >= 0.0 && hi[a] < 1.0)) fits = false;
  }
  if (!fits) return false;
  lv = 0;  // deepest level whose cells are ≥ span·emax (span 2: ≤ 2 cells per axis; 1: ≤ 3; 0.35: ≤ 7)
  while (lv < kMaxLevel && G.size / (double)(1 << (lv + 1)) >= G.span * emax) ++lv;
  const double s = (double)(1 << lv);
  for (int a = 0; a < 3; ++a) clo[a] = chi[a] = 0;
  for (int a = 0; a < d; ++a) {
    clo[a] = min((int)floor(lo[a] * s), (1 << lv) - 1);
    chi[a] = min((int)floor(hi[a] * s), (1 << lv) - 1);
  }
  return true;
}

__global__ void k_idx_count(IdxGeom G, const double* rec, int n, int* cnt, int* ovf, unsigned* lmask) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int lv, clo[3], chi[3];
  bool fits = record_cells(G, rec + (size_t)r * record_size(G.dim), lv, clo, chi);
  int c = 0;
  if (fits) {
    c = (chi[0] - clo[0] + 1) * (chi[1] - clo[1] + 1) * (chi[2] - clo[2] + 1);
    atomicOr(lmask, 1u << lv);
  }
  cnt[r] = c;
  ovf[r] = fits ? 0 : 1;
}

// Cell key: level k above key_shift = d·(deepest occupied level), then the cell's linear
// index (z·2^k + y)·2^k + x — as short as the occupied levels allow, so the radix sort runs
// over key_shift + 5 bits.
__global__ void k_idx_emit(IdxGeom G, const double* rec, int n, const int* off, int key_shift,
                           unsigned long long* keys, int* vals, int r0) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int lv, clo[3], chi[3];
  if (!record_cells(G, rec + (size_t)r * record_size(G.dim), lv, clo, chi)) return;
  int o = off[r];
  for (int z = clo[2]; z <= chi[2]; ++z)
    for (int y = clo[1]; y <= chi[1]; ++y)
      for (int x = clo[0]; x <= chi[0]; ++x) {
        const unsigned long long cell = (((unsigned long long)z << lv | (unsigned long long)y) << lv) | x;
        keys[o] = (unsigned long long)lv << key_shift | cell;
        vals[o] = r0 + r;
        ++o;
      }
}

// One thread per sorted entry: the first entry of each cell run inserts the cell into the
// open-addressing table with its [start, end) range.
__global__ void k_idx_hash(const unsigned long long* keys, int T, int hbits, unsigned long long* hkey,
                           int2* hrange) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const unsigned long long k = keys[t];
  if (t > 0 && keys[t - 1] == k) return;
  int end = t + 1;
  while (end < T && keys[end] == k) ++end;
  const unsigned hm = (1u << hbits) - 1u;
  for (unsigned h = hash_slot(k, hbits);; h = (h + 1) & hm) {
    const unsigned long long prev = atomicCAS(hkey + h, ~0ULL, k);
    if (prev == ~0ULL) {
      hrange[h] = make_int2(t, end);
      return;
    }
  }
}

// rows[t] = side[items[t]]: the rejection rows in entry order (contiguous scans)
__global__ void k_idx_rows(const int* items, int T, const float4* side, float4* rows) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)T * kSide) return;
  const long long t = i / kSide;
  rows[i] = side[(size_t)items[t] * kSide + (i - t * kSide)];
}

// float32 rejection rows (vc_cache.cuh, DevCache::side).  tol bounds |q32 − q| for points with
// q ≤ 1, i.e. |Δ| ≤ √d·r_max: rounding x, p and their difference to float32 (≤ u(|x| + |p| + |Δ|)
// per axis), M to float32 and the products / sums (≤ 5u·|Δ|·Σ_i|M_ij| per axis j), then
// |q32 − q| ≤ Σ_j (2e_j + e_j²) + 8u; doubled.  Non-finite M → tol = +inf (never rejects).
__global__ void k_idx_side(const double* rec, int n, int dim, float4* side) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const double* R = rec + (size_t)r * record_size(dim);
  const double* ax = R + dim + 3 + 3 * dim;
  const double* rad = ax + dim * dim;
  double M[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  double rmax = 0.0, pmax = 0.0;
  for (int j = 0; j < dim; ++j) rmax = fmax(rmax, fabs(rad[j]));
  for (int i = 0; i < dim; ++i) pmax = fmax(pmax, fabs(R[i]));
  bool finite = true;
  for (int i = 0; i < dim; ++i)
    for (int j = 0; j < dim; ++j) {
      M[i][j] = ax[i * dim + j] / rad[j];  // sphere records: identity axes, equal radii
      finite &= isfinite(M[i][j]);
    }
  const double u = 5.9604644775390625e-08;  // 2^-24
  const double dmax = sqrt((double)dim) * rmax;
  const double B = u * (2.0 * pmax + 3.0 * dmax);
  double tol = 8.0 * u;
  for (int j = 0; j < dim; ++j) {
    double ms = 0.0;
    for (int i = 0; i < dim; ++i) ms += fabs(M[i][j]);
    const double e = (B + 5.0 * u * dmax) * ms;
    tol += 2.0 * e + e * e;
  }
  tol *= 2.0;
  if (!finite || !isfinite(tol) || !isfinite(pmax)) tol = INFINITY;
  float4* o = side + (size_t)r * kSide;
  if (dim == 3) {
    o[0] = make_float4((float)R[0], (float)R[1], (float)R[2], (float)tol);
    o[1] = make_float4((float)M[0][0], (float)M[0][1], (float)M[0][2], (float)M[1][0]);
    o[2] = make_float4((float)M[1][1], (float)M[1][2], (float)M[2][0], (float)M[2][1]);
    o[3] = make_float4((float)M[2][2], 0.0f, 0.0f, 0.0f);
  } else {
    o[0] = make_float4((float)R[0], (float)R[1], (float)tol, (float)M[0][0]);
    o[1] = make_float4((float)M[0][1], (float)M[1][0], (float)M[1][1], 0.0f);
  }
}

__global__ void k_cache_gather(const double* src, size_t stride, const int* sel, const long long* tags, int k, int RS,
                               double* dst, long long* dtag) {
  int j = blockIdx.y;
  if (j >= k) return;
  const double* s = src + (size_t)sel[j] * stride;
  for (int t = threadIdx.x; t < RS; t += blockDim.x) dst[(size_t)j * RS + t] = s[t];
  if (threadIdx.x == 0) dtag[j] = tags ? tags[j] : -1;
}

__global__ void k_iota(int* v, int n, int first = 0) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = first + i;
}

__global__ void k_fill_tags(long long* tag, int n, long long v) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) tag[i] = v;
}

int make_dev_camera(const vc_camera& C0, DevCamera* out) {
  DevCamera cam{};
  // camera frame (src/renderer.py:158-170)
  double f[3], r[3], u[3];
  double fn = 0.0;
  for (int a = 0; a < 3; ++a) {
    f[a] = C0.look_at[a] - C0.position[a];
    fn += f[a] * f[a];
  }
  fn = std::sqrt(fn);
  if (fn == 0.0) return fail(VC_EINVAL, "camera look_at must differ from position");
  for (int a = 0; a < 3; ++a) f[a] /= fn;
  r[0] = f[1] * C0.up[2] - f[2] * C0.up[1];
  r[1] = f[2] * C0.up[0] - f[0] * C0.up[2];
  r[2] = f[0] * C0.up[1] - f[1] * C0.up[0];
  double rn = std::sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  if (rn < 1e-9) return fail(VC_EINVAL, "camera up must not be parallel to the view direction");
  for (int a = 0; a < 3; ++a) r[a] /= rn;
  u[0] = r[1] * f[2] - r[2] * f[1];
  u[1] = r[2] * f[0] - r[0] * f[2];
  u[2] = r[0] * f[1] - r[1] * f[0];
  for (int a = 0; a < 3; ++a) {
    cam.pos[a] = C0.position[a];
    cam.fwd[a] = f[a];
    cam.right[a] = r[a];
    cam.up[a] = u[a];
  }
  cam.tan_half = std::tan(C0.fov_degrees * (3.141592653589793 / 180.0) * 0.5);
  cam.aspect = (double)C0.width / (double)C0.height;
  cam.w = C0.width;
  cam.h = C0.height;
  cam.row0 = C0.row0;
  cam.rows = C0.rows > 0 ? C0.rows : C0.height - C0.row0;
  cam.col0 = C0.col0;
  cam.cols = C0.cols > 0 ? C0.cols : C0.width - C0.col0;
  if (cam.w < 1 || cam.h < 1) return fail(VC_EINVAL, "camera resolution must be positive");
  if (cam.row0 < 0 || cam.col0 < 0 || cam.row0 + cam.rows > cam.h || cam.col0 + cam.cols > cam.w)
    return fail(VC_EINVAL, "crop outside the image");
  *out = cam;
  return VC_OK;
}

int cache_init(vc_cache* c, int dim, const double* bmin, const double* bmax) {
  c->dim = dim;
  c->n = 0;
  // root cube of the reference tree (src/cache.py:284-288)
  double diag = 0.0, mx = 0.0;
  for (int a = 0; a < dim; ++a) {
    diag += (bmax[a] - bmin[a]) * (bmax[a] - bmin[a]);
    mx = std::max(mx, bmax[a] - bmin[a]);
  }
  diag = std::sqrt(diag);
  double half = 0.5 * mx + 0.25 * diag;
  for (int a = 0; a < dim; ++a) c->origin[a] = 0.5 * (bmin[a] + bmax[a]) - half;
  c->size = 2.0 * half;
  cudaError_t e = cudaSuccess;
  for (CacheIndex& X : c->ix) {
    X.hbits = 10;
    X.hcap = 1u << X.hbits;
    if (e == cudaSuccess) e = cudaMalloc(&X.hkey, X.hcap * 8);
    if (e == cudaSuccess) e = cudaMemset(X.hkey, 0xff, X.hcap * 8);
    if (e == cudaSuccess) e = cudaMalloc(&X.hrange, X.hcap * sizeof(int2));
    if (e == cudaSuccess) e = cudaMalloc(&X.items, 16);
    if (e == cudaSuccess) e = cudaMalloc(&X.rows, 16 * kSide);
    if (e == cudaSuccess) e = cudaMalloc(&X.overflow, 16);
    X.items_cap = 1;
    X.ovf_cap = 4;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cache index allocation");
  return VC_OK;
}

int cache_reserve(vc_cache* c, size_t n_records, cudaStream_t st) {
  if (n_records <= c->rec_cap) return VC_OK;
  size_t cap = std::max<size_t>(n_records, std::max<size_t>(1024, c->rec_cap * 2));
  const size_t RS = record_size(c->dim);
  double* r = nullptr;
  long long* t = nullptr;
  cudaError_t e = cudaMalloc(&r, cap * RS * 8);
  if (e == cudaSuccess) e = cudaMalloc(&t, cap * 8);
  if (e == cudaSuccess && c->n) e = cudaMemcpyAsync(r, c->d_rec, (size_t)c->n * RS * 8, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess && c->n) e = cudaMemcpyAsync(t, c->d_tag, (size_t)c->n * 8, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    cudaFree(r);
    cudaFree(t);
    return cuda_fail(e, "cache growth");
  }
  cudaFree(c->d_rec);
  cudaFree(c->d_tag);
  c->d_rec = r;
  c->d_tag = t;
  // rejection rows: an incremental rebuild recomputes only the appended records' rows
  float4* sd = nullptr;
  e = cudaMalloc(&sd, cap * kSide * sizeof(float4));
  if (e == cudaSuccess && c->n && c->d_side)
    e = cudaMemcpyAsync(sd, c->d_side, (size_t)c->n * kSide * sizeof(float4), cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    cudaFree(sd);
    return cuda_fail(e, "cache growth");
  }
  cudaFree(c->d_side);
  c->d_side = sd;
  c->rec_cap = cap;
  return VC_OK;
}

int cache_append(vc_cache* c, const double* src, size_t stride, const int* d_sel, const long long* d_tags, int k,
                 cudaStream_t st) {
  if (k <= 0) return VC_OK;
  int rc = cache_reserve(c, (size_t)c->n + k, st);
  if (rc) return rc;
  const int RS = record_size(c->dim);
  k_cache_gather<<<dim3(1, k), 32, 0, st>>>(src, stride, d_sel, d_tags, k, RS, c->d_rec + (size_t)c->n * RS,
                                            c->d_tag + c->n);
  count_launches(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "cache append");
  c->n += k;
  return VC_OK;
}

int cache_truncate(vc_cache* c, int n, cudaStream_t st) {
  (void)st;
  if (n < c->n) c->n = n;
  return VC_OK;
}

// Index records [r0, r0 + nr) into X (scratch in c->ws; the index arrays grow only).
static int index_build(vc_cache* c, CacheIndex& X, int r0, int nr, cudaStream_t st) {
  cudaError_t e = cudaSuccess;
  auto alloc = [&](int slot, size_t bytes) { return c->ws.get(slot, bytes, &e); };
  X.clear();
  if (nr == 0) return VC_OK;
  const int RS = record_size(c->dim);
  const double* rec = c->d_rec + (size_t)r0 * RS;
  IdxGeom G{};
  G.dim = c->dim;
  for (int a = 0; a < 3; ++a) G.origin[a] = c->origin[a];
  G.size = c->size;
  G.inv_size = 1.0 / c->size;
  G.span = c->cell_span;
  if (const char* es = getenv("VOLCACHE_IDX_SPAN"))  // tuning knob: the lookup span (the engine's 2 stays)
    if (c->cell_span < 2.0) G.span = atof(es);
  const int n = nr;
  int* cnt = (int*)alloc(0, (size_t)n * 4);
  int* ovf = (int*)alloc(1, (size_t)n * 4);
  int* off = (int*)alloc(2, ((size_t)n + 1) * 4);
  int* cnt1 = (int*)alloc(3, ((size_t)n + 1) * 4);
  int* n_sel = (int*)alloc(6, 16);
  int* ovf_list = (int*)alloc(5, (size_t)n * 4);
  int* iota = (int*)alloc(12, (size_t)n * 4);
  if (e != cudaSuccess) return cuda_fail(e, "cache index scratch");
  unsigned* lmask = (unsigned*)(n_sel + 2);
  e = cudaMemsetAsync(lmask, 0, 4, st);
  const int nb = (n + 127) / 128;
  k_idx_side<<<nb, 128, 0, st>>>(rec, n, c->dim, c->d_side + (size_t)r0 * kSide);
  k_idx_count<<<nb, 128, 0, st>>>(G, rec, n, cnt, ovf, lmask);
  // scan n+1 entries (the last one a zero slot) → per-record entry offsets and the total
  if (e == cudaSuccess) e = cudaMemcpyAsync(cnt1, cnt, (size_t)n * 4, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(cnt1 + n, 0, 4, st);
  size_t tb = 0, sb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt1, off, n + 1, st);
  cub::DeviceSelect::Flagged(nullptr, sb, iota, ovf, ovf_list, n_sel, n, st);
  void* tmp = alloc(4, std::max(tb, sb));
  if (e != cudaSuccess) return cuda_fail(e, "cache index scan");
  cub::DeviceScan::ExclusiveSum(tmp, tb, cnt1, off, n + 1, st);
  // overflow list (record order) and its count
  k_iota<<<nb, 128, 0, st>>>(iota, n, r0);
  cub::DeviceSelect::Flagged(tmp, sb, iota, ovf, ovf_list, n_sel, n, st);
  int hv[3] = {0, 0, 0};
  if (e == cudaSuccess) e = cudaMemcpyAsync(&hv[0], off + n, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&hv[1], n_sel, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&hv[2], lmask, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "cache index sizes");
  const int T = hv[0];
  X.n_overflow = hv[1];
  X.level_mask = (unsigned)hv[2];
  unsigned long long* keys = (unsigned long long*)alloc(8, (size_t)T * 8 + 8);
  int* vals = (int*)alloc(9, (size_t)T * 4 + 4);
  unsigned long long* keys2 = (unsigned long long*)alloc(10, (size_t)T * 8 + 8);
  if (X.items_cap < (size_t)T + 1) {
    cudaFree(X.items);
    cudaFree(X.rows);
    X.items = nullptr;
    X.rows = nullptr;
    size_t cap = std::max<size_t>((size_t)T + 1, X.items_cap * 2);
    if (e == cudaSuccess) e = cudaMalloc(&X.items, cap * 4);
    if (e == cudaSuccess) e = cudaMalloc(&X.rows, cap * kSide * sizeof(float4));
    X.items_cap = e == cudaSuccess ? cap : 0;
  }
  // hash table: ≥ 2 slots per entry (≥ 2 per occupied cell), power of two
  int hbits = 10;
  while (hbits < 30 && (1ULL << hbits) < 2ULL * (unsigned long long)T) ++hbits;
  if ((1ULL << hbits) > X.hcap) {
    cudaFree(X.hkey);
    cudaFree(X.hrange);
    X.hkey = nullptr;
    X.hrange = nullptr;
    X.hcap = 1ULL << hbits;
    if (e == cudaSuccess) e = cudaMalloc(&X.hkey, X.hcap * 8);
    if (e == cudaSuccess) e = cudaMalloc(&X.hrange, X.hcap * sizeof(int2));
  }
  X.hbits = hbits;
  if (X.ovf_cap < (size_t)X.n_overflow + 1) {  // grows only (no per-rebuild free)
    cudaFree(X.overflow);
    X.overflow = nullptr;
    X.ovf_cap = std::max<size_t>((size_t)X.n_overflow + 1, 2 * X.ovf_cap);
    if (e == cudaSuccess) e = cudaMalloc(&X.overflow, X.ovf_cap * 4);
  }
  if (e == cudaSuccess && X.n_overflow)
    e = cudaMemcpyAsync(X.overflow, ovf_list, (size_t)X.n_overflow * 4, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(X.hkey, 0xff, (1ULL << hbits) * 8, st);
  if (e != cudaSuccess) return cuda_fail(e, "cache index buffers");
  int kmax = 0;
  for (int k = 0; k <= kMaxLevel; ++k)
    if ((X.level_mask >> k) & 1u) kmax = k;
  X.key_shift = c->dim * kmax;
  const int end_bit = X.key_shift + 5;
  k_idx_emit<<<nb, 128, 0, st>>>(G, rec, n, off, X.key_shift, keys, vals, r0);
  // stable sort by cell keeps records in insertion order within a cell
  size_t rb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, rb, keys, keys2, vals, X.items, T, 0, end_bit, st);
  void* rtmp = alloc(11, rb);
  if (e != cudaSuccess) return cuda_fail(e, "cache index sort scratch");
  if (T > 0) {
    cub::DeviceRadixSort::SortPairs(rtmp, rb, keys, keys2, vals, X.items, T, 0, end_bit, st);
    k_idx_hash<<<(T + 127) / 128, 128, 0, st>>>(keys2, T, hbits, X.hkey, X.hrange);
    k_idx_rows<<<(int)(((long long)T * kSide + 255) / 256), 256, 0, st>>>(X.items, T, c->d_side, X.rows);
  }
  count_launches(9);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "cache index build");
  return VC_OK;
}

// Index after an append / truncation: the records since the last full index go to ix[1]
// alone while they number ≤ max(4096, n_main / 4); otherwise (or after a truncation below
// n_main) everything is re-indexed into ix[0].  Either way a query sees every record, in
// the order of one index over all of them (vc_cache.cuh, DevCache).
int cache_rebuild(vc_cache* c, cudaStream_t st) {
  const int n = c->n;
  const int delta = n - c->n_main;
  if (delta >= 0 && delta <= std::max(4096, c->n_main / 4) && c->n_main > 0) {
    return index_build(c, c->ix[1], c->n_main, delta, st);
  }
  c->n_main = n;
  c->ix[1].clear();
  return index_build(c, c->ix[0], 0, n, st);
}

// Both parts re-indexed as one (after a populate run: lookups then scan a single index).
int cache_rebuild_full(vc_cache* c, cudaStream_t st) {
  c->n_main = c->n;
  c->ix[1].clear();
  return index_build(c, c->ix[0], 0, c->n, st);
}

template <int D>
__global__ void k_interpolate(DevCache C, int m, const double* xq, double* J, int* count) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double x[3];
#pragma unroll
  for (int a = 0; a < D; ++a) x[a] = xq[(size_t)i * D + a];
  double j[3];
  int c = 0;
  bool ok = cache_interpolate<D>(C, x, j, &c);
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  J[(size_t)i * 3 + 0] = ok ? j[0] : nan;
  J[(size_t)i * 3 + 1] = ok ? j[1] : nan;
  J[(size_t)i * 3 + 2] = ok ? j[2] : nan;
  if (count) count[i] = c;
}

// ---------------------------------------------------------------------------
// Camera march (src/renderer.py:133-193, :382-394, :440-484)
// ---------------------------------------------------------------------------

struct MarchOut {
  double* image;          // h × w × 3
  long long* miss_cnt;    // per crop pixel (pass 1)
  long long* miss_off;    // per crop pixel exclusive prefix (pass 2)
  double* miss_x;         // miss points (pass 1b)
  uint32_t* miss_words;   // miss seeds (seed, 211, k, i, m)
  const double* miss_J;   // direct-evaluation results (pass 2)
  long long* hits;        // per crop pixel cache hits
  const long long* first; // mode 3: first march-point ordinal per (pass, pixel)
  const long long* c_ord; // mode 3: ordinals of the points that inserted records (sorted)
  const double* c_val;    // mode 3: their direct values
  long long c_n;
};

// mode 0: count misses and hits, and finish every pixel without a miss (its image is the
// hit-only accumulation; a frame over a populated cache is done in this one pass);
// mode 1: write miss points + seeds; mode 2: final accumulation of the pixels with misses;
// mode 3: final accumulation after insertion (frozen=False): each point reads the caches
// as they were when it was reached (records of tag ≤ its ordinal), src/renderer.py:361-368
// REFL = false: the hit's L_o is its emission (no direct-lighting code in the kernel, as k_primary)
#ifndef VC_MARCH_BS
#define VC_MARCH_BS 128
#endif
#ifndef VC_MARCH_TILE
#define VC_MARCH_TILE 1  // cfg5 frame 204.7 -> 172.5 ms against 32 x 1 pixel strips per warp
#endif
#ifndef VC_MARCH_TW
#define VC_MARCH_TW 8    // tile width in pixels (a power of two ≤ 32)
#endif
#ifndef VC_MARCH_MINB
#define VC_MARCH_MINB 8  // resident 128-thread CTAs per SM (≤ 64 registers): cfg5 frame 235 / 230 / 216 / 190 ms at 4 / 5 / 6 / 8
#endif
template <bool REFL>
__global__ void __launch_bounds__(VC_MARCH_BS, VC_MARCH_MINB * 128 / VC_MARCH_BS)
    k_march(DevScene S, DevCache Cs, DevCache Cm, DevCamera cam, int spp, double step, int seed,
            const uint64_t* jit_state, JumpTables jt, int n_light_dummy, MarchOut out, int mode) {
#if VC_MARCH_TILE
  // a warp marches a TW × 32/TW pixel tile (8 × 4): its rays stay within a few cells of one another, so the
  // lanes probe the same index cells and scan similar candidate lists
  constexpr int TW = VC_MARCH_TW, TH = 32 / TW;
  const int tiles_x = (cam.cols + TW - 1) / TW;
  const int tile = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int ty = tile / tiles_x, tx = tile - ty * tiles_x;
  const int ry = ty * TH + lane / TW, rx = tx * TW + lane % TW;
  if (ry >= cam.rows || rx >= cam.cols) return;
  const int t = ry * cam.cols + rx;
  const int py = cam.row0 + ry, px = cam.col0 + rx;
#else
  const int npx = cam.rows * cam.cols;
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= npx) return;
  const int py = cam.row0 + t / cam.cols, px = cam.col0 + t % cam.cols;
#endif
  const long long i = (long long)py * cam.w + px;
  if ((mode == 1 || mode == 2) && out.miss_cnt[t] == 0) return;  // finished by pass 0
  const double four_pi = 4.0 * kPi;
  double img[3] = {0.0, 0.0, 0.0};
  long long nm = 0, hits = 0;
  long long slot = (mode == 1 || mode == 2) ? out.miss_off[t] : 0;
  const bool accum = mode != 1;
  for (int k = 0; k < spp; ++k) {
    double jx = 0.5, jy = 0.5;
    if (spp > 1) {  // rng.random((h, w, 2)) per k from SeedSequence(seed, 101)
      Pcg64 g = pcg_load(jit_state);
      pcg_advance(g, (unsigned long long)((long long)k * cam.h * cam.w * 2 + i * 2), jt);
      jx = g.next_double();
      jy = g.next_double();
    }
    double o[3], d[3];
    camera_ray(cam, px, py, jx, jy, o, d);
    double ts;
    int id;
    trace_closest<3>(S, o, d, ts, id);
    double hp[3], lo[3];
    double tt = isfinite(ts) ? ts : 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) hp[a] = add(o[a], mul(tt, d[a]));
    if (accum) {
      if constexpr (REFL) {
        surface_radiance<3>(S, id, hp, d, lo);
      } else {
        lo[0] = lo[1] = lo[2] = 0.0;
        if (id >= 0)
          for (int c = 0; c < 3; ++c) lo[c] = S.emission[(size_t)id * 3 + c];
      }
    }
    double t_in, t_out;
    bool valid;
    bounds_span(S, o, d, t_in, t_out, valid);
    double acc[3] = {0.0, 0.0, 0.0};
    if (!valid) {
      if (accum && id >= 0) {
        img[0] += lo[0];
        img[1] += lo[1];
        img[2] += lo[2];
      }
      continue;
    }
    double t_end = fmin(ts, t_out);
    if (isnan(ts)) t_end = ts;
    int steps = (int)floor(__ddiv_rn(sub(t_end, t_in), step) + 0.5);
    for (int m = 1; m <= steps; ++m) {
      double tk = add(t_in, mul((double)m - 0.5, step));
      double y[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) y[a] = add(o[a], mul(tk, d[a]));
      double Js[3], Jm[3];
      long long lim = LLONG_MAX;
      if (mode == 3) lim = out.first[(long long)k * cam.w * cam.h + i] + m;
      bool cs = cache_interpolate<3>(Cs, y, Js, nullptr, lim);
      bool cm = cs && cache_interpolate<3>(Cm, y, Jm, nullptr, lim);
      double J[3];
      if (cs && cm) {
        ++hits;
        J[0] = add(Js[0], Jm[0]);
        J[1] = add(Js[1], Jm[1]);
        J[2] = add(Js[2], Jm[2]);
      } else if (mode == 3) {  // inserted, blend still None: the direct value
        const long long ord = lim - 1;
        long long lo = 0, hi = out.c_n;
        while (lo < hi) {
          long long mid = (lo + hi) >> 1;
          if (out.c_ord[mid] < ord) lo = mid + 1;
          else hi = mid;
        }
        const bool f = lo < out.c_n && out.c_ord[lo] == ord;
        for (int c = 0; c < 3; ++c) J[c] = f ? out.c_val[lo * 3 + c] : 0.0;
      } else {
        if (mode == 1) {
          for (int a = 0; a < 3; ++a) out.miss_x[slot * 3 + a] = y[a];
          uint32_t* w = out.miss_words + slot * 5;
          w[0] = (uint32_t)seed;
          w[1] = 211u;
          w[2] = (uint32_t)k;
          w[3] = (uint32_t)i;
          w[4] = (uint32_t)m;
        }
        if (mode == 2) {
          J[0] = out.miss_J[slot * 3 + 0];
          J[1] = out.miss_J[slot * 3 + 1];
          J[2] = out.miss_J[slot * 3 + 2];
        } else {
          J[0] = J[1] = J[2] = 0.0;  // pass 0: this pixel is redone by pass 2
        }
        ++slot;
        ++nm;
      }
      if (accum) {
        double f = mul(mul(exp(-S.sigma_t * sub(tk, t_in)), four_pi), 1.0);
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[c] = add(acc[c], mul(mul(f, J[c]), step));
      }
    }
    if (accum) {
      if (id >= 0) {
        double T = exp(-S.sigma_t * fmax(0.0, sub(t_end, t_in)));
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[c] = add(acc[c], mul(T, lo[c]));
      }
      img[0] += acc[0];
      img[1] += acc[1];
      img[2] += acc[2];
    }
  }
  if (mode == 0) {
    out.miss_cnt[t] = nm;
    out.hits[t] = hits;
  }
  if ((mode == 0 && nm == 0) || mode >= 2) {
#pragma unroll
    for (int c = 0; c < 3; ++c) out.image[i * 3 + c] = __ddiv_rn(img[c], (double)spp);
    if (mode == 3) out.hits[t] = hits;
  }
  (void)n_light_dummy;
}

__global__ void k_misses_J(int m, const double* moments, int MS, double* J) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double* M = moments + (size_t)i * 2 * MS;
  for (int c = 0; c < 3; ++c) J[(size_t)i * 3 + c] = add(M[c], M[MS + c]);
}

}  // namespace vc

using namespace vc;

extern "C" {

int vc_cache_create(int dim, const double* bmin, const double* bmax, int n, const double* records,
                    vc_cache** out) {
  if (!out) return fail(VC_EINVAL, "null output handle");
  *out = nullptr;
  if (dim != 2 && dim != 3) return fail(VC_EINVAL, "bounds must be matching 2- or 3-vectors");
  for (int a = 0; a < dim; ++a)
    if (!(bmax[a] > bmin[a])) return fail(VC_EINVAL, "bounds_max must exceed bounds_min");
  if (n < 0) return fail(VC_EINVAL, "negative record count");
  vc_cache* c = new vc_cache();
  int rc = cache_init(c, dim, bmin, bmax);
  if (!rc) rc = cache_reserve(c, (size_t)std::max(n, 1), 0);
  if (!rc && n > 0) {
    cudaError_t e = cudaMemcpy(c->d_rec, records, (size_t)n * record_size(dim) * 8, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) rc = cuda_fail(e, "cache upload");
    k_fill_tags<<<(n + 255) / 256, 256>>>(c->d_tag, n, -1LL);
    c->n = n;
  }
  if (!rc) rc = cache_rebuild(c, 0);
  if (!rc) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) rc = cuda_fail(e, "cache build");
  }
  if (rc) {
    delete c;
    return rc;
  }
  *out = c;
  return VC_OK;
}

void vc_cache_destroy(vc_cache* c) { delete c; }

int vc_cache_insert(vc_cache* c, int n, const double* records, int flags, void* stream) {
  if (!c) return fail(VC_EINVAL, "null cache");
  if (n < 0) return fail(VC_EINVAL, "negative record count");
  if (n == 0) return VC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t RS = record_size(c->dim);
  int rc = cache_reserve(c, (size_t)c->n + n, st);
  if (rc) return rc;
  cudaError_t e = cudaMemcpyAsync(c->d_rec + (size_t)c->n * RS, records, (size_t)n * RS * 8,
                                  (flags & VC_MEM_HOST) ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "cache insert upload");
  k_fill_tags<<<(n + 255) / 256, 256, 0, st>>>(c->d_tag + c->n, n, -1LL);
  count_launches(1);
  c->n += n;
  rc = cache_rebuild(c, st);
  if (rc) return rc;
  e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? VC_OK : cuda_fail(e, "cache insert");
}

int vc_cache_set_blend(vc_cache* c, int log_space) {
  if (!c) return fail(VC_EINVAL, "null cache");
  c->blend = log_space ? 1 : 0;
  return VC_OK;
}

int vc_cache_interpolate(vc_cache* c, int m, const double* xq, double* J, int32_t* count, int flags,
                         void* stream) {
  if (!c) return fail(VC_EINVAL, "null cache");
  if (m <= 0) return VC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const bool host = flags & VC_MEM_HOST;
  const int D = c->dim;
  const double* dx = xq;
  double* dJ = J;
  int* dc = count;
  std::vector<void*> tmp;
  cudaError_t e = cudaSuccess;
  if (host) {
    double* a = nullptr;
    double* b = nullptr;
    int* cc = nullptr;
    e = cudaMalloc(&a, (size_t)m * D * 8);
    if (e == cudaSuccess) e = cudaMalloc(&b, (size_t)m * 24);
    if (e == cudaSuccess && count) e = cudaMalloc(&cc, (size_t)m * 4);
    if (e == cudaSuccess) e = cudaMemcpyAsync(a, xq, (size_t)m * D * 8, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "interpolate staging");
    dx = a;
    dJ = b;
    dc = cc;
    tmp = {a, b, cc};
  }
  DevCache C = c->dev();
  if (D == 2) k_interpolate<2><<<(m + 127) / 128, 128, 0, st>>>(C, m, dx, dJ, dc);
  else k_interpolate<3><<<(m + 127) / 128, 128, 0, st>>>(C, m, dx, dJ, dc);
  count_launches(1);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "interpolate launch");
  if (host) {
    e = cudaMemcpyAsync(J, dJ, (size_t)m * 24, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && count) e = cudaMemcpyAsync(count, dc, (size_t)m * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    for (void* p : tmp) cudaFree(p);
    if (e != cudaSuccess) return cuda_fail(e, "interpolate download");
  }
  return VC_OK;
}

#define VC_MARCH(refl) ((refl) ? k_march<true> : k_march<false>)

int vc_render(vc_scene* sc, vc_cache* cs, vc_cache* cm, const vc_camera* camp, const vc_render_params* rp,
              double* image, int64_t* stats, int flags, void* stream) {
  if (!sc || !cs || !cm || !camp || !rp || !image) return fail(VC_EINVAL, "null argument");
  if (sc->dim != 3 || cs->dim != 3 || cm->dim != 3) return fail(VC_EINVAL, "Camera rendering requires a 3D scene");
  if (!(rp->march_step > 0.0)) return fail(VC_EINVAL, "march_step must be positive");
  if (rp->spp < 1) return fail(VC_EINVAL, "spp must be at least 1");
  cudaStream_t st = (cudaStream_t)stream;
  const vc_camera& C0 = *camp;
  DevCamera cam{};
  int rc = make_dev_camera(*camp, &cam);
  if (rc) return rc;
  const int npx = cam.rows * cam.cols;
  rc = ensure_emitters(sc, rp->n_light_samples);
  if (rc) return rc;
  DevScene S = dev_scene(sc);
  cudaError_t e = cudaSuccess;
  // jitter stream: default_rng(SeedSequence([seed, 101]))
  uint32_t jw[2] = {(uint32_t)rp->seed, 101u};
  uint64_t jst[4];
  seedseq_pcg64(jw, 2, jst);
  JumpTables jt{jump_tables(&e)};
  if (!jt.tab) return cuda_fail(e, "jump tables");
  Workspace& ws = sc->ws;
  auto alloc = [&](int slot, size_t bytes) { return ws.get(slot, bytes, &e); };
  uint64_t* djit = (uint64_t*)alloc(22, 32);
  long long* mcnt = (long long*)alloc(23, ((size_t)npx + 1) * 8);
  long long* moff = (long long*)alloc(24, ((size_t)npx + 1) * 8);
  long long* hits = (long long*)alloc(25, (size_t)npx * 8);
  double* dimg = (double*)alloc(26, (size_t)cam.w * cam.h * 24);
  if (e != cudaSuccess) return cuda_fail(e, "render workspace");
  e = cudaMemcpyAsync(djit, jst, 32, cudaMemcpyHostToDevice, st);
  MarchOut mo{};
  mo.image = dimg;
  mo.miss_cnt = mcnt;
  mo.miss_off = moff;
  mo.hits = hits;
#if VC_MARCH_TILE
  const int grid = (int)(((long long)((cam.rows + 32 / VC_MARCH_TW - 1) / (32 / VC_MARCH_TW)) *
                              ((cam.cols + VC_MARCH_TW - 1) / VC_MARCH_TW) * 32 + VC_MARCH_BS - 1) / VC_MARCH_BS);
#else
  const int grid = (npx + VC_MARCH_BS - 1) / VC_MARCH_BS;
#endif
  if (rp->grow) {  // frozen = False: misses insert in (pass, pixel, step) order (src/renderer.py:361-368)
    if (rp->estimator == VC_EST_PATH) return fail(VC_EINVAL, "the path mode has no cache to grow");
    if (cam.rows != cam.h || cam.cols != cam.w) return fail(VC_EINVAL, "frozen=False renders the full image (no crop)");
    vc_populate_params pp{};
    pp.target = VC_TARGET_CAMERA;
    pp.camera = C0;
    pp.march_step = rp->march_step;
    pp.seed = rp->seed;
    pp.n_angular = rp->n_angular;
    pp.n_inner = rp->n_inner;
    pp.n_light_samples = rp->n_light_samples;
    pp.epsilon = rp->epsilon > 0 ? rp->epsilon : 0.05;
    pp.isotropic = rp->isotropic;
    pp.estimator = rp->estimator;
    pp.max_media_bounces = rp->max_media_bounces;
    pp.baseline_alpha = rp->baseline_alpha;
    RenderStream rs;
    int64_t pst[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    rc = populate_run(sc, &pp, 2, cs, cm, pst, st, nullptr, rp->spp, &rs);
    if (rc) return rc;
    mo.first = rs.first;
    mo.c_ord = rs.c_ord;
    mo.c_val = rs.c_val;
    mo.c_n = rs.c_n;
    VC_MARCH(S.reflective)<<<grid, VC_MARCH_BS, 0, st>>>(S, cs->dev(), cm->dev(), cam, rp->spp, rp->march_step, rp->seed, djit, jt, 0, mo,
                                  3);
    count_launches(1);
    e = cudaGetLastError();
    for (int y = 0; y < cam.h && e == cudaSuccess; ++y)
      e = cudaMemcpyAsync(image + (size_t)y * cam.w * 3, dimg + (size_t)y * cam.w * 3, (size_t)cam.w * 24,
                          (flags & VC_MEM_HOST) ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "render download");
    if (stats) {
      stats[0] = rs.total - pst[7];
      stats[1] = pst[7];
    }
    return VC_OK;
  }
  DevCache Cs = cs->dev(), Cm = cm->dev();
  prof_begin(KC_MARCH, st);
  VC_MARCH(S.reflective)<<<grid, VC_MARCH_BS, 0, st>>>(S, Cs, Cm, cam, rp->spp, rp->march_step, rp->seed, djit, jt, 0, mo, 0);
  prof_end(st);
  // miss offsets (device scan over npx + 1 counts, the last one zero) and the hit total
  long long* hsum = (long long*)alloc(50, 16);
  e = cudaMemsetAsync(mcnt + npx, 0, 8, st);
  size_t tb = 0, tr = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, mcnt, moff, npx + 1, st);
  cub::DeviceReduce::Sum(nullptr, tr, hits, hsum, npx, st);
  void* tmp = alloc(51, std::max(tb, tr));
  if (e != cudaSuccess) return cuda_fail(e, "march scan scratch");
  cub::DeviceScan::ExclusiveSum(tmp, tb, mcnt, moff, npx + 1, st);
  cub::DeviceReduce::Sum(tmp, tr, hits, hsum, npx, st);
  e = cudaMemcpyAsync(hsum + 1, moff + npx, 8, cudaMemcpyDeviceToDevice, st);
  long long hv[2] = {0, 0};
  if (e == cudaSuccess) e = cudaMemcpyAsync(hv, hsum, 16, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "march pass 1");
  const long long nmiss = hv[1];
  long long launches = 3;
  if (nmiss > 0) {
    double* mx = (double*)alloc(27, (size_t)nmiss * 24);
    uint32_t* mw = (uint32_t*)alloc(28, (size_t)nmiss * 20);
    double* mmom = (double*)alloc(29, (size_t)nmiss * 2 * moment_size(3) * 8);
    long long* mst = (long long*)alloc(30, (size_t)nmiss * kStats * 8);
    double* mJ = (double*)alloc(31, (size_t)nmiss * 24);
    if (e != cudaSuccess) return cuda_fail(e, "miss workspace");
    mo.miss_x = mx;
    mo.miss_words = mw;
    VC_MARCH(S.reflective)<<<grid, VC_MARCH_BS, 0, st>>>(S, Cs, Cm, cam, rp->spp, rp->march_step, rp->seed, djit, jt, 0, mo, 1);
    vc_build_params bp{};
    bp.n_angular = rp->n_angular;
    bp.march_step = rp->march_step;
    bp.n_inner = rp->n_inner;
    bp.n_light_samples = rp->n_light_samples;
    bp.epsilon = rp->epsilon > 0 ? rp->epsilon : 0.05;
    bp.flags = VC_SEED_WORDS;
    bp.seed_words = 5;
    // direct evaluations at cache misses (src/renderer.py:361-368, frozen)
    int stride = moment_size(3);
    if (rp->estimator == VC_EST_PATH) {  // _point_value, mode "path" (src/renderer.py:337-346)
      stride = 3;
      rc = path_impl(sc, (int)nmiss, mx, mw, rp->path_samples, rp->max_media_bounces, rp->n_light_samples,
                     VC_SEED_WORDS, 5, mmom, st);
    } else if (rp->estimator == VC_EST_BASELINE) {  // CacheSet.compute, mode "baseline"
      vc_baseline_params blp{};
      blp.n_angular = rp->n_angular;
      blp.max_media_bounces = rp->max_media_bounces;
      blp.n_light_samples = rp->n_light_samples;
      blp.alpha = 1.0;
      blp.flags = VC_SEED_WORDS;
      blp.seed_words = 5;
      stride = 3 + 3 * 3;
      rc = baseline_impl(sc, (int)nmiss, mx, mw, &blp, mmom, nullptr, nullptr, st);
    } else {
      rc = build_impl(sc, (int)nmiss, mx, mw, nullptr, &bp, mmom, (int64_t*)mst, nullptr, st, nullptr);
    }
    if (rc) return rc;
    k_misses_J<<<(int)((nmiss + 127) / 128), 128, 0, st>>>((int)nmiss, mmom, stride, mJ);
    mo.miss_J = mJ;
    prof_begin(KC_MARCH, st);
    VC_MARCH(S.reflective)<<<grid, VC_MARCH_BS, 0, st>>>(S, Cs, Cm, cam, rp->spp, rp->march_step, rp->seed, djit, jt, 0, mo, 2);
    prof_end(st);
    launches += 3;
  }
  count_launches(launches);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "march launch");
  const bool host = flags & VC_MEM_HOST;
  // the crop rows (pitched copy)
  const size_t pitch = (size_t)cam.w * 24;
  e = cudaMemcpy2DAsync(image + ((size_t)cam.row0 * cam.w + cam.col0) * 3, pitch,
                        dimg + ((size_t)cam.row0 * cam.w + cam.col0) * 3, pitch, (size_t)cam.cols * 24, cam.rows,
                        host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "render download");
  if (stats) {
    stats[0] = hv[0];
    stats[1] = nmiss;
  }
  return VC_OK;
}

}  // extern "C"
