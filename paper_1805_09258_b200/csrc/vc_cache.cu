// Record cache on device: multi-level grid index, interpolation, frozen-cache camera march.
//
// Index: the reference keeps records in an MX-CIF tree whose point query returns
// exactly the records with support > 0 (src/cache.py:262-334, ≡ linear scan).  Here a
// record of bounding radius r lives on the coarsest-needed level ℓ of a pyramid of
// dense grids over the same padded root cube (cell size h_ℓ ≥ 2r, so its box touches
// ≤ 2^d cells); a query visits one cell per level plus the overflow list of records
// whose box leaves the root cube, and applies the reference's strict support test —
// the covering set is identical to the linear scan.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "vc_api_internal.h"
#include "vc_build.h"
#include "vc_device.cuh"

namespace vc {

struct DevCache {
  int dim, n, L0, n_overflow;
  double origin[3];
  double size;
  const long long* level_off;  // L0+2 entries: first cell index of each level
  const int* cell_start;       // per cell start into items (+1 sentinel)
  const int* items;
  const int* overflow;
  const double* rec;           // n × record_size(dim), reference layout
};

}  // namespace vc

struct vc_cache {
  int dim = 0, n = 0, L0 = 0;
  double origin[3] = {0, 0, 0}, size = 0.0;
  long long n_cells = 0;
  std::vector<long long> level_off;
  long long* d_level_off = nullptr;
  int* d_cell_start = nullptr;
  int* d_items = nullptr;
  int* d_overflow = nullptr;
  int n_overflow = 0;
  double* d_rec = nullptr;
  vc::DevCache dev() const {
    vc::DevCache c{};
    c.dim = dim;
    c.n = n;
    c.L0 = L0;
    c.n_overflow = n_overflow;
    for (int a = 0; a < 3; ++a) c.origin[a] = origin[a];
    c.size = size;
    c.level_off = d_level_off;
    c.cell_start = d_cell_start;
    c.items = d_items;
    c.overflow = d_overflow;
    c.rec = d_rec;
    return c;
  }
  ~vc_cache() {
    cudaFree(d_level_off);
    cudaFree(d_cell_start);
    cudaFree(d_items);
    cudaFree(d_overflow);
    cudaFree(d_rec);
  }
};

namespace vc {

// support coordinate, first-order estimate, cubic weight (src/cache.py:49-56, :112-121)
template <int D>
__device__ __forceinline__ void blend_record(const double* R, const double* x, double num[3], double& den,
                                             int& hits) {
  const double* pos = R;
  const double* val = R + D;
  const double* grd = R + D + 3;
  const double* ax = R + D + 3 + 3 * D;
  const double* rad = R + D + 3 + 3 * D + D * D;
  double dl[D];
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
  double sup = sub(1.0, sqrt(q));
  if (!(sup > 0.0)) return;
  ++hits;
  double d = fmin(fmax(sup, 0.0), 1.0);
  double w = sub(mul(mul(3.0, d), d), mul(mul(mul(2.0, d), d), d));
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

template <int D>
__device__ inline bool cache_interpolate(const DevCache& C, const double* x, double J[3], int* count) {
  double num[3] = {0.0, 0.0, 0.0}, den = 0.0;
  int hits = 0;
  const int RS = record_size(D);
  for (int lv = C.L0; lv >= 0; --lv) {  // coarse → fine (tree order: root first)
    const int N = 1 << (C.L0 - lv);
    const double h = C.size / N;
    long long cell = 0;
    bool inside = true;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      double f = floor((x[a] - C.origin[a]) / h);
      if (!(f >= 0.0 && f < (double)N)) inside = false;
      cell = cell * N + (inside ? (long long)f : 0);
    }
    if (!inside) continue;
    long long ci = C.level_off[lv] + cell;
    int b = C.cell_start[ci], e = C.cell_start[ci + 1];
    for (int t = b; t < e; ++t) blend_record<D>(C.rec + (size_t)C.items[t] * RS, x, num, den, hits);
  }
  for (int t = 0; t < C.n_overflow; ++t) blend_record<D>(C.rec + (size_t)C.overflow[t] * RS, x, num, den, hits);
  if (count) *count = hits;
  if (hits == 0 || !(den > 0.0)) return false;
  J[0] = __ddiv_rn(num[0], den);
  J[1] = __ddiv_rn(num[1], den);
  J[2] = __ddiv_rn(num[2], den);
  return true;
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

struct DevCamera {
  double pos[3], fwd[3], right[3], up[3];
  double tan_half, aspect;
  int w, h, row0, rows, col0, cols;
};

struct MarchOut {
  double* image;          // h × w × 3
  long long* miss_cnt;    // per crop pixel (pass 1)
  long long* miss_off;    // per crop pixel exclusive prefix (pass 2)
  double* miss_x;         // miss points (pass 1b)
  uint32_t* miss_words;   // miss seeds (seed, 211, k, i, m)
  const double* miss_J;   // direct-evaluation results (pass 2)
  long long* hits;        // per crop pixel cache hits
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

// mode 0: count misses; mode 1: write miss points + seeds; mode 2: final accumulation
__global__ void __launch_bounds__(128) k_march(DevScene S, DevCache Cs, DevCache Cm, DevCamera cam, int spp,
                                               double step, int seed, const uint64_t* jit_state, JumpTables jt,
                                               int n_light_dummy, MarchOut out, int mode) {
  const int npx = cam.rows * cam.cols;
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= npx) return;
  const int py = cam.row0 + t / cam.cols, px = cam.col0 + t % cam.cols;
  const long long i = (long long)py * cam.w + px;
  const double four_pi = 4.0 * kPi;
  double img[3] = {0.0, 0.0, 0.0};
  long long nm = 0, hits = 0;
  long long slot = (mode >= 1) ? out.miss_off[t] : 0;
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
    if (mode == 2) surface_radiance<3>(S, id, hp, d, lo);
    double t_in, t_out;
    bool valid;
    bounds_span(S, o, d, t_in, t_out, valid);
    double acc[3] = {0.0, 0.0, 0.0};
    if (!valid) {
      if (mode == 2 && id >= 0) {
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
      bool cs = cache_interpolate<3>(Cs, y, Js, nullptr);
      bool cm = cs && cache_interpolate<3>(Cm, y, Jm, nullptr);
      double J[3];
      if (cs && cm) {
        ++hits;
        J[0] = add(Js[0], Jm[0]);
        J[1] = add(Js[1], Jm[1]);
        J[2] = add(Js[2], Jm[2]);
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
        }
        ++slot;
        ++nm;
      }
      if (mode == 2) {
        double f = mul(mul(exp(-S.sigma_t * sub(tk, t_in)), four_pi), 1.0);
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[c] = add(acc[c], mul(mul(f, J[c]), step));
      }
    }
    if (mode == 2) {
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
  if (mode == 0) out.miss_cnt[t] = nm;
  if (mode == 2) {
#pragma unroll
    for (int c = 0; c < 3; ++c) out.image[i * 3 + c] = __ddiv_rn(img[c], (double)spp);
    out.hits[t] = hits;
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
  c->dim = dim;
  c->n = n;
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
  c->L0 = dim == 3 ? 7 : 10;
  const int RS = record_size(dim);
  // levels: N_ℓ = 2^(L0−ℓ) cells per axis
  c->level_off.assign(c->L0 + 2, 0);
  long long tot = 0;
  for (int lv = 0; lv <= c->L0; ++lv) {
    c->level_off[lv] = tot;
    long long N = 1LL << (c->L0 - lv);
    tot += (dim == 3) ? N * N * N : N * N;
  }
  c->level_off[c->L0 + 1] = tot;
  c->n_cells = tot;
  std::vector<int> cnt(tot + 1, 0);
  std::vector<std::pair<long long, int>> ins;  // (cell, record)
  std::vector<int> overflow;
  ins.reserve((size_t)n * (1 << dim));
  for (int r = 0; r < n; ++r) {
    const double* R = records + (size_t)r * RS;
    const double* rad = R + dim + 3 + 3 * dim + dim * dim;
    double br = 0.0;
    for (int a = 0; a < dim; ++a) br = std::max(br, rad[a]);
    br = br * (1.0 + 1e-9) + 1e-12 * c->size;
    bool fits = std::isfinite(br);
    double lo[3], hi[3];
    for (int a = 0; a < dim; ++a) {
      lo[a] = R[a] - br;
      hi[a] = R[a] + br;
      if (!(lo[a] >= c->origin[a] && hi[a] <= c->origin[a] + c->size)) fits = false;
    }
    if (!fits) {
      overflow.push_back(r);
      continue;
    }
    int lv = 0;
    while (lv < c->L0 && c->size / (double)(1LL << (c->L0 - lv)) < 2.0 * br) ++lv;
    long long N = 1LL << (c->L0 - lv);
    double h = c->size / (double)N;
    long long clo[3] = {0, 0, 0}, chi[3] = {0, 0, 0};
    for (int a = 0; a < dim; ++a) {
      clo[a] = std::min(std::max((long long)std::floor((lo[a] - c->origin[a]) / h), 0LL), N - 1);
      chi[a] = std::min(std::max((long long)std::floor((hi[a] - c->origin[a]) / h), 0LL), N - 1);
    }
    for (long long z = (dim == 3 ? clo[2] : 0); z <= (dim == 3 ? chi[2] : 0); ++z)
      for (long long y = clo[1]; y <= chi[1]; ++y)
        for (long long x = clo[0]; x <= chi[0]; ++x) {
          long long cell = (dim == 3) ? (z * N + y) * N + x : y * N + x;
          ins.push_back({c->level_off[lv] + cell, r});
          cnt[c->level_off[lv] + cell]++;
        }
  }
  std::vector<int> start(tot + 1, 0);
  for (long long i = 0; i < tot; ++i) start[i + 1] = start[i] + cnt[i];
  std::vector<int> items(ins.size() + 1);
  std::vector<int> fillp(start.begin(), start.end() - 1);
  for (auto& p : ins) items[fillp[p.first]++] = p.second;  // records stay in insertion order
  c->n_overflow = (int)overflow.size();
  cudaError_t e = cudaSuccess;
  auto up = [&](void** dst, const void* src, size_t bytes) {
    if (e != cudaSuccess) return;
    if (bytes == 0) bytes = 8;
    e = cudaMalloc(dst, bytes);
    if (e == cudaSuccess && src) e = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
  };
  up((void**)&c->d_level_off, c->level_off.data(), c->level_off.size() * 8);
  up((void**)&c->d_cell_start, start.data(), start.size() * 4);
  up((void**)&c->d_items, items.data(), items.size() * 4);
  up((void**)&c->d_overflow, overflow.empty() ? nullptr : overflow.data(), overflow.size() * 4);
  up((void**)&c->d_rec, n ? records : nullptr, (size_t)n * RS * 8);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cache upload");
  }
  *out = c;
  return VC_OK;
}

void vc_cache_destroy(vc_cache* c) { delete c; }

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

int vc_render(vc_scene* sc, vc_cache* cs, vc_cache* cm, const vc_camera* camp, const vc_render_params* rp,
              double* image, int64_t* stats, int flags, void* stream) {
  if (!sc || !cs || !cm || !camp || !rp || !image) return fail(VC_EINVAL, "null argument");
  if (sc->dim != 3 || cs->dim != 3 || cm->dim != 3) return fail(VC_EINVAL, "Camera rendering requires a 3D scene");
  if (!(rp->march_step > 0.0)) return fail(VC_EINVAL, "march_step must be positive");
  if (rp->spp < 1) return fail(VC_EINVAL, "spp must be at least 1");
  cudaStream_t st = (cudaStream_t)stream;
  const vc_camera& C0 = *camp;
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
  if (cam.row0 < 0 || cam.col0 < 0 || cam.row0 + cam.rows > cam.h || cam.col0 + cam.cols > cam.w)
    return fail(VC_EINVAL, "crop outside the image");
  const int npx = cam.rows * cam.cols;
  int rc = ensure_emitters(sc, rp->n_light_samples);
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
  long long* mcnt = (long long*)alloc(23, (size_t)npx * 8);
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
  DevCache Cs = cs->dev(), Cm = cm->dev();
  const int grid = (npx + 127) / 128;
  k_march<<<grid, 128, 0, st>>>(S, Cs, Cm, cam, rp->spp, rp->march_step, rp->seed, djit, jt, 0, mo, 0);
  std::vector<long long> hc(npx), ho(npx + 1, 0);
  e = cudaMemcpyAsync(hc.data(), mcnt, (size_t)npx * 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "march pass 1");
  for (int t = 0; t < npx; ++t) ho[t + 1] = ho[t] + hc[t];
  const long long nmiss = ho[npx];
  e = cudaMemcpyAsync(moff, ho.data(), (size_t)(npx + 1) * 8, cudaMemcpyHostToDevice, st);
  long long launches = 1;
  if (nmiss > 0) {
    double* mx = (double*)alloc(27, (size_t)nmiss * 24);
    uint32_t* mw = (uint32_t*)alloc(28, (size_t)nmiss * 20);
    double* mmom = (double*)alloc(29, (size_t)nmiss * 2 * moment_size(3) * 8);
    long long* mst = (long long*)alloc(30, (size_t)nmiss * kStats * 8);
    double* mJ = (double*)alloc(31, (size_t)nmiss * 24);
    if (e != cudaSuccess) return cuda_fail(e, "miss workspace");
    mo.miss_x = mx;
    mo.miss_words = mw;
    k_march<<<grid, 128, 0, st>>>(S, Cs, Cm, cam, rp->spp, rp->march_step, rp->seed, djit, jt, 0, mo, 1);
    vc_build_params bp{};
    bp.n_angular = rp->n_angular;
    bp.march_step = rp->march_step;
    bp.n_inner = rp->n_inner;
    bp.n_light_samples = rp->n_light_samples;
    bp.epsilon = rp->epsilon > 0 ? rp->epsilon : 0.05;
    bp.flags = VC_SEED_WORDS;
    bp.seed_words = 5;
    // direct evaluations at cache misses (src/renderer.py:361-368, frozen)
    rc = build_impl(sc, (int)nmiss, mx, mw, nullptr, &bp, mmom, (int64_t*)mst, nullptr, st, nullptr);
    if (rc) return rc;
    k_misses_J<<<(int)((nmiss + 127) / 128), 128, 0, st>>>((int)nmiss, mmom, moment_size(3), mJ);
    mo.miss_J = mJ;
    launches += 2;
  }
  k_march<<<grid, 128, 0, st>>>(S, Cs, Cm, cam, rp->spp, rp->march_step, rp->seed, djit, jt, 0, mo, 2);
  launches += 1;
  count_launches(launches);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "march launch");
  const bool host = flags & VC_MEM_HOST;
  std::vector<long long> hh(npx);
  e = cudaMemcpyAsync(hh.data(), hits, (size_t)npx * 8, cudaMemcpyDeviceToHost, st);
  if (host) {
    // copy the crop rows back
    for (int y = cam.row0; y < cam.row0 + cam.rows && e == cudaSuccess; ++y)
      e = cudaMemcpyAsync(image + ((size_t)y * cam.w + cam.col0) * 3, dimg + ((size_t)y * cam.w + cam.col0) * 3,
                          (size_t)cam.cols * 24, cudaMemcpyDeviceToHost, st);
  } else {
    for (int y = cam.row0; y < cam.row0 + cam.rows && e == cudaSuccess; ++y)
      e = cudaMemcpyAsync(image + ((size_t)y * cam.w + cam.col0) * 3, dimg + ((size_t)y * cam.w + cam.col0) * 3,
                          (size_t)cam.cols * 24, cudaMemcpyDeviceToDevice, st);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "render download");
  if (stats) {
    long long h = 0;
    for (long long v : hh) h += v;
    stats[0] = h;
    stats[1] = nmiss;
  }
  return VC_OK;
}

}  // extern "C"
