// Cache pre-population on the device: populate_cache (src/renderer.py:282-327).
//
// The reference marches view points in scanline order and, at each point whose
// single or multiple cache lacks coverage, builds a record pair and inserts it
// (which = per-cache miss).  That greedy loop is sequential: whether point t needs a
// record depends on every record inserted before t.  This engine reproduces it
// exactly with speculative windows:
//
//   1. cover   — the next L points (the lookahead) are tested against the committed
//                caches; the uncovered ones form U (ordered).
//   2. select  — a speculative build set: the first point of U, every point that
//                already has a pooled build, and the first point of U in each cell of
//                a grid of predicted record size (first C by ordinal).
//   3. build   — record pairs for the new selections (one record-build wave).
//   4. resolve — the sequential rule among the built points, by one warp over C×C
//                coverage bitsets: built point e takes a record in cache c iff it was
//                uncovered in c and no earlier accepted record of c covers it.
//   5. stop    — accepted records are appended (tag = ordinal) and indexed; the first
//                point of U that was not built but is still uncovered by records of
//                smaller ordinal is the stop point.  Decisions before it are final;
//                records with larger tags are rolled back and their builds pooled.
//
// Every decision uses the reference's coverage predicate on the exact record set the
// sequential loop would have seen, so the committed caches equal the reference's
// (record for record, in insertion order).  Misprediction costs only time: a stop
// ends the window early, an unneeded speculative build is discarded.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "vc_build.h"
#include "vc_cache.cuh"

namespace vc {

// Ordered march-point stream (src/renderer.py:282-299).
struct MarchStream {
  int kind;  // 0: FieldGrid cell centers, 1: camera march
  int nx, ny;
  double fmin[2], fmax[2];
  double pos[3];             // camera origin
  const double* ray;         // per pixel: d.xyz, t_in
  const long long* first;    // per pixel: first point ordinal (n_rays + 1 entries)
  int n_rays;
  double step;
};

template <int D>
__device__ inline void stream_point(const MarchStream& S, long long ord, double* x) {
  if (S.kind == 0) {  // FieldGrid.cell_center (src/renderer.py:112-121)
    const int iy = (int)(ord / S.nx), ix = (int)(ord % S.nx);
    const double dx = __ddiv_rn(sub(S.fmax[0], S.fmin[0]), (double)S.nx);
    const double dy = __ddiv_rn(sub(S.fmax[1], S.fmin[1]), (double)S.ny);
    x[0] = add(S.fmin[0], mul(add((double)ix, 0.5), dx));
    x[1] = sub(S.fmax[1], mul(add((double)iy, 0.5), dy));
    return;
  }
  int lo = 0, hi = S.n_rays;  // first[lo] ≤ ord < first[hi]
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (S.first[mid] <= ord) lo = mid;
    else hi = mid;
  }
  const double* R = S.ray + (size_t)lo * 4;
  const long long k = ord - S.first[lo] + 1;
  const double t = add(R[3], mul((double)k - 0.5, S.step));
#pragma unroll
  for (int a = 0; a < D; ++a) x[a] = add(S.pos[a], mul(t, R[a]));
}

// Pixel-center rays, first hit and medium span → march steps (src/renderer.py:290-299).
// Pass k of a render with spp > 1 jitters pixel i by rng.random((h, w, 2)) of the stream
// SeedSequence(seed, 101) (src/renderer.py:446-450): draws k·h·w·2 + 2i, +1.
__global__ void k_pop_rays(DevScene S, DevCamera cam, double step, int spp, const uint64_t* jit_state,
                           JumpTables jt, double* ray, long long* steps) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long npx = (long long)cam.w * cam.h;
  if (r >= npx * spp) return;
  const int k = (int)(r / npx);
  const long long i = r - (long long)k * npx;
  const int py = (int)(i / cam.w), px = (int)(i % cam.w);
  double jx = 0.5, jy = 0.5;
  if (spp > 1) {
    Pcg64 g = pcg_load(jit_state);
    pcg_advance(g, (unsigned long long)((long long)k * npx * 2 + i * 2), jt);
    jx = g.next_double();
    jy = g.next_double();
  }
  double o[3], d[3];
  camera_ray(cam, px, py, jx, jy, o, d);
  double ts;
  int id;
  trace_closest<3>(S, o, d, ts, id);
  double t_in, t_out;
  bool valid;
  bounds_span(S, o, d, t_in, t_out, valid);
  long long n = 0;
  if (valid) {
    double t_end = fmin(ts, t_out);
    if (isnan(ts)) t_end = ts;
    double f = floor(__ddiv_rn(sub(t_end, t_in), step) + 0.5);
    if (f > 0.0) n = (long long)f;
  }
  ray[(size_t)r * 4 + 0] = d[0];
  ray[(size_t)r * 4 + 1] = d[1];
  ray[(size_t)r * 4 + 2] = d[2];
  ray[(size_t)r * 4 + 3] = t_in;
  steps[r] = n;
}

// 1. points [pos, pos+L) and their per-cache miss bits against records of smaller tag
template <int D>
__global__ void k_pop_cover(MarchStream M, DevCache Cs, DevCache Cm, long long pos, int L, double* X,
                            unsigned char* need) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= L) return;
  const long long ord = pos + j;
  double x[3];
  stream_point<D>(M, ord, x);
#pragma unroll
  for (int a = 0; a < D; ++a) X[(size_t)j * D + a] = x[a];
  const bool cs = cache_covers<D>(Cs, x, ord);
  const bool cm = cache_covers<D>(Cm, x, ord);
  need[j] = (unsigned char)((cs ? 0 : 1) | (cm ? 0 : 2));
}

__global__ void k_pop_iota(int* v, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

__global__ void k_pop_first(const unsigned long long* keys, const int* vals, int nu, unsigned char* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nu) return;
  if (i == 0 || keys[i] != keys[i - 1]) flag[vals[i]] = 1;
}

// SeedSequence entropy of a march point: populate (seed, 401, i) (src/renderer.py:317),
// field render (seed, 307, iy, ix) (:432-434), camera render (seed, 211, k, i, m) (:471)
__global__ void k_pop_words(MarchStream M, long long pos, const int* js, int n, uint32_t seed, int kind, int npx,
                            uint32_t* words) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const long long ord = pos + js[e];
  const int nw = kind == 0 ? 3 : (kind == 1 ? 4 : 5);
  uint32_t* w = words + (size_t)e * nw;
  w[0] = seed;
  if (kind == 0) {
    w[1] = 401u;
    w[2] = (uint32_t)(ord & 0xffffffffLL);
  } else if (kind == 1) {
    w[1] = 307u;
    w[2] = (uint32_t)(ord / M.nx);
    w[3] = (uint32_t)(ord % M.nx);
  } else {
    int lo = 0, hi = M.n_rays;
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (M.first[mid] <= ord) lo = mid;
      else hi = mid;
    }
    w[1] = 211u;
    w[2] = (uint32_t)(lo / npx);
    w[3] = (uint32_t)(lo % npx);
    w[4] = (uint32_t)(ord - M.first[lo] + 1);
  }
}

// committed builds of a camera render: (ordinal, L_s + L_m), appended in ordinal order
__global__ void k_pop_commit_list(const double* WR, const int* slot, const long long* ord, int k, int D, int RS,
                                  long long* c_ord, double* c_val) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= k) return;
  const double* R = WR + (size_t)slot[q] * 2 * RS;
  c_ord[q] = ord[q];
  for (int c = 0; c < 3; ++c) c_val[(size_t)q * 3 + c] = add(R[D + c], R[RS + D + c]);
}

template <int D>
__global__ void k_pop_gather_x(const double* X, const int* js, int n, double* out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
#pragma unroll
  for (int a = 0; a < D; ++a) out[(size_t)e * D + a] = X[(size_t)js[e] * D + a];
}

// new record pairs (2·RS doubles each) → window slots
__global__ void k_pop_scatter(const double* src, int n, const int* slot, int RS2, double* WR) {
  const int e = blockIdx.y;
  if (e >= n) return;
  for (int t = threadIdx.x; t < RS2; t += blockDim.x) WR[(size_t)slot[e] * RS2 + t] = src[(size_t)e * RS2 + t];
}

// need bits of pooled builds against the committed caches (records of tag < pos ≤ ord)
template <int D>
__global__ void k_pool_need(const double* WR, const int* slot, const long long* ords, int E, DevCache Cs,
                            DevCache Cm, unsigned char* needP) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const double* x = WR + (size_t)slot[e] * 2 * record_size(D);  // record position = march point
  const bool cs = cache_covers<D>(Cs, x, ords[e]);
  const bool cm = cache_covers<D>(Cm, x, ords[e]);
  needP[e] = (unsigned char)((cs ? 0 : 1) | (cm ? 0 : 2));
}

// coverage bits: bit b of word (c, e, w) = record c of pooled build b (b < e) covers x_e
template <int D>
__global__ void k_pop_bits(const double* WR, const int* slot, int E, int W, int blend, unsigned long long* bits) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 2LL * E * W) return;
  const int c = (int)(t / ((long long)E * W));
  const int rem = (int)(t % ((long long)E * W));
  const int e = rem / W, w = rem % W;
  const int RS = record_size(D);
  const double* x = WR + (size_t)slot[e] * 2 * RS;
  unsigned long long word = 0;
  const int b1 = min(w * 64 + 64, e);
  for (int b = w * 64; b < b1; ++b) {
    const double* R = WR + (size_t)slot[b] * 2 * RS + (size_t)c * RS;
    double dl[D];
    bool cov;
    if (blend == 0) {
      const double sup = record_support<D>(R, x, dl);
      cov = sup > 0.0 && support_weight(sup) > 0.0;
    } else {  // log_space_interpolate coverage: sphere support and a positive channel
      const double sup = sphere_support<D>(R, x, dl);
      cov = sup > 0.0 && support_weight(sup) > 0.0 && (R[D] > 0.0 || R[D + 1] > 0.0 || R[D + 2] > 0.0);
    }
    if (cov) word |= 1ULL << (b - w * 64);
  }
  bits[((size_t)c * E + e) * W + w] = word;
}

// sequential acceptance among the pooled builds, in ordinal order (one warp; E ≤ 4096)
__global__ void k_pop_resolve(const unsigned long long* bits, const unsigned char* needP, int E, int W,
                              unsigned char* acc) {
  const int lane = threadIdx.x;
  unsigned long long as[2] = {0, 0}, am[2] = {0, 0};
  for (int e = 0; e < E; ++e) {
    bool hs = false, hm = false;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int w = lane + 32 * k;
      if (w < W) {
        hs |= (bits[(size_t)e * W + w] & as[k]) != 0;
        hm |= (bits[((size_t)E + e) * W + w] & am[k]) != 0;
      }
    }
    const bool cov_s = __any_sync(0xffffffffu, hs);
    const bool cov_m = __any_sync(0xffffffffu, hm);
    const int nd = needP[e];
    const bool a_s = (nd & 1) && !cov_s;
    const bool a_m = (nd & 2) && !cov_m;
    const int w = e >> 6;
    if ((w & 31) == lane) {
      if (a_s) as[w >> 5] |= 1ULL << (e & 63);
      if (a_m) am[w >> 5] |= 1ULL << (e & 63);
    }
    if (lane == 0) acc[e] = (unsigned char)((a_s ? 1 : 0) | (a_m ? 2 : 0));
  }
}

// Uncovered lookahead points that have no build, against every record of smaller tag
// (committed + tentatively accepted pooled builds): need2 flags and the stop ordinal.
template <int D>
__global__ void k_pop_need2(const double* X, const int* U, int nu, const unsigned char* need, long long pos,
                            const long long* pool, int np, DevCache Cs, DevCache Cm, unsigned char* need2,
                            unsigned long long* stop) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nu) return;
  const int j = U[p];
  const long long ord = pos + j;
  int lo = 0, hi = np;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (pool[mid] < ord) lo = mid + 1;
    else hi = mid;
  }
  if (lo < np && pool[lo] == ord) {
    need2[p] = 0;
    return;
  }
  double x[3];
#pragma unroll
  for (int a = 0; a < D; ++a) x[a] = X[(size_t)j * D + a];
  const int nd = need[j];
  const bool ms = (nd & 1) && !cache_covers<D>(Cs, x, ord);
  const bool mm = !ms && (nd & 2) && !cache_covers<D>(Cm, x, ord);
  need2[p] = (ms || mm) ? 1 : 0;
  if (ms || mm) atomicMin(stop, (unsigned long long)ord);
}

// cell key per need2 candidate (V = positions in U)
template <int D>
__global__ void k_pop_keys(const double* X, const int* U, const int* V, int nv, double o0, double o1, double o2,
                           double inv_h, unsigned long long* keys, int* vals) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nv) return;
  const double* x = X + (size_t)U[V[i]] * D;
  const double o[3] = {o0, o1, o2};
  unsigned long long k = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double f = floor((x[a] - o[a]) * inv_h);
    long long c = (long long)fmin(fmax(f, 0.0), 2097151.0);
    k |= (unsigned long long)c << (21 * a);
  }
  keys[i] = k;
  vals[i] = i;
}

// selected V entries → lookahead indices j
__global__ void k_pop_sel_j(const int* sel, const int* V, const int* U, int E, int* sel_j) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  sel_j[e] = U[V[sel[e]]];
}

__global__ void k_pop_commit_J(const double* WR, const int* slot, const long long* ord, int k, int D, int RS,
                               double* J) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= k) return;
  const double* R = WR + (size_t)slot[q] * 2 * RS;
  for (int c = 0; c < 3; ++c) J[(size_t)ord[q] * 3 + c] = add(R[D + c], R[RS + D + c]);
}

}  // namespace vc

using namespace vc;

namespace {

struct Engine {
  vc_scene* sc;
  vc_cache* cs;
  vc_cache* cm;
  MarchStream M{};
  long long N = 0;
  int D = 0;
  vc_build_params bp{};
  uint32_t seed = 0;
  int seed_kind = 0;  // 0: populate (seed, 401, i); 1: field render (seed, 307, iy, ix); 2: camera render
  int npx = 1;        // camera pixels (seed kind 2)
  int estimator = VC_EST_SUBDIVISION;
  int (*hook)(void*, int, const double*, const uint32_t*, int, double*, int64_t*, void*) = nullptr;
  void* hook_user = nullptr;
  vc_baseline_params blp{};
  double* commit_J = nullptr;  // optional N × 3: direct value (L_s + L_m) of every point that built
  bool commit_list = false;    // camera render: (ordinal, value) of every point that built
  long long* c_ord = nullptr;
  double* c_val = nullptr;
  long long c_n = 0, c_cap = 0;
  ~Engine() {
    cudaFree(c_ord);
    cudaFree(c_val);
  }
  cudaStream_t st = nullptr;
  Workspace ws;
  int C = 2048;
  long long L = 65536, Lmax = 1LL << 24;
  double kappa = 1.0, h_sel = INFINITY;
  double waste_ratio = 0.3;  // VOLCACHE_POP_WASTE: target discarded / committed builds per window
  int64_t stats[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaError_t e = cudaSuccess;

  void* get(int slot, size_t bytes) { return ws.get(slot, bytes, &e); }

  int run();
};

int Engine::run() {
  const int RS = record_size(D);
  const int RS2 = 2 * RS;
  const int n_slots = 2 * C;  // pooled builds (built, not yet resolved)
  double* WR = (double*)get(0, (size_t)n_slots * RS2 * 8);
  if (e != cudaSuccess) return cuda_fail(e, "populate pool");
  std::vector<int> free_slots;
  for (int s = n_slots - 1; s >= 0; --s) free_slots.push_back(s);
  std::map<long long, int> pool;  // ordinal → slot
  std::vector<double> hrec((size_t)n_slots * RS2);
  // VOLCACHE_POP_TIMING=1: host wall time per phase (each phase ends in a stream sync) on stderr
  const bool timing = getenv("VOLCACHE_POP_TIMING") && getenv("VOLCACHE_POP_TIMING")[0] == '1';
  double tph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  double wave_s[5] = {0, 0, 0, 0, 0};  // build waves by size: <16, <128, <512, <1536, ≥1536
  long long wave_n[5] = {0, 0, 0, 0, 0}, wave_rec[5] = {0, 0, 0, 0, 0};
  auto tnow = [&]() {
    if (timing) cudaStreamSynchronize(st);
    return std::chrono::steady_clock::now();
  };
  auto tacc = [&](int k, std::chrono::steady_clock::time_point& t0) {
    if (!timing) return;
    auto t1 = tnow();
    tph[k] += std::chrono::duration<double>(t1 - t0).count();
    t0 = t1;
  };
  long long pos = 0;
  while (pos < N) {
    auto tp = tnow();
    const int Lw = (int)std::min<long long>(L, N - pos);
    // 1. lookahead points and their misses against the committed caches
    double* X = (double*)get(1, (size_t)Lw * D * 8);
    unsigned char* need = (unsigned char*)get(2, (size_t)Lw);
    int* iota = (int*)get(3, (size_t)Lw * 4);
    int* U = (int*)get(4, (size_t)Lw * 4);
    int* cnt = (int*)get(5, 64);
    if (e != cudaSuccess) return cuda_fail(e, "populate lookahead buffers");
    const int nb = (Lw + 127) / 128;
    if (D == 2) k_pop_cover<2><<<nb, 128, 0, st>>>(M, cs->dev(), cm->dev(), pos, Lw, X, need);
    else k_pop_cover<3><<<nb, 128, 0, st>>>(M, cs->dev(), cm->dev(), pos, Lw, X, need);
    k_pop_iota<<<nb, 128, 0, st>>>(iota, Lw);
    size_t tb = 0;
    cub::DeviceSelect::Flagged(nullptr, tb, iota, need, U, cnt, Lw, st);
    void* tmp = get(6, tb);
    if (e != cudaSuccess) return cuda_fail(e, "populate select scratch");
    cub::DeviceSelect::Flagged(tmp, tb, iota, need, U, cnt, Lw, st);
    int nu = 0;
    e = cudaMemcpyAsync(&nu, cnt, 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "populate cover");
    count_launches(4);
    stats[3] += 1;
    tacc(0, tp);
    // 2. sequential acceptance among the pooled builds inside the lookahead
    std::vector<long long> pords;
    std::vector<int> pslots;
    for (auto& kv : pool) {
      if (kv.first >= pos + Lw) break;
      pords.push_back(kv.first);
      pslots.push_back(kv.second);
    }
    const int E = (int)pords.size();
    long long* dords = (long long*)get(9, (size_t)(E + 1) * 8);
    int* dslot = (int*)get(19, (size_t)(E + 1) * 4);
    unsigned char* acc = (unsigned char*)get(28, (size_t)E + 1);
    if (e != cudaSuccess) return cuda_fail(e, "populate pool buffers");
    std::vector<unsigned char> hacc(E, 0);
    if (E > 0) {
      unsigned char* needP = (unsigned char*)get(10, (size_t)E);
      const int W = (E + 63) / 64;
      unsigned long long* bits = (unsigned long long*)get(27, (size_t)2 * E * W * 8);
      if (e != cudaSuccess) return cuda_fail(e, "populate resolve buffers");
      e = cudaMemcpyAsync(dords, pords.data(), (size_t)E * 8, cudaMemcpyHostToDevice, st);
      if (e == cudaSuccess) e = cudaMemcpyAsync(dslot, pslots.data(), (size_t)E * 4, cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) return cuda_fail(e, "populate pool upload");
      const long long nt = 2LL * E * W;
      if (D == 2) {
        k_pool_need<2><<<(E + 127) / 128, 128, 0, st>>>(WR, dslot, dords, E, cs->dev(), cm->dev(), needP);
        k_pop_bits<2><<<(int)((nt + 127) / 128), 128, 0, st>>>(WR, dslot, E, W, cs->blend, bits);
      } else {
        k_pool_need<3><<<(E + 127) / 128, 128, 0, st>>>(WR, dslot, dords, E, cs->dev(), cm->dev(), needP);
        k_pop_bits<3><<<(int)((nt + 127) / 128), 128, 0, st>>>(WR, dslot, E, W, cs->blend, bits);
      }
      k_pop_resolve<<<1, 32, 0, st>>>(bits, needP, E, W, acc);
      count_launches(3);
      e = cudaMemcpyAsync(hacc.data(), acc, E, cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) return cuda_fail(e, "populate resolve");
    }
    tacc(1, tp);
    // 3. tentative insertion of the accepted builds (tag = ordinal)
    const int n0s = cs->n, n0m = cm->n;
    std::vector<int> rows_s, rows_m;
    std::vector<long long> tags_s, tags_m;
    for (int q = 0; q < E; ++q) {
      if (hacc[q] & 1) {
        rows_s.push_back(2 * pslots[q]);
        tags_s.push_back(pords[q]);
      }
      if (hacc[q] & 2) {
        rows_m.push_back(2 * pslots[q] + 1);
        tags_m.push_back(pords[q]);
      }
    }
    auto append = [&](vc_cache* c, const std::vector<int>& rows, const std::vector<long long>& tags, int s0) -> int {
      if (rows.empty()) return VC_OK;
      int* dr = (int*)get(s0, rows.size() * 4);
      long long* dt = (long long*)get(s0 + 1, tags.size() * 8);
      if (e != cudaSuccess) return cuda_fail(e, "populate append buffers");
      e = cudaMemcpyAsync(dr, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice, st);
      if (e == cudaSuccess) e = cudaMemcpyAsync(dt, tags.data(), tags.size() * 8, cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) return cuda_fail(e, "populate append upload");
      int rc = cache_append(c, WR, RS, dr, dt, (int)rows.size(), st);
      if (rc) return rc;
      return cache_rebuild(c, st);
    };
    int rc = append(cs, rows_s, tags_s, 29);
    if (!rc) rc = append(cm, rows_m, tags_m, 31);
    if (rc) return rc;
    tacc(2, tp);
    // 4. unbuilt points still uncovered by every record of smaller tag; the first is the stop
    unsigned char* need2 = (unsigned char*)get(7, (size_t)nu + 1);
    unsigned long long* dstop = (unsigned long long*)get(33, 8);
    if (e != cudaSuccess) return cuda_fail(e, "populate stop buffers");
    unsigned long long hstop = (unsigned long long)(pos + Lw);
    e = cudaMemcpyAsync(dstop, &hstop, 8, cudaMemcpyHostToDevice, st);
    const int nbu = (nu + 127) / 128;
    if (nu > 0) {
      if (D == 2) k_pop_need2<2><<<nbu, 128, 0, st>>>(X, U, nu, need, pos, dords, E, cs->dev(), cm->dev(), need2, dstop);
      else k_pop_need2<3><<<nbu, 128, 0, st>>>(X, U, nu, need, pos, dords, E, cs->dev(), cm->dev(), need2, dstop);
      count_launches(1);
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hstop, dstop, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "populate stop");
    const long long stop = std::min<long long>((long long)hstop, pos + Lw);
    tacc(3, tp);
    // 5. next speculative builds: need2 points thinned to one per cell of the predicted size
    std::vector<int> hj;
    if (stop < pos + Lw) {
      int* iota_u = (int*)get(15, (size_t)nu * 4);
      int* V = (int*)get(16, (size_t)nu * 4);
      if (e != cudaSuccess) return cuda_fail(e, "populate selection buffers");
      k_pop_iota<<<nbu, 128, 0, st>>>(iota_u, nu);
      size_t tb2 = 0;
      cub::DeviceSelect::Flagged(nullptr, tb2, iota_u, need2, V, cnt + 1, nu, st);
      void* tmp2 = get(17, tb2);
      if (e != cudaSuccess) return cuda_fail(e, "populate select scratch");
      cub::DeviceSelect::Flagged(tmp2, tb2, iota_u, need2, V, cnt + 1, nu, st);
      int nv = 0;
      e = cudaMemcpyAsync(&nv, cnt + 1, 4, cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) return cuda_fail(e, "populate candidates");
      count_launches(3);
      int* sel = (int*)get(18, (size_t)nv * 4 + 4);
      int ns = 1;
      if (std::isfinite(h_sel) && h_sel > 0.0 && nv > 1) {
        unsigned long long* keys = (unsigned long long*)get(11, (size_t)nv * 8);
        unsigned long long* keys2 = (unsigned long long*)get(12, (size_t)nv * 8);
        int* vals = (int*)get(13, (size_t)nv * 4);
        int* vals2 = (int*)get(14, (size_t)nv * 4);
        unsigned char* flagv = (unsigned char*)get(8, (size_t)nv);
        int* iota_v = (int*)get(20, (size_t)nv * 4);
        if (e != cudaSuccess) return cuda_fail(e, "populate key buffers");
        const double inv_h = 1.0 / h_sel;
        const int nbv = (nv + 127) / 128;
        if (D == 2)
          k_pop_keys<2><<<nbv, 128, 0, st>>>(X, U, V, nv, sc->bmin[0], sc->bmin[1], 0.0, inv_h, keys, vals);
        else
          k_pop_keys<3><<<nbv, 128, 0, st>>>(X, U, V, nv, sc->bmin[0], sc->bmin[1], sc->bmin[2], inv_h, keys, vals);
        size_t rb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, rb, keys, keys2, vals, vals2, nv, 0, 21 * D, st);
        void* rtmp = get(21, rb);
        if (e != cudaSuccess) return cuda_fail(e, "populate sort scratch");
        cub::DeviceRadixSort::SortPairs(rtmp, rb, keys, keys2, vals, vals2, nv, 0, 21 * D, st);
        e = cudaMemsetAsync(flagv, 0, nv, st);
        k_pop_first<<<nbv, 128, 0, st>>>(keys2, vals2, nv, flagv);
        k_pop_iota<<<nbv, 128, 0, st>>>(iota_v, nv);
        size_t tb3 = 0;
        cub::DeviceSelect::Flagged(nullptr, tb3, iota_v, flagv, sel, cnt + 2, nv, st);
        void* tmp3 = get(22, tb3);
        if (e != cudaSuccess) return cuda_fail(e, "populate thinning scratch");
        cub::DeviceSelect::Flagged(tmp3, tb3, iota_v, flagv, sel, cnt + 2, nv, st);
        e = cudaMemcpyAsync(&ns, cnt + 2, 4, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return cuda_fail(e, "populate thinning");
        count_launches(6);
      } else {
        const int zero = 0;
        e = cudaMemcpyAsync(sel, &zero, 4, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return cuda_fail(e, "populate selection");
      }
      const int Es = std::min(ns, C);
      int* sel_j = (int*)get(23, (size_t)Es * 4);
      if (e != cudaSuccess) return cuda_fail(e, "populate selection list");
      k_pop_sel_j<<<(Es + 127) / 128, 128, 0, st>>>(sel, V, U, Es, sel_j);
      count_launches(1);
      hj.resize(Es);
      e = cudaMemcpyAsync(hj.data(), sel_j, (size_t)Es * 4, cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) return cuda_fail(e, "populate selection download");
    }
    tacc(4, tp);
    // 6. decisions before the stop are final: keep them, roll back the rest
    int keep_s = 0, keep_m = 0, committed = 0, covered = 0;
    for (int q = 0; q < E; ++q) {
      if (pords[q] >= stop) break;
      keep_s += (hacc[q] & 1) ? 1 : 0;
      keep_m += (hacc[q] & 2) ? 1 : 0;
      if (hacc[q]) ++committed;
      else ++covered;
    }
    stats[5] += covered;
    stats[7] += committed;
    if (commit_J && committed > 0) {  // the value _point_value returns when the blend is None
      std::vector<int> cs_slot;
      std::vector<long long> cs_ord;
      for (int q = 0; q < E && pords[q] < stop; ++q)
        if (hacc[q]) {
          cs_slot.push_back(pslots[q]);
          cs_ord.push_back(pords[q]);
        }
      int* d1 = (int*)get(38, cs_slot.size() * 4);
      long long* d2 = (long long*)get(39, cs_ord.size() * 8);
      if (e != cudaSuccess) return cuda_fail(e, "populate commit buffers");
      e = cudaMemcpyAsync(d1, cs_slot.data(), cs_slot.size() * 4, cudaMemcpyHostToDevice, st);
      if (e == cudaSuccess) e = cudaMemcpyAsync(d2, cs_ord.data(), cs_ord.size() * 8, cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) return cuda_fail(e, "populate commit upload");
      k_pop_commit_J<<<((int)cs_slot.size() + 127) / 128, 128, 0, st>>>(WR, d1, d2, (int)cs_slot.size(), D, RS,
                                                                       commit_J);
      count_launches(1);
    }
    if (commit_list && committed > 0) {
      std::vector<int> cs_slot;
      std::vector<long long> cs_ord;
      for (int q = 0; q < E && pords[q] < stop; ++q)
        if (hacc[q]) {
          cs_slot.push_back(pslots[q]);
          cs_ord.push_back(pords[q]);
        }
      const long long k = (long long)cs_slot.size();
      if (c_n + k > c_cap) {  // grow (ordinals arrive sorted)
        const long long cap = std::max<long long>(c_n + k, std::max<long long>(4096, 2 * c_cap));
        long long* no = nullptr;
        double* nv = nullptr;
        e = cudaMalloc(&no, cap * 8);
        if (e == cudaSuccess) e = cudaMalloc(&nv, cap * 24);
        if (e == cudaSuccess && c_n) e = cudaMemcpyAsync(no, c_ord, c_n * 8, cudaMemcpyDeviceToDevice, st);
        if (e == cudaSuccess && c_n) e = cudaMemcpyAsync(nv, c_val, c_n * 24, cudaMemcpyDeviceToDevice, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
          cudaFree(no);
          cudaFree(nv);
          return cuda_fail(e, "render commit list");
        }
        cudaFree(c_ord);
        cudaFree(c_val);
        c_ord = no;
        c_val = nv;
        c_cap = cap;
      }
      int* d1 = (int*)get(38, cs_slot.size() * 4);
      long long* d2 = (long long*)get(39, cs_ord.size() * 8);
      if (e != cudaSuccess) return cuda_fail(e, "render commit buffers");
      e = cudaMemcpyAsync(d1, cs_slot.data(), cs_slot.size() * 4, cudaMemcpyHostToDevice, st);
      if (e == cudaSuccess) e = cudaMemcpyAsync(d2, cs_ord.data(), cs_ord.size() * 8, cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) return cuda_fail(e, "render commit upload");
      k_pop_commit_list<<<(int)((k + 127) / 128), 128, 0, st>>>(WR, d1, d2, (int)k, D, RS, c_ord + c_n,
                                                                c_val + (size_t)c_n * 3);
      count_launches(1);
      c_n += k;
    }
    if (keep_s < (int)rows_s.size()) {
      cache_truncate(cs, n0s + keep_s, st);
      rc = cache_rebuild(cs, st);
      if (rc) return rc;
    }
    if (keep_m < (int)rows_m.size()) {
      cache_truncate(cm, n0m + keep_m, st);
      rc = cache_rebuild(cm, st);
      if (rc) return rc;
    }
    if (committed > 0) {  // committed radii → next cell size
      e = cudaMemcpyAsync(hrec.data(), WR, hrec.size() * 8, cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) return cuda_fail(e, "populate radii");
      std::vector<double> rmin;
      for (int q = 0; q < E && pords[q] < stop; ++q)
        for (int c = 0; c < 2; ++c) {
          if (!(hacc[q] & (1 << c))) continue;
          const double* rad = hrec.data() + (size_t)pslots[q] * RS2 + (size_t)c * RS + D + 3 + 3 * D + D * D;
          double r = rad[0];
          for (int a = 1; a < D; ++a) r = std::min(r, rad[a]);
          if (std::isfinite(r) && r > 0.0) rmin.push_back(r);
        }
      if (!rmin.empty()) {
        std::nth_element(rmin.begin(), rmin.begin() + rmin.size() / 2, rmin.end());
        // controller: grow the selection cell while speculative builds that turned out
        // covered exceed waste_ratio × committed ones, shrink it otherwise
        if (covered > waste_ratio * committed) kappa *= 1.25;
        else kappa *= 0.9;
        kappa = std::min(8.0, std::max(0.1, kappa));
        h_sel = kappa * rmin[rmin.size() / 2];
      }
    }
    for (int q = 0; q < E && pords[q] < stop; ++q) {
      pool.erase(pords[q]);
      free_slots.push_back(pslots[q]);
    }
    tacc(5, tp);
    // 7. build the new selections into the pool
    const int nn = (int)hj.size();
    if (nn > 0) {
      std::vector<int> new_slot;
      std::vector<int> js;
      for (int q = 0; q < nn; ++q) {
        if (free_slots.empty()) {  // evict the furthest pooled build
          if (pool.empty()) break;
          auto last = std::prev(pool.end());
          free_slots.push_back(last->second);
          pool.erase(last);
        }
        new_slot.push_back(free_slots.back());
        free_slots.pop_back();
        js.push_back(hj[q]);
      }
      const int nb2 = (int)js.size();
      int* djs = (int*)get(24, (size_t)nb2 * 4);
      int* dns = (int*)get(25, (size_t)nb2 * 4);
      double* xb = (double*)get(26, (size_t)nb2 * D * 8);
      uint32_t* dw = (uint32_t*)get(34, (size_t)nb2 * 20);
      double* rec = (double*)get(35, (size_t)nb2 * RS2 * 8);
      double* mom = (double*)get(36, (size_t)nb2 * 2 * moment_size(D) * 8);
      long long* bst = (long long*)get(37, (size_t)nb2 * kStats * 8);
      if (e != cudaSuccess) return cuda_fail(e, "populate build buffers");
      e = cudaMemcpyAsync(djs, js.data(), (size_t)nb2 * 4, cudaMemcpyHostToDevice, st);
      if (e == cudaSuccess) e = cudaMemcpyAsync(dns, new_slot.data(), (size_t)nb2 * 4, cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) return cuda_fail(e, "populate build upload");
      k_pop_words<<<(nb2 + 127) / 128, 128, 0, st>>>(M, pos, djs, nb2, seed, seed_kind, npx, dw);
      if (D == 2) k_pop_gather_x<2><<<(nb2 + 127) / 128, 128, 0, st>>>(X, djs, nb2, xb);
      else k_pop_gather_x<3><<<(nb2 + 127) / 128, 128, 0, st>>>(X, djs, nb2, xb);
      count_launches(1);
      auto tb0 = tnow();
      if (estimator == VC_EST_BASELINE) {  // CacheSet.compute, mode "baseline" (src/renderer.py:233-244)
        rc = baseline_impl(sc, nb2, xb, dw, &blp, nullptr, rec, nullptr, st);
      } else if (hook) {  // multi-GPU: the wave is sharded over ranks and all-gathered by the caller
        rc = hook(hook_user, nb2, xb, dw, bp.seed_words, rec, (int64_t*)bst, (void*)st);
        if (rc) return fail(VC_EHOOK, "populate build hook failed (code " + std::to_string(rc) + ")");
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "populate build hook");
      } else {
        rc = build_impl(sc, nb2, xb, dw, nullptr, &bp, mom, (int64_t*)bst, rec, st, nullptr);
      }
      if (rc) return rc;
      if (timing) {
        const double dt = std::chrono::duration<double>(tnow() - tb0).count();
        const int b = nb2 < 16 ? 0 : nb2 < 128 ? 1 : nb2 < 512 ? 2 : nb2 < 1536 ? 3 : 4;
        wave_n[b] += 1;
        wave_rec[b] += nb2;
        wave_s[b] += dt;
      }
      k_pop_scatter<<<dim3(1, nb2), 64, 0, st>>>(rec, nb2, dns, RS2, WR);
      count_launches(1);
      if (D == 3 && estimator != VC_EST_BASELINE) {
        std::vector<long long> hs((size_t)nb2 * kStats);
        e = cudaMemcpyAsync(hs.data(), bst, hs.size() * 8, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return cuda_fail(e, "populate build");
        for (int i = 0; i < nb2; ++i)
          if (hs[(size_t)i * kStats + 5] != 0)
            return fail(VC_ETRI, "spherical Delaunay triangulation failed at march point " +
                                     std::to_string(pos + js[i]));
      }
      for (int i = 0; i < nb2; ++i) pool[pos + js[i]] = new_slot[i];
      stats[4] += nb2;
    }
    tacc(6, tp);
    // 8. advance
    if (stop >= pos + Lw) {
      pos += Lw;
      L = std::min(Lmax, L * 2);
    } else {
      if (stop > pos) stats[6] += 1;
      pos = stop;
    }
  }
  stats[0] = N;
  stats[1] = cs->n;
  stats[2] = cm->n;
  if (timing)
    fprintf(stderr,
            "populate phases (s): cover %.3f resolve %.3f append %.3f stop %.3f select %.3f commit %.3f build %.3f"
            " | windows %lld builds %lld\n",
            tph[0], tph[1], tph[2], tph[3], tph[4], tph[5], tph[6], (long long)stats[3], (long long)stats[4]);
  if (timing)
    for (int b = 0; b < 5; ++b)
      fprintf(stderr, "  waves %s: %lld waves, %lld records, %.3f s\n",
              b == 0 ? "<16" : b == 1 ? "<128" : b == 2 ? "<512" : b == 3 ? "<1536" : ">=1536", wave_n[b],
              wave_rec[b], wave_s[b]);
  return VC_OK;
}

}  // namespace

// Stream setup + engine run on existing caches (records with tag −1 pre-exist).
// seed_kind 2 (camera render with insertion) marches spp jittered passes and hands the
// ray prefix and the committed direct values to the caller through `rs`.
static int populate_run_impl(vc_scene* sc, const vc_populate_params* pp, int seed_kind, vc_cache* cs, vc_cache* cm,
                             int64_t* stats, cudaStream_t st, double* commit_J, int spp, RenderStream* rs);

// The engine rebuilds the indexes after every window with the coarser cell span; the
// finished caches are re-indexed at the lookup span (vc_cache::cell_span).
int vc::populate_run(vc_scene* sc, const vc_populate_params* pp, int seed_kind, vc_cache* cs, vc_cache* cm,
                     int64_t* stats, cudaStream_t st, double* commit_J, int spp, RenderStream* rs) {
  const double span_s = cs->cell_span, span_m = cm->cell_span;
  cs->cell_span = cm->cell_span = 2.0;
  int rc = populate_run_impl(sc, pp, seed_kind, cs, cm, stats, st, commit_J, spp, rs);
  cs->cell_span = span_s;
  cm->cell_span = span_m;
  if (!rc) rc = cache_rebuild_full(cs, st);
  if (!rc) rc = cache_rebuild_full(cm, st);
  return rc;
}

static int populate_run_impl(vc_scene* sc, const vc_populate_params* pp, int seed_kind, vc_cache* cs, vc_cache* cm,
                             int64_t* stats, cudaStream_t st, double* commit_J, int spp, RenderStream* rs) {
  if (!(pp->march_step > 0.0)) return fail(VC_EINVAL, "march_step must be positive");
  if (!(pp->epsilon > 0.0)) return fail(VC_EINVAL, "epsilon must be positive");
  Engine g;
  g.sc = sc;
  g.D = sc->dim;
  g.st = st;
  g.seed = (uint32_t)pp->seed;
  g.seed_kind = seed_kind;
  g.commit_J = commit_J;
  g.bp.n_angular = pp->n_angular;
  g.bp.march_step = pp->march_step;
  g.bp.n_inner = pp->n_inner;
  g.bp.n_light_samples = pp->n_light_samples;
  g.bp.epsilon = pp->epsilon;
  g.bp.flags = VC_SEED_WORDS | VC_MAKE_RECORDS | (pp->isotropic ? VC_ISOTROPIC : 0);
  g.bp.seed_words = seed_kind == 0 ? 3 : (seed_kind == 1 ? 4 : 5);
  g.commit_list = rs != nullptr;
  g.estimator = pp->estimator == VC_EST_BASELINE ? VC_EST_BASELINE : VC_EST_SUBDIVISION;
  g.hook = pp->build_hook;
  if (const char* ew = getenv("VOLCACHE_POP_WASTE")) g.waste_ratio = std::max(0.05, atof(ew));
  g.hook_user = pp->build_hook_user;
  g.blp.n_angular = pp->n_angular;
  g.blp.max_media_bounces = pp->max_media_bounces;
  g.blp.n_light_samples = pp->n_light_samples;
  g.blp.alpha = pp->baseline_alpha;
  g.blp.flags = VC_SEED_WORDS;
  g.blp.seed_words = g.bp.seed_words;
  cs->blend = cm->blend = (g.estimator == VC_EST_BASELINE) ? 1 : 0;
  if (pp->window > 0) g.C = std::min(pp->window, 2048);
  if (pp->lookahead > 0) g.L = pp->lookahead;
  MarchStream& M = g.M;
  M.step = pp->march_step;
  struct Bufs {
    double* ray = nullptr;
    long long* first = nullptr;
    long long* steps = nullptr;
    void* tmp = nullptr;
    ~Bufs() {
      cudaFree(ray);
      cudaFree(first);
      cudaFree(steps);
      cudaFree(tmp);
    }
  } bf;
  if (pp->target == VC_TARGET_FIELD) {
    if (sc->dim != 2) return fail(VC_EINVAL, "FieldGrid rendering requires a 2D scene");
    if (pp->field_nx < 1 || pp->field_ny < 1) return fail(VC_EINVAL, "FieldGrid resolution must be positive");
    for (int a = 0; a < 2; ++a)
      if (!(pp->field_max[a] > pp->field_min[a])) return fail(VC_EINVAL, "FieldGrid bounds must have positive extent");
    M.kind = 0;
    M.nx = pp->field_nx;
    M.ny = pp->field_ny;
    for (int a = 0; a < 2; ++a) {
      M.fmin[a] = pp->field_min[a];
      M.fmax[a] = pp->field_max[a];
    }
    g.N = (long long)M.nx * M.ny;
  } else if (pp->target == VC_TARGET_CAMERA) {
    if (sc->dim != 3) return fail(VC_EINVAL, "Camera rendering requires a 3D scene");
    if (seed_kind == 1) return fail(VC_EINVAL, "field seeds on a camera target");
    if (seed_kind == 0) spp = 1;
    DevCamera cam{};
    vc_camera c0 = pp->camera;
    c0.row0 = c0.col0 = 0;
    c0.rows = c0.cols = 0;
    int rc = make_dev_camera(c0, &cam);
    if (rc) return rc;
    const int npx = cam.w * cam.h;
    const long long nr = (long long)npx * spp;
    if (nr > (1LL << 31) - 2) return fail(VC_EINVAL, "too many camera rays");
    cudaError_t e = cudaMalloc(&bf.ray, (size_t)nr * 32);
    if (e == cudaSuccess) e = cudaMalloc(&bf.steps, ((size_t)nr + 1) * 8);
    if (e == cudaSuccess) e = cudaMalloc(&bf.first, ((size_t)nr + 1) * 8);
    if (e != cudaSuccess) return cuda_fail(e, "populate ray buffers");
    rc = ensure_emitters(sc, pp->n_light_samples);
    if (rc) return rc;
    DevScene S = dev_scene(sc);
    uint64_t* djit = nullptr;
    JumpTables jt{jump_tables(&e)};
    if (!jt.tab) return cuda_fail(e, "jump tables");
    if (spp > 1) {  // jitter stream default_rng(SeedSequence([seed, 101])) (src/renderer.py:446)
      uint32_t jw[2] = {(uint32_t)pp->seed, 101u};
      uint64_t jst[4];
      seedseq_pcg64(jw, 2, jst);
      e = cudaMalloc(&djit, 32);
      if (e == cudaSuccess) e = cudaMemcpy(djit, jst, 32, cudaMemcpyHostToDevice);
      if (e != cudaSuccess) {
        cudaFree(djit);
        return cuda_fail(e, "jitter state");
      }
    }
    k_pop_rays<<<(int)((nr + 127) / 128), 128, 0, st>>>(S, cam, pp->march_step, spp, djit, jt, bf.ray, bf.steps);
    e = cudaMemsetAsync(bf.steps + nr, 0, 8, st);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, bf.steps, bf.first, nr + 1, st);
    if (e == cudaSuccess) e = cudaMalloc(&bf.tmp, tb + 16);
    if (e == cudaSuccess) cub::DeviceScan::ExclusiveSum(bf.tmp, tb, bf.steps, bf.first, nr + 1, st);
    long long total = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&total, bf.first + nr, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(djit);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    count_launches(2);
    if (e != cudaSuccess) return cuda_fail(e, "populate rays");
    M.kind = 1;
    for (int a = 0; a < 3; ++a) M.pos[a] = cam.pos[a];
    M.ray = bf.ray;
    M.first = bf.first;
    M.n_rays = (int)nr;
    g.npx = npx;
    g.N = total;
  } else {
    return fail(VC_EINVAL, "target must be VC_TARGET_FIELD or VC_TARGET_CAMERA");
  }
  g.cs = cs;
  g.cm = cm;
  int rc = g.run();
  if (!rc) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_fail(e, "populate");
  }
  if (!rc && stats)
    for (int k = 0; k < 8; ++k) stats[k] = g.stats[k];
  if (!rc && rs) {  // hand over the ray prefix and the committed direct values
    rs->first = bf.first;
    bf.first = nullptr;
    rs->c_ord = g.c_ord;
    rs->c_val = g.c_val;
    rs->c_n = g.c_n;
    g.c_ord = nullptr;
    g.c_val = nullptr;
    rs->total = g.N;
  }
  return rc;
}

__global__ void k_field_values(MarchStream M, DevCache Cs, DevCache Cm, int n, int tagged, const double* direct,
                               double* J, unsigned char* miss) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double x[2];
  stream_point<2>(M, j, x);
  const long long lim = tagged ? (long long)j + 1 : LLONG_MAX;
  double Js[3], Jm[3];
  const bool cs = cache_interpolate<2>(Cs, x, Js, nullptr, lim);
  const bool cm = cache_interpolate<2>(Cm, x, Jm, nullptr, lim);
  const bool hit = cs && cm;
  for (int c = 0; c < 3; ++c) J[(size_t)j * 3 + c] = hit ? add(Js[c], Jm[c]) : 0.0;
  if (!hit && direct && !isnan(direct[(size_t)j * 3]))  // inserted, blend still None: the direct value
    for (int c = 0; c < 3; ++c) J[(size_t)j * 3 + c] = direct[(size_t)j * 3 + c];
  miss[j] = hit ? 0 : 1;
}

__global__ void k_field_points(MarchStream M, const int* cells, int n, double* x, uint32_t* words, uint32_t seed) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int j = cells[e];
  stream_point<2>(M, j, x + (size_t)e * 2);
  uint32_t* w = words + (size_t)e * 4;
  w[0] = seed;
  w[1] = 307u;
  w[2] = (uint32_t)(j / M.nx);
  w[3] = (uint32_t)(j % M.nx);
}

__global__ void k_field_direct(const double* mom, int MS, const int* cells, int n, double* J) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const double* m = mom + (size_t)e * 2 * MS;
  for (int c = 0; c < 3; ++c) J[(size_t)cells[e] * 3 + c] = add(m[c], m[MS + c]);
}

extern "C" {

int vc_populate(vc_scene* sc, const vc_populate_params* pp, vc_cache** single, vc_cache** multiple, int64_t* stats,
                void* stream) {
  if (!sc || !pp || !single || !multiple) return fail(VC_EINVAL, "null argument");
  *single = *multiple = nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  double bmin[3], bmax[3];
  for (int a = 0; a < 3; ++a) {
    bmin[a] = sc->bmin[a];
    bmax[a] = sc->bmax[a];
  }
  vc_cache* cs = new vc_cache();
  vc_cache* cm = new vc_cache();
  int rc = cache_init(cs, sc->dim, bmin, bmax);
  if (!rc) rc = cache_init(cm, sc->dim, bmin, bmax);
  if (!rc) rc = cache_reserve(cs, 1024, st);
  if (!rc) rc = cache_reserve(cm, 1024, st);
  if (!rc) rc = cache_rebuild(cs, st);
  if (!rc) rc = cache_rebuild(cm, st);
  if (!rc) rc = populate_run(sc, pp, 0, cs, cm, stats, st, nullptr, 1, nullptr);
  if (rc) {
    delete cs;
    delete cm;
    return rc;
  }
  *single = cs;
  *multiple = cm;
  return VC_OK;
}

int vc_render_field(vc_scene* sc, vc_cache* cs, vc_cache* cm, const vc_populate_params* pp, int frozen,
                    double* image, int64_t* stats, int flags, void* stream) {
  if (!sc || !cs || !cm || !pp || !image) return fail(VC_EINVAL, "null argument");
  if (sc->dim != 2 || cs->dim != 2 || cm->dim != 2) return fail(VC_EINVAL, "FieldGrid rendering requires a 2D scene");
  if (pp->target != VC_TARGET_FIELD) return fail(VC_EINVAL, "vc_render_field needs a VC_TARGET_FIELD target");
  if (pp->field_nx < 1 || pp->field_ny < 1) return fail(VC_EINVAL, "FieldGrid resolution must be positive");
  if (!(pp->march_step > 0.0)) return fail(VC_EINVAL, "march_step must be positive");
  if (!(pp->epsilon > 0.0)) return fail(VC_EINVAL, "epsilon must be positive");
  cudaStream_t st = (cudaStream_t)stream;
  const int n = pp->field_nx * pp->field_ny;
  if (pp->estimator == VC_EST_PATH) frozen = 1;  // no cache in the path mode
  MarchStream M{};
  M.kind = 0;
  M.nx = pp->field_nx;
  M.ny = pp->field_ny;
  for (int a = 0; a < 2; ++a) {
    M.fmin[a] = pp->field_min[a];
    M.fmax[a] = pp->field_max[a];
  }
  int64_t pst[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  Workspace ws;
  cudaError_t e = cudaSuccess;
  double* direct = nullptr;
  if (!frozen) {  // misses insert as the render proceeds (src/renderer.py:361-368)
    direct = (double*)ws.get(7, (size_t)n * 24, &e);
    if (e == cudaSuccess) e = cudaMemsetAsync(direct, 0xff, (size_t)n * 24, st);  // NaN: no direct value
    if (e != cudaSuccess) return cuda_fail(e, "field direct buffer");
    int rc = populate_run(sc, pp, 1, cs, cm, pst, st, direct, 1, nullptr);
    if (rc) return rc;
  }
  double* J = (double*)ws.get(0, (size_t)n * 24, &e);
  unsigned char* miss = (unsigned char*)ws.get(1, (size_t)n, &e);
  if (e != cudaSuccess) return cuda_fail(e, "field buffers");
  k_field_values<<<(n + 127) / 128, 128, 0, st>>>(M, cs->dev(), cm->dev(), n, frozen ? 0 : 1, direct, J, miss);
  count_launches(1);
  std::vector<unsigned char> hm(n);
  e = cudaMemcpyAsync(hm.data(), miss, n, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "field lookup");
  long long n_direct = 0;
  if (frozen) {  // direct evaluation, no insertion
    std::vector<int> cells;
    for (int j = 0; j < n; ++j)
      if (hm[j]) cells.push_back(j);
    const int nm = (int)cells.size();
    n_direct = nm;
    if (nm > 0) {
      const int MS = moment_size(2);
      int* dc = (int*)ws.get(2, (size_t)nm * 4, &e);
      double* x = (double*)ws.get(3, (size_t)nm * 16, &e);
      uint32_t* w = (uint32_t*)ws.get(4, (size_t)nm * 16, &e);
      double* mom = (double*)ws.get(5, (size_t)nm * 2 * MS * 8, &e);
      long long* bst = (long long*)ws.get(6, (size_t)nm * kStats * 8, &e);
      if (e == cudaSuccess) e = cudaMemcpyAsync(dc, cells.data(), (size_t)nm * 4, cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) return cuda_fail(e, "field miss buffers");
      k_field_points<<<(nm + 127) / 128, 128, 0, st>>>(M, dc, nm, x, w, (uint32_t)pp->seed);
      vc_build_params bp{};
      bp.n_angular = pp->n_angular;
      bp.march_step = pp->march_step;
      bp.n_inner = pp->n_inner;
      bp.n_light_samples = pp->n_light_samples;
      bp.epsilon = pp->epsilon;
      bp.flags = VC_SEED_WORDS;
      bp.seed_words = 4;
      int rc;
      int stride = MS;
      if (pp->estimator == VC_EST_PATH) {  // _point_value, mode "path" (src/renderer.py:337-346)
        stride = 3;
        rc = path_impl(sc, nm, x, w, pp->path_samples, pp->max_media_bounces, pp->n_light_samples, VC_SEED_WORDS,
                       4, mom, st);
      } else if (pp->estimator == VC_EST_BASELINE) {  // value = est_single + est_multiple
        vc_baseline_params blp{};
        blp.n_angular = pp->n_angular;
        blp.max_media_bounces = pp->max_media_bounces;
        blp.n_light_samples = pp->n_light_samples;
        blp.alpha = pp->baseline_alpha;
        blp.flags = VC_SEED_WORDS;
        blp.seed_words = 4;
        stride = 3 + 3 * 2;
        rc = baseline_impl(sc, nm, x, w, &blp, mom, nullptr, nullptr, st);
      } else {
        rc = build_impl(sc, nm, x, w, nullptr, &bp, mom, (int64_t*)bst, nullptr, st, nullptr);
      }
      if (rc) return rc;
      k_field_direct<<<(nm + 127) / 128, 128, 0, st>>>(mom, stride, dc, nm, J);
      count_launches(2);
    }
  } else {
    n_direct = pst[7];
  }
  // image = full_angle(2) · J (src/renderer.py:428-436)
  std::vector<double> hJ((size_t)n * 3);
  e = cudaMemcpyAsync(hJ.data(), J, (size_t)n * 24, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "field download");
  const double scale = 2.0 * 3.141592653589793;
  std::vector<double> out((size_t)n * 3);
  for (size_t i = 0; i < out.size(); ++i) out[i] = scale * hJ[i];
  if (flags & VC_MEM_HOST) {
    std::copy(out.begin(), out.end(), image);
  } else {
    e = cudaMemcpyAsync(image, out.data(), out.size() * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "field upload");
  }
  if (stats) {
    stats[0] = n - n_direct;
    stats[1] = n_direct;
  }
  return VC_OK;
}

int64_t vc_cache_size(const vc_cache* c) { return c ? (int64_t)c->n : -1; }

int vc_cache_records(const vc_cache* c, double* records, int64_t* tags, int flags, void* stream) {
  if (!c) return fail(VC_EINVAL, "null cache");
  cudaStream_t st = (cudaStream_t)stream;
  const cudaMemcpyKind k = (flags & VC_MEM_HOST) ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  cudaError_t e = cudaSuccess;
  if (c->n > 0 && records) e = cudaMemcpyAsync(records, c->d_rec, (size_t)c->n * record_size(c->dim) * 8, k, st);
  if (e == cudaSuccess && c->n > 0 && tags) e = cudaMemcpyAsync(tags, c->d_tag, (size_t)c->n * 8, k, st);
  if (e == cudaSuccess && (flags & VC_MEM_HOST)) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "cache download");
  return VC_OK;
}

}  // extern "C"
