// C ABI of libvolcache_b200: scene upload, workspace management, wave orchestration.
#include <algorithm>
#include <cfloat>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/volcache_b200.h"
#include "vc_build.h"
#include "vc_device.cuh"
#include "vc_api_internal.h"

namespace vc {

thread_local std::string g_err;
std::atomic<long long> g_launches{0};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(VC_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

void* Workspace::get(int slot, size_t bytes, cudaError_t* err) {
  if (bytes == 0) bytes = 16;
  if (cap[slot] < bytes) {
    if (ptr[slot]) cudaFree(ptr[slot]);
    ptr[slot] = nullptr;
    cap[slot] = 0;
    cudaError_t e = cudaMalloc(&ptr[slot], bytes);
    if (e != cudaSuccess) {
      *err = e;
      return nullptr;
    }
    cap[slot] = bytes;
  }
  return ptr[slot];
}

__global__ void k_outside(const double* x, long long N, int D, double3 lo, double3 hi, int* flag) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    bool out = false;
    for (int a = 0; a < D; ++a) {
      const double v = x[i * D + a];
      const double l = a == 0 ? lo.x : (a == 1 ? lo.y : lo.z), h = a == 0 ? hi.x : (a == 1 ? hi.y : hi.z);
      out |= !(v >= l && v <= h);  // NaN counts as outside, as on the host
    }
    if (out) atomicOr(flag, 1);
  }
}

// Device inputs: k_outside raises a device flag (read by k_rings, which then skips every
// ring so no kernel indexes past the r_ub-sized buffers) and copies it to pinned memory
// behind an event; the caller enqueues its work first and waits only at check_end, so the
// check never drains the stream ahead of the wave.
int check_begin(const vc_scene* sc, long long N, const double* x, bool host, const char* what, cudaStream_t st,
                InsideCheck* ck) {
  ck->pending = false;
  ck->dflag = nullptr;
  const int D = sc->dim;
  const double eps = 1e-12 * sc->scale;
  if (host) {
    for (long long i = 0; i < N; ++i)
      for (int a = 0; a < D; ++a) {
        const double v = x[(size_t)i * D + a];
        if (!(v >= sc->bmin[a] - eps && v <= sc->bmax[a] + eps)) return fail(VC_EOUTSIDE, what);
      }
    return VC_OK;
  }
  static thread_local int* dflag = nullptr;
  static thread_local int* hflag = nullptr;
  static thread_local cudaEvent_t ev = nullptr;
  cudaError_t e = cudaSuccess;
  if (!dflag) e = cudaMalloc(&dflag, 4);
  if (e == cudaSuccess && !hflag) e = cudaMallocHost(&hflag, 4);
  if (e == cudaSuccess && !ev) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaMemsetAsync(dflag, 0, 4, st);
  if (e != cudaSuccess) return cuda_fail(e, "bounds check");
  const double3 lo = make_double3(sc->bmin[0] - eps, sc->bmin[1] - eps, sc->bmin[2] - eps);
  const double3 hi = make_double3(sc->bmax[0] + eps, sc->bmax[1] + eps, sc->bmax[2] + eps);
  const int grid = (int)std::max<long long>(1, std::min<long long>((N + 255) / 256, 4 * 148));
  k_outside<<<grid, 256, 0, st>>>(x, N, D, lo, hi, dflag);
  count_launches(1);
  e = cudaMemcpyAsync(hflag, dflag, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaEventRecord(ev, st);
  if (e != cudaSuccess) return cuda_fail(e, "bounds check");
  ck->pending = true;
  ck->dflag = dflag;
  ck->hflag = hflag;
  ck->ev = ev;
  ck->what = what;
  return VC_OK;
}

// Deferred form (VC_DEFER_CHECK): the wave's flag is OR-ed into a sticky per-thread device word on
// the stream and the call returns without waiting; vc_check_deferred reads and clears the word.
__global__ void k_flag_or(int* sticky, const int* flag) {
  if (*flag) atomicOr(sticky, 1);
}

static int* sticky_flag() {
  static thread_local int* d = nullptr;
  if (!d && cudaMalloc(&d, 4) == cudaSuccess) cudaMemset(d, 0, 4);
  return d;
}

int check_defer(InsideCheck* ck, cudaStream_t st) {
  if (!ck->pending) return VC_OK;
  ck->pending = false;
  int* sticky = sticky_flag();
  if (!sticky) return fail(VC_ECUDA, "bounds check (deferred flag allocation)");
  k_flag_or<<<1, 1, 0, st>>>(sticky, ck->dflag);
  count_launches(1);
  return VC_OK;
}

int check_deferred_read(cudaStream_t st) {
  int* sticky = sticky_flag();
  if (!sticky) return fail(VC_ECUDA, "bounds check (deferred flag allocation)");
  int h = 0;
  cudaError_t e = cudaMemcpyAsync(&h, sticky, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(sticky, 0, 4, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "bounds check");
  return h ? fail(VC_EOUTSIDE, "subdivision center lies outside the medium bounds (deferred check)") : VC_OK;
}

int check_end(InsideCheck* ck) {
  if (!ck->pending) return VC_OK;
  ck->pending = false;
  const cudaError_t e = cudaEventSynchronize(ck->ev);
  if (e != cudaSuccess) return cuda_fail(e, "bounds check");
  return *ck->hflag ? fail(VC_EOUTSIDE, ck->what) : VC_OK;
}

int check_inside(const vc_scene* sc, long long N, const double* x, bool host, const char* what,
                 cudaStream_t st) {
  InsideCheck ck;
  const int rc = check_begin(sc, N, x, host, what, st, &ck);
  return rc ? rc : check_end(&ck);
}

Workspace::~Workspace() {
  for (int i = 0; i < kSlots; ++i)
    if (ptr[i]) cudaFree(ptr[i]);
}

// PCG64 jump tables, built once per device.
const unsigned long long* jump_tables(cudaError_t* err) {
  static const unsigned long long* dev_tab[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev_tab[dev]) return dev_tab[dev];
  std::vector<unsigned long long> h(3 * 1024 * 4);
  u128 M = pcg_mult();
  u128 bA = M, bG = 1;  // jump by 1
  for (int lv = 0; lv < 3; ++lv) {
    u128 A = 1, G = 0;  // jump by 0
    for (int k = 0; k < 1024; ++k) {
      unsigned long long* e = &h[((size_t)lv * 1024 + k) * 4];
      e[0] = (unsigned long long)(A >> 64);
      e[1] = (unsigned long long)A;
      e[2] = (unsigned long long)(G >> 64);
      e[3] = (unsigned long long)G;
      G = bA * G + bG;  // then jump by base
      A = bA * A;
    }
    // base for next level: jump by 1024^(lv+1) = current (A, G) after 1024 steps
    bA = A;
    bG = G;
  }
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMalloc(&d, h.size() * 8);
  if (e == cudaSuccess) e = cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    *err = e;
    return nullptr;
  }
  dev_tab[dev] = d;
  return d;
}

bool grid_shape_3d(int n, int* rows, int* cols) {
  // src/scene.py:370-385
  double target = std::sqrt(n / 2.0);
  int best = -1;
  int lim = (int)std::sqrt((double)n);
  for (int r = 2; r <= lim; ++r) {
    if (n % r) continue;
    if (n / r < 3) continue;
    if (best < 0 || std::fabs(r - target) < std::fabs(best - target)) best = r;
  }
  if (best < 0) return false;
  *rows = best;
  *cols = n / best;
  return true;
}

int ensure_emitters(vc_scene* sc, int n_light) {
  if (sc->es_nlight == n_light) return VC_OK;
  const int D = sc->dim;
  std::vector<double> pos, w;
  std::vector<int> surf;
  for (int k = 0; k < sc->K; ++k) {
    const double* E = &sc->emission[3 * (size_t)k];
    if (!(E[0] > 0.0 || E[1] > 0.0 || E[2] > 0.0)) continue;
    const double* V = &sc->verts[(size_t)k * D * D];
    if (D == 2) {  // src/transport.py:139-146
      double e0 = V[2] - V[0], e1 = V[3] - V[1];
      double len = std::sqrt(e0 * e0 + e1 * e1);
      for (int j = 0; j < n_light; ++j) {
        double u = (j + 0.5) / n_light;
        pos.push_back(V[0] + u * e0);
        pos.push_back(V[1] + u * e1);
        w.push_back(len / n_light);
        surf.push_back(k);
      }
    } else {  // src/transport.py:147-160
      int m = std::max(2, (int)std::lround(std::sqrt((double)n_light)));
      double e1[3], e2[3];
      for (int a = 0; a < 3; ++a) {
        e1[a] = V[3 + a] - V[a];
        e2[a] = V[6 + a] - V[a];
      }
      double c0 = e1[1] * e2[2] - e1[2] * e2[1], c1 = e1[2] * e2[0] - e1[0] * e2[2],
             c2 = e1[0] * e2[1] - e1[1] * e2[0];
      double area = 0.5 * std::sqrt(c0 * c0 + c1 * c1 + c2 * c2);
      for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) {
          double u = (i + 0.5) / m, v = (j + 0.5) / m;
          if (u + v > 1.0) {
            u = 1.0 - u;
            v = 1.0 - v;
          }
          for (int a = 0; a < 3; ++a) pos.push_back(V[a] + u * e1[a] + v * e2[a]);
          w.push_back(area / (m * m));
          surf.push_back(k);
        }
    }
  }
  cudaFree(sc->d_es_pos);
  cudaFree(sc->d_es_w);
  cudaFree(sc->d_es_surf);
  sc->d_es_pos = nullptr;
  sc->d_es_w = nullptr;
  sc->d_es_surf = nullptr;
  sc->n_es = (int)w.size();
  if (sc->n_es) {
    cudaError_t e = cudaMalloc(&sc->d_es_pos, pos.size() * 8);
    if (e == cudaSuccess) e = cudaMalloc(&sc->d_es_w, w.size() * 8);
    if (e == cudaSuccess) e = cudaMalloc(&sc->d_es_surf, surf.size() * 4);
    if (e == cudaSuccess) e = cudaMemcpy(sc->d_es_pos, pos.data(), pos.size() * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(sc->d_es_w, w.data(), w.size() * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(sc->d_es_surf, surf.data(), surf.size() * 4, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "emitter upload");
  }
  sc->es_nlight = n_light;
  return VC_OK;
}

DevScene dev_scene(const vc_scene* sc) {
  DevScene S{};
  S.dim = sc->dim;
  S.K = sc->K;
  S.geo = sc->geo.dev();
  S.emit = sc->emit.dev();
  S.ep = sc->ep;
  S.n_es = sc->n_es;
  S.reflective = sc->reflective;
  for (int a = 0; a < 3; ++a) {
    S.bmin[a] = sc->bmin[a];
    S.bmax[a] = sc->bmax[a];
  }
  S.scale = sc->scale;
  S.t_eps = 1e-6 * sc->scale;
  S.sigma_s = sc->sigma_s;
  S.sigma_a = sc->sigma_a;
  S.sigma_t = sc->sigma_s + sc->sigma_a;
  S.max_emission = sc->max_emission;
  S.normal = sc->d_normal;
  S.emission = sc->d_emission;
  S.albedo = sc->d_albedo;
  S.es_pos = sc->d_es_pos;
  S.es_w = sc->d_es_w;
  S.es_surf = sc->d_es_surf;
  S.n_lights = sc->n_lights;
  S.lights = sc->d_lights;
  return S;
}

void count_launches(long long n) { g_launches += n; }

// Optional per-kernel CUDA-event profile: events are recorded on the launching stream
// around every kernel while enabled; vc_profile_read sums elapsed time per class.
namespace {
struct ProfRec {
  int kc;
  cudaEvent_t a, b;
};
struct Profiler {
  bool on = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  struct Open {
    cudaStream_t st;
    int kc;
    cudaEvent_t ev;
  };
  std::vector<Open> open;  // one open interval per stream (the wave forks the triangulation)
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};
Profiler g_prof;
}  // namespace

void prof_begin(int kc, cudaStream_t st) {
  if (!g_prof.on) return;
  cudaEvent_t a = g_prof.get();
  cudaEventRecord(a, st);
  for (auto& o : g_prof.open)
    if (o.st == st) {
      o.kc = kc;
      o.ev = a;
      return;
    }
  g_prof.open.push_back({st, kc, a});
}

void prof_end(cudaStream_t st) {
  if (!g_prof.on) return;
  for (size_t i = 0; i < g_prof.open.size(); ++i)
    if (g_prof.open[i].st == st) {
      cudaEvent_t b = g_prof.get();
      cudaEventRecord(b, st);
      g_prof.recs.push_back({g_prof.open[i].kc, g_prof.open[i].ev, b});
      g_prof.open.erase(g_prof.open.begin() + i);
      return;
    }
}

// ---------------------------------------------------------------------------
// The record build, in waves sized by the scratch budget.
// ---------------------------------------------------------------------------

// Candidate windows of the hull triangulation, per stratum row: the smallest window
// (rows r ± h, columns c ± w, h ≤ 3) whose border lies at least 2 mean spacings from every
// point of the row's strata, with at most kHullK candidates.  The window only sets the
// cost: every cell the kernel keeps passes its own security test (k_delaunay_hull).
// VOLCACHE_DEL_HULL=0 sends every row to the clipping kernel.
static void del_row_table(BuildParams& P) {
  const char* env = getenv("VOLCACHE_DEL_HULL");
  const bool on = !(env && env[0] == '0');
  const char* ek = getenv("VOLCACHE_HULL_KMAX");
  const int kcap = ek ? std::max(8, std::min(kHullK, atoi(ek))) : kHullK;
  const int rows = P.rows, cols = P.cols;
  P.del_kmax = 0;
  const double pi = 3.141592653589793;
  const char* ea = getenv("VOLCACHE_HULL_ALPHA");  // window margin in mean spacings (default 2)
  const double alpha = (ea ? std::max(0.5, std::min(4.0, atof(ea))) : 2.0) * std::sqrt(4.0 * pi / P.n_angular);
  for (int r = 0; r < std::min(rows, kDelRowsMax); ++r) {
    const double tht = std::acos(1.0 - 2.0 * r / rows), thb = std::acos(1.0 - 2.0 * (r + 1) / rows);
    const double smin = std::min(std::sin(tht), std::sin(thb));
    int best = 1 << 30, code = 0;
    for (int h = 1; on && h <= 3; ++h) {
      if (r - h < 0 || r + h >= rows) continue;
      const double drow = std::min(tht - std::acos(1.0 - 2.0 * (r - h) / rows),
                                   std::acos(1.0 - 2.0 * (r + h + 1) / rows) - thb);
      if (drow < alpha) continue;
      for (int w = 1; w <= 15 && 2 * (2 * w + 1) < cols; ++w) {
        const double dw = w * 2.0 * pi / cols;
        if (dw >= 0.5 * pi) break;
        if (std::asin(std::min(1.0, std::sin(dw) * smin)) >= alpha) {
          const int K = (2 * h + 1) * (2 * w + 1) - 1;
          if (K <= kcap && K < best) {
            best = K;
            code = (h << 6) | w;
          }
          break;
        }
      }
    }
    P.del_hw[r] = (unsigned char)code;
    P.del_kmax = std::max(P.del_kmax, code ? best : 0);
  }
  static const int kClassMax[3] = {34, 44, kHullK};
  int nr = 0;
  for (int k = 0; k < 3; ++k) {
    P.del_cls[k] = nr;
    P.del_cls_k[k] = 0;
    for (int r = 0; r < std::min(rows, kDelRowsMax); ++r) {
      const int code = P.del_hw[r];
      if (!code) continue;
      const int K = (2 * (code >> 6) + 1) * (2 * (code & 63) + 1) - 1;
      if (K <= kClassMax[k] && (k == 0 || K > kClassMax[k - 1])) {
        P.del_rows[nr++] = (unsigned short)r;
        P.del_cls_k[k] = std::max(P.del_cls_k[k], K);
      }
    }
  }
  P.del_cls[3] = nr;
  // polar rows: candidates within δ = 3 spacings (2·R_cell ≤ δ holds for all but ~1% of
  // the cap cells; ≤ 40 candidates), kept in 16-bit column indices
  P.del_zstep = 2.0 / rows;
  const double delta = 3.0 * std::sqrt(4.0 * pi / P.n_angular);
  P.del_cap = (on && P.del_kmax > 0 && rows >= 4 && 2 * cols <= 65535) ? 1 : 0;
  P.del_cap_cos = (float)std::cos(delta);
  P.del_cap_sin = (float)std::sin(delta);
  P.del_cap_c2 = std::cos(0.5 * delta) * std::cos(0.5 * delta);
  P.del_cap_s2 = std::sin(0.5 * delta) * std::sin(0.5 * delta);
  P.del_warp_delta = 3.2 * std::sqrt(4.0 * pi / P.n_angular);
  P.del_dbg_cell = getenv("VOLCACHE_DEL_DEBUG_CELL") ? atoi(getenv("VOLCACHE_DEL_DEBUG_CELL")) : -1;
}

int build_impl(vc_scene* sc, int N, const double* x, const void* rng, const int32_t* adjacency,
               const vc_build_params* prm, double* moments, int64_t* stats, double* records,
               cudaStream_t st, Inspect* insp) {
  if (!sc || !prm) return fail(VC_EINVAL, "null scene or params");
  if (N < 0) return fail(VC_EINVAL, "n_records must be non-negative");
  if (N == 0) return VC_OK;
  const int D = sc->dim;
  const int n = prm->n_angular;
  if (!(prm->march_step > 0.0)) return fail(VC_EINVAL, "march_step must be positive");
  if (prm->n_inner < 1) return fail(VC_EINVAL, "n_inner must be >= 1");
  if (prm->n_light_samples < 1) return fail(VC_EINVAL, "n_light_samples must be >= 1");
  const bool host = prm->flags & VC_MEM_HOST;
  const bool words = prm->flags & VC_SEED_WORDS;
  BuildParams P{};
  P.n_angular = n;
  P.march_step = prm->march_step;
  P.n_inner = prm->n_inner;
  if (prm->media_bounces < 0 || prm->media_bounces > 8) return fail(VC_EINVAL, "media_bounces must be in [0, 8]");
  P.media_bounces = std::max(1, prm->media_bounces);
  if (!(prm->hg_g > -1.0 && prm->hg_g < 1.0)) return fail(VC_EINVAL, "hg_g must lie in (-1, 1)");
  P.hg_g = D == 3 ? prm->hg_g : 0.0;
  P.epsilon = prm->epsilon;
  P.anisotropic = (prm->flags & VC_ISOTROPIC) ? 0 : 1;
  P.make_records = (records != nullptr) || (prm->flags & VC_MAKE_RECORDS);
  if (P.make_records && !(prm->epsilon > 0.0)) return fail(VC_EINVAL, "epsilon must be positive");
  if (D == 2) {
    if (n < 3) return fail(VC_EINVAL, "2D stratification needs n >= 3");
    P.rows = 1;
    P.cols = n;
    P.n_tris = n;
  } else {
    if (!grid_shape_3d(n, &P.rows, &P.cols))
      return fail(VC_EINVAL, "n=" + std::to_string(n) + " is not expressible as rows x cols with rows >= 2 and cols >= 3");
    P.n_tris = 2 * n - 4;
  }
  P.host_adjacency = (D == 3 && adjacency != nullptr) ? 1 : 0;
  P.r_ub = (int)std::floor(sc->scale * (1.0 + 1e-9) / prm->march_step + 0.5) + 2;
  {  // triangulation search radii: α₀ = 2.8 × mean direction spacing, ×1.5 per retry, ≤ 1.5
    double a = 2.8 * std::sqrt(4.0 * 3.141592653589793 / n);
    for (int k = 0; k < kDelLevels; ++k) {
      P.del[k] = DelAngle{a, std::sin(a), std::cos(a), std::tan(0.5 * a)};
      a = std::min(1.5 * a, 1.5);
    }
  }
  if (D == 3) del_row_table(P);
  // ValueError (src/subdivision.py:155-158), host and device inputs alike: host inputs are
  // checked before any work; device inputs by a flag kernel whose result is read after the
  // wave is enqueued (a flagged wave does no ring work; the call then fails)
  InsideCheck inside;
  {
    const int rc = check_begin(sc, N, x, host, "subdivision center lies outside the medium bounds", st, &inside);
    if (rc) return rc;
  }
  int rc = ensure_emitters(sc, prm->n_light_samples);
  if (rc) return rc;
  cudaError_t err = cudaSuccess;
  JumpTables jt{jump_tables(&err)};
  if (!jt.tab) return cuda_fail(err, "jump tables");
  DevScene S = dev_scene(sc);

  // per-record scratch bytes
  const size_t MS = moment_size(D), RS = record_size(D);
  const size_t media_per = (size_t)n * P.r_ub;
  size_t per = (size_t)n * (D * 8 + 8 + 4 * 5 + 24) + media_per * 12 + 64 + 2 * MS * 8 + 2 * RS * 8 +
               kStats * 8 + 32 + 8;
  if (D == 3) per += (size_t)P.n_tris * 12 + (P.host_adjacency ? 0 : (size_t)n * 32 * 8);
  per += media_per / 10 * 80;                     // two-pass gather queue
  per += (media_per / 16 + 1) * 4;                // gather run → direction table
  per += (size_t)n * 8 * ((P.r_ub + 63) / 64);  // live-sample bit masks
  per += (size_t)n * 16;                          // float32 directions
  per += (size_t)n * 16 + kAsmParts * 96 * 8;     // DirInfo + assembly partials
  // assembly item lists: surface items ≤ 2n, media items ≤ valence × live samples; lists that
  // outgrow their share fall back to the fused kernel
  long long item_cap = 4LL * n + (long long)(media_per / 4) + 1024;
  if (const char* e = getenv("VOLCACHE_ASM_ITEM_CAP")) item_cap = std::max(0LL, atoll(e));
  per += (size_t)item_cap * 8 + kAsmParts * 8 + 4;
  if (sc->budget <= 0) {  // default scratch budget: 1/3 of HBM (B200: 60 GB), ≤ 64 GiB
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    sc->budget = std::min<long long>((long long)(tot / 3), 64LL << 30);
    if (sc->budget < (1LL << 30)) sc->budget = 1LL << 30;
  }
  long long B = (long long)(sc->budget / (long long)per);
  if (B < 1) B = 1;
  if (B > N) B = N;
  if (B > 65535) B = 65535;
  if (insp) B = 1;
  Workspace& ws = sc->ws;
  auto alloc = [&](int slot, size_t bytes) { return ws.get(slot, bytes, &err); };
  Wave W{};
  double* dx = (double*)alloc(0, B * D * 8);
  uint64_t* drng = (uint64_t*)alloc(1, B * 4 * 8);
  W.dirs = (double*)alloc(2, B * n * D * 8);
  W.s = (double*)alloc(3, B * n * 8);
  W.idx = (int*)alloc(4, B * n * 4);
  W.cnt = (int*)alloc(5, B * n * 4);
  W.pre = (int*)alloc(6, B * n * 4);
  W.run_stride = (int)(media_per / 16 + 1);
  W.run_dir = (int*)alloc(48, (size_t)B * W.run_stride * 4);
  W.lo = (double*)alloc(7, B * n * 24);
  W.emit_tab = sc->reflective ? nullptr : sc->d_emission;  // non-reflective: L_o = emission[idx], lo unused
  W.rec_R = (int*)alloc(8, B * 4);
  W.rec_P = (int*)alloc(9, B * 4);
  W.rec_maxc = (int*)alloc(10, B * 4);
  W.rec_base = (long long*)alloc(11, (B + 1) * 8);
  W.media = (float*)alloc(12, B * media_per * 12);
  W.media_cap = (long long)(B * media_per);
  W.tris = (int*)alloc(13, D == 3 ? B * P.n_tris * 12 : 16);
  W.deg = (int*)alloc(14, B * n * 4);
  W.tri_status = (int*)alloc(15, B * 4);
  double* dmom = (double*)alloc(16, B * 2 * MS * 8);
  long long* dstat = (long long*)alloc(17, B * kStats * 8);
  double* drec = (double*)alloc(18, B * 2 * RS * 8);
  int* own = (int*)alloc(19, (D == 3 && !P.host_adjacency) ? B * n * 32 * 8 : 16);
  W.own_stride = (long long)B * n;
  int* own_cnt = (int*)alloc(20, B * n * 4);
  uint32_t* dwords = (uint32_t*)alloc(21, words ? B * prm->seed_words * 4 + 4 : 16);
  W.dirs32 = (float4*)alloc(35, D == 3 ? B * n * 16 : 16);
  W.info = (DirInfo*)alloc(36, B * n * sizeof(DirInfo));
  W.del_retry_cap = (int)std::min<long long>(B * n, 1LL << 16);
  W.del_retry = (int*)alloc(38, (size_t)W.del_retry_cap * 4);
  W.del_retry_count = (unsigned int*)alloc(39, 8);
  W.del_scratch = (double*)alloc(40, D == 3 ? (size_t)W.del_retry_cap * 48 * 3 * 8 : 16);
  W.del_fb = (int*)alloc(44, (D == 3 && !P.host_adjacency) ? (size_t)B * n * 4 : 16);
  W.del_fb_count = (unsigned int*)alloc(45, 8);
  W.del_fb2 = (int*)alloc(46, (D == 3 && !P.host_adjacency) ? (size_t)B * n * 4 : 16);
  W.del_fb2_count = (unsigned int*)alloc(47, 8);
  W.cap_bin_stride = kCapGMax * kCapGMax + 1 + P.cols;  // bin starts + 2·cols 16-bit indices
  W.cap_bins = (int*)alloc(49, (D == 3 && !P.host_adjacency && P.cols <= kCapGCols) ? (size_t)B * 2 * W.cap_bin_stride * 4 : 16);
  W.partial = (double*)alloc(37, B * kAsmParts * 64 * 8 + B * kAsmParts * 5 * 8);  // sums + 5 counters
  W.item_cap = item_cap;
  W.asm_items = item_cap > 0 ? (uint2*)alloc(41, (size_t)B * item_cap * 8) : nullptr;
  W.item_n = (int*)alloc(42, B * kAsmParts * 8);
  W.asm_fb = (int*)alloc(43, B * 4);
  W.live_words = (P.r_ub + 63) / 64;
  W.dense_media = insp ? 1 : 0;
  W.live = (unsigned long long*)alloc(34, B * (size_t)W.live_words * n * 8);
  // two-pass gather queue (emitter hits; overflow falls back to in-place resolution)
  // ~5% of cfg3 gather rays hit a window: room for ≥ 10% of the wave's media capacity
  W.gather_q_cap = std::min<long long>(W.media_cap, std::max<long long>(1LL << 24, W.media_cap / 10));
  if (const char* e = getenv("VOLCACHE_GATHER_QCAP")) W.gather_q_cap = std::min<long long>(W.gather_q_cap, atoll(e));
  W.gather_q = alloc(32, (size_t)W.gather_q_cap * 80);
  W.gather_q_count = (unsigned long long*)alloc(33, 16);  // [1]: the occlusion pass's fetch cursor
  W.surv_cnt = (int*)alloc(52, (size_t)B * 8);  // slots 22-30, 50-51: vc_render around its miss builds
  W.redo = W.surv_cnt + B;
  W.ray_cursor = (unsigned long long*)alloc(53, 16);
  if (err != cudaSuccess) return cuda_fail(err, "workspace allocation");

  W.outside = inside.dflag;
  KernelCounter kc;
  for (long long w0 = 0; w0 < N; w0 += B) {
    const int b = (int)std::min<long long>(B, N - w0);
    W.B = b;
    // inputs
    if (host) {
      err = cudaMemcpyAsync(dx, x + w0 * D, b * D * 8, cudaMemcpyHostToDevice, st);
      W.x = dx;
    } else {
      W.x = x + w0 * D;
    }
    if (err != cudaSuccess) return cuda_fail(err, "x upload");
    if (words) {
      const uint32_t* wsrc = (const uint32_t*)rng + w0 * prm->seed_words;
      if (host) {
        err = cudaMemcpyAsync(dwords, wsrc, (size_t)b * prm->seed_words * 4, cudaMemcpyHostToDevice, st);
        wsrc = dwords;
      }
      launch_seedseq(b, wsrc, prm->seed_words, drng, st);
      kc.launches += 1;
      W.rng = drng;
    } else if (host) {
      err = cudaMemcpyAsync(drng, (const uint64_t*)rng + w0 * 4, (size_t)b * 32, cudaMemcpyHostToDevice, st);
      W.rng = drng;
    } else {
      W.rng = (const uint64_t*)rng + w0 * 4;
    }
    if (err != cudaSuccess) return cuda_fail(err, "rng upload");
    if (P.host_adjacency) {
      const size_t tb = (size_t)b * P.n_tris * 12;
      err = cudaMemcpyAsync(W.tris, adjacency + w0 * P.n_tris * 3, tb,
                            host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st);
      if (err != cudaSuccess) return cuda_fail(err, "adjacency upload");
    }
    W.moments = (host || !moments) ? dmom : moments + w0 * 2 * MS;
    W.stats = (host || !stats) ? dstat : (long long*)stats + w0 * kStats;
    W.records = (host || !records) ? drec : records + w0 * 2 * RS;
    launch_wave(S, P, W, jt, own, own_cnt, sc->sm_count, st, &kc);
    err = cudaGetLastError();
    if (err != cudaSuccess) return cuda_fail(err, "record-build launch");
    if (host) {
      if (moments) err = cudaMemcpyAsync(moments + w0 * 2 * MS, W.moments, b * 2 * MS * 8, cudaMemcpyDeviceToHost, st);
      if (err == cudaSuccess && stats)
        err = cudaMemcpyAsync(stats + w0 * kStats, W.stats, b * kStats * 8, cudaMemcpyDeviceToHost, st);
      if (err == cudaSuccess && records)
        err = cudaMemcpyAsync(records + w0 * 2 * RS, W.records, b * 2 * RS * 8, cudaMemcpyDeviceToHost, st);
      if (err != cudaSuccess) return cuda_fail(err, "result download");
    }
    if (insp) {
      err = cudaStreamSynchronize(st);
      if (err != cudaSuccess) return cuda_fail(err, "inspect sync");
      if (insp->dirs) cudaMemcpy(insp->dirs, W.dirs, (size_t)n * D * 8, cudaMemcpyDeviceToHost);
      if (insp->s) cudaMemcpy(insp->s, W.s, (size_t)n * 8, cudaMemcpyDeviceToHost);
      if (insp->idx) cudaMemcpy(insp->idx, W.idx, (size_t)n * 4, cudaMemcpyDeviceToHost);
      if (insp->counts) cudaMemcpy(insp->counts, W.cnt, (size_t)n * 4, cudaMemcpyDeviceToHost);
      if (insp->tris && D == 3) cudaMemcpy(insp->tris, W.tris, (size_t)P.n_tris * 12, cudaMemcpyDeviceToHost);
      long long base[2];
      cudaMemcpy(base, W.rec_base, 16, cudaMemcpyDeviceToHost);
      long long Pn = base[1] - base[0];
      if (insp->P) *insp->P = Pn;
      if (insp->media && insp->media_cap > 0)
        cudaMemcpy(insp->media, W.media, (size_t)std::min<long long>(Pn, insp->media_cap) * 12,
                   cudaMemcpyDeviceToHost);
      err = cudaGetLastError();
      if (err != cudaSuccess) return cuda_fail(err, "inspect copy");
    }
  }
  g_launches += kc.launches;
  if (!host && (prm->flags & VC_DEFER_CHECK)) {
    if (const int rc = check_defer(&inside, st)) return rc;
  } else if (const int rc = check_end(&inside)) {
    return rc;
  }
  if (host) {
    err = cudaStreamSynchronize(st);
    if (err != cudaSuccess) return cuda_fail(err, "record build");
    if (stats && D == 3)
      for (int i = 0; i < N; ++i)
        if (stats[(size_t)i * kStats + 5] != 0)
          return fail(VC_ETRI, "spherical Delaunay triangulation failed for record " + std::to_string(i));
  }
  return VC_OK;
}

}  // namespace vc

using namespace vc;

struct vc_scene_deleter {};

extern "C" {

int vc_version(void) { return 1; }

const char* vc_last_error(void) { return g_err.c_str(); }

int64_t vc_kernel_launches(void) { return (int64_t)g_launches.load(); }

int vc_profile(int on) {
  for (auto& r : g_prof.recs) {
    g_prof.pool.push_back(r.a);
    g_prof.pool.push_back(r.b);
  }
  g_prof.recs.clear();
  g_prof.open.clear();
  g_prof.on = on != 0;
  return VC_OK;
}

int vc_profile_read(double* ms, int64_t* launches, int max_classes) {
  const int n = std::min<int>(max_classes, KC_COUNT);
  for (int k = 0; k < n; ++k) {
    ms[k] = 0.0;
    launches[k] = 0;
  }
  for (auto& r : g_prof.recs) {
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e != cudaSuccess) return cuda_fail(e, "profile sync");
    float t = 0.0f;
    cudaEventElapsedTime(&t, r.a, r.b);
    if (r.kc < n) {
      ms[r.kc] += t;
      launches[r.kc] += 1;
    }
  }
  return KC_COUNT;
}

// Emitter plane grids (3D): triangles grouped by plane (normals and offsets equal to
// 1e-9, every vertex within 1e-9·scale of the group plane), at most kEmitPlanes groups;
// per group a grid of cells 1/16 of the mean triangle box over the triangles'
// in-plane boxes, each padded by 1e-5·scale — far beyond the distance (≤ 1e-6·scale for
// rays at ≥ 1e-3 of grazing) between the plane point a ray lands on and the point of a
// triangle the float64 hit test accepts.  Returns false when the emitters need more planes,
// or when an emitter vertex lies outside the bounds padded by 0.005·scale: the grid walk
// skips landings beyond 1.01·scale (any hit from a point of the medium on an emitter inside
// the bounds is nearer), and the float32 gather pre-filter's error bounds assume plane
// offsets and grid origins of magnitude ≲ scale about the bounds centre.
static bool build_emit_planes(const std::vector<double>& prim, const std::vector<int>& order, double scale,
                              const double* bmin, const double* bmax, vc::EmitPlanes* ep,
                              std::vector<int>* start, std::vector<int>* tri, std::vector<unsigned>* occ) {
  using vc::kEmitPlanes;
  *ep = vc::EmitPlanes{};
  const int K = (int)order.size();
  if (K == 0) return false;
  for (int k = 0; k < K; ++k) {
    const double* P = &prim[(size_t)order[k] * 9];
    for (int v = 0; v < 3; ++v)
      for (int a = 0; a < 3; ++a) {
        const double x = P[a] + (v == 1 ? P[3 + a] : 0.0) + (v == 2 ? P[6 + a] : 0.0);
        if (!(x >= bmin[a] - 5e-3 * scale && x <= bmax[a] + 5e-3 * scale)) return false;
      }
  }
  std::vector<int> grp(K);
  int ng = 0;
  for (int k = 0; k < K; ++k) {
    const double* P = &prim[(size_t)order[k] * 9];
    const double* e1 = P + 3;
    const double* e2 = P + 6;
    double nv[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
    const double nn = std::sqrt(nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2]);
    if (!(nn > 0.0)) return false;
    int big = 0;
    for (int a = 0; a < 3; ++a) {
      nv[a] /= nn;
      if (std::fabs(nv[a]) > std::fabs(nv[big])) big = a;
    }
    if (nv[big] < 0.0)
      for (int a = 0; a < 3; ++a) nv[a] = -nv[a];
    const double c = nv[0] * P[0] + nv[1] * P[1] + nv[2] * P[2];
    int g = -1;
    for (int h = 0; h < ng && g < 0; ++h) {
      bool same = std::fabs(c - ep->c[h]) <= 1e-9 * scale;
      for (int a = 0; a < 3; ++a) same &= std::fabs(nv[a] - ep->n[h][a]) <= 1e-9;
      for (int v = 0; v < 3 && same; ++v) {  // every vertex on the group plane
        double x[3];
        for (int a = 0; a < 3; ++a) x[a] = P[a] + (v == 1 ? P[3 + a] : 0.0) + (v == 2 ? P[6 + a] : 0.0);
        same &= std::fabs(ep->n[h][0] * x[0] + ep->n[h][1] * x[1] + ep->n[h][2] * x[2] - ep->c[h]) <= 1e-9 * scale;
      }
      if (same) g = h;
    }
    if (g < 0) {
      if (ng == kEmitPlanes) return false;
      g = ng++;
      for (int a = 0; a < 3; ++a) ep->n[g][a] = nv[a];
      ep->c[g] = c;
      // in-plane frame: a1 ⟂ n from the axis least aligned with n, a2 = n × a1
      double ax[3] = {0.0, 0.0, 0.0};
      ax[(big + 1) % 3] = 1.0;
      double d = ax[0] * nv[0] + ax[1] * nv[1] + ax[2] * nv[2];
      double a1[3] = {ax[0] - d * nv[0], ax[1] - d * nv[1], ax[2] - d * nv[2]};
      const double l1 = std::sqrt(a1[0] * a1[0] + a1[1] * a1[1] + a1[2] * a1[2]);
      for (int a = 0; a < 3; ++a) ep->a1[g][a] = a1[a] / l1;
      const double* u = ep->a1[g];
      ep->a2[g][0] = nv[1] * u[2] - nv[2] * u[1];
      ep->a2[g][1] = nv[2] * u[0] - nv[0] * u[2];
      ep->a2[g][2] = nv[0] * u[1] - nv[1] * u[0];
    }
    grp[k] = g;
  }
  ep->ng = ng;
  ep->axis_only = 1;
  for (int g = 0; g < ng; ++g) {
    ep->axis[g] = -1;
    for (int a = 0; a < 3; ++a)
      if (std::fabs(ep->n[g][a]) == 1.0 && ep->n[g][(a + 1) % 3] == 0.0 && ep->n[g][(a + 2) % 3] == 0.0) ep->axis[g] = a;
    if (ep->axis[g] < 0) ep->axis_only = 0;
  }
  const double pad = 1e-5 * scale;
  std::vector<double> box((size_t)K * 4);  // in-plane (x0, y0, x1, y1), padded
  for (int k = 0; k < K; ++k) {
    const double* P = &prim[(size_t)order[k] * 9];
    const int g = grp[k];
    double x0 = INFINITY, y0 = INFINITY, x1 = -INFINITY, y1 = -INFINITY;
    for (int v = 0; v < 3; ++v) {
      double x[3];
      for (int a = 0; a < 3; ++a) x[a] = P[a] + (v == 1 ? P[3 + a] : 0.0) + (v == 2 ? P[6 + a] : 0.0);
      double px = 0.0, py = 0.0;
      for (int a = 0; a < 3; ++a) {
        px += ep->a1[g][a] * x[a];
        py += ep->a2[g][a] * x[a];
      }
      x0 = std::min(x0, px); x1 = std::max(x1, px);
      y0 = std::min(y0, py); y1 = std::max(y1, py);
    }
    box[4 * k] = x0 - pad; box[4 * k + 1] = y0 - pad;
    box[4 * k + 2] = x1 + pad; box[4 * k + 3] = y1 + pad;
  }
  int ncell = 0;
  std::vector<std::vector<int>> cells;
  for (int g = 0; g < ng; ++g) {
    double x0 = INFINITY, y0 = INFINITY, x1 = -INFINITY, y1 = -INFINITY, area = 0.0;
    int cnt = 0;
    for (int k = 0; k < K; ++k)
      if (grp[k] == g) {
        x0 = std::min(x0, box[4 * k]); y0 = std::min(y0, box[4 * k + 1]);
        x1 = std::max(x1, box[4 * k + 2]); y1 = std::max(y1, box[4 * k + 3]);
        area += (box[4 * k + 2] - box[4 * k]) * (box[4 * k + 3] - box[4 * k + 1]);
        ++cnt;
      }
    // cells of ~1/16 of a triangle's box: landings between or beside the emitters meet
    // empty cells, a landing on one meets about its own pair of triangles
    const double cs = std::sqrt(std::max(area / (16.0 * cnt), 1e-30));
    const int gx = std::min(128, std::max(1, (int)std::ceil((x1 - x0) / cs)));
    const int gy = std::min(128, std::max(1, (int)std::ceil((y1 - y0) / cs)));
    ep->lo[g][0] = x0; ep->lo[g][1] = y0;
    ep->inv[g][0] = gx / (x1 - x0); ep->inv[g][1] = gy / (y1 - y0);
    ep->gx[g] = gx; ep->gy[g] = gy; ep->cell0[g] = ncell;
    cells.resize((size_t)ncell + (size_t)gx * gy);
    for (int k = 0; k < K; ++k) {
      if (grp[k] != g) continue;
      const int i0 = std::max(0, (int)std::floor((box[4 * k] - x0) * ep->inv[g][0]));
      const int i1 = std::min(gx - 1, (int)std::floor((box[4 * k + 2] - x0) * ep->inv[g][0]));
      const int j0 = std::max(0, (int)std::floor((box[4 * k + 1] - y0) * ep->inv[g][1]));
      const int j1 = std::min(gy - 1, (int)std::floor((box[4 * k + 3] - y0) * ep->inv[g][1]));
      for (int j = j0; j <= j1; ++j)
        for (int i = i0; i <= i1; ++i) cells[(size_t)ncell + (size_t)j * gx + i].push_back(k);
    }
    ncell += gx * gy;
  }
  start->assign((size_t)ncell + 1, 0);
  tri->clear();
  for (int c = 0; c < ncell; ++c) {
    (*start)[c] = (int)tri->size();
    tri->insert(tri->end(), cells[c].begin(), cells[c].end());
  }
  (*start)[ncell] = (int)tri->size();
  if (tri->empty()) tri->push_back(0);
  // coarse occupancy (blocks of fx × fy cells, ≤ 32 × 32 blocks per plane)
  occ->assign((size_t)kEmitPlanes * 32, 0u);
  for (int g = 0; g < ng; ++g) {
    const int gx = ep->gx[g], gy = ep->gy[g];
    const int fx = (gx + 31) / 32, fy = (gy + 31) / 32;
    ep->occ_w[g] = (gx + fx - 1) / fx;
    ep->occ_h[g] = (gy + fy - 1) / fy;
    ep->occ_inv[g][0] = ep->inv[g][0] / fx;
    ep->occ_inv[g][1] = ep->inv[g][1] / fy;
    for (int j = 0; j < gy; ++j)
      for (int i = 0; i < gx; ++i) {
        const int c = ep->cell0[g] + j * gx + i;
        if ((*start)[c + 1] > (*start)[c]) (*occ)[(size_t)g * 32 + j / fy] |= 1u << (i / fx);
      }
  }
  return true;
}

int vc_scene_create(int dim, int n_surfaces, const double* vertices, const double* emission,
                    const double* albedo, const double* bounds_min, const double* bounds_max,
                    double sigma_s, double sigma_a, vc_scene** out) {
  if (!out) return fail(VC_EINVAL, "null output handle");
  *out = nullptr;
  if (dim != 2 && dim != 3) return fail(VC_EINVAL, "dimensionality must be 2 or 3");
  if (n_surfaces < 0) return fail(VC_EINVAL, "negative surface count");
  if (!(sigma_s >= 0.0) || !(sigma_a >= 0.0)) return fail(VC_EINVAL, "medium coefficients must be non-negative");
  for (int a = 0; a < dim; ++a)
    if (!(bounds_max[a] > bounds_min[a])) return fail(VC_EINVAL, "bounds max must exceed min on every axis");
  vc_scene* sc = new vc_scene();
  sc->dim = dim;
  sc->K = n_surfaces;
  sc->verts.assign(vertices, vertices + (size_t)n_surfaces * dim * dim);
  sc->emission.assign(emission, emission + (size_t)n_surfaces * 3);
  sc->albedo.assign(albedo, albedo + (size_t)n_surfaces * 3);
  double sq = 0.0;
  for (int a = 0; a < 3; ++a) {
    sc->bmin[a] = a < dim ? bounds_min[a] : 0.0;
    sc->bmax[a] = a < dim ? bounds_max[a] : 0.0;
    if (a < dim) sq += (bounds_max[a] - bounds_min[a]) * (bounds_max[a] - bounds_min[a]);
  }
  sc->scale = std::sqrt(sq);
  sc->sigma_s = sigma_s;
  sc->sigma_a = sigma_a;
  sc->max_emission = 0.0;
  sc->reflective = 0;
  for (size_t i = 0; i < sc->emission.size(); ++i) sc->max_emission = std::max(sc->max_emission, sc->emission[i]);
  for (size_t i = 0; i < sc->albedo.size(); ++i)
    if (sc->albedo[i] > 0.0) sc->reflective = 1;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sc->sm_count, cudaDevAttrMultiProcessorCount, dev);
  if (sc->sm_count <= 0) sc->sm_count = 148;
  // primitives: float64 (v0, e1, e2) or (a, e), normals (src/scene.py:124-143)
  const int K = n_surfaces, ps = prim_stride(dim);
  std::vector<double> prim((size_t)K * ps), normal((size_t)K * dim);
  for (int k = 0; k < K; ++k) {
    const double* V = &sc->verts[(size_t)k * dim * dim];
    double* P = &prim[(size_t)k * ps];
    if (dim == 2) {
      P[0] = V[0];
      P[1] = V[1];
      P[2] = V[2] - V[0];
      P[3] = V[3] - V[1];
      double len = std::sqrt(P[2] * P[2] + P[3] * P[3]);
      normal[2 * k] = -P[3] / len;
      normal[2 * k + 1] = P[2] / len;
    } else {
      for (int a = 0; a < 3; ++a) {
        P[a] = V[a];
        P[3 + a] = V[3 + a] - V[a];
        P[6 + a] = V[6 + a] - V[a];
      }
      const double* e1 = P + 3;
      const double* e2 = P + 6;
      double c[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
      double nn = std::sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
      for (int a = 0; a < 3; ++a) normal[3 * k + a] = c[a] / nn;
    }
  }
  cudaError_t e = cudaSuccess;
  auto up = [&](void** dst, const void* src, size_t bytes) {
    if (e != cudaSuccess) return;
    if (bytes == 0) bytes = 8;
    e = cudaMalloc(dst, bytes);
    if (e == cudaSuccess && src) e = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
  };
  // a primitive subset (original ids `ids`) → BVH (when large enough) + leaf-order prims
  // a primitive subset (original ids `ids`) → BVH (when large enough) + leaf-order prims.
  // Node boxes and the float32 primitive rows are taken relative to the bounds centre (in
  // float64, then rounded), so float32 magnitudes stay ≲ scale wherever the scene sits.
  double ctr[3] = {0, 0, 0};
  for (int a = 0; a < dim; ++a) ctr[a] = 0.5 * (sc->bmin[a] + sc->bmax[a]);
  auto up32 = [](double v) {  // float32 ≥ v
    float f = (float)v;
    return (double)f < v ? std::nextafter(f, FLT_MAX) : f;
  };
  auto make_set = [&](const std::vector<int>& ids, int bvh_min, GpuBvh& g, int leaf_max) {
    const int Ks = (int)ids.size();
    g.K = Ks;
    for (int a = 0; a < 3; ++a) g.ctr[a] = ctr[a];
    std::vector<int> order(ids);
    std::vector<unsigned char> last((size_t)std::max(Ks, 1), 0);
    HostBVH bvh;
    if (Ks > bvh_min) {
      std::vector<double> vs((size_t)Ks * dim * dim);
      for (int i = 0; i < Ks; ++i)
        for (int v = 0; v < dim; ++v)
          for (int a = 0; a < dim; ++a)
            vs[((size_t)i * dim + v) * dim + a] = sc->verts[((size_t)ids[i] * dim + v) * dim + a] - ctr[a];
      build_bvh(dim, Ks, vs.data(), 1e-5 * sc->scale, &bvh, leaf_max);
      for (int i = 0; i < Ks; ++i) order[i] = ids[bvh.order[i]];
      std::memcpy(last.data(), bvh.leaf_last, (size_t)Ks);
      g.stack_need = std::max(1, bvh.max_depth);
    }
    std::vector<double> leaf((size_t)Ks * ps);
    for (int i = 0; i < Ks; ++i) std::memcpy(&leaf[(size_t)i * ps], &prim[(size_t)order[i] * ps], ps * 8);
    std::vector<float4> p32((size_t)std::max(Ks, 1) * 3);
    for (int i = 0; i < Ks; ++i) {
      const double* P = &leaf[(size_t)i * ps];
      float4* q = &p32[(size_t)i * 3];
      const unsigned idf = (unsigned)order[i] | (last[i] ? 0x80000000u : 0u);
      float fid;
      std::memcpy(&fid, &idf, 4);
      if (dim == 3) {
        double r[3], vb = 0.0, E = 0.0;
        for (int a = 0; a < 3; ++a) {
          r[a] = P[a] - ctr[a];
          vb = std::max(vb, std::fabs(r[a]));
          E = std::max(E, std::max(std::fabs(P[3 + a]), std::fabs(P[6 + a])));
        }
        // tiny or non-finite edges: no pre-test (its relative error bounds assume normal floats)
        const bool pre = std::isfinite(E) && std::isfinite(vb) && E > 1e-9 * sc->scale && vb < 1e30;
        q[0] = make_float4((float)r[0], (float)r[1], (float)r[2], (float)up32(vb * (1.0 + 1e-6)));
        q[1] = make_float4((float)P[3], (float)P[4], (float)P[5], pre ? (float)up32(E * (1.0 + 1e-6)) : -1.0f);
        q[2] = make_float4((float)P[6], (float)P[7], (float)P[8], fid);
      } else {
        q[0] = make_float4((float)(P[0] - ctr[0]), (float)(P[1] - ctr[1]), 0.0f, 0.0f);
        q[1] = make_float4((float)P[2], (float)P[3], 0.0f, -1.0f);
        q[2] = make_float4(0.0f, 0.0f, 0.0f, fid);
      }
    }
    up((void**)&g.prim, Ks ? leaf.data() : nullptr, leaf.size() * 8);
    up((void**)&g.prim_id, Ks ? order.data() : nullptr, order.size() * 4);
    up((void**)&g.prim32, Ks ? p32.data() : nullptr, p32.size() * sizeof(float4));
    if (bvh.n_nodes) {
      up((void**)&g.nodes, bvh.nodes, sizeof(float4) * 4 * bvh.n_nodes);
      g.n_nodes = bvh.n_nodes;
      free_bvh(&bvh);
    }
  };
  std::vector<int> all(K), em;
  for (int k = 0; k < K; ++k) {
    all[k] = k;
    const double* E = &sc->emission[3 * (size_t)k];
    if (E[0] > 0.0 || E[1] > 0.0 || E[2] > 0.0) em.push_back(k);
  }
  auto leaf_env = [](const char* name, int dflt) {
    const char* v = getenv(name);
    return v ? atoi(v) : dflt;
  };
  make_set(all, 16, sc->geo, leaf_env("VOLCACHE_LEAF_GEO", 2));  // leaf ≤ 2: fewer float64 tests
  make_set(em, 4, sc->emit, leaf_env("VOLCACHE_LEAF_EMIT", 2));
  if (dim == 3 && !(getenv("VOLCACHE_EMIT_PLANES") && getenv("VOLCACHE_EMIT_PLANES")[0] == '0')) {
    // leaf order of the emitter set (as make_set laid it out)
    std::vector<int> eorder((size_t)sc->emit.K);
    if (sc->emit.K) cudaMemcpy(eorder.data(), sc->emit.prim_id, eorder.size() * 4, cudaMemcpyDeviceToHost);
    std::vector<int> start, tri;
    std::vector<unsigned> occ;
    if (build_emit_planes(prim, eorder, sc->scale, sc->bmin, sc->bmax, &sc->ep, &start, &tri, &occ)) {
      up((void**)&sc->d_ep_start, start.data(), start.size() * 4);
      up((void**)&sc->d_ep_tri, tri.data(), tri.size() * 4);
      up((void**)&sc->d_ep_occ, occ.data(), occ.size() * 4);
      sc->ep.cell_start = sc->d_ep_start;
      sc->ep.cell_tri = sc->d_ep_tri;
      const char* ef = getenv("VOLCACHE_EMIT_FILTER");
      sc->ep.occ = (ef && ef[0] == '0') ? nullptr : sc->d_ep_occ;
    } else {
      sc->ep.ng = 0;
    }
  }
  up((void**)&sc->d_normal, K ? normal.data() : nullptr, normal.size() * 8);
  up((void**)&sc->d_emission, K ? sc->emission.data() : nullptr, sc->emission.size() * 8);
  up((void**)&sc->d_albedo, K ? sc->albedo.data() : nullptr, sc->albedo.size() * 8);
  if (e != cudaSuccess) {
    delete sc;
    return cuda_fail(e, "scene upload");
  }
  *out = sc;
  return VC_OK;
}

void vc_scene_destroy(vc_scene* sc) { delete sc; }

int vc_scene_set_lights(vc_scene* sc, int n_lights, const double* rows) {
  if (!sc || n_lights < 0 || (n_lights > 0 && !rows)) return fail(VC_EINVAL, "invalid lights");
  for (int l = 0; l < n_lights; ++l) {
    const double* r = rows + 8 * (size_t)l;
    if (!(r[0] == 0.0 || r[0] == 1.0)) return fail(VC_EINVAL, "light kind must be 0 (point) or 1 (directional)");
    if (!(r[4] >= 0.0 && r[5] >= 0.0 && r[6] >= 0.0)) return fail(VC_EINVAL, "light strength must be non-negative");
    if (r[0] == 1.0) {
      double n2 = 0.0;
      for (int a = 0; a < sc->dim; ++a) n2 += r[1 + a] * r[1 + a];
      if (!(std::fabs(n2 - 1.0) <= 1e-12)) return fail(VC_EINVAL, "directional light vector must be unit length");
    }
  }
  cudaFree(sc->d_lights);
  sc->d_lights = nullptr;
  sc->n_lights = 0;
  if (n_lights == 0) return VC_OK;
  cudaError_t e = cudaMalloc((void**)&sc->d_lights, sizeof(double) * 8 * (size_t)n_lights);
  if (e == cudaSuccess) e = cudaMemcpy(sc->d_lights, rows, sizeof(double) * 8 * (size_t)n_lights, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "lights upload");
  sc->n_lights = n_lights;
  return VC_OK;
}

int vc_check_deferred(void* stream) { return check_deferred_read((cudaStream_t)stream); }

int vc_scene_set_budget(vc_scene* sc, int64_t bytes) {
  if (!sc || bytes <= 0) return fail(VC_EINVAL, "invalid budget");
  sc->budget = bytes;
  return VC_OK;
}

int vc_build_records(vc_scene* sc, int n_records, const double* x, const void* rng, const int32_t* adjacency,
                     const vc_build_params* params, double* moments, int64_t* stats, double* records,
                     void* stream) {
  return build_impl(sc, n_records, x, rng, adjacency, params, moments, stats, records, (cudaStream_t)stream,
                    nullptr);
}

int vc_build_inspect(vc_scene* sc, const double* x, const void* rng, const int32_t* adjacency,
                     const vc_build_params* params, double* dirs, double* s, int32_t* idx, int32_t* counts,
                     int32_t* tris, float* media, int64_t media_cap, int64_t* P, double* moments,
                     int64_t* stats) {
  if (!params) return fail(VC_EINVAL, "null params");
  vc_build_params p = *params;
  p.flags |= VC_MEM_HOST;
  Inspect in{dirs, s, idx, counts, tris, media, media_cap, P};
  return build_impl(sc, 1, x, rng, adjacency, &p, moments, stats, nullptr, 0, &in);
}

int vc_make_records(int n, int dim, const double* x, const double* moments, double epsilon, double scene_scale,
                    double max_emission, int flags, double* records, void* stream) {
  if (dim != 2 && dim != 3) return fail(VC_EINVAL, "dim must be 2 or 3");
  if (!(epsilon > 0.0)) return fail(VC_EINVAL, "epsilon must be positive");
  if (n <= 0) return VC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const bool host = flags & VC_MEM_HOST;
  const size_t MS = moment_size(dim), RS = record_size(dim);
  DevScene S{};
  S.dim = dim;
  S.scale = scene_scale;
  S.max_emission = max_emission;
  BuildParams P{};
  P.epsilon = epsilon;
  P.anisotropic = (flags & VC_ISOTROPIC) ? 0 : 1;
  Wave W{};
  W.B = n;
  cudaError_t e = cudaSuccess;
  double *dx = nullptr, *dm = nullptr, *dr = nullptr;
  if (host) {
    e = cudaMalloc(&dx, (size_t)n * dim * 8);
    if (e == cudaSuccess) e = cudaMalloc(&dm, (size_t)n * 2 * MS * 8);
    if (e == cudaSuccess) e = cudaMalloc(&dr, (size_t)n * 2 * RS * 8);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dx, x, (size_t)n * dim * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dm, moments, (size_t)n * 2 * MS * 8, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "make_records staging");
    W.x = dx;
    W.moments = dm;
    W.records = dr;
  } else {
    W.x = x;
    W.moments = const_cast<double*>(moments);
    W.records = records;
  }
  launch_make_records(S, P, W, st);
  count_launches(1);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "make_records launch");
  if (host) {
    e = cudaMemcpyAsync(records, dr, (size_t)n * 2 * RS * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(dx);
    cudaFree(dm);
    cudaFree(dr);
    if (e != cudaSuccess) return cuda_fail(e, "make_records download");
  }
  return VC_OK;
}

int vc_trace(vc_scene* sc, int m, const double* o, const double* d, double* t, int32_t* idx, int flags,
             void* stream) {
  if (!sc) return fail(VC_EINVAL, "null scene");
  if (m <= 0) return VC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const bool host = flags & VC_MEM_HOST;
  const int D = sc->dim;
  const double* dO = o;
  const double* dD = d;
  double* dt = t;
  int* di = idx;
  void* buf = nullptr;
  cudaError_t e = cudaSuccess;
  if (host) {
    e = cudaMalloc(&buf, (size_t)m * (2 * D * 8 + 12));
    if (e != cudaSuccess) return cuda_fail(e, "trace staging");
    double* b = (double*)buf;
    dO = b;
    dD = b + (size_t)m * D;
    dt = b + (size_t)2 * m * D;
    di = (int*)(b + (size_t)2 * m * D + m);
    e = cudaMemcpyAsync((void*)dO, o, (size_t)m * D * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync((void*)dD, d, (size_t)m * D * 8, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "trace upload");
  }
  launch_trace(dev_scene(sc), m, dO, dD, dt, di, (flags & VC_TRACE_BOUNDS) ? 1 : 0, st);
  g_launches += 1;
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "trace launch");
  if (host) {
    e = cudaMemcpyAsync(t, dt, (size_t)m * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(idx, di, (size_t)m * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(buf);
    if (e != cudaSuccess) return cuda_fail(e, "trace download");
  }
  return VC_OK;
}

int vc_surface_radiance(vc_scene* sc, int m, const double* points, const double* dirs, const int32_t* idx,
                        int n_light_samples, double* out, int flags, void* stream) {
  if (!sc) return fail(VC_EINVAL, "null scene");
  if (n_light_samples < 1) return fail(VC_EINVAL, "n_light_samples must be >= 1");
  if (m <= 0) return VC_OK;
  int rc = ensure_emitters(sc, n_light_samples);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const bool host = flags & VC_MEM_HOST;
  const int D = sc->dim;
  const double *dp = points, *dd = dirs;
  const int* di = idx;
  double* dout = out;
  void* buf = nullptr;
  cudaError_t e = cudaSuccess;
  if (host) {
    e = cudaMalloc(&buf, (size_t)m * (2 * D * 8 + 24 + 8));
    if (e != cudaSuccess) return cuda_fail(e, "surface radiance staging");
    double* b = (double*)buf;
    dp = b;
    dd = b + (size_t)m * D;
    dout = b + (size_t)2 * m * D;
    di = (const int*)(b + (size_t)2 * m * D + 3 * (size_t)m);
    e = cudaMemcpyAsync((void*)dp, points, (size_t)m * D * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync((void*)dd, dirs, (size_t)m * D * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync((void*)di, idx, (size_t)m * 4, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) {
      cudaFree(buf);
      return cuda_fail(e, "surface radiance upload");
    }
  }
  launch_surface_radiance(dev_scene(sc), m, dp, dd, di, dout, st);
  g_launches += 1;
  e = cudaGetLastError();
  if (e == cudaSuccess && host) {
    e = cudaMemcpyAsync(out, dout, (size_t)m * 24, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  cudaFree(buf);
  return e == cudaSuccess ? VC_OK : cuda_fail(e, "surface radiance");
}

int vc_seed_states(int n, const uint32_t* words, int nw, uint64_t* states) {
  if (n < 0 || nw < 1 || nw > 16) return fail(VC_EINVAL, "seed words per record must be in [1, 16]");
  for (int i = 0; i < n; ++i) seedseq_pcg64(words + (size_t)i * nw, nw, states + (size_t)i * 4);
  return VC_OK;
}

}  // extern "C"
