// Record-build kernels: one wave of B cache points → moments (+ records).
//
// Pipeline per wave (reference: estimate_moments, src/subdivision.py:136-393):
//   k_primary    thread per (record, direction): PCG64 jitter → stratified direction,
//                nearest hit (BVH, float64 decision), surface radiance (+shadow rays)
//   k_rings      CTA per record: R = ⌊max s/step + ½⌋, live-ring counts, exclusive prefix
//   k_wave_scan  single CTA: media-sample offsets across the wave
//   k_gather     grid-stride over media samples: PCG64 jump to the sample's draws,
//                gather ray, σs·mean T·L_o  (src/transport.py:288-310)
//   k_delaunay   thread per direction (3D): spherical Voronoi cell by half-space
//                clipping with a security radius → canonical Delaunay triangles
//   k_own_scan + k_tri_scatter: owned triangles in point order → triangle list
//   k_assemble   CTA per record: ring elements with live representative vertex are
//                queued per warp (ballot compaction) and evaluated 32 at a time;
//                moments summed with shuffles + shared-memory tree, no atomics
//   k_make_record thread per (record, kind): eigen + radii (src/cache.py:146-189)
#include <cfloat>
#include <type_traits>
#include <cstdio>
#include <vector>
#include <mutex>

#include "vc_device.cuh"
#include "vc_eigen.cuh"
#include "vc_build.h"

namespace vc {

// ---------------------------------------------------------------------------
// Directions + primary rays
// ---------------------------------------------------------------------------

#ifndef VC_LB_TRACE
#define VC_LB_TRACE 3  // min resident 256-thread CTAs per SM for the ray kernels
#endif
// the BVH-latency-bound kernels run better at 4 CTAs (≤ 64 registers): primary 1.92 →
// 1.64 ms, occlusion 1.70 → 1.48 ms per 512 records
#ifndef VC_PRIMARY_BS
#define VC_PRIMARY_BS 128  // threads per k_primary CTA: 5.44 ms per 2048 records vs 5.77 at 256 (a CTA frees its slots when its slowest warp ends; 64: 5.43, 32: 5.50)
#endif
#ifndef VC_LB_PRIMARY
#define VC_LB_PRIMARY 4
#endif
#ifndef VC_LB_OCCL
#define VC_LB_OCCL 4
#endif
// the emitter pass, since its float32 pre-filter: 4 CTAs (64 registers) 1.99 ms vs 3 CTAs
// 2.05 ms vs 2 CTAs 2.43 ms per 512 records
#ifndef VC_EMIT_BS
#define VC_EMIT_BS 128  // threads per CTA of the emitter filter / fused pass (gather 11.56 vs 11.60 ms at 256)
#endif
#ifndef VC_EVAL_BS
#define VC_EVAL_BS 128  // threads per CTA of the survivor evaluation (gather 11.55 vs 11.60 ms at 256)
#endif
#ifndef VC_EMIT_CTAS
#define VC_EMIT_CTAS 16  // 256-thread CTA equivalents per record in the emitter filter
#endif
#ifndef VC_EVAL_CTAS
#define VC_EVAL_CTAS 16  // ... and in the survivor evaluation
#endif
#ifndef VC_LB_EMIT
#define VC_LB_EMIT 4
#endif

// Thread → direction map: each warp takes a 4-row × 8-column tile of the stratum grid
// (≈7°×11° at the equator) instead of 32 columns of one row (≈2°×45°), so the lanes'
// rays and cells are spatially coherent.  Falls back to row-major when the grid does
// not tile.
#ifndef VC_TILE_R
#define VC_TILE_R 4  // stratum rows per warp tile (VC_TILE_R × 32/VC_TILE_R); 4×8: 1.65 ms, 2×16: 1.71, 8×4: 1.69 per 512 records
#endif
__device__ __forceinline__ int tiled_direction(int t, const BuildParams& P) {
  constexpr int TR = VC_TILE_R, TC = 32 / VC_TILE_R;
  if ((P.rows % TR) || (P.cols % TC) || P.rows == 1) return t;
  const int tile = t >> 5, lane = t & 31;
  const int tiles_per_row = P.cols / TC;
  const int tr = tile / tiles_per_row, tc = tile - tr * tiles_per_row;
  return (tr * TR + lane / TC) * P.cols + tc * TC + lane % TC;
}

// VC_SMEM_STACK: BVH traversal stacks in dynamic shared memory (DevBvh::stack_need entries
// per thread) instead of per-thread local arrays.  Measured per 2048-record wave (r2): shared
// 7.77 ms primary / 14.02 ms gather vs local 6.15 / 13.45 — the 40 KB-per-CTA carve-out
// shrinks the L1 that caches BVH nodes and primitives, which costs more than the local
// stack traffic it removes (the stack's live lines stay in L1 anyway)
#ifndef VC_SMEM_STACK
#define VC_SMEM_STACK 0
#endif
#if VC_SMEM_STACK
#define VC_RAY_STACK                     \
  extern __shared__ uint2 trav_stack[]; \
  SharedStack<256> stk{trav_stack + threadIdx.x}
#else
#define VC_RAY_STACK LocalStack stk
#endif

// REFL = false (no surface reflects): L_o is the emission, so the direct-lighting code —
// shadow rays through a second inlined BVH traversal — is not compiled into the kernel
// (its register demand made the traversal spill: 308 → 16 bytes of spill stores).
template <int D, bool REFL>
__global__ void __launch_bounds__(VC_PRIMARY_BS, VC_LB_PRIMARY * 256 / VC_PRIMARY_BS)
    k_primary(DevScene S, BuildParams P, Wave W, JumpTables jt) {
  VC_RAY_STACK;
  const int n = P.n_angular;
  long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)W.B * n) return;
  int rec = (int)(gid / n);
  int k = tiled_direction((int)(gid - (long long)rec * n), P);
  Pcg64 g0 = pcg_load(W.rng + 4 * rec);
  double d[3], o[3];
  stratum_direction<D>(k, P, g0, jt, d);
#pragma unroll
  for (int a = 0; a < D; ++a) o[a] = W.x[rec * D + a];
  double s;
  int id;
  trace_or_bounds<D>(S, o, d, s, id, &stk);
  double hit[3];
#pragma unroll
  for (int a = 0; a < D; ++a) hit[a] = add(o[a], mul(s, d[a]));
  double L[3];
  if constexpr (REFL) {
    surface_radiance<D>(S, id, hit, d, L, &stk);
  } else {  // surface_radiance of a non-reflective scene (src/transport.py:240-254)
    L[0] = L[1] = L[2] = 0.0;
    if (id >= 0) {
      const double* E = S.emission + (size_t)id * 3;
      L[0] = E[0];
      L[1] = E[1];
      L[2] = E[2];
    }
  }
  size_t base = (size_t)rec * n + k;
#pragma unroll
  for (int a = 0; a < D; ++a) W.dirs[base * D + a] = d[a];
  if constexpr (D == 3) W.dirs32[base] = make_float4((float)d[0], (float)d[1], (float)d[2], 0.0f);
  W.s[base] = s;
  W.idx[base] = id;
  if (REFL || !W.emit_tab) {  // (non-reflective: the readers take emission[idx] themselves)
    W.lo[base * 3 + 0] = L[0];
    W.lo[base * 3 + 1] = L[1];
    W.lo[base * 3 + 2] = L[2];
  }
}

// Persistent-lane primary pass (non-reflective scenes with a BVH; VC_PRIMARY_PT): the
// directions first (thread per direction), then every lane owns one primary ray at a time
// and advances its nearest-hit traversal leaf by leaf, fetching the next ray index (tile
// order) through a warp-aggregated cursor when its ray is done.  Same traversal, culling
// and (t, index) decision per ray as trace_or_bounds; the results do not depend on the
// schedule.  Off: 6.03 ms vs 5.77 ms per 2048 records for the thread-per-direction kernel
// (lane efficiency 15.4/32 — the tiled primary rays are coherent, fetching breaks that).
#ifndef VC_PRIMARY_PT
#define VC_PRIMARY_PT 0
#endif
template <int D>
__global__ void __launch_bounds__(256) k_directions(BuildParams P, Wave W, JumpTables jt) {
  const int n = P.n_angular;
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)W.B * n) return;
  const int rec = (int)(gid / n);
  const int k = (int)(gid - (long long)rec * n);
  Pcg64 g0 = pcg_load(W.rng + 4 * rec);
  double d[3];
  stratum_direction<D>(k, P, g0, jt, d);
  const size_t base = (size_t)rec * n + k;
#pragma unroll
  for (int a = 0; a < D; ++a) W.dirs[base * D + a] = d[a];
  if constexpr (D == 3) W.dirs32[base] = make_float4((float)d[0], (float)d[1], (float)d[2], 0.0f);
}

template <int D>
__global__ void __launch_bounds__(256, VC_LB_PRIMARY) k_primary_pt(DevScene S, BuildParams P, Wave W,
                                                                 unsigned long long* cursor) {
  const int n = P.n_angular;
  const long long total = (long long)W.B * n;
  const DevBvh& H = S.geo;
  const int lane = threadIdx.x & 31;
  const float slack = 1e-5f * (float)S.scale;
  auto tlim = [&](double t) { return isfinite(t) ? __double2float_ru(t) * 1.0001f + slack : INFINITY; };
  LocalStack stk;
  long long ray = -1;
  bool exhausted = false;
  double o[3] = {0, 0, 0}, d[3] = {0, 0, 0}, t_best = INFINITY;
  int id_best = -1;
  float2 inv2[3], noi2[3];
  float tbf = INFINITY;
  int sp = 0;
  unsigned cur = 0;
  size_t base = 0;
  auto finish = [&]() {
    double s = isfinite(t_best) ? t_best : bounds_exit<D>(S, o, d);
    W.s[base] = s;
    W.idx[base] = id_best;
    double L[3] = {0.0, 0.0, 0.0};  // surface_radiance of a non-reflective scene: the emission
    if (id_best >= 0) {
      const double* E = S.emission + (size_t)id_best * 3;
      L[0] = E[0];
      L[1] = E[1];
      L[2] = E[2];
    }
    W.lo[base * 3 + 0] = L[0];
    W.lo[base * 3 + 1] = L[1];
    W.lo[base * 3 + 2] = L[2];
    ray = -1;
  };
  auto pop = [&]() -> bool {
    while (sp > 0) {
      const uint2 e = stk.get(--sp);
      if (__uint_as_float(e.y) <= tbf) {
        cur = e.x;
        return true;
      }
    }
    return false;
  };
  while (true) {
    const bool need = ray < 0 && !exhausted;
    const unsigned mneed = __ballot_sync(0xffffffffu, need);
    if (mneed) {
      const int leader = __ffs(mneed) - 1;
      unsigned long long b0 = 0;
      if (lane == leader) b0 = atomicAdd(cursor, (unsigned long long)__popc(mneed));
      b0 = __shfl_sync(0xffffffffu, b0, leader);
      if (need) {
        const long long g = (long long)b0 + __popc(mneed & ((1u << lane) - 1u));
        if (g >= total) {
          exhausted = true;
        } else {
          ray = g;
          const int rec = (int)(g / n);
          const int k = tiled_direction((int)(g - (long long)rec * n), P);
          base = (size_t)rec * n + k;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            o[a] = a < D ? W.x[rec * D + a] : 0.0;
            d[a] = a < D ? W.dirs[base * D + a] : 0.0;
            float inv = 0.0f, noi = 0.0f;
            if (a < D) {
              const float orl = (float)(o[a] - H.ctr[a]);
              asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"((float)d[a]));
              noi = -orl * inv;
            }
            inv2[a] = make_float2(inv, inv);
            noi2[a] = make_float2(noi, noi);
          }
          t_best = INFINITY;
          id_best = -1;
          tbf = INFINITY;
          sp = 0;
          cur = 0;
        }
      }
    }
    if (!__any_sync(0xffffffffu, ray >= 0)) {
      if (__all_sync(0xffffffffu, exhausted)) break;
      continue;
    }
    if (ray >= 0) {  // one step: descend to the next leaf, test it
      bool alive = true;
      while (!(cur & 0x80000000u)) {
        const float4* N = H.nodes + 4 * (size_t)cur;
        const float4 A = __ldg(N), B = __ldg(N + 1), C = __ldg(N + 2), R = __ldg(N + 3);
        float tl, tr;
        bool hl, hr;
        box_hit2<D>(A, B, C, inv2, noi2, tbf, hl, hr, tl, tr);
        if (hl && hr) {
          const bool lf = tl <= tr;
          stk.put(sp++, make_uint2(__float_as_uint(lf ? R.z : R.x), __float_as_uint(lf ? tr : tl)));
          cur = __float_as_uint(lf ? R.x : R.z);
        } else if (hl || hr) {
          cur = __float_as_uint(hl ? R.x : R.z);
        } else if (!pop()) {
          alive = false;
          break;
        }
      }
      if (alive) {
        for (int k = (int)(cur & 0x7fffffffu);; ++k) {
          const int idf = __float_as_int(__ldg(&H.prim32[3 * (size_t)k + 2].w));
          const double t = hit_prim<D>(H.prim + (size_t)k * prim_stride(D), o, d, S.t_eps);
          if (t != INFINITY) {
            const int id = idf & 0x7fffffff;
            if (t < t_best || (t == t_best && id < id_best)) {
              t_best = t;
              id_best = id;
              tbf = tlim(t_best);
            }
          }
          if (idf < 0) break;
        }
        if (!pop()) finish();
      } else {
        finish();
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Ring counts (src/subdivision.py:172-176)
// ---------------------------------------------------------------------------

__device__ __forceinline__ double ring_radius(int i, double step) {
  // (np.arange(1, R+1) − 0.5)·step, element i (0-based)
  return mul((double)(i + 1) - 0.5, step);
}

__device__ __forceinline__ int live_rings(double s, int R, double step) {
  double est = floor(__ddiv_rn(s, step) + 0.5);
  int c = (int)fmin(fmax(est, 0.0), (double)R);
  while (c > 0 && !(ring_radius(c - 1, step) < s)) --c;
  while (c < R && ring_radius(c, step) < s) ++c;
  return c;
}

template <int BS>
__device__ inline long long block_exscan(long long v, long long& total, long long* sm) {
  // sm: BS/32 + 1 entries
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm[wid] = x;
  __syncthreads();
  if (wid == 0) {
    long long w = (lane < BS / 32) ? sm[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < BS / 32) sm[lane] = w;
  }
  __syncthreads();
  long long pre = (wid > 0 ? sm[wid - 1] : 0) + x - v;
  total = sm[BS / 32 - 1];
  __syncthreads();
  return pre;
}

#ifndef VC_GATHER_RUN
#define VC_GATHER_RUN 16
#endif
constexpr int kGatherRun = VC_GATHER_RUN;  // consecutive samples per thread in pass 1
static_assert(kGatherRun == 16, "run table stride (vc_api.cu)");

constexpr int kRingBS = 512;

__global__ void __launch_bounds__(kRingBS) k_rings(BuildParams P, Wave W) {
  __shared__ long long sm[kRingBS / 32 + 1];
  __shared__ double smax[kRingBS / 32];
  const int rec = blockIdx.x, n = P.n_angular;
  const double* s = W.s + (size_t)rec * n;
  double mx = 0.0;
  for (int k = threadIdx.x; k < n; k += kRingBS) mx = fmax(mx, s[k]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) smax[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < kRingBS / 32 ? smax[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) smax[0] = v;
  }
  __syncthreads();
  const double max_s = smax[0];
  // a wave whose points failed the device bounds check does no ring work (the call fails);
  // R ≤ r_ub − 2 holds for every point inside the bounds
  const int R = (W.outside && *W.outside) ? 0 : min((int)floor(__ddiv_rn(max_s, P.march_step) + 0.5), P.r_ub);
  long long run = 0;
  int maxc = 0;
  for (int base = 0; base < n; base += kRingBS) {
    int k = base + threadIdx.x;
    int c = (k < n) ? live_rings(s[k], R, P.march_step) : 0;
    maxc = max(maxc, c);
    long long tot;
    long long pre = block_exscan<kRingBS>(c, tot, sm);
    if (k < n) {
      const size_t g = (size_t)rec * n + k;
      W.cnt[g] = c;
      W.pre[g] = (int)(run + pre);
      // gather runs (kGatherRun consecutive samples) that start in this direction
      const int j0 = (int)(run + pre);
      for (int m = (j0 + kGatherRun - 1) / kGatherRun; m * kGatherRun < j0 + c; ++m)
        W.run_dir[(size_t)rec * W.run_stride + m] = k;
      const double* lo = W.lo + g * 3;
      if (W.emit_tab) {  // non-reflective scene: the surface radiance is the hit's emission
        const int id = W.idx[g];
        lo = id >= 0 ? W.emit_tab + (size_t)id * 3 : nullptr;
      }
      DirInfo di;
      di.s = s[k];
      di.cnt = c;
      di.surf_live = (lo && (lo[0] > 0.0 || lo[1] > 0.0 || lo[2] > 0.0)) ? 1 : 0;
      W.info[g] = di;
    }
    run += tot;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) maxc = max(maxc, __shfl_xor_sync(0xffffffffu, maxc, o));
  __shared__ int smc[kRingBS / 32];
  if ((threadIdx.x & 31) == 0) smc[threadIdx.x >> 5] = maxc;
  __syncthreads();
  if (threadIdx.x == 0) {
    int m = 0;
    for (int w = 0; w < kRingBS / 32; ++w) m = max(m, smc[w]);
    W.rec_R[rec] = R;
    W.rec_P[rec] = (int)run;
    W.rec_maxc[rec] = m;
  }
}

__global__ void __launch_bounds__(1024) k_wave_scan(Wave W, int gather_on) {
  __shared__ long long sm[1024 / 32 + 1];
  long long run = 0;
  for (int base = 0; base < W.B; base += 1024) {
    int r = base + threadIdx.x;
    long long v = (r < W.B && gather_on) ? W.rec_P[r] : 0;
    long long tot;
    long long pre = block_exscan<1024>(v, tot, sm);
    if (r < W.B) W.rec_base[r] = run + pre;
    run += tot;
  }
  if (threadIdx.x == 0) W.rec_base[W.B] = run;
}

// ---------------------------------------------------------------------------
// Media-sample gather (src/subdivision.py:177-195, src/transport.py:288-310)
// ---------------------------------------------------------------------------

// Live-sample bit of media sample (k, ring) of record rec (read by the assembly scan);
// set by whoever computes a positive radiance, on masks zeroed before the gather.
__device__ __forceinline__ void mark_live(const Wave& W, int n, int rec, int k, int ring) {
  unsigned long long* w = W.live + ((size_t)rec * W.live_words + (ring >> 6)) * n + k;
  atomicOr(w, 1ULL << (ring & 63));
}

// Extension helpers (oracle hg_phase / hg_sample, same float64 operation order).
__device__ __forceinline__ double hg_phase(double g, double c) {
  const double num = sub(1.0, mul(g, g));
  const double b = sub(add(1.0, mul(g, g)), mul(mul(2.0, g), c));
  return __ddiv_rn(num, mul(4.0 * kPi, pow(b, 1.5)));
}

// cd ← a direction about cd with cos θ ~ HG(g) from u0, azimuth 2π·u1 (Duff et al. basis)
__device__ __forceinline__ void hg_sample(double g, double* cd, double u0, double u1) {
  const double s = __ddiv_rn(sub(1.0, mul(g, g)), add(sub(1.0, g), mul(mul(2.0, g), u0)));
  const double ct = __ddiv_rn(sub(add(1.0, mul(g, g)), mul(s, s)), mul(2.0, g));
  const double st = sqrt(fmax(0.0, sub(1.0, mul(ct, ct))));
  const double phi = mul(2.0 * kPi, u1);
  const double x = cd[0], y = cd[1], z = cd[2];
  const double sg = copysign(1.0, z);
  const double a = __ddiv_rn(-1.0, add(sg, z));
  const double b = mul(mul(x, y), a);
  const double t1[3] = {add(1.0, mul(mul(mul(sg, x), x), a)), mul(sg, b), mul(-sg, x)};
  const double t2[3] = {b, add(sg, mul(mul(y, y), a)), -y};
  const double ca = mul(st, cos(phi)), sa = mul(st, sin(phi));
#pragma unroll
  for (int c = 0; c < 3; ++c) cd[c] = add(add(mul(ca, t1[c]), mul(sa, t2[c])), mul(ct, cd[c]));
}

// Extension (oracle delta_inscatter): mean incident radiance over the sphere (circle) at a
// media point from the delta lights, Σ_l term_l·I_l / 4π (2π); g ≠ 0 weighs each light by
// 4π·p_g(d_l·toward).
template <int D>
__device__ inline void delta_inscatter(const DevScene& S, const double* p, double g, const double* toward,
                                       double out[3]) {
  out[0] = out[1] = out[2] = 0.0;
  const double norm = (D == 3) ? 4.0 * kPi : 2.0 * kPi;
  for (int l = 0; l < S.n_lights; ++l) {
    const double* L8 = S.lights + 8 * (size_t)l;
    double d[3];
    const double val = delta_term<D>(S, L8, p, d);
    if (!(val > 0.0)) continue;
    double w = __ddiv_rn(val, norm);
    if (g != 0.0)
      w = mul(w, mul(4.0 * kPi, hg_phase(g, add(add(mul(d[0], toward[0]), mul(d[1], toward[1])),
                                                  mul(d[2], toward[2])))));
    out[0] = add(out[0], mul(w, L8[4]));
    out[1] = add(out[1], mul(w, L8[5]));
    out[2] = add(out[2], mul(w, L8[6]));
  }
}

template <int D>
__global__ void __launch_bounds__(256, VC_LB_TRACE) k_gather(DevScene S, BuildParams P, Wave W, JumpTables jt) {
  const long long total = W.rec_base[W.B];
  const int n = P.n_angular;
  const long long draws0 = (D == 3) ? 2LL * P.rows * P.cols : (long long)n;
  const int per = (D == 3 ? 2 : 1) * P.n_inner;
  const int nb = P.media_bounces - 1;  // extension: further media events per gather path
  const double hg = (D == 3) ? P.hg_g : 0.0;  // extension: Henyey–Greenstein media
  const bool emitter_first = !S.reflective && 2 * S.emit.K <= S.geo.K && nb == 0 && hg == 0.0;
  const double albedo = S.sigma_t > 0.0 ? __ddiv_rn(S.sigma_s, S.sigma_t) : 0.0;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < total;
       j += (long long)gridDim.x * blockDim.x) {
    // record: last r with base[r] ≤ j
    int lo = 0, hi = W.B - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (W.rec_base[mid] <= j) lo = mid; else hi = mid - 1;
    }
    const int rec = lo;
    const int jl = (int)(j - W.rec_base[rec]);
    const int* pre = W.pre + (size_t)rec * n;
    int a = 0, b = n - 1;
    while (a < b) {
      int mid = (a + b + 1) >> 1;
      if (pre[mid] <= jl) a = mid; else b = mid - 1;
    }
    const int k = a, i = jl - pre[k];
    const double ri = ring_radius(i, P.march_step);
    double y[3], dk[3];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      dk[c] = W.dirs[((size_t)rec * n + k) * D + c];
      y[c] = add(W.x[rec * D + c], mul(ri, dk[c]));
    }
    Pcg64 g = pcg_load(W.rng + 4 * rec);
    pcg_advance(g, (unsigned long long)(draws0 + (long long)per * jl), jt);
    double acc[3] = {0.0, 0.0, 0.0};
    for (int t = 0; t < P.n_inner; ++t) {
      double gd[3];
      if constexpr (D == 2) {
        double th = mul(2.0 * kPi, g.next_double());
        gd[0] = cos(th);
        gd[1] = sin(th);
      } else {
        double u0 = g.next_double(), u1 = g.next_double();
        double z = sub(1.0, mul(2.0, u0));
        double phi = mul(2.0 * kPi, u1);
        double sq = sqrt(fmax(sub(1.0, mul(z, z)), 0.0));
        gd[0] = mul(sq, cos(phi));
        gd[1] = mul(sq, sin(phi));
        gd[2] = z;
      }
      double s2;
      int id2;
      if (emitter_first) {
        // Non-reflective scene: L_o(hit) = emission, so only a nearest hit on an emitter
        // carries radiance.  Find the nearest emitter, then ask the BVH whether any
        // primitive precedes it in (t, index) order — same (s2, idx2) decision as the
        // full nearest-hit search whenever the result can be non-zero.
        nearest_emitter<D>(S, y, gd, s2, id2);
        if (id2 >= 0 && occluded<D>(S, y, gd, s2, id2)) id2 = -1;
      } else {
        trace_or_bounds<D>(S, y, gd, s2, id2);
      }
      double path[3] = {0.0, 0.0, 0.0};
      if (id2 >= 0) {
        double hp[3], L[3];
#pragma unroll
        for (int c = 0; c < D; ++c) hp[c] = add(y[c], mul(s2, gd[c]));
        surface_radiance<D>(S, id2, hp, gd, L);
        double T = exp(-S.sigma_t * s2);
        path[0] = mul(T, L[0]);
        path[1] = mul(T, L[1]);
        path[2] = mul(T, L[2]);
      }
      double w0 = 1.0;
      if (hg != 0.0) {  // extension: HG scattering at y toward x (oracle gather_mean_bounces)
        double dx[3], wk[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) dx[c] = sub(y[c], W.x[rec * D + c]);
        const double nrm = sqrt(add(add(mul(dx[0], dx[0]), mul(dx[1], dx[1])), mul(dx[2], dx[2])));
#pragma unroll
        for (int c = 0; c < 3; ++c) wk[c] = __ddiv_rn(dx[c], nrm);
        w0 = mul(4.0 * kPi, hg_phase(hg, add(add(mul(gd[0], wk[0]), mul(gd[1], wk[1])), mul(gd[2], wk[2]))));
#pragma unroll
        for (int c = 0; c < 3; ++c) path[c] = mul(path[c], w0);
      }
      if (nb > 0 && S.sigma_t > 0.0) {
        // Extension: the multiple-scattering loop of path_trace_radiance (src/transport.py:
        // 362-388) from y along the gather ray — collision at −log1p(−u)/σt inside the current
        // segment, weight σs/σt, uniform new direction, T·L_o at its hit — with this path's
        // draws from the record stream after every reference draw (oracle: gather_mean_bounces)
        constexpr int pb = (D == 3) ? 3 : 2;
        Pcg64 gx = pcg_load(W.rng + 4 * rec);
        pcg_advance(gx, (unsigned long long)(draws0 + (long long)per * W.rec_P[rec] +
                                             ((long long)jl * P.n_inner + t) * nb * pb), jt);
        double pos[3] = {y[0], y[1], y[2]}, cd[3] = {gd[0], gd[1], gd[2]}, cs = s2, w = w0;
        for (int bb = 0; bb < nb; ++bb) {
          const double ud = gx.next_double();
          const double ua = gx.next_double();
          const double ub = (D == 3) ? gx.next_double() : 0.0;
          const double tc = __ddiv_rn(-log1p(-ud), S.sigma_t);
          if (!(tc < cs)) break;  // the path leaves this segment through its surface / bounds
#pragma unroll
          for (int c = 0; c < D; ++c) pos[c] = add(pos[c], mul(tc, cd[c]));
          w = mul(w, albedo);
          const double pd[3] = {cd[0], cd[1], cd[2]};  // the direction the path arrived along
          if constexpr (D == 2) {
            const double th = mul(2.0 * kPi, ua);
            cd[0] = cos(th);
            cd[1] = sin(th);
          } else if (hg != 0.0) {
            hg_sample(hg, cd, ua, ub);
          } else {
            const double z = sub(1.0, mul(2.0, ua));
            const double phi = mul(2.0 * kPi, ub);
            const double sq = sqrt(fmax(sub(1.0, mul(z, z)), 0.0));
            cd[0] = mul(sq, cos(phi));
            cd[1] = mul(sq, sin(phi));
            cd[2] = z;
          }
          int id3;
          trace_or_bounds<D>(S, pos, cd, cs, id3);
          if (id3 >= 0) {
            double hp[3], L[3];
#pragma unroll
            for (int c = 0; c < D; ++c) hp[c] = add(pos[c], mul(cs, cd[c]));
            surface_radiance<D>(S, id3, hp, cd, L);
            const double wT = mul(w, exp(-S.sigma_t * cs));
#pragma unroll
            for (int c = 0; c < 3; ++c) path[c] = add(path[c], mul(wT, L[c]));
          }
          if (S.n_lights > 0) {  // extension: the delta lights scattered at this collision
            double dl[3];
            delta_inscatter<D>(S, pos, hg, pd, dl);
#pragma unroll
            for (int c = 0; c < 3; ++c) path[c] = add(path[c], mul(w, dl[c]));
          }
        }
      }
      acc[0] = add(acc[0], path[0]);
      acc[1] = add(acc[1], path[1]);
      acc[2] = add(acc[2], path[2]);
    }
    float* out = W.media + (size_t)(W.rec_base[rec] + jl) * 3;
    bool pos = false;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double v = mul(S.sigma_s, __ddiv_rn(acc[c], (double)P.n_inner));
      float f = (float)v;
      if (v > 0.0 && !(f > 0.0f)) f = FLT_TRUE_MIN;  // keep the liveness bit exact
      out[c] = f;
      pos |= f > 0.0f;
    }
    if (pos) mark_live(W, n, rec, k, i);
  }
}

#ifndef VC_DELTA_PT
#define VC_DELTA_PT 0  // persistent-lane shadow rays for the delta lights: measured slower (221 vs 194 ms per
                       // 2048 lamp-lit cfg3 records) — the shadow rays of consecutive samples are coherent
#endif
// Extension: the delta lights' in-scatter at every live-ring media sample, added to the
// gathered radiance after either gather path (thread per sample; a sample no gather ray lit
// has an undefined row in the two-pass path, so the live bit decides add vs. write).
template <int D>
__global__ void __launch_bounds__(256) k_gather_delta(DevScene S, BuildParams P, Wave W) {
  const long long total = W.rec_base[W.B];
  const int n = P.n_angular;
  const double hg = (D == 3) ? P.hg_g : 0.0;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < total;
       j += (long long)gridDim.x * blockDim.x) {
    int lo = 0, hi = W.B - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (W.rec_base[mid] <= j) lo = mid; else hi = mid - 1;
    }
    const int rec = lo;
    const int jl = (int)(j - W.rec_base[rec]);
    const int* pre = W.pre + (size_t)rec * n;
    int a = 0, b = n - 1;
    while (a < b) {
      int mid = (a + b + 1) >> 1;
      if (pre[mid] <= jl) a = mid; else b = mid - 1;
    }
    const int k = a, i = jl - pre[k];
    const double ri = ring_radius(i, P.march_step);
    double y[3] = {0.0, 0.0, 0.0}, wk[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double dk = W.dirs[((size_t)rec * n + k) * D + c];
      y[c] = add(W.x[rec * D + c], mul(ri, dk));
    }
    if (hg != 0.0) {
      double dx[3], n2 = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        dx[c] = sub(y[c], W.x[rec * D + c]);
        n2 = add(n2, mul(dx[c], dx[c]));
      }
      const double nrm = sqrt(n2);
#pragma unroll
      for (int c = 0; c < 3; ++c) wk[c] = __ddiv_rn(dx[c], nrm);
    }
    double dl[3];
    delta_inscatter<D>(S, y, hg, wk, dl);
    if (!(dl[0] > 0.0 || dl[1] > 0.0 || dl[2] > 0.0)) continue;
    const unsigned long long word = W.live[((size_t)rec * W.live_words + (i >> 6)) * n + k];
    const bool live = (word >> (i & 63)) & 1ULL;
    float* out = W.media + (size_t)(W.rec_base[rec] + jl) * 3;
    bool pos = false;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double v = mul(S.sigma_s, dl[c]);
      float f = (float)v;
      if (v > 0.0 && !(f > 0.0f)) f = FLT_TRUE_MIN;
      f += live ? out[c] : 0.0f;
      out[c] = f;
      pos |= f > 0.0f;
    }
    if (pos && !live) mark_live(W, n, rec, k, i);
  }
}

// Extension (oracle delta_single): the delta lights' own single scattering at the cache
// point, f̄·I·φ(x)/4π (2π) with its closed-form gradient and Hessian (visibility held
// constant), added to the single moments.
template <int D>
__global__ void k_delta_single(DevScene S, Wave W) {
  const int rec = blockIdx.x * blockDim.x + threadIdx.x;
  if (rec >= W.B) return;
  if (D == 3 && W.tri_status[rec] != 0) return;
  if (W.outside && *W.outside) return;
  const double norm = (D == 3) ? 4.0 * kPi : 2.0 * kPi;
  const double c0 = S.sigma_s / norm / norm;  // f̄ / norm
  const double sig = S.sigma_t;
  constexpr int kk = D - 1;
  double x[3] = {0.0, 0.0, 0.0};
  for (int a = 0; a < D; ++a) x[a] = W.x[rec * D + a];
  double* M = W.moments + ((size_t)rec * 2) * moment_size(D);
  for (int l = 0; l < S.n_lights; ++l) {
    const double* L8 = S.lights + 8 * (size_t)l;
    double d[3];
    const double phi = delta_term<D>(S, L8, x, d);
    if (!(phi > 0.0)) continue;
    double g[3] = {0.0, 0.0, 0.0}, h[9] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (L8[0] == 0.0) {
      double w[3], r2 = 0.0;
      for (int a = 0; a < D; ++a) {
        w[a] = x[a] - L8[1 + a];
        r2 += w[a] * w[a];
      }
      const double r = sqrt(r2);
      const double a1 = sig + kk / r;
      const double d1 = -a1 * phi, d2 = (a1 * a1 + kk / (r * r)) * phi;
      for (int a = 0; a < D; ++a) {
        const double ua = w[a] / r;
        g[a] = d1 * ua;
        for (int b = 0; b < D; ++b) {
          const double ub = w[b] / r;
          h[a * D + b] = d2 * ua * ub + d1 / r * ((a == b ? 1.0 : 0.0) - ua * ub);
        }
      }
    } else {
      int ax = 0;
      double best = 0.0;
      for (int a = 0; a < D; ++a) {
        const double t1 = (S.bmin[a] - x[a]) / d[a], t2 = (S.bmax[a] - x[a]) / d[a];
        const double far = isnan(t1) ? INFINITY : np_max(t1, t2);
        if (a == 0 || far < best) {
          best = far;
          ax = a;
        }
      }
      const double e = 1.0 / d[ax];
      g[ax] = sig * phi * e;
      h[ax * D + ax] = sig * sig * phi * e * e;
    }
    for (int c = 0; c < 3; ++c) {
      const double I = c0 * L8[4 + c];
      M[c] += I * phi;
      for (int a = 0; a < D; ++a) M[3 + c * D + a] += I * g[a];
      for (int e2 = 0; e2 < D * D; ++e2) M[3 + 3 * D + c * D * D + e2] += I * h[e2];
    }
  }
}

// Two-pass gather for non-reflective scenes with one gather direction per sample.
// Pass 1 (k_gather_emit): CTA rows = records, each thread walks a run of consecutive
// samples (direction found once by binary search, then advanced; PCG64 jumped once and
// stepped), tests the gather ray against the emitter BVH only, writes zero radiance
// for misses and queues emitter hits.  Pass 2 (k_gather_occl): one thread per queued
// ray runs the any-hit occlusion query on the full BVH in (t, index) order — full warps
// for the divergent traversal, and the same (s, idx) decision as a nearest-hit search.
struct GatherItem {
  double y[3], d[3], te;
  long long slot;  // media row
  int ie, rec, k, ring;
};

static_assert(sizeof(GatherItem) == 80, "queue entry layout (workspace sizing)");




__device__ __forceinline__ void store_media(float* out, const double* v) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    float f = (float)v[c];
    if (v[c] > 0.0 && !(f > 0.0f)) f = FLT_TRUE_MIN;  // keep the liveness bit exact
    out[c] = f;
  }
}

// Media radiance of an unoccluded emitter hit in the two-pass gather: σs · T · L_o / n_inner
// with n_inner = 1 and L_o = emission (non-reflective scene); extension hg ≠ 0: the path is
// weighted 4π·p_g(d·w), w = (y − x)/|y − x| (k_gather's first-event weight).
template <int D>
__device__ __forceinline__ void emitter_radiance(const DevScene& S, const Wave& W, double hg, int rec,
                                                 const double* y, const double* d, double te, int ie, double* v) {
  const double* E = S.emission + (size_t)ie * 3;
  const double T = exp(-S.sigma_t * te);
  double w0 = 1.0;
  if (D == 3 && hg != 0.0) {
    double dx[3], n2 = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      dx[c] = sub(y[c], W.x[rec * D + c]);
      n2 = add(n2, mul(dx[c], dx[c]));
    }
    const double nrm = sqrt(n2);
    double cs = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) cs = add(cs, mul(d[c], __ddiv_rn(dx[c], nrm)));
    w0 = mul(4.0 * kPi, hg_phase(hg, cs));
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) v[c] = mul(S.sigma_s, mul(mul(T, E[c]), w0));
}

#ifndef VC_QCHUNK
#define VC_QCHUNK 32
#endif
constexpr int kQChunk = VC_QCHUNK;  // queue slots a warp reserves with one atomic
static_assert(kQChunk >= 32, "a step's hits (≤ 32) must fit one fresh chunk");

// Could the gather ray with draws (u0, u1) from y reach an emitter?  False only when
// every emitter plane is axis-aligned and the ray certainly moves away from each of them
// (the sign of the direction's axis component follows from u0 or u1 alone:
// d = (√(1−z²)·cos 2πu1, √(1−z²)·sin 2πu1, 1 − 2u0)); a hit needs the landing distance
// (c − n·y)/(n·d) above −1e-5·scale, impossible for an origin farther than that from the
// plane when n·d has the other sign.
// Per-launch constants of that test (registers; no indexing by plane or axis).
struct Toward {
  int ng;                 // 0: every ray may reach an emitter
  int ax[kEmitPlanes];    // plane axis
  double nz[kEmitPlanes]; // n_axis (±1)
  double c[kEmitPlanes];
  __device__ __forceinline__ explicit Toward(const EmitPlanes& E) {
    ng = E.axis_only ? E.ng : 0;
#pragma unroll
    for (int g = 0; g < kEmitPlanes; ++g) {
      const int a = g < E.ng ? E.axis[g] : 0;
      ax[g] = a;
      nz[g] = g < E.ng ? (a == 0 ? E.n[g][0] : (a == 1 ? E.n[g][1] : E.n[g][2])) : 1.0;
      c[g] = g < E.ng ? E.c[g] : 0.0;
    }
  }
  __device__ __forceinline__ bool operator()(const double* y, double u0, double u1, double tol) const {
    if (ng == 0) return true;
    bool any = false;
#pragma unroll
    for (int g = 0; g < kEmitPlanes; ++g) {
      if (g >= ng) break;
      const int a = ax[g];
      const double ya = a == 0 ? y[0] : (a == 1 ? y[1] : y[2]);
      const double s = c[g] - nz[g] * ya;  // c − n·y with n = ±e_a
      int sd;                              // sign of d_a (0: zero or not decided)
      if (a == 2) sd = u0 < 0.5 ? 1 : (u0 > 0.5 ? -1 : 0);
      else if (u0 == 0.0) sd = 0;
      else if (a == 0) sd = (u1 < 0.25 || u1 > 0.75) ? 1 : ((u1 > 0.25 && u1 < 0.75) ? -1 : 0);
      else sd = (u1 > 0.0 && u1 < 0.5) ? 1 : (u1 > 0.5 ? -1 : 0);
      any |= fabs(s) <= tol || sd == 0 || (nz[g] > 0.0 ? sd : -sd) == (s > 0.0 ? 1 : -1);
    }
    return any;
  }
};

// Float32 pre-filter of the gather rays (3D, emitter plane grids with occupancy): could the
// ray with draws (u0, u1) from the media sample y meet an emitter triangle?  Every position
// (sample point, plane offsets, grid origins) is taken relative to the bounds centre in
// float64 before rounding, so magnitudes stay ≲ scale wherever the scene sits.  The direction
// and the landing point on each emitter plane are computed in float32 with a bound on
// their error against the float64 values (y: ≤ ey = 2e-6·scale; direction components:
// ≤ ed = 2e-6, from z = 1 − 2u0 and sin θ = 2√(u0(1 − u0)) taken from float64 and
// sincospi of 2u1); a plane is skipped only when the landing distance is certainly
// negative or every coarse occupancy block within the landing point's error radius is
// empty.  A triangle the float64 test accepts holds the float64 landing point, whose fine
// cell lists it (cells cover the triangles' padded boxes), so its block is occupied:
// "false" is exact, the survivors take the float64 path unchanged.  Rays within 2e-3 of
// grazing a plane are always kept.
struct alignas(16) FilterPlane {  // four 16-byte shared-memory loads per plane
  float4 nc;   // normal, offset
  float4 a1;   // in-plane axis 1, grid origin x
  float4 a2;   // in-plane axis 2, grid origin y
  float4 cc;   // 1 / block size (x, y), blocks (x, y) as int bits
};

// Direction inputs of the filter: u0f = (float)u0, om = (float)(1 − u0), z = (float)(1 − 2u0)
// (each the correctly rounded float of the exact float64 value) and (cos, sin)(2π·u1) to
// within 1e-6.
struct FilterDir {
  float u0f, om, z, cp, sp;
};

// From the float64 draws (the fused pass): sincospif of 2·(float)u1.
__device__ __forceinline__ FilterDir filter_dir(double u0, double u1) {
  FilterDir f;
  f.u0f = (float)u0;
  f.om = (float)(1.0 - u0);
  f.z = (float)(1.0 - 2.0 * u0);
  sincospif(2.0f * (float)u1, &f.sp, &f.cp);
  return f;
}

// From the raw 53-bit draw mantissas m (u = m·2⁻⁵³, numpy's double): the same u0f / om / z
// by integer → float conversions of the exact values (bit-identical to filter_dir), and
// MUFU sine / cosine of φ = 2π(u1 − ½) ∈ [−π, π) with (cos, sin)(φ + π) = −(cos, sin)φ:
// argument error ≤ 2π·2⁻²⁴ (u1 rounded to float, u1 − ½ exact or within 2⁻²⁵), MUFU error
// ≤ 2⁻²¹·⁴¹ on [−π, π] — ≤ 1e-6 in all, inside the filter's ed = 2e-6.
__device__ __forceinline__ FilterDir filter_dir_raw(unsigned long long m0, unsigned long long m1) {
  constexpr float k53 = 1.1102230246251565e-16f;  // 2⁻⁵³
  FilterDir f;
  f.u0f = __ull2float_rn(m0) * k53;
  f.om = __ull2float_rn((1ULL << 53) - m0) * k53;
  f.z = __ll2float_rn((long long)(1ULL << 53) - 2LL * (long long)m0) * k53;
  const float phi = 6.283185307179586f * (__ull2float_rn(m1) * k53 - 0.5f);
  float s, c;
  __sincosf(phi, &s, &c);
  f.sp = -s;
  f.cp = -c;
  return f;
}

__device__ __forceinline__ bool emitter_may_hit(const FilterPlane* fp, const unsigned* occ, int ng,
                                                const float* y, const FilterDir& fd, float ey, float mpad) {
  const float z = fd.z;
  const float sq = sqrtf(4.0f * fd.u0f * fd.om);
  const float sp = fd.sp, cp = fd.cp;
  const float d[3] = {sq * cp, sq * sp, z};
  constexpr float ed = 2e-6f;
  for (int g = 0; g < ng; ++g) {
    const float4 nc = fp[g].nc;
    const float dn = nc.x * d[0] + nc.y * d[1] + nc.z * d[2];
    const float adn = fabsf(dn);
    if (adn < 2e-3f) return true;
    const float tp = (nc.w - (nc.x * y[0] + nc.y * y[1] + nc.z * y[2])) / dn;
    const float e = ey + fabsf(tp) * ed;
    if (tp + 2.0f * e / adn < 0.0f) continue;  // behind the sample
    const float X[3] = {y[0] + tp * d[0], y[1] + tp * d[1], y[2] + tp * d[2]};
    const float4 a1 = fp[g].a1, a2 = fp[g].a2, cc = fp[g].cc;
    const int cw = __float_as_int(cc.z), ch = __float_as_int(cc.w);
    const float px = a1.x * X[0] + a1.y * X[1] + a1.z * X[2];
    const float py = a2.x * X[0] + a2.y * X[1] + a2.z * X[2];
    const float m = 4.0f * e * (1.0f + 1.0f / adn) + mpad;
    int i0 = (int)floorf((px - m - a1.w) * cc.x), i1 = (int)floorf((px + m - a1.w) * cc.x);
    int j0 = (int)floorf((py - m - a2.w) * cc.y), j1 = (int)floorf((py + m - a2.w) * cc.y);
    if (i1 < 0 || j1 < 0 || i0 >= cw || j0 >= ch) continue;  // beside every emitter
    i0 = max(i0, 0); j0 = max(j0, 0);
    i1 = min(i1, cw - 1); j1 = min(j1, ch - 1);
    if (i1 - i0 > 1 || j1 - j0 > 1) return true;
    const unsigned mask = (i1 > i0 ? 3u : 1u) << i0;
    for (int j = j0; j <= j1; ++j)
      if (occ[g * 32 + j] & mask) return true;
  }
  return false;
}

// Pass 1 of the two-pass gather.  Each lane walks runs of kGatherRun consecutive samples
// (PCG64 jumped once per run, then stepped); the draws of samples whose ray cannot reach an
// emitter are consumed and dropped at once, the others are compacted into a per-warp queue
// in shared memory and evaluated 32 at a time (direction, nearest emitter through the plane
// grids), so the expensive part runs on full warps.
struct PendSample {
  double u0, u1;
  int j, k, i, pad;
};
constexpr int kPendCap = 64;  // per warp: ≤ 31 left over + one step's 32
// emitter pass split into filter → survivor evaluation (k_gather_eval); 0: one fused kernel
#ifndef VC_GATHER_SPLIT
#define VC_GATHER_SPLIT 1
#endif

// MODE 0: filter + evaluate fused.  MODE 1 (split): the filter only — survivors' sample
// indices are appended to the record's survivor list (stored in its own media rows, which
// hold ≥ 3 ints per sample and are written only later, for live samples), evaluated by
// k_gather_eval; the loop then carries no BVH / queue code and fits the register budget
// without spills.  MODE 2: the fused pass again for records whose evaluation found the
// queue full (W.redo) — the others exit at once.
template <int D, int MODE>
__global__ void __launch_bounds__(VC_EMIT_BS, VC_LB_EMIT * 256 / VC_EMIT_BS) k_gather_emit(DevScene S, BuildParams P, Wave W, JumpTables jt,
                                                               GatherItem* q, unsigned long long* q_count,
                                                               long long q_cap) {
  if (MODE == 2 && !W.redo[blockIdx.y]) return;
  __shared__ PendSample pend_all[VC_EMIT_BS / 32][kPendCap];
  __shared__ FilterPlane fplane[kEmitPlanes];
  __shared__ unsigned focc[kEmitPlanes * 32];
  const bool filt = D == 3 && S.ep.ng > 0 && S.ep.occ != nullptr;
  if (filt) {
    for (int t = threadIdx.x; t < kEmitPlanes * 32; t += blockDim.x) focc[t] = S.ep.occ[t];
    if (threadIdx.x < S.ep.ng) {
      const int g = threadIdx.x;
      const EmitPlanes& E = S.ep;
      // offsets and grid origins relative to the bounds centre (float64, then rounded)
      double ctr[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) ctr[a] = 0.5 * (S.bmin[a] + S.bmax[a]);
      auto dotc = [&](const double* v) { return v[0] * ctr[0] + v[1] * ctr[1] + v[2] * ctr[2]; };
      fplane[g].nc = make_float4((float)E.n[g][0], (float)E.n[g][1], (float)E.n[g][2], (float)(E.c[g] - dotc(E.n[g])));
      fplane[g].a1 = make_float4((float)E.a1[g][0], (float)E.a1[g][1], (float)E.a1[g][2],
                                 (float)(E.lo[g][0] - dotc(E.a1[g])));
      fplane[g].a2 = make_float4((float)E.a2[g][0], (float)E.a2[g][1], (float)E.a2[g][2],
                                 (float)(E.lo[g][1] - dotc(E.a2[g])));
      fplane[g].cc = make_float4((float)E.occ_inv[g][0], (float)E.occ_inv[g][1], __int_as_float(E.occ_w[g]),
                                 __int_as_float(E.occ_h[g]));
    }
    __syncthreads();
  }
  const float f_ey = (float)(2e-6 * S.scale), f_pad = (float)(1e-6 * S.scale);
  const float f_step = (float)P.march_step;
  const int rec = blockIdx.y;
  const long long base = W.rec_base[rec];
  const int Pr = (int)(W.rec_base[rec + 1] - base);
  const int n = P.n_angular;
  const long long draws0 = (D == 3) ? 2LL * P.rows * P.cols : (long long)n;
  const int* pre = W.pre + (size_t)rec * n;
  const int* cnt = W.cnt + (size_t)rec * n;
  const int lane = threadIdx.x & 31;
  PendSample* pend = pend_all[threadIdx.x >> 5];
  double x[3] = {0.0, 0.0, 0.0};
  float xr[3] = {0.0f, 0.0f, 0.0f};  // the filter's sample origin relative to the bounds centre
#pragma unroll
  for (int c = 0; c < D; ++c) {
    x[c] = W.x[rec * D + c];
    xr[c] = (float)(x[c] - 0.5 * (S.bmin[c] + S.bmax[c]));
  }
  const uint64_t* st = W.rng + 4 * rec;
  const double tol = 1e-5 * S.scale;
  const Toward toward(S.ep);
  // the warp appends emitter hits into queue chunks it reserves kQChunk slots at a time
  // (one atomic per chunk instead of one per step); unused slots are marked empty
  long long cbase = 0;
  int cused = kQChunk;  // warp-uniform
  auto seal = [&]() {   // mark the rest of the current chunk empty
    for (int t = cused + lane; t < kQChunk; t += 32)
      if (cbase + t < q_cap) q[cbase + t].slot = -1;
  };
  auto origin = [&](int k, int i, double* y) {
    const double ri = ring_radius(i, P.march_step);
#pragma unroll
    for (int c = 0; c < D; ++c) y[c] = add(x[c], mul(ri, W.dirs[((size_t)rec * n + k) * D + c]));
  };
  int* surv = (int*)(W.media + (size_t)base * 3);  // MODE 1: the record's survivor list
  // evaluate pend[0, m) (lane l takes entry l); every lane takes part in the queue ballot
  auto evaluate = [&](int m) {
    if constexpr (MODE == 1) {
      int sb = 0;
      if (lane == 0) sb = atomicAdd(W.surv_cnt + rec, m);
      sb = __shfl_sync(0xffffffffu, sb, 0);
      if (lane < m) surv[sb + lane] = pend[lane].j;
      return;
    }
    const bool active = lane < m;
    double y[3] = {0.0, 0.0, 0.0}, gd[3] = {0.0, 0.0, 0.0}, te = 0.0;
    int ie = -1, j = 0, k = 0, i = 0;
    if (active) {
      const PendSample ps = pend[lane];
      j = ps.j;
      k = ps.k;
      i = ps.i;
      origin(k, i, y);
      if constexpr (D == 2) {
        double th = mul(2.0 * kPi, ps.u0);
        gd[0] = cos(th);
        gd[1] = sin(th);
      } else {
        double z = sub(1.0, mul(2.0, ps.u0));
        double sq = sqrt(fmax(sub(1.0, mul(z, z)), 0.0));
        // cos, sin of φ = 2π·u1 (src/transport.py:274-285) without the range reduction of
        // sincos(φ): equal to the reference's cos(fl(2π·u1)) within an ulp of φ
        double sp, cp;
        sincospi(2.0 * ps.u1, &sp, &cp);
        gd[0] = mul(sq, cp);
        gd[1] = mul(sq, sp);
        gd[2] = z;
      }
      nearest_emitter<D>(S, y, gd, te, ie);
      if (ie < 0 && W.dense_media) {  // dead samples are read only by inspection
        const double zero[3] = {0.0, 0.0, 0.0};
        store_media(W.media + (size_t)(base + j) * 3, zero);
      }
    }
    const bool hit = active && ie >= 0;
    const unsigned hits = __ballot_sync(0xffffffffu, hit);
    if (hits) {
      const int nh = __popc(hits);
      if (cused + nh > kQChunk) {  // new chunk
        seal();
        unsigned long long nb = 0;
        if (lane == 0) nb = atomicAdd(q_count, (unsigned long long)kQChunk);
        cbase = (long long)__shfl_sync(0xffffffffu, nb, 0);
        cused = 0;
      }
      if (hit) {
        const long long slot = cbase + cused + __popc(hits & ((1u << lane) - 1u));
        if (slot < q_cap) {
          GatherItem& it = q[slot];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            it.y[c] = c < D ? y[c] : 0.0;
            it.d[c] = c < D ? gd[c] : 0.0;
          }
          it.te = te;
          it.ie = ie;
          it.slot = base + j;
          it.rec = rec;
          it.k = k;
          it.ring = i;
        } else {  // queue full: resolve in place (same result, less coherent)
          double v[3] = {0.0, 0.0, 0.0};
          if (!occluded<D>(S, y, gd, te, ie)) emitter_radiance<D>(S, W, P.hg_g, rec, y, gd, te, ie, v);
          store_media(W.media + (size_t)(base + j) * 3, v);
          if (v[0] > 0.0 || v[1] > 0.0 || v[2] > 0.0) mark_live(W, n, rec, k, i);
        }
      }
      cused += nh;
    }
  };
  int qn = 0;  // warp-uniform queue length
  const int stride = gridDim.x * blockDim.x * kGatherRun;
  // warp-uniform loop: lane runs [j0, j0 + kGatherRun) of the record's samples
  for (int j0w = (blockIdx.x * blockDim.x + (threadIdx.x & ~31)) * kGatherRun; j0w < Pr; j0w += stride) {
    const int j0 = j0w + lane * kGatherRun;
    int k = 0, i = 0, ck = 0;  // ck = cnt[k]
    Pcg64 g;
    if (j0 < Pr) {
      // direction of the first sample (run table written by k_rings)
      k = W.run_dir[(size_t)rec * W.run_stride + j0 / kGatherRun];
      i = j0 - pre[k];
      g = pcg_load(st);
      pcg_advance(g, (unsigned long long)(draws0 + (long long)(D == 3 ? 2 : 1) * j0), jt);
      ck = cnt[k];
    }
    for (int step = 0; step < kGatherRun; ++step) {
      const int j = j0 + step;
      const bool active = j < Pr;
      bool keep = false;
      double u0 = 0.0, u1 = 0.0;
      if (active) {
        while (i >= ck) {  // next direction with live rings
          ++k;
          i = 0;
          ck = cnt[k];
        }
        FilterDir fd{};
        if (MODE == 1 && D == 3 && filt) {  // the survivors redraw their doubles (k_gather_eval)
          const unsigned long long m0 = g.next64() >> 11, m1 = g.next64() >> 11;
          fd = filter_dir_raw(m0, m1);
        } else {
          u0 = g.next_double();
          if constexpr (D == 3) {
            u1 = g.next_double();
            if (filt) fd = filter_dir(u0, u1);
          }
        }
        if constexpr (D == 3) {
          if (filt) {
            // the filter's float32 sample point (error ≤ f_ey against origin())
            const float4 dk = W.dirs32[(size_t)rec * n + k];
            const float ri = ((float)i + 0.5f) * f_step;
            const float y32[3] = {xr[0] + ri * dk.x, xr[1] + ri * dk.y, xr[2] + ri * dk.z};
            keep = emitter_may_hit(fplane, focc, S.ep.ng, y32, fd, f_ey, f_pad);
          } else {
            double y[3];
            origin(k, i, y);
            keep = toward(y, u0, u1, tol);
          }
          if (!keep && W.dense_media) {
            const double zero[3] = {0.0, 0.0, 0.0};
            store_media(W.media + (size_t)(base + j) * 3, zero);
          }
        } else {
          keep = true;
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) pend[qn + __popc(m & ((1u << lane) - 1u))] = PendSample{u0, u1, j, k, i, 0};
      qn += __popc(m);
      if (qn >= 32) {
        __syncwarp();
        evaluate(32);
        __syncwarp();
        if (lane < qn - 32) pend[lane] = pend[32 + lane];
        __syncwarp();
        qn -= 32;
      }
      if (active) ++i;
    }
  }
  if (qn > 0) {
    __syncwarp();
    evaluate(qn);
  }
  seal();
}

// Evaluation of the survivors of k_gather_emit<D, 1>: thread per survivor — its direction
// and ring from the run table, its draws by a PCG64 jump (the same values the fused pass
// draws), the nearest emitter through the plane grids, emitter hits appended to the
// occlusion queue in warp chunks.  A full queue flags the record for the fused redo pass.
template <int D>
__global__ void __launch_bounds__(VC_EVAL_BS, VC_LB_EMIT * 256 / VC_EVAL_BS) k_gather_eval(DevScene S, BuildParams P, Wave W, JumpTables jt,
                                                               GatherItem* q, unsigned long long* q_count,
                                                               long long q_cap) {
  const int rec = blockIdx.y;
  const long long base = W.rec_base[rec];
  const int ns = W.surv_cnt[rec];
  const int* surv = (const int*)(W.media + (size_t)base * 3);
  const int n = P.n_angular;
  const long long draws0 = (D == 3) ? 2LL * P.rows * P.cols : (long long)n;
  const int* pre = W.pre + (size_t)rec * n;
  const int* cnt = W.cnt + (size_t)rec * n;
  const int lane = threadIdx.x & 31;
  long long cbase = 0;
  int cused = kQChunk;  // warp-uniform
  const int stride = gridDim.x * blockDim.x;
  for (int t0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31); t0 < ns; t0 += stride) {
    const int t = t0 + lane;
    const bool active = t < ns;
    double y[3] = {0.0, 0.0, 0.0}, gd[3] = {0.0, 0.0, 0.0}, te = 0.0;
    int ie = -1, j = 0, k = 0, i = 0;
    if (active) {
      j = surv[t];
      k = W.run_dir[(size_t)rec * W.run_stride + j / kGatherRun];
      while (j >= pre[k] + cnt[k]) ++k;  // the run's first direction, then on to j's
      i = j - pre[k];
      Pcg64 g = pcg_load(W.rng + 4 * rec);
      pcg_advance(g, (unsigned long long)(draws0 + (long long)(D == 3 ? 2 : 1) * j), jt);
      const double u0 = g.next_double();
      const double ri = ring_radius(i, P.march_step);
#pragma unroll
      for (int c = 0; c < D; ++c) y[c] = add(W.x[rec * D + c], mul(ri, W.dirs[((size_t)rec * n + k) * D + c]));
      if constexpr (D == 2) {
        const double th = mul(2.0 * kPi, u0);
        gd[0] = cos(th);
        gd[1] = sin(th);
      } else {
        const double u1 = g.next_double();
        const double z = sub(1.0, mul(2.0, u0));
        const double sq = sqrt(fmax(sub(1.0, mul(z, z)), 0.0));
        double sp, cp;
        sincospi(2.0 * u1, &sp, &cp);  // as the fused pass (k_gather_emit)
        gd[0] = mul(sq, cp);
        gd[1] = mul(sq, sp);
        gd[2] = z;
      }
      nearest_emitter<D>(S, y, gd, te, ie);
    }
    const bool hit = active && ie >= 0;
    const unsigned hits = __ballot_sync(0xffffffffu, hit);
    if (hits) {
      const int nh = __popc(hits);
      if (cused + nh > kQChunk) {  // new chunk
        for (int u = cused + lane; u < kQChunk; u += 32)
          if (cbase + u < q_cap) q[cbase + u].slot = -1;
        unsigned long long nb = 0;
        if (lane == 0) nb = atomicAdd(q_count, (unsigned long long)kQChunk);
        cbase = (long long)__shfl_sync(0xffffffffu, nb, 0);
        cused = 0;
      }
      if (hit) {
        const long long slot = cbase + cused + __popc(hits & ((1u << lane) - 1u));
        if (slot < q_cap) {
          GatherItem& it = q[slot];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            it.y[c] = c < D ? y[c] : 0.0;
            it.d[c] = c < D ? gd[c] : 0.0;
          }
          it.te = te;
          it.ie = ie;
          it.slot = base + j;
          it.rec = rec;
          it.k = k;
          it.ring = i;
        } else {
          atomicOr(W.redo + rec, 1);  // queue full: the record takes the fused redo pass
        }
      }
      cused += nh;
    }
  }
  for (int u = cused + lane; u < kQChunk; u += 32)
    if (cbase + u < q_cap) q[cbase + u].slot = -1;
}

template <int D, bool HG = false>
__global__ void __launch_bounds__(256, VC_LB_OCCL) k_gather_occl(DevScene S, Wave W, int n, const GatherItem* q,
                                                               const unsigned long long* q_count, long long q_cap,
                                                               float* media, double hg) {
  VC_RAY_STACK;
  const long long nq = min((long long)*q_count, q_cap);
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < nq;
       t += (long long)gridDim.x * blockDim.x) {
    if (q[t].slot < 0) continue;  // unused tail of a warp's chunk
    const GatherItem it = q[t];
    double v[3] = {0.0, 0.0, 0.0};
    if (!occluded<D>(S, it.y, it.d, it.te, it.ie, &stk))
      emitter_radiance<D>(S, W, HG ? hg : 0.0, it.rec, it.y, it.d, it.te, it.ie, v);
    store_media(media + (size_t)it.slot * 3, v);
    if (v[0] > 0.0 || v[1] > 0.0 || v[2] > 0.0) mark_live(W, n, it.rec, it.k, it.ring);
  }
}

// Occlusion pass with persistent lanes: every lane owns one queued ray at a time and advances
// its traversal leaf by leaf; a lane whose ray is decided writes the result and fetches the
// next ray (warp-aggregated atomic cursor) at the next step, so lanes no longer idle until
// the slowest ray of a grid-stride batch finishes (k_gather_occl: 9 of 32 lanes active per
// instruction).  The traversal is bvh_query's any-hit mode, resumable: the same node order,
// culling and (t, index) decision per ray.
#ifndef VC_OCCL_PT
#define VC_OCCL_PT 1
#endif
template <int D, bool HG = false>
__global__ void __launch_bounds__(256, VC_LB_OCCL) k_gather_occl_pt(DevScene S, Wave W, int n, const GatherItem* q,
                                                                  unsigned long long* q_count, long long q_cap,
                                                                  float* media, double hg) {
  const long long nq = min((long long)q_count[0], q_cap);
  unsigned long long* cursor = q_count + 1;
  const DevBvh& H = S.geo;
  const int lane = threadIdx.x & 31;
  const float slack = 1e-5f * (float)S.scale;
  LocalStack stk;
  long long cur_item = -1;
  bool exhausted = false;
  double o[3] = {0, 0, 0}, d[3] = {0, 0, 0}, thr = 0.0;
  int id_thr = 0;
  float2 inv2[3], noi2[3];
  float tbf = 0.0f;
  int sp = 0;
  unsigned cur = 0;
  auto finish = [&](bool occl) {
    const GatherItem& it = q[cur_item];
    double v[3] = {0.0, 0.0, 0.0};
    if (!occl) emitter_radiance<D>(S, W, HG ? hg : 0.0, it.rec, it.y, it.d, it.te, it.ie, v);
    store_media(media + (size_t)it.slot * 3, v);
    if (v[0] > 0.0 || v[1] > 0.0 || v[2] > 0.0) mark_live(W, n, it.rec, it.k, it.ring);
    cur_item = -1;
  };
  auto pop = [&]() -> bool {
    while (sp > 0) {
      const uint2 e = stk.get(--sp);
      if (__uint_as_float(e.y) <= tbf) {
        cur = e.x;
        return true;
      }
    }
    return false;
  };
  while (true) {
    // lanes without a ray fetch the next ones
    const bool need = cur_item < 0 && !exhausted;
    const unsigned mneed = __ballot_sync(0xffffffffu, need);
    if (mneed) {
      const int leader = __ffs(mneed) - 1;
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(cursor, (unsigned long long)__popc(mneed));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (need) {
        const long long t = (long long)base + __popc(mneed & ((1u << lane) - 1u));
        if (t >= nq) {
          exhausted = true;
        } else if (q[t].slot >= 0) {  // (negative: an unused tail slot of a producer's chunk)
          cur_item = t;
          const GatherItem& it = q[t];
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            o[a] = it.y[a];
            d[a] = it.d[a];
          }
          thr = it.te;
          id_thr = it.ie;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            float inv = 0.0f, noi = 0.0f;
            if (a < D) {
              const float orl = (float)(o[a] - H.ctr[a]);
              asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"((float)d[a]));
              noi = -orl * inv;
            }
            inv2[a] = make_float2(inv, inv);
            noi2[a] = make_float2(noi, noi);
          }
          tbf = __double2float_ru(thr) * 1.0001f + slack;  // thr finite: an emitter hit distance
          sp = 0;
          cur = 0;
        }
      }
    }
    if (!__any_sync(0xffffffffu, cur_item >= 0)) {
      if (__all_sync(0xffffffffu, exhausted)) break;
      continue;
    }
    if (cur_item >= 0) {
      // one step: descend to the next leaf, test it
      bool alive = true;
      while (!(cur & 0x80000000u)) {
        const float4* N = H.nodes + 4 * (size_t)cur;
        const float4 A = __ldg(N), B = __ldg(N + 1), C = __ldg(N + 2), R = __ldg(N + 3);
        float tl, tr;
        bool hl, hr;
        box_hit2<D>(A, B, C, inv2, noi2, tbf, hl, hr, tl, tr);
        if (hl && hr) {
          const bool lf = tl <= tr;
          stk.put(sp++, make_uint2(__float_as_uint(lf ? R.z : R.x), __float_as_uint(lf ? tr : tl)));
          cur = __float_as_uint(lf ? R.x : R.z);
        } else if (hl || hr) {
          cur = __float_as_uint(hl ? R.x : R.z);
        } else if (!pop()) {
          alive = false;
          break;
        }
      }
      if (!alive) {
        finish(false);
      } else {
        bool occl = false;
        for (int k = (int)(cur & 0x7fffffffu);; ++k) {
          const int idf = __float_as_int(__ldg(&H.prim32[3 * (size_t)k + 2].w));
          const double t = hit_prim<D>(H.prim + (size_t)k * prim_stride(D), o, d, S.t_eps);
          if (t != INFINITY) {
            const int id = idf & 0x7fffffff;
            if (t < thr || (t == thr && id < id_thr)) {
              occl = true;
              break;
            }
          }
          if (idf < 0) break;
        }
        if (occl) finish(true);
        else if (!pop()) finish(false);
      }
    }
  }
}

// k_gather_delta with persistent lanes (scenes with a BVH): a lane owns one media sample at
// a time, walks its lights one shadow ray after the other — each advanced leaf by leaf, as
// k_gather_occl_pt — and fetches the next sample through a warp-aggregated cursor once the
// last light is decided.  Same per-sample arithmetic and light order as k_gather_delta.
template <int D>
__global__ void __launch_bounds__(256, 3) k_gather_delta_pt(DevScene S, BuildParams P, Wave W,
                                                            unsigned long long* cursor) {
  const long long total = W.rec_base[W.B];
  const int n = P.n_angular;
  const double hg = (D == 3) ? P.hg_g : 0.0;
  const DevBvh& H = S.geo;
  const int lane = threadIdx.x & 31;
  const float slack = 1e-5f * (float)S.scale;
  const double off = 1e-6 * S.scale;
  const double norm = (D == 3) ? 4.0 * kPi : 2.0 * kPi;
  LocalStack stk;
  long long j = -1;  // the lane's sample (−1: none)
  bool exhausted = false, ray = false;
  int rec = 0, k = 0, i = 0, l = 0;
  double y[3] = {0.0, 0.0, 0.0}, dl[3] = {0.0, 0.0, 0.0};
  double d[3] = {0.0, 0.0, 0.0}, thr = 0.0, rr = 0.0;  // rr: distance to a point light
  float2 inv2[3], noi2[3];
  float tbf = 0.0f;
  int sp = 0;
  unsigned cur = 0;
  auto pop = [&]() -> bool {
    while (sp > 0) {
      const uint2 e = stk.get(--sp);
      if (__uint_as_float(e.y) <= tbf) {
        cur = e.x;
        return true;
      }
    }
    return false;
  };
  auto decided = [&](bool occl) {
    if (!occl) {
      const double* L8 = S.lights + 8 * (size_t)l;
      double val;
      if (L8[0] == 0.0) {
        const double rm = fmax(rr, off);
        val = __ddiv_rn(exp(-S.sigma_t * rr), D == 3 ? mul(rm, rm) : rm);
      } else {
        val = exp(-S.sigma_t * bounds_exit<D>(S, y, d));
      }
      if (val > 0.0) {
        double w = __ddiv_rn(val, norm);
        if (hg != 0.0) {
          double dx[3], n2 = 0.0;
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            dx[c] = sub(y[c], W.x[rec * D + c]);
            n2 = add(n2, mul(dx[c], dx[c]));
          }
          const double nrm = sqrt(n2);
          double cs = 0.0;  // d·w in delta_inscatter's order
#pragma unroll
          for (int c = 0; c < 3; ++c) cs = add(cs, mul(d[c], __ddiv_rn(dx[c], nrm)));
          w = mul(w, mul(4.0 * kPi, hg_phase(hg, cs)));
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) dl[c] = add(dl[c], mul(w, L8[4 + c]));
      }
    }
    ray = false;
    ++l;
  };
  while (true) {
    const bool need = j < 0 && !exhausted;
    const unsigned mneed = __ballot_sync(0xffffffffu, need);
    if (mneed) {
      const int leader = __ffs(mneed) - 1;
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(cursor, (unsigned long long)__popc(mneed));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (need) {
        const long long t = (long long)base + __popc(mneed & ((1u << lane) - 1u));
        if (t >= total) {
          exhausted = true;
        } else {
          j = t;
          int lo = 0, hi = W.B - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (W.rec_base[mid] <= j) lo = mid; else hi = mid - 1;
          }
          rec = lo;
          const int jl = (int)(j - W.rec_base[rec]);
          const int* pre = W.pre + (size_t)rec * n;
          int a = 0, b = n - 1;
          while (a < b) {
            const int mid = (a + b + 1) >> 1;
            if (pre[mid] <= jl) a = mid; else b = mid - 1;
          }
          k = a;
          i = jl - pre[k];
          const double ri = ring_radius(i, P.march_step);
#pragma unroll
          for (int c = 0; c < D; ++c) y[c] = add(W.x[rec * D + c], mul(ri, W.dirs[((size_t)rec * n + k) * D + c]));
          l = 0;
          dl[0] = dl[1] = dl[2] = 0.0;
        }
      }
    }
    if (j >= 0 && !ray) {
      while (l < S.n_lights) {  // the sample's next shadow ray
        const double* L8 = S.lights + 8 * (size_t)l;
        bool ok = true;
        if (L8[0] == 0.0) {
          double to[3], r2 = 0.0;
#pragma unroll
          for (int a = 0; a < D; ++a) {
            to[a] = sub(L8[1 + a], y[a]);
            r2 = add(r2, mul(to[a], to[a]));
          }
          const double r = sqrt(r2);
          ok = r > off;
          if (ok) {
#pragma unroll
            for (int a = 0; a < D; ++a) d[a] = __ddiv_rn(to[a], r);
            thr = mul(r, 1.0 - 1e-6);
            rr = r;
          }
        } else {
#pragma unroll
          for (int a = 0; a < D; ++a) d[a] = L8[1 + a];
          thr = INFINITY;
          rr = 0.0;
        }
        if (ok) {
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            float inv = 0.0f, noi = 0.0f;
            if (a < D) {
              const float orl = (float)(y[a] - H.ctr[a]);
              asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"((float)d[a]));
              noi = -orl * inv;
            }
            inv2[a] = make_float2(inv, inv);
            noi2[a] = make_float2(noi, noi);
          }
          tbf = isfinite(thr) ? __double2float_ru(thr) * 1.0001f + slack : INFINITY;
          sp = 0;
          cur = 0;
          ray = true;
          break;
        }
        ++l;
      }
      if (!ray) {  // every light decided: merge into the sample's media row
        if (dl[0] > 0.0 || dl[1] > 0.0 || dl[2] > 0.0) {
          const unsigned long long word = W.live[((size_t)rec * W.live_words + (i >> 6)) * n + k];
          const bool live = (word >> (i & 63)) & 1ULL;
          float* out = W.media + (size_t)j * 3;
          bool pos = false;
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double v = mul(S.sigma_s, dl[c]);
            float f = (float)v;
            if (v > 0.0 && !(f > 0.0f)) f = FLT_TRUE_MIN;
            f += live ? out[c] : 0.0f;
            out[c] = f;
            pos |= f > 0.0f;
          }
          if (pos && !live) mark_live(W, n, rec, k, i);
        }
        j = -1;
      }
    }
    if (!__any_sync(0xffffffffu, ray)) {
      if (__all_sync(0xffffffffu, exhausted && j < 0)) break;
      continue;
    }
    if (ray) {  // one step: descend to the next leaf, test it
      bool alive = true;
      while (!(cur & 0x80000000u)) {
        const float4* N = H.nodes + 4 * (size_t)cur;
        const float4 A = __ldg(N), B = __ldg(N + 1), C = __ldg(N + 2), R = __ldg(N + 3);
        float tl, tr;
        bool hl, hr;
        box_hit2<D>(A, B, C, inv2, noi2, tbf, hl, hr, tl, tr);
        if (hl && hr) {
          const bool lf = tl <= tr;
          stk.put(sp++, make_uint2(__float_as_uint(lf ? R.z : R.x), __float_as_uint(lf ? tr : tl)));
          cur = __float_as_uint(lf ? R.x : R.z);
        } else if (hl || hr) {
          cur = __float_as_uint(hl ? R.x : R.z);
        } else if (!pop()) {
          alive = false;
          break;
        }
      }
      if (!alive) {
        decided(false);
      } else {
        bool occl = false;
        for (int kk = (int)(cur & 0x7fffffffu);; ++kk) {
          const int idf = __float_as_int(__ldg(&H.prim32[3 * (size_t)kk + 2].w));
          const double t = hit_prim<D>(H.prim + (size_t)kk * prim_stride(D), y, d, S.t_eps);
          if (t < thr) {  // (id_thr = −1: no tie clause)
            occl = true;
            break;
          }
          if (idf < 0) break;
        }
        if (occl) decided(true);
        else if (!pop()) decided(false);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Spherical Delaunay (3D connectivity, src/scene.py:388-399)
// ---------------------------------------------------------------------------

constexpr int kMaxV = 24;

// Owned triangle t of cell `base` (wave-global direction index): slot-major int2 rows
// (stride W.own_stride cells), so the lanes of a warp (consecutive cells) write and
// k_tri_scatter reads one coalesced row per slot.
__device__ __forceinline__ void own_put(const Wave& W, int* own, size_t base, int t, int a, int b) {
  ((int2*)own)[(size_t)t * W.own_stride + base] = make_int2(a, b);
}

struct Line {
  double A, B, C;
};

__device__ __forceinline__ Line cell_line(int lab, const double* p, const double* e1, const double* e2,
                                          const double* dirs, double L) {
  if (lab < 0) {
    switch (lab) {
      case -1: return {-1.0, 0.0, L};
      case -2: return {0.0, -1.0, L};
      case -3: return {1.0, 0.0, L};
      default: return {0.0, 1.0, L};
    }
  }
  const double* q = dirs + 3 * (size_t)lab;
  double d[3] = {p[0] - q[0], p[1] - q[1], p[2] - q[2]};
  return {e1[0] * d[0] + e1[1] * d[1] + e1[2] * d[2], e2[0] * d[0] + e2[1] * d[1] + e2[2] * d[2],
          p[0] * d[0] + p[1] * d[1] + p[2] * d[2]};
}

__device__ __forceinline__ void meet(const Line& l1, const Line& l2, double& a, double& b) {
  const double det = l1.A * l2.B - l2.A * l1.B;
  const double inv = 1.0 / det;
  a = (l1.B * l2.C - l2.B * l1.C) * inv;
  b = (l2.A * l1.C - l1.A * l2.C) * inv;
}

// Cell polygon held in shared memory, [vertex][thread] layout (bank-conflict free): the
// per-thread working set of the clipping loop would otherwise live in local memory and,
// at full occupancy, overflow L1 into L2.
constexpr int kDelBS = 128;
// Polygon capacity in shared memory.  On the stratum grids the largest polygon met while
// clipping has 11 vertices (n = 16384, measured); a cell that outgrows the capacity is
// recomputed by k_delaunay_retry with a 48-vertex polygon in global memory.
#ifndef VC_POLYV
#define VC_POLYV 14
#endif
constexpr int kPolyV = VC_POLYV;
constexpr int kRetryV = 48;

template <int STRIDE, int CAP>
struct PolyT {
  static constexpr int kCap = CAP;
  double* a;
  double* b;
  int* lab;
  __device__ __forceinline__ double& A(int v) { return a[v * STRIDE]; }
  __device__ __forceinline__ double& B(int v) { return b[v * STRIDE]; }
  __device__ __forceinline__ int& L(int v) { return lab[v * STRIDE]; }
};
using Poly = PolyT<kDelBS, kPolyV>;
using PolyRetry = PolyT<1, kRetryV>;

// Voronoi cell of point i over candidates within angle alpha (exact if the cell radius
// stays below alpha/2).  Returns 0 secure, 1 needs a larger alpha, 2 polygon overflow.
template <class Poly>
__device__ int voronoi_cell_poly(const double* __restrict__ dirs, const float4* __restrict__ dirs32, int rows,
                                 int cols, int i, const DelAngle& ang, Poly poly, int& m) {
  const double alpha = ang.alpha;
  const double* p = dirs + 3 * (size_t)i;
  const double px = p[0], py = p[1], pz = p[2];
  const float4 p32 = dirs32[i];
  double h[3] = {0.0, 0.0, 1.0};
  if (fabs(pz) >= 0.9) { h[0] = 1.0; h[2] = 0.0; }
  double e1[3] = {h[1] * pz - h[2] * py, h[2] * px - h[0] * pz, h[0] * py - h[1] * px};
  const double ne = rsqrt(e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2]);
  e1[0] *= ne; e1[1] *= ne; e1[2] *= ne;
  const double e2[3] = {py * e1[2] - pz * e1[1], pz * e1[0] - px * e1[2], px * e1[1] - py * e1[0]};
  const double pp[3] = {px, py, pz};
  // initial square of half-size tan(α/2): a cell reaching beyond it fails the security
  // test (2·R_cell ≤ α) anyway, and the tighter start shrinks the candidate cut early
  const double L = ang.tan_half * 1.001;
  m = 4;
  poly.A(0) = L;  poly.B(0) = -L; poly.L(0) = -1;
  poly.A(1) = L;  poly.B(1) = L;  poly.L(1) = -2;
  poly.A(2) = -L; poly.B(2) = L;  poly.L(2) = -3;
  poly.A(3) = -L; poly.B(3) = -L; poly.L(3) = -4;
  double t2R = 2.0 * L * L;
  // a candidate q can cut the cell only if ∠(p, q) < 2·R_cell, i.e. p·q > cos 2R =
  // (1 − tan²R)/(1 + tan²R); tested in float32 with a margin (2e-6) far above the
  // rounding of the float32 directions, dot and bound — a looser cut only costs time
  auto cutf_of = [](double t) {
    const float tf = (float)t;
    return __fdividef(1.0f - tf, 1.0f + tf) - 2e-6f;
  };
  float cutf = cutf_of(t2R);
  // candidate rows: bands meeting z ∈ [cos(θ+α), cos(θ−α)]; columns: azimuth half-width
  // asin(sin α / sin θ)
  const double sa = ang.sin_a, ca = ang.cos_a;
  const double st = sqrt(fmax(0.0, 1.0 - pz * pz));
  const double z_hi = pz * ca + st * sa;  // cos(θ − α) (pole cap when θ ≤ α)
  const double z_lo = pz * ca - st * sa;  // cos(θ + α)
  const bool cap_n = st <= sa && pz > 0.0, cap_s = st <= sa && pz < 0.0;
  const int r0 = i / cols, c0 = i - r0 * cols;
  auto row_of = [&](double z) {
    int r = (int)floor((1.0 - z) * rows * 0.5);
    return min(max(r, 0), rows - 1);
  };
  const int rlo = cap_n ? 0 : min(row_of(z_hi), r0);
  const int rhi = cap_s ? rows - 1 : max(row_of(z_lo), r0);
  int half = cols;
  if (!cap_n && !cap_s) {
    const double dphi = asin(fmin(sa / st, 1.0));
    half = (int)ceil(dphi * cols / (2.0 * kPi)) + 1;
    if (2 * half + 1 >= cols) half = cols;
  }
  const int span = max(r0 - rlo, rhi - r0);
  const int ncol_iter = (half >= cols) ? cols : 2 * half + 1;
  // clip the cell by the bisector of (p, q_j); 2 = polygon overflow
  auto consider = [&](const int j) -> int {
    // float32 pre-test (one 16-byte load); its margin 2e-6 ≫ the float32 rounding error
    const float4 q4 = __ldg(dirs32 + j);
    if (!(p32.x * q4.x + p32.y * q4.y + p32.z * q4.z > cutf)) return 0;
    const double* q = dirs + 3 * (size_t)j;
    const double qx = q[0], qy = q[1], qz = q[2];
    const double d0 = px - qx, d1 = py - qy, d2 = pz - qz;
    const Line ln = {e1[0] * d0 + e1[1] * d1 + e1[2] * d2, e2[0] * d0 + e2[1] * d1 + e2[2] * d2,
                     px * d0 + py * d1 + pz * d2};
    unsigned out = 0;
    double kept = 0.0;  // largest squared radius among the vertices the cut keeps
    for (int v = 0; v < m; ++v) {
      const double va = poly.A(v), vb = poly.B(v);
      if (ln.A * va + ln.B * vb + ln.C < 0.0) out |= 1u << v;
      else kept = fmax(kept, va * va + vb * vb);
    }
    if (!out) return 0;
    const unsigned full = (1u << m) - 1u;
    if (out == full) return 2;  // cannot happen: p (the origin) is inside every bisector
    // convex polygon: the outside vertices form one cyclic run [s, e]
    const unsigned prev = ((out << 1) | (out >> (m - 1))) & full;  // bit v: out[v−1]
    const unsigned next = ((out >> 1) | (out << (m - 1))) & full;  // bit v: out[v+1]
    const int s = __ffs(out & ~prev) - 1;
    const int e = __ffs(out & ~next) - 1;
    const int sp = (s + m - 1) % m;  // inside vertex before the run
    const int L_out = __popc(out);
    const int m_new = m - L_out + 2;
    if (m_new > Poly::kCap) return 2;
    // X = edge(sp) ∩ bisector, Y = bisector ∩ edge(e); cyclic order … sp, X, Y, e+1 …
    const int lab_e = poly.L(e);
    double xa, xb, ya, yb;
    meet(cell_line(poly.L(sp), pp, e1, e2, dirs, L), ln, xa, xb);
    meet(ln, cell_line(lab_e, pp, e1, e2, dirs, L), ya, yb);
    if (s <= e) {
      // run inside the array: [0, s) X Y [e+1, m) — shift the tail by 2 − L_out in place
      const int shift = 2 - L_out;
      if (shift < 0) {
        for (int v = e + 1; v < m; ++v) {
          poly.A(v + shift) = poly.A(v); poly.B(v + shift) = poly.B(v); poly.L(v + shift) = poly.L(v);
        }
      } else if (shift > 0) {
        for (int v = m - 1; v > e; --v) {
          poly.A(v + shift) = poly.A(v); poly.B(v + shift) = poly.B(v); poly.L(v + shift) = poly.L(v);
        }
      }
      poly.A(s) = xa; poly.B(s) = xb; poly.L(s) = j;
      poly.A(s + 1) = ya; poly.B(s + 1) = yb; poly.L(s + 1) = lab_e;
    } else {
      // run wraps: keep [e+1, s) moved to the front, then X Y
      const int nk = s - e - 1;
      for (int v = 0; v < nk; ++v) {
        poly.A(v) = poly.A(e + 1 + v); poly.B(v) = poly.B(e + 1 + v); poly.L(v) = poly.L(e + 1 + v);
      }
      poly.A(nk) = xa; poly.B(nk) = xb; poly.L(nk) = j;
      poly.A(nk + 1) = ya; poly.B(nk + 1) = yb; poly.L(nk + 1) = lab_e;
    }
    m = m_new;
    // the new polygon = kept vertices + X + Y: its radius without another pass
    t2R = fmax(kept, fmax(xa * xa + xb * xb, ya * ya + yb * yb));
    cutf = cutf_of(t2R);
    return 0;
  };
  // regular cells first take their 8 stratum neighbours, which are nearly always Delaunay
  // neighbours: the lanes of a warp (adjacent cells of one row) then clip together, and
  // the later, farther candidates mostly fail the cut pre-test
  const bool pro = half < cols;
  if (pro) {
    for (int t = 0; t < 8; ++t) {
      const int dr = (t < 2) ? 0 : ((t < 4) ? ((t & 1) ? 1 : -1) : ((t < 6) ? -1 : 1));
      const int dc = (t < 2) ? ((t & 1) ? 1 : -1) : ((t < 4) ? 0 : ((t & 1) ? 1 : -1));
      const int row = r0 + dr;
      if (row < rlo || row > rhi) continue;
      int col = c0 + dc;
      if (col < 0) col += cols;
      else if (col >= cols) col -= cols;
      if (consider(row * cols + col) == 2) return 2;
    }
  }
  // after the neighbours the cell is usually well inside half the search radius: sweep
  // only the window of its current 2·R_cell (same bounds as for α; R only shrinks, so a
  // point outside it can never cut)
  int rlo2 = rlo, rhi2 = rhi, ncol2 = ncol_iter, span2 = span;
  if (pro) {
    const double t = t2R;
    const double c2 = (1.0 - t) / (1.0 + t) - 1e-12, s2 = 2.0 * sqrt(t) / (1.0 + t) + 1e-12;
    if (c2 > ca && s2 < sa) {
      const bool capn2 = st <= s2 && pz > 0.0, caps2 = st <= s2 && pz < 0.0;
      rlo2 = max(rlo, capn2 ? 0 : min(row_of(pz * c2 + st * s2), r0));
      rhi2 = min(rhi, caps2 ? rows - 1 : max(row_of(pz * c2 - st * s2), r0));
      if (!capn2 && !caps2) {
        const int h2 = (int)ceil(asin(fmin(s2 / st, 1.0)) * cols / (2.0 * kPi)) + 1;
        if (2 * h2 + 1 < ncol2) ncol2 = 2 * h2 + 1;
      }
      span2 = max(r0 - rlo2, rhi2 - r0);
    }
  }
  for (int rr = 0; rr <= 2 * span2; ++rr) {
    // rows outward from r0 (nearest first), skipping rows outside [rlo2, rhi2]
    int dr = (rr + 1) >> 1;
    int row = (rr & 1) ? r0 - dr : r0 + dr;
    if (row < rlo2 || row > rhi2) continue;
    for (int cc = 0; cc < ncol2; ++cc) {
      int dc = (cc + 1) >> 1;
      if (pro && dr <= 1 && dc <= 1) continue;  // taken above
      int col = (cc & 1) ? c0 - dc : c0 + dc;
      if (col < 0) col += cols;
      else if (col >= cols) col -= cols;
      const int j = row * cols + col;
      if (j == i) continue;
      if (consider(j) == 2) return 2;
    }
  }
  for (int v = 0; v < m; ++v)
    if (poly.L(v) < 0) return 1;
  const double th2 = ang.tan_half;
  return (t2R <= th2 * th2) ? 0 : 1;
}

// One direction's cell → valence and owned canonical triangles (i < both neighbours).
// Returns 0 ok, 2 polygon overflow (nothing written); 1 (not closed after every retry)
// marks the record as failed.
template <class PolyType>
__device__ int delaunay_point(const BuildParams& P, const Wave& W, int rec, int i, PolyType poly, int* own,
                              int* own_cnt) {
  const int n = P.n_angular;
  const double* dirs = W.dirs + (size_t)rec * n * 3;
  int m = 0;
  // search radius α = 2.8 × mean spacing: the security test needs α ≥ 2·R_cell, and on the
  // jittered stratum grid R_cell ≤ 1.4 spacing for > 99.8% of directions (max ≈ 1.6);
  // the rest retry with 1.5α
  int st = 1;
  for (int attempt = 0; attempt < kDelLevels && st == 1; ++attempt)
    st = voronoi_cell_poly(dirs, W.dirs32 + (size_t)rec * n, P.rows, P.cols, i, P.del[attempt], poly, m);
  if (st == 2) return 2;
  const size_t base = ((size_t)rec * n + i);
  W.deg[base] = (st == 0) ? m : 0;
  int c = 0;
  if (st == 0) {
    for (int t = 0; t < m; ++t) {
      int a = poly.L(t), b = poly.L(t + 1 == m ? 0 : t + 1);
      if (i < a && i < b) {
        if (c == kMaxV) {
          atomicMax(W.tri_status + rec, 2);
          break;
        }
        own_put(W, own, base, c, a, b);
        ++c;
      }
    }
  } else {
    atomicMax(W.tri_status + rec, st);
  }
  own_cnt[base] = c;
  return 0;
}

#ifndef VC_LB_DEL2
#define VC_LB_DEL2 5
#endif

__global__ void __launch_bounds__(kDelBS, VC_LB_DEL2) k_delaunay_smem(BuildParams P, Wave W, int* own, int* own_cnt) {
  extern __shared__ unsigned char dsm[];
  double* sa = (double*)dsm;
  double* sb = sa + kPolyV * kDelBS;
  int* sl = (int*)(sb + kPolyV * kDelBS);
  const int n = P.n_angular;
  long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)W.B * n) return;
  const int rec = (int)(gid / n);
  const int i = (int)(gid - (long long)rec * n);  // row-major: a warp shares one row's window shape
  Poly poly{sa + threadIdx.x, sb + threadIdx.x, sl + threadIdx.x};
  const int st = delaunay_point(P, W, rec, i, poly, own, own_cnt);
  if (st == 2) {  // polygon outgrew shared memory: queue for k_delaunay_retry
    const unsigned slot = atomicAdd(W.del_retry_count, 1u);
    if ((int)slot < W.del_retry_cap) W.del_retry[slot] = rec * n + i;
    else atomicMax(W.tri_status + rec, 2);
  }
}

// Cells that outgrew the shared-memory polygon, recomputed with a 48-vertex polygon in
// global memory (one slot per queued cell).
__global__ void __launch_bounds__(128) k_delaunay_retry(BuildParams P, Wave W, int* own, int* own_cnt,
                                                        double* scratch) {
  const unsigned nr = min(*W.del_retry_count, (unsigned)W.del_retry_cap);
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < nr; t += gridDim.x * blockDim.x) {
    const int gid = W.del_retry[t];
    const int rec = gid / P.n_angular, i = gid - rec * P.n_angular;
    double* a = scratch + (size_t)t * kRetryV * 3;
    PolyRetry poly{a, a + kRetryV, (int*)(a + 2 * kRetryV)};
    if (delaunay_point(P, W, rec, i, poly, own, own_cnt) != 0) atomicMax(W.tri_status + rec, 2);
  }
}

constexpr size_t kDelSmem = (size_t)kPolyV * kDelBS * (8 + 8 + 4);

// Clipping kernel over the cells the hull kernel handed back (grid-stride over the list).
__global__ void __launch_bounds__(kDelBS, VC_LB_DEL2) k_delaunay_list(BuildParams P, Wave W, int* own, int* own_cnt) {
  extern __shared__ unsigned char dsm[];
  double* sa = (double*)dsm;
  double* sb = sa + kPolyV * kDelBS;
  int* sl = (int*)(sb + kPolyV * kDelBS);
  const int n = P.n_angular;
  const unsigned cnt = *W.del_fb2_count;
  Poly poly{sa + threadIdx.x, sb + threadIdx.x, sl + threadIdx.x};
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
    const int gid = W.del_fb2[t];
    const int rec = gid / n, i = gid - rec * n;
    if (delaunay_point(P, W, rec, i, poly, own, own_cnt) == 2) {
      const unsigned slot = atomicAdd(W.del_retry_count, 1u);
      if ((int)slot < W.del_retry_cap) W.del_retry[slot] = gid;
      else atomicMax(W.tri_status + rec, 2);
    }
  }
}

// ---------------------------------------------------------------------------
// Stratum-window triangulation.  The Delaunay neighbours of p are the vertices of the
// convex hull of the other directions mapped by the stereographic projection from p,
//   u(q) = (e1·q, e2·q) / (1 − p·q),      1 − p·q = |p − q|² / 2,
// (circles through p become lines; a point inside the circumcircle of (p, a, b) lands
// beyond the line through u(a), u(b)), in counter-clockwise order about p.  One thread
// per direction gift-wraps the hull of the candidates of a fixed stratum window (rows
// r ± h, columns c ± w; uniform loop bounds across a warp, whose lanes share a row).
// The wrap compares orientations in float32 and flags any test within its error bound
// (|cross| ≤ 128·2⁻²⁴·max|u|²), so every decision it keeps is the exact one.  The cell is
// kept only if it is secure: for every Voronoi vertex v (circumcentre of p and two
// consecutive neighbours, radius R) the spherical cap of radius R about v stays inside
// the window — rows beyond the window lie beyond the parallels of its border rows, and
// columns beyond it in the two hemispheres cut off by its border meridians — so no
// direction outside the window can lie in any of the star's circumcircles.  Flagged,
// insecure or unclosed cells, and rows without a window (the polar caps), go to the
// clipping kernel (k_delaunay_list) through a list.
// ---------------------------------------------------------------------------
#ifndef VC_HULL_BS
#define VC_HULL_BS 128  // 64 / 256: 3.16 / 3.20 ms vs 3.15 ms per 512 records (Delaunay kernels)
#endif
constexpr int kHullBS = VC_HULL_BS;
constexpr int kHullH = 16;             // hull vertices
constexpr int kHullSlots = kHullK + 1;  // window candidates including the centre

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Stereographic projection of q from p onto the (e1, e2) plane, in float32 (five
// roundings relative to |u|); q = p gives NaN, which every later test ignores.
struct Proj {
  double px, py, pz, e1x, e1y, e1z, e2x, e2y, e2z;
  __device__ __forceinline__ Proj(double x, double y, double z) : px(x), py(y), pz(z) {
    double hx = 0.0, hy = 0.0, hz = 1.0;
    if (fabs(pz) >= 0.9) { hx = 1.0; hz = 0.0; }
    e1x = hy * pz - hz * py; e1y = hz * px - hx * pz; e1z = hx * py - hy * px;
    const double ne = rsqrt(e1x * e1x + e1y * e1y + e1z * e1z);
    e1x *= ne; e1y *= ne; e1z *= ne;
    e2x = py * e1z - pz * e1y; e2y = pz * e1x - px * e1z; e2z = px * e1y - py * e1x;
  }
  __device__ __forceinline__ float2 operator()(const double* q) const {
    const double d0 = px - q[0], d1 = py - q[1], d2 = pz - q[2];
    const float inv = 2.0f * rcp_approx((float)(d0 * d0 + d1 * d1 + d2 * d2));
    return make_float2((float)(-(e1x * d0 + e1y * d1 + e1z * d2)) * inv,
                       (float)(-(e2x * d0 + e2y * d1 + e2z * d2)) * inv);
  }
  // float64 projection (the fallback wrap)
  __device__ __forceinline__ double2 d2(const double* q) const {
    const double d0 = px - q[0], d1 = py - q[1], d2 = pz - q[2];
    const double inv = 2.0 / (d0 * d0 + d1 * d1 + d2 * d2);
    return make_double2(-(e1x * d0 + e1y * d1 + e1z * d2) * inv, -(e2x * d0 + e2y * d1 + e2z * d2) * inv);
  }
};

template <class T> struct Vec2;
template <> struct Vec2<float> {
  using V = float2;
  static constexpr float kEps = 5.9604645e-8f;  // 2⁻²⁴
  __device__ static V nan() { return make_float2(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000)); }
  __device__ static V proj(const Proj& pr, const double* q) { return pr(q); }
};
template <> struct Vec2<double> {
  using V = double2;
  static constexpr double kEps = 1.1102230246251565e-16;  // 2⁻⁵³
  __device__ static V nan() { return make_double2(__longlong_as_double(0x7ff8000000000000LL), __longlong_as_double(0x7ff8000000000000LL)); }
  __device__ static V proj(const Proj& pr, const double* q) { return pr.d2(q); }
};

// Counter-clockwise gift wrap of the projections us[0..K) (stride kHullBS) from `start`
// (a hull vertex).  Every orientation is compared in float32 and the smallest |cross| met
// must exceed `margin` (the float32 error bound), else the wrap fails (returns 0).  The
// current vertex and the initial candidate are parked as NaN during a scan, so the loop
// body is the same for every candidate (NaN never wins and never trips the bound).
// the wrap's candidate scan: u − a as one packed add and 8 candidates per loop trip — Delaunay
// class 12.05 → 11.71 ms per 2048 records (packed add alone 11.88, unroll 8 alone 11.77, 16: 11.71,
// 2: 12.82)
#ifndef VC_HULL_ADD2
#define VC_HULL_ADD2 1
#endif
#ifndef VC_HULL_UNROLL
#define VC_HULL_UNROLL 8
#endif
constexpr int kHullUnroll = VC_HULL_UNROLL;
template <class T, int BS>
__device__ __forceinline__ int gift_wrap(typename Vec2<T>::V* us, int K, int start, T nmax, unsigned char* hs) {
  using V = typename Vec2<T>::V;
  const V nan2 = Vec2<T>::nan();
  int hn = 0, cur = start;
  for (;;) {
    hs[hn * BS] = (unsigned char)cur;
    ++hn;
    const V a = us[cur * BS];
    T mn = (T)FLT_MAX;
    int b0 = cur;
    V b = nan2;
    do {  // the next candidate that is not NaN (the centre) as the initial best
      b0 = (b0 + 1 == K) ? 0 : b0 + 1;
      b = us[b0 * BS];
    } while (b.x != b.x && b0 != cur);
    us[cur * BS] = nan2;
    us[b0 * BS] = nan2;
    T bx = b.x - a.x, by = b.y - a.y;
    int best = b0;
#if VC_HULL_ADD2
    if constexpr (sizeof(T) == 4) {  // u − a as one packed add (sm_100a add.f32x2, same rounding)
      const float2 na = make_float2(-a.x, -a.y);
#pragma unroll kHullUnroll
      for (int c = 0; c < K; ++c) {
        const float2 u = us[c * BS];
        unsigned long long r;
        asm("add.rn.f32x2 %0, %1, %2;"
            : "=l"(r)
            : "l"(*reinterpret_cast<const unsigned long long*>(&u)),
              "l"(*reinterpret_cast<const unsigned long long*>(&na)));
        const float2 cc = *reinterpret_cast<float2*>(&r);
        const T cr = bx * cc.y - by * cc.x;
        mn = fmin(mn, fabs(cr));
        if (cr < (T)0) { best = c; bx = cc.x; by = cc.y; }
      }
    } else
#endif
    {
#pragma unroll kHullUnroll
    for (int c = 0; c < K; ++c) {
      const V u = us[c * BS];
      const T cx = u.x - a.x, cy = u.y - a.y;
      const T cr = bx * cy - by * cx;
      mn = fmin(mn, fabs(cr));
      if (cr < (T)0) { best = c; bx = cx; by = cy; }
    }
    }
    // float32 error bound of this step's orientations: each projection carries ≤ 5
    // roundings relative to its norm, so |err(cross)| ≤ 30·2⁻²⁴·(|a| + |b|)(|a| + |c|)
    // ≤ 32·2⁻²⁴·(|a|₁ + max|u|₁)²
    const T na = fabs(a.x) + fabs(a.y), la = na + nmax;
    if (!(mn > (T)32 * Vec2<T>::kEps * la * la)) {
      // rare: the step's tests again, each against its own bound 32·2⁻²⁴·(|a|₁+|b|₁)(|a|₁+|c|₁)
      // (every test outside its bound decides exactly, so both scans agree)
      T vx = b.x - a.x, vy = b.y - a.y, nb = fabs(b.x) + fabs(b.y);
      bool bad = false;
      for (int c = 0; c < K; ++c) {
        const V u = us[c * BS];
        const T cx = u.x - a.x, cy = u.y - a.y;
        const T cr = vx * cy - vy * cx;
        const T nc = fabs(u.x) + fabs(u.y);
        bad |= fabs(cr) <= (T)32 * Vec2<T>::kEps * (na + nb) * (na + nc);
        if (cr < (T)0) { vx = cx; vy = cy; nb = nc; }
      }
      if (bad) {
        us[cur * BS] = a;
        us[b0 * BS] = b;
        return 0;
      }
    }
    us[cur * BS] = a;
    us[b0 * BS] = b;
    if (best == start) break;
    if (hn == kHullH) return 0;
    cur = best;
  }
  return hn;
}

// X ≥ √Q  ⇔  X ≥ 0 ∧ X² ≥ Q
__device__ __forceinline__ bool ge_root(double X, double Q) { return X >= 0.0 && X * X >= Q; }

// Security and output of a wrapped star.  `gidx(slot)` maps a candidate slot to its
// direction, `secure(c, cp, Q, tol)` tests one Voronoi vertex (c ∝ v; |c| cos R = c·p,
// |c|² sin² R = Q).  Writes the valence and the owned triangles (i < both neighbours),
// as delaunay_point; false leaves the cell to the clipping kernel.
template <int BS, class GIdx, class Secure>
__device__ __forceinline__ bool hull_star(const Wave& W, const double* dirs, const Proj& pr, size_t base, int i,
                                          const unsigned char* hs, int hn, GIdx gidx, Secure secure, int* own,
                                          int* own_cnt) {
  if (hn < 3 || hn > kMaxV) return false;
  const double px = pr.px, py = pr.py, pz = pr.pz;
  const int g0 = gidx(hs[0]);
  int gb = g0;
  double bxd = dirs[3 * (size_t)gb] - px, byd = dirs[3 * (size_t)gb + 1] - py, bzd = dirs[3 * (size_t)gb + 2] - pz;
  for (int t = 0; t < hn; ++t) {
    const double ax = bxd, ay = byd, az = bzd;
    gb = (t + 1 == hn) ? g0 : gidx(hs[(t + 1) * BS]);
    bxd = dirs[3 * (size_t)gb] - px; byd = dirs[3 * (size_t)gb + 1] - py; bzd = dirs[3 * (size_t)gb + 2] - pz;
    const double cx = ay * bzd - az * byd, cy = az * bxd - ax * bzd, cz = ax * byd - ay * bxd;
    const double cp = cx * px + cy * py + cz * pz;
    const double xx = cy * pz - cz * py, xy = cz * px - cx * pz, xz = cx * py - cy * px;
    const double Q = xx * xx + xy * xy + xz * xz;
    const double tol = 1e-6 * (fabs(cx) + fabs(cy) + fabs(cz));
    if (!(cp > tol && secure(cx, cy, cz, cp, Q, tol))) return false;
  }
  int c = 0, ga = g0;
  for (int t = 0; t < hn; ++t) {
    const int gn = (t + 1 == hn) ? g0 : gidx(hs[(t + 1) * BS]);
    if (i < ga && i < gn) {
      own_put(W, own, base, c, ga, gn);
      ++c;
    }
    ga = gn;
  }
  W.deg[base] = hn;
  own_cnt[base] = c;
  return true;
}

template <class T, int BS>
__device__ __forceinline__ bool hull_cell(const BuildParams& P, const Wave& W, int rec, int i, typename Vec2<T>::V* us,
                                          unsigned char* hs, int* own, int* own_cnt) {
  const int n = P.n_angular, rows = P.rows, cols = P.cols;
  const int r0 = i / cols, c0 = i - r0 * cols;
  const int hw = r0 < kDelRowsMax ? P.del_hw[r0] : 0;
  if (!hw) return false;
  const int h = hw >> 6, w = hw & 63, wc = 2 * w + 1;
  const double* dirs = W.dirs + (size_t)rec * n * 3;
  const Proj pr(dirs[3 * (size_t)i], dirs[3 * (size_t)i + 1], dirs[3 * (size_t)i + 2]);
  // projected window candidates, row-major (the centre projects to NaN)
  int col0 = c0 - w;
  col0 += (col0 < 0) ? cols : 0;
  int K = 0, start = 0;
  T m2 = 0, n1 = 0;
  for (int dr = -h; dr <= h; ++dr) {
    const double* rowp = dirs + 3 * (size_t)(r0 + dr) * cols;
    const double* q = rowp + 3 * col0;
    const double* rowe = rowp + 3 * cols;
    for (int dc = 0; dc < wc; ++dc) {
      const auto u = Vec2<T>::proj(pr, q);
      us[K * BS] = u;
      const T r2 = u.x * u.x + u.y * u.y;
      if (r2 > m2) { m2 = r2; start = K; }
      n1 = fmax(n1, fabs(u.x) + fabs(u.y));
      ++K;
      q += 3;
      q = (q == rowe) ? rowp : q;
    }
  }
  const int hn = gift_wrap<T, BS>(us, K, start, n1, hs);
  // candidate k → direction index (k / wc by a 16-bit reciprocal, exact for k < 2¹⁶/wc²)
  const unsigned rwc = (65536u + wc - 1) / wc;
  auto gidx = [&](int k) {
    const int a = (int)(((unsigned)k * rwc) >> 16);
    int col = col0 + (k - a * wc);
    col -= (col >= cols) ? cols : 0;
    return (r0 - h + a) * cols + col;
  };
  // security: the cap about each Voronoi vertex stays on the window side of both border
  // meridians (distance asin(v·n) ≥ R) and between the border parallels (|θ_v − θ| ≥ R)
  const bool top = r0 - h > 0, bot = r0 + h < rows - 1;
  const double zt = 1.0 - P.del_zstep * (r0 - h), zb = 1.0 - P.del_zstep * (r0 + h + 1);
  const double st2 = fmax(0.0, 1.0 - zt * zt), sb2 = fmax(0.0, 1.0 - zb * zb);
  double shi, chi, slo, clo;
  sincospi(2.0 * (c0 + w + 1) / cols, &shi, &chi);
  sincospi(2.0 * (c0 - w) / cols, &slo, &clo);
  auto secure = [&](double cx, double cy, double cz, double cp, double Q, double tol) {
    bool ok = ge_root(cx * shi - cy * chi - tol, Q) && ge_root(cy * clo - cx * slo - tol, Q);
    if (top) ok &= ge_root(zt * cp - cz - tol, st2 * Q);
    if (bot) ok &= ge_root(cz - zb * cp - tol, sb2 * Q);
    return ok;
  };
  return hull_star<BS>(W, dirs, pr, (size_t)rec * n + i, i, hs, hn, gidx, secure, own, own_cnt);
}

// One launch per window class: thread → (record, row of the class, column).
__global__ void __launch_bounds__(kHullBS) k_delaunay_hull(BuildParams P, Wave W, int* own, int* own_cnt, int cls) {
  extern __shared__ float2 hsm[];
  unsigned char* hs = (unsigned char*)(hsm + (P.del_cls_k[cls] + 1) * kHullBS) + threadIdx.x;
  const int n = P.n_angular, cols = P.cols;
  const int nr = P.del_cls[cls + 1] - P.del_cls[cls];
  const long long gid = (long long)blockIdx.x * kHullBS + threadIdx.x;
  bool fb = false;
  int cell = 0;
  if (gid < (long long)W.B * nr * cols) {
    const int rec = (int)(gid / ((long long)nr * cols));
    const int rem = (int)(gid - (long long)rec * nr * cols);
    const int rs = rem / cols;
    const int i = (int)P.del_rows[P.del_cls[cls] + rs] * cols + (rem - rs * cols);
    cell = rec * n + i;
    fb = !hull_cell<float, kHullBS>(P, W, rec, i, hsm + threadIdx.x, hs, own, own_cnt);
  }
  const unsigned m = __ballot_sync(0xffffffffu, fb);
  if (m) {
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    unsigned slot = 0;
    if (lane == leader) slot = atomicAdd(W.del_fb_count, (unsigned)__popc(m));
    slot = __shfl_sync(0xffffffffu, slot, leader);
    if (fb) W.del_fb[slot + __popc(m & ((1u << lane) - 1u))] = cell;
  }
}

// Rows that neither the hull classes nor the cap kernel take (no window, cap kernel off)
// go to the clipping kernel directly.
__global__ void k_delaunay_rest(BuildParams P, Wave W) {
  const int n = P.n_angular, cols = P.cols;
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  bool fb = false;
  int cell = 0;
  if (gid < (long long)W.B * n) {
    const int rec = (int)(gid / n);
    const int i = (int)(gid - (long long)rec * n);
    const int r0 = i / cols;
    const bool cap = P.del_cap && (r0 == 0 || r0 == P.rows - 1);
    fb = !cap && (r0 >= kDelRowsMax || P.del_hw[r0] == 0);
    cell = rec * n + i;
  }
  const unsigned m = __ballot_sync(0xffffffffu, fb);
  if (m) {
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    unsigned slot = 0;
    if (lane == leader) slot = atomicAdd(W.del_fb_count, (unsigned)__popc(m));
    slot = __shfl_sync(0xffffffffu, slot, leader);
    if (fb) W.del_fb[slot + __popc(m & ((1u << lane) - 1u))] = cell;
  }
}

// The polar rows (0 and rows − 1), whose strata meet at the pole: the candidates are the
// directions of the two cap rows within angle δ of p (a float32 dot pre-test with margin,
// compacted into shared memory with their indices); besides the parallel below the two
// rows, the security test asks R ≤ δ/2 of every Voronoi vertex, so no skipped direction
// (farther than δ from p) can reach a circumcircle.
constexpr int kCapSlots = 40;
constexpr size_t kCapSmem = (size_t)kHullBS * (kCapSlots * (sizeof(float2) + 2) + kHullH);

// Candidate radius δ of a cap cell: cos δ and sin δ (pre-test, column range) and
// cos²(δ/2), sin²(δ/2) (security R ≤ δ/2).
struct CapRadius {
  float cos_d, sin_d;
  double c2, s2;
};

// One polar-row cell i of record rec (see k_delaunay_cap) with up to `slots` candidates.
// One polar-row cell i of record rec (see k_delaunay_cap) with up to `slots` candidates.
template <class T, int BS>
__device__ __forceinline__ bool cap_cell(const BuildParams& P, const Wave& W, int rec, int i, const CapRadius& cr,
                                         int slots, typename Vec2<T>::V* us, unsigned short* ix, unsigned char* hs,
                                         int* own, int* own_cnt) {
  const int n = P.n_angular, rows = P.rows, cols = P.cols;
  const bool north = i < cols;
  const int rlo = north ? 0 : rows - 2;  // the two cap rows
  const double* dirs = W.dirs + (size_t)rec * n * 3;
  const float4* d32 = W.dirs32 + (size_t)rec * n;
  const Proj pr(dirs[3 * (size_t)i], dirs[3 * (size_t)i + 1], dirs[3 * (size_t)i + 2]);
  const float4 p32 = d32[i];
  const float cutf = cr.cos_d - 1e-6f;
  int K = 0, start = 0;
  T m2 = 0, n1 = 0;
  // columns within the azimuth half-width asin(sin δ / sin θ_p) of p's stratum column
  // (the whole row when the δ-disc holds the pole), one column of slack either side
  const int c0 = i - (north ? 0 : (rows - 1) * cols);
  const float stp = sqrtf(p32.x * p32.x + p32.y * p32.y);
  int half = cols;
  if (stp > 1.01f * cr.sin_d) half = (int)ceilf(asinf(cr.sin_d / stp) * (float)cols * 0.15915494f) + 1;
  const int span = (2 * half + 1 >= cols) ? cols : 2 * half + 1;
  int cstart = (span == cols) ? 0 : c0 - half;
  cstart += (cstart < 0) ? cols : 0;
  for (int rr = rlo; rr < rlo + 2; ++rr) {
    int col = cstart;
    for (int t = 0; t < span; ++t) {
      const int j = rr * cols + col;
      col = (col + 1 == cols) ? 0 : col + 1;
      const float4 q = d32[j];
      if (p32.x * q.x + p32.y * q.y + p32.z * q.z > cutf) {
        if (K == slots) return false;
        const auto u = Vec2<T>::proj(pr, dirs + 3 * (size_t)j);
        us[K * BS] = u;
        ix[K * BS] = (unsigned short)(j - rlo * cols);
        const T r2 = u.x * u.x + u.y * u.y;
        if (r2 > m2) { m2 = r2; start = K; }
        n1 = fmax(n1, fabs(u.x) + fabs(u.y));
        ++K;
      }
    }
  }
  const int hn = gift_wrap<T, BS>(us, K, start, n1, hs);
  auto gidx = [&](int s) { return rlo * cols + (int)ix[s * BS]; };
  // the parallel below (north) / above (south) the two cap rows
  const double zb = north ? 1.0 - 2.0 * P.del_zstep : 1.0 - P.del_zstep * (rows - 2);
  const double sb2 = fmax(0.0, 1.0 - zb * zb);
  auto secure = [&](double cx, double cy, double cz, double cp, double Q, double tol) {
    bool ok = (cp - tol) * (cp - tol) * cr.s2 >= cr.c2 * Q;  // R ≤ δ/2
    ok &= north ? ge_root(cz - zb * cp - tol, sb2 * Q) : ge_root(zb * cp - cz - tol, sb2 * Q);
    return ok;
  };
  return hull_star<BS>(W, dirs, pr, (size_t)rec * n + i, i, hs, hn, gidx, secure, own, own_cnt);
}

__global__ void __launch_bounds__(kHullBS) k_delaunay_cap(BuildParams P, Wave W, int* own, int* own_cnt) {
  extern __shared__ float2 csm[];
  unsigned short* ix0 = (unsigned short*)(csm + kCapSlots * kHullBS);
  unsigned char* hs = (unsigned char*)(ix0 + kCapSlots * kHullBS) + threadIdx.x;
  const int n = P.n_angular, rows = P.rows, cols = P.cols;
  const long long gid = (long long)blockIdx.x * kHullBS + threadIdx.x;  // over B × 2 × cols
  bool fb = false;
  int cell = -1;
  if (gid < (long long)W.B * 2 * cols) {
    const int rec = (int)(gid / (2 * cols));
    const int k = (int)(gid - (long long)rec * 2 * cols);
    const int i = k < cols ? k : (rows - 1) * cols + (k - cols);
    cell = rec * n + i;
    const CapRadius cr{P.del_cap_cos, P.del_cap_sin, P.del_cap_c2, P.del_cap_s2};
    fb = !cap_cell<float, kHullBS>(P, W, rec, i, cr, kCapSlots, csm + threadIdx.x, ix0 + threadIdx.x, hs, own,
                                   own_cnt);
  }
  const unsigned m = __ballot_sync(0xffffffffu, fb);
  if (m) {
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    unsigned slot = 0;
    if (lane == leader) slot = atomicAdd(W.del_fb_count, (unsigned)__popc(m));
    slot = __shfl_sync(0xffffffffu, slot, leader);
    if (fb) W.del_fb[slot + __popc(m & ((1u << lane) - 1u))] = cell;
  }
}

// Binned cap kernel.  k_cap_bin (one CTA per record and pole): the 2·cols directions of
// the two cap rows are counting-sorted into a G × G grid over their (x, y) coordinates (cells at least
// ρ wide, ρ ≥ the chord length of the δ pre-test), so a polar cell scans the ≤ 3 × 3 bins
// around it instead of every column within its azimuth range — the whole two rows for the
// ~11 % of cells whose δ-disc holds the pole, which set the pace of nearly every warp.
// k_delaunay_capg (thread per polar cell): same candidate set (the float32 pre-test
// decides), same wrap and security test as k_delaunay_cap.
constexpr int kCapGBS = 128;
constexpr size_t kCapBinSmem = sizeof(int) * (2 * kCapGMax * kCapGMax + 1) + 2 * sizeof(unsigned short) * 2 * kCapGCols;

struct CapGrid {
  int G;
  float x0, inv, rho;
  __device__ __forceinline__ int bin(float v) const {  // monotone in v (clamped)
    const int b = (int)floorf((v - x0) * inv);
    return min(max(b, 0), G - 1);
  }
};

// Grid of the binned cap kernel (false: use the column-range kernel).  ρ bounds the
// float32 chord |p − q| of every pair passing the pre-test p·q > cos δ − 1e-6 (with margin);
// the grid spans the cap rows' |x|, |y| ≤ sin θ of their lower parallel.
static bool cap_grid(const BuildParams& P, CapGrid& cg) {
  const char* env = getenv("VOLCACHE_CAP_GRID");
  if ((env && env[0] == '0') || P.cols > kCapGCols || P.host_adjacency) return false;
  const double cd = (double)P.del_cap_cos;
  const double rho = 1.001 * std::sqrt(2.0 * (1.0 - cd) + 4e-6);
  const double zl = 1.0 - 2.0 * P.del_zstep;
  const double gr = 1.001 * std::sqrt(std::max(0.0, 1.0 - zl * zl)) + 1e-6;
  const int G = std::min(kCapGMax, std::max(1, (int)std::floor(2.0 * gr / rho)));
  cg.G = G;
  cg.x0 = (float)-gr;
  cg.inv = (float)(G / (2.0 * gr));
  cg.rho = (float)rho;
  return true;
}

template <class T, int BS>
__device__ __forceinline__ bool cap_cell_binned(const BuildParams& P, const Wave& W, int rec, int i,
                                                const CapRadius& cr, const CapGrid& cg, const int* bstart,
                                                const unsigned short* sorted, typename Vec2<T>::V* us,
                                                unsigned short* ix, unsigned char* hs, int* own, int* own_cnt) {
  const int n = P.n_angular, rows = P.rows, cols = P.cols;
  const bool north = i < cols;
  const int rlo = north ? 0 : rows - 2;
  const double* dirs = W.dirs + (size_t)rec * n * 3;
  const float4* d32 = W.dirs32 + (size_t)rec * n;
  const float4* c32 = d32 + (size_t)rlo * cols;
  const Proj pr(dirs[3 * (size_t)i], dirs[3 * (size_t)i + 1], dirs[3 * (size_t)i + 2]);
  const float4 p32 = d32[i];
  const float cutf = cr.cos_d - 1e-6f;
  int K = 0, start = 0;
  T m2 = 0, n1 = 0;
  const int bx0 = cg.bin(p32.x - cg.rho), bx1 = cg.bin(p32.x + cg.rho);
  const int by0 = cg.bin(p32.y - cg.rho), by1 = cg.bin(p32.y + cg.rho);
  for (int by = by0; by <= by1; ++by) {
    // bins bx0..bx1 of one grid row are contiguous in the sorted list
    const int a = bstart[by * cg.G + bx0], b = bstart[by * cg.G + bx1 + 1];
    for (int t = a; t < b; ++t) {
      const int jl = sorted[t];
      const float4 q = c32[jl];
      if (p32.x * q.x + p32.y * q.y + p32.z * q.z > cutf) {
        if (K == kCapSlots) return false;
        const auto u = Vec2<T>::proj(pr, dirs + 3 * ((size_t)rlo * cols + jl));
        us[K * BS] = u;
        ix[K * BS] = (unsigned short)jl;
        const T r2 = u.x * u.x + u.y * u.y;
        if (r2 > m2) { m2 = r2; start = K; }
        n1 = fmax(n1, fabs(u.x) + fabs(u.y));
        ++K;
      }
    }
  }
  const int hn = gift_wrap<T, BS>(us, K, start, n1, hs);
  auto gidx = [&](int s) { return rlo * cols + (int)ix[s * BS]; };
  const double zb = north ? 1.0 - 2.0 * P.del_zstep : 1.0 - P.del_zstep * (rows - 2);
  const double sb2 = fmax(0.0, 1.0 - zb * zb);
  auto secure = [&](double cx, double cy, double cz, double cp, double Q, double tol) {
    bool ok = (cp - tol) * (cp - tol) * cr.s2 >= cr.c2 * Q;  // R ≤ δ/2
    ok &= north ? ge_root(cz - zb * cp - tol, sb2 * Q) : ge_root(zb * cp - cz - tol, sb2 * Q);
    return ok;
  };
  return hull_star<BS>(W, dirs, pr, (size_t)rec * n + i, i, hs, hn, gidx, secure, own, own_cnt);
}

// Counting sort of one (record, pole)'s cap-row directions by bin → W.cap_bins:
// G² + 1 bin starts, then the 2·cols row-local indices in bin order.
__global__ void __launch_bounds__(kCapGBS) k_cap_bin(BuildParams P, Wave W, CapGrid cg) {
  extern __shared__ int bsm[];
  int* bcur = bsm;                                   // G²
  unsigned short* binof = (unsigned short*)(bsm + kCapGMax * kCapGMax);
  const int n = P.n_angular, rows = P.rows, cols = P.cols;
  const int rec = blockIdx.x >> 1;
  const bool north = !(blockIdx.x & 1);
  const int rlo = north ? 0 : rows - 2;
  const int np = 2 * cols, nb = cg.G * cg.G;
  const float4* c32 = W.dirs32 + (size_t)rec * n + (size_t)rlo * cols;
  int* out = W.cap_bins + (size_t)blockIdx.x * W.cap_bin_stride;
  unsigned short* sorted = (unsigned short*)(out + kCapGMax * kCapGMax + 1);
  for (int b = threadIdx.x; b < nb; b += kCapGBS) bcur[b] = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < np; j += kCapGBS) {
    const float4 q = c32[j];
    const int b = cg.bin(q.y) * cg.G + cg.bin(q.x);
    binof[j] = (unsigned short)b;
    atomicAdd(&bcur[b], 1);
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive scan of the bin counts (warp 0, 32 bins per pass)
    const int lane = threadIdx.x;
    int base = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int v = (b0 + lane < nb) ? bcur[b0 + lane] : 0;
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (b0 + lane < nb) {
        out[b0 + lane] = base + x - v;
        bcur[b0 + lane] = base + x - v;
      }
      base += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) out[nb] = base;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < np; j += kCapGBS) sorted[atomicAdd(&bcur[binof[j]], 1)] = (unsigned short)j;
}

// Thread per polar cell (as k_delaunay_cap), candidates from the bins of k_cap_bin.
__global__ void __launch_bounds__(kHullBS) k_delaunay_capg(BuildParams P, Wave W, int* own, int* own_cnt,
                                                           CapGrid cg) {
  extern __shared__ float2 csm[];
  unsigned short* ix0 = (unsigned short*)(csm + kCapSlots * kHullBS);
  unsigned char* hs = (unsigned char*)(ix0 + kCapSlots * kHullBS) + threadIdx.x;
  const int n = P.n_angular, rows = P.rows, cols = P.cols;
  const long long gid = (long long)blockIdx.x * kHullBS + threadIdx.x;  // over B × 2 × cols
  bool fb = false;
  int cell = -1;
  if (gid < (long long)W.B * 2 * cols) {
    const int rec = (int)(gid / (2 * cols));
    const int k = (int)(gid - (long long)rec * 2 * cols);
    const bool north = k < cols;
    const int i = north ? k : (rows - 1) * cols + (k - cols);
    cell = rec * n + i;
    const int* bins = W.cap_bins + (size_t)(2 * rec + (north ? 0 : 1)) * W.cap_bin_stride;
    const CapRadius cr{P.del_cap_cos, P.del_cap_sin, P.del_cap_c2, P.del_cap_s2};
    fb = !cap_cell_binned<float, kHullBS>(P, W, rec, i, cr, cg, bins,
                                          (const unsigned short*)(bins + kCapGMax * kCapGMax + 1),
                                          csm + threadIdx.x, ix0 + threadIdx.x, hs, own, own_cnt);
  }
  const unsigned m = __ballot_sync(0xffffffffu, fb);
  if (m) {
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    unsigned slot = 0;
    if (lane == leader) slot = atomicAdd(W.del_fb_count, (unsigned)__popc(m));
    slot = __shfl_sync(0xffffffffu, slot, leader);
    if (fb) W.del_fb[slot + __popc(m & ((1u << lane) - 1u))] = cell;
  }
}

// Cells the float32 kernels hand back (an orientation within the float32 error bound, a
// star not certified by its window or disc, a polar cell past the cap kernel's radius):
// one warp per cell in float64.  Candidates are the directions within δ of p (lanes over
// the stratum rows and columns that can hold them, ballot-compacted into the warp's
// shared memory); each gift-wrap step is a warp reduction under the orientation order
// (from a hull vertex every other projection lies in a half-plane, so "more clockwise" is
// a strict order); the star is kept when every circumradius R ≤ δ/2, else δ grows towards
// 2.05·max R (by 1.2× to 1.6×) and the cell is redone (at most 5 radii, ≤ kWarpK
// candidates).  Cells still
// open go to the clipping kernel (second list).
constexpr int kWarpK = 320;
constexpr int kWarpBS = 256;
constexpr size_t kWarpSmem = (size_t)(kWarpBS / 32) * (kWarpK * (sizeof(double2) + 4) + kHullH * 4);

__device__ bool warp_cell(const BuildParams& P, const Wave& W, int rec, int i, double2* us, int* ix, int* hs,
                          int* own, int* own_cnt) {
  const int lane = threadIdx.x & 31;
  const int n = P.n_angular, rows = P.rows, cols = P.cols;
  const double* dirs = W.dirs + (size_t)rec * n * 3;
  const float4* d32 = W.dirs32 + (size_t)rec * n;
  const double px = dirs[3 * (size_t)i], py = dirs[3 * (size_t)i + 1], pz = dirs[3 * (size_t)i + 2];
  const Proj pr(px, py, pz);
  const float4 p32 = d32[i];
  const double st = sqrt(fmax(0.0, 1.0 - pz * pz));
  double delta = P.del_warp_delta;
  for (int attempt = 0; attempt < 5; ++attempt) {
    const double cd = cos(delta), sd = sin(delta);
    const float cutf = (float)cd - 1e-6f;
    // stratum rows meeting z ∈ [cos(θ + δ), cos(θ − δ)], columns within asin(sin δ / sin θ)
    const bool pole_n = st <= sd && pz > 0.0, pole_s = st <= sd && pz < 0.0;
    auto row_of = [&](double z) { return min(max((int)floor((1.0 - z) * rows * 0.5), 0), rows - 1); };
    const int ra = pole_n ? 0 : row_of(pz * cd + st * sd + 1e-9);
    const int rb = pole_s ? rows - 1 : row_of(pz * cd - st * sd - 1e-9);
    const int c0 = i % cols;
    int half = cols;
    if (!pole_n && !pole_s) half = (int)ceil(asin(fmin(1.0, sd / st)) * cols * 0.15915494309189535) + 1;
    const int span = (2 * half + 1 >= cols) ? cols : 2 * half + 1;
    int cstart = (span == cols) ? 0 : c0 - half;
    cstart += (cstart < 0) ? cols : 0;
    const int total = (rb - ra + 1) * span;
    int K = 0;
    for (int t0 = 0; t0 < total; t0 += 32) {
      const int t = t0 + lane;
      bool take = false;
      int j = 0;
      if (t < total) {
        const int rr = ra + t / span;
        int col = cstart + t % span;
        col -= (col >= cols) ? cols : 0;
        j = rr * cols + col;
        const float4 q = d32[j];
        take = p32.x * q.x + p32.y * q.y + p32.z * q.z > cutf && j != i;
      }
      const unsigned m = __ballot_sync(0xffffffffu, take);
      const int pos = K + __popc(m & ((1u << lane) - 1u));
      if (take && pos < kWarpK) {
        us[pos] = pr.d2(dirs + 3 * (size_t)j);
        ix[pos] = j;
      }
      K += __popc(m);
    }
    if (K > kWarpK || K < 3) {
      if (P.del_dbg_cell == rec * n + i && lane == 0) printf("warp_cell: K=%d delta=%g\n", K, delta);
      return false;
    }
    __syncwarp();
    // start: the largest projection (nearest direction), a hull vertex; L1 bound N
    double best_r = -1.0, nmax = 0.0;
    int start = -1;
    for (int c = lane; c < K; c += 32) {
      const double2 u = us[c];
      const double r = u.x * u.x + u.y * u.y;
      nmax = fmax(nmax, fabs(u.x) + fabs(u.y));
      if (r > best_r) { best_r = r; start = c; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double r2 = __shfl_xor_sync(0xffffffffu, best_r, o);
      const int s2 = __shfl_xor_sync(0xffffffffu, start, o);
      if (r2 > best_r || (r2 == best_r && s2 < start)) { best_r = r2; start = s2; }
      nmax = fmax(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
    }
    // gift wrap, one warp reduction per step
    int hn = 0, cur = start;
    bool bad = false;
    for (;;) {
      if (lane == 0) hs[hn] = cur;
      ++hn;
      const double2 a = us[cur];
      const double la = fabs(a.x) + fabs(a.y) + nmax;
      const double margin = 32.0 * 1.1102230246251565e-16 * la * la;
      int b = -1;
      double bx = 0.0, by = 0.0;
      for (int c = lane; c < K; c += 32) {
        if (c == cur) continue;
        const double2 u = us[c];
        const double cx = u.x - a.x, cy = u.y - a.y;
        if (b < 0) { b = c; bx = cx; by = cy; continue; }
        const double cr = bx * cy - by * cx;
        bad |= fabs(cr) <= margin;
        if (cr < 0.0) { b = c; bx = cx; by = cy; }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const int b2 = __shfl_xor_sync(0xffffffffu, b, o);
        const double x2 = __shfl_xor_sync(0xffffffffu, bx, o), y2 = __shfl_xor_sync(0xffffffffu, by, o);
        if (b2 >= 0) {
          if (b < 0) { b = b2; bx = x2; by = y2; }
          else if (b2 != b) {
            const double cr = bx * y2 - by * x2;
            bad |= fabs(cr) <= margin;
            // keep the more clockwise; both lanes of a pair must agree
            if (cr < 0.0 || (cr == 0.0 && b2 < b)) { b = b2; bx = x2; by = y2; }
          }
        }
      }
      if (__any_sync(0xffffffffu, bad)) {
        if (P.del_dbg_cell == rec * n + i && lane == 0) printf("warp_cell: flagged step %d K=%d\n", hn, K);
        return false;
      }
      if (b == start) break;
      if (hn == kHullH) {
        if (P.del_dbg_cell == rec * n + i && lane == 0) printf("warp_cell: hull overflow K=%d\n", K);
        return false;
      }
      cur = b;
    }
    __syncwarp();
    if (hn < 3 || hn > kMaxV) {
      if (P.del_dbg_cell == rec * n + i && lane == 0) printf("warp_cell: hn=%d\n", hn);
      return false;
    }
    // security: every circumradius R ≤ δ/2 (c ∝ Voronoi vertex: tan² R = Q / (c·p)²)
    const double c2 = cos(0.5 * delta) * cos(0.5 * delta), s2 = sin(0.5 * delta) * sin(0.5 * delta);
    bool ok = true;
    double tmax = 0.0;
    if (lane < hn) {
      const int ga = ix[hs[lane]], gb = ix[hs[lane + 1 == hn ? 0 : lane + 1]];
      const double ax = dirs[3 * (size_t)ga] - px, ay = dirs[3 * (size_t)ga + 1] - py, az = dirs[3 * (size_t)ga + 2] - pz;
      const double bx = dirs[3 * (size_t)gb] - px, by = dirs[3 * (size_t)gb + 1] - py, bz = dirs[3 * (size_t)gb + 2] - pz;
      const double cx = ay * bz - az * by, cy = az * bx - ax * bz, cz = ax * by - ay * bx;
      const double cp = cx * px + cy * py + cz * pz;
      const double xx = cy * pz - cz * py, xy = cz * px - cx * pz, xz = cx * py - cy * px;
      const double Q = xx * xx + xy * xy + xz * xz;
      const double tol = 1e-6 * (fabs(cx) + fabs(cy) + fabs(cz));
      ok = cp > tol && (cp - tol) * (cp - tol) * s2 >= c2 * Q;
      tmax = cp > tol ? Q / (cp * cp) : INFINITY;
    }
    const bool all_ok = __all_sync(0xffffffffu, ok);
#pragma unroll
    for (int o = 16; o; o >>= 1) tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
    if (all_ok) {
      if (lane == 0) {
        const size_t base = (size_t)rec * n + i;
        int c = 0;
        for (int t = 0; t < hn; ++t) {
          const int ga = ix[hs[t]], gn = ix[hs[t + 1 == hn ? 0 : t + 1]];
          if (i < ga && i < gn) {
            own_put(W, own, base, c, ga, gn);
            ++c;
          }
        }
        W.deg[base] = hn;
        own_cnt[base] = c;
      }
      __syncwarp();
      return true;
    }
    if ((P.del_dbg_cell == rec * n + i && lane == 0)) printf("warp_cell: insecure delta=%g tmax=%g hn=%d K=%d\n", delta, tmax, hn, K);
    if (!(tmax < INFINITY)) return false;
    // a far circumcentre usually means a neighbour beyond δ: grow by at most 1.6×
    delta = fmin(1.6 * delta, fmax(1.2 * delta, 2.05 * atan(sqrt(tmax))));
    if (delta > 1.5) return false;
    __syncwarp();
  }
  return false;
}

__global__ void __launch_bounds__(kWarpBS) k_delaunay_warp(BuildParams P, Wave W, int* own, int* own_cnt) {
  extern __shared__ unsigned char wsm[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* us = (double2*)wsm + wid * kWarpK;
  int* ix = (int*)((double2*)wsm + (kWarpBS / 32) * kWarpK) + wid * kWarpK;
  int* hs = (int*)((double2*)wsm + (kWarpBS / 32) * kWarpK) + (kWarpBS / 32) * kWarpK + wid * kHullH;
  const int n = P.n_angular;
  const unsigned cnt = *W.del_fb_count;
  for (unsigned t = blockIdx.x * (kWarpBS / 32) + wid; t < cnt; t += gridDim.x * (kWarpBS / 32)) {
    const int cell = W.del_fb[t];
    const int rec = cell / n, i = cell - rec * n;
    if (!warp_cell(P, W, rec, i, us, ix, hs, own, own_cnt) && lane == 0) {
      const unsigned slot = atomicAdd(W.del_fb2_count, 1u);
      W.del_fb2[slot] = cell;
    }
    __syncwarp();
  }
}

constexpr int kCompactBS = 512;

// Canonical triangle list in two launches: k_own_scan (CTA per record) turns the owned
// counts into exclusive offsets (4 cells per thread, one block scan per 4·kCompactBS
// cells), k_tri_scatter (thread per cell) copies each cell's owned triangles to its offset.
__global__ void __launch_bounds__(kCompactBS) k_own_scan(BuildParams P, Wave W, const int* own_cnt, int* off) {
  __shared__ long long sm[kCompactBS / 32 + 1];
  const int rec = blockIdx.x, n = P.n_angular;
  const int* cnt = own_cnt + (size_t)rec * n;
  int* o = off + (size_t)rec * n;
  long long run = 0;
  for (int base = 0; base < n; base += 4 * kCompactBS) {
    const int i = base + 4 * threadIdx.x;
    int c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) c[u] = (i + u < n) ? cnt[i + u] : 0;
    long long tot;
    long long pre = run + block_exscan<kCompactBS>(c[0] + c[1] + c[2] + c[3], tot, sm);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (i + u < n) o[i + u] = (int)pre;
      pre += c[u];
    }
    run += tot;
  }
  if (threadIdx.x == 0 && run != P.n_tris) atomicMax(W.tri_status + rec, 3);
}

__global__ void k_tri_scatter(BuildParams P, Wave W, const int* own, const int* own_cnt, const int* off) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int n = P.n_angular;
  if (gid >= (long long)W.B * n) return;
  const int rec = (int)(gid / n), i = (int)(gid - (long long)rec * n);
  const int c = own_cnt[gid];
  const int o0 = off[gid];
  int* tris = W.tris + (size_t)rec * P.n_tris * 3;
  const int2* o2 = (const int2*)own + gid;
  for (int t = 0; t < c; ++t) {
    const int o = o0 + t;
    if (o < P.n_tris) {
      const int2 ab = o2[(size_t)t * W.own_stride];
      tris[o * 3 + 0] = i;
      tris[o * 3 + 1] = ab.x;
      tris[o * 3 + 2] = ab.y;
    }
  }
}

// Vertex valence of caller-supplied triangles (star counting).
__global__ void k_degree(BuildParams P, Wave W) {
  long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long tot = (long long)W.B * P.n_tris;
  if (gid >= tot) return;
  int rec = (int)(gid / P.n_tris);
  const int* t = W.tris + gid * 3;
  for (int v = 0; v < 3; ++v) atomicAdd(W.deg + (size_t)rec * P.n_angular + t[v], 1);
}

// ---------------------------------------------------------------------------
// Moment assembly (src/subdivision.py:287-370)
// ---------------------------------------------------------------------------

constexpr int kQCap = 64;
// 3D element math in float32 (float64 ok-mask; per-round warp sums in float32, accumulated
// over rounds in float64); 0: float64 throughout
#ifndef VC_ASM_F32
#define VC_ASM_F32 1
#endif
template <int D>
using AsmT = typename std::conditional<D == 3 && VC_ASM_F32, float, double>::type;
#ifndef VC_ASM_MINB
#define VC_ASM_MINB (512 / VC_ASM_BS)  // resident CTAs per SM → ≤ 128 registers
#endif

template <int D>
struct ElemView {
  int v[D];
};

template <int D>
__device__ __forceinline__ void elem_vertices(const Wave& W, const BuildParams& P, int rec, int e, int* v) {
  if constexpr (D == 2) {
    v[0] = e;
    v[1] = (e + 1 == P.n_angular) ? 0 : e + 1;
  } else {
    const int* t = W.tris + ((size_t)rec * P.n_tris + e) * 3;
    v[0] = t[0];
    v[1] = t[1];
    v[2] = t[2];
  }
}


// Per-record inputs of the element contributions.
template <int D>
struct AsmCtx {
  const double* dirs;
  const DirInfo* info;   // s and live-ring count of a direction in one 16-byte load
  const double* sv;
  const int* cnt;
  const int* pre;
  const double* lo;
  const int* idx;          // with emit: surface radiance = emit[idx[v]] (non-reflective scenes)
  const double* emit;
  const float* media;
  double x[3];
  double step;
};

template <int D>
__device__ __forceinline__ AsmCtx<D> asm_ctx(const BuildParams& P, const Wave& W, int rec) {
  const size_t rb = (size_t)rec * P.n_angular;
  AsmCtx<D> c;
  c.dirs = W.dirs + rb * D;
  c.info = W.info + rb;
  c.sv = W.s + rb;
  c.cnt = W.cnt + rb;
  c.pre = W.pre + rb;
  c.lo = W.lo + rb * 3;
  c.idx = W.idx + rb;
  c.emit = W.emit_tab;
  c.media = W.media + (size_t)W.rec_base[rec] * 3;
#pragma unroll
  for (int a = 0; a < D; ++a) c.x[a] = W.x[rec * D + a];
  c.step = P.march_step;
  return c;
}

// Contribution (3·NQ components, c·NQ + t) of element v[] at `ring` with representative
// vertex slot `rep` (src/subdivision.py:318-366); false = degenerate element (dropped).
template <int D, class CT>
__device__ __forceinline__ bool asm_item(const DevScene& S, const AsmCtx<D>& C, int kind, double wt, const int* v,
                                         int ring, int rep, CT (&cvec)[32]) {
  constexpr int NQ = 1 + D + D * (D + 1) / 2;
  double rv[D][3];
  double dist[D];
  const double ri = (kind == 1) ? ring_radius(ring, C.step) : 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const DirInfo di = C.info[v[j]];
    const bool live = (kind == 1) && (ring < di.cnt);
    dist[j] = live ? ri : di.s;
#pragma unroll
    for (int a = 0; a < D; ++a) rv[j][a] = dist[j] * C.dirs[(size_t)v[j] * D + a];
  }
  double rad[3];
  const int vrep = rep == 0 ? v[0] : (rep == 1 || D == 2 ? v[1] : v[D - 1]);
  if (kind == 0) {
    const double* lo = C.lo + (size_t)vrep * 3;
    if (C.emit) {
      const int id = C.idx[vrep];
      lo = C.emit + (size_t)(id >= 0 ? id : 0) * 3;  // (a surface item's representative is live: id ≥ 0)
    }
    rad[0] = lo[0];
    rad[1] = lo[1];
    rad[2] = lo[2];
  } else {
    const float* m = C.media + (size_t)(C.pre[vrep] + ring) * 3;
    rad[0] = m[0];
    rad[1] = m[1];
    rad[2] = m[2];
  }
#if VC_ASM_F32
  if constexpr (D == 3) {
    // float32 element math (the 3D form is fp32-safe) on lengths scaled by
    // 1/L, L = the largest vertex distance; the ok-mask stays the float64 one: decided here
    // when |A| clears its threshold by far more than the float32 error (≤ 12u·Πr_i against
    // 1e-5·Πr_i), else by ff_triangle_ok.  A non-finite float32 result takes the float64 path.
    const double L = fmax(dist[0], fmax(dist[1], dist[2]));
    const double iL = 1.0 / L;
    float r32[3][3], rr[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
#pragma unroll
      for (int a = 0; a < 3; ++a) r32[j][a] = (float)(rv[j][a] * iL);
      rr[j] = sqrtf(r32[j][0] * r32[j][0] + r32[j][1] * r32[j][1] + r32[j][2] * r32[j][2]);
    }
    const float A32 = r32[0][0] * (r32[1][1] * r32[2][2] - r32[1][2] * r32[2][1]) +
                      r32[0][1] * (r32[1][2] * r32[2][0] - r32[1][0] * r32[2][2]) +
                      r32[0][2] * (r32[1][0] * r32[2][1] - r32[1][1] * r32[2][0]);
    const bool sure = rr[0] > 0.0f && rr[1] > 0.0f && rr[2] > 0.0f && fabsf(A32) >= 1e-5f * rr[0] * rr[1] * rr[2];
    if (!sure && !ff_triangle_ok(rv[0], rv[1], rv[2])) return false;
    float F32, g32[3], H32[6], q32[10];
    ff_triangle_f32(r32[0], r32[1], r32[2], F32, g32, H32);
    float w32[3];  // −r32[rep] by selects (no local-memory indexing)
#pragma unroll
    for (int a = 0; a < 3; ++a) w32[a] = -(rep == 0 ? r32[0][a] : (rep == 1 ? r32[1][a] : r32[2][a]));
    const double drep = rep == 0 ? dist[0] : (rep == 1 ? dist[1] : dist[2]);
    element_q_f32(w32, (float)(drep * iL), (float)(S.sigma_t * L), F32, g32, H32, q32);
    bool fin = true;
#pragma unroll
    for (int t = 0; t < 10; ++t) fin = fin && isfinite(q32[t]);
    if (fin) {
      const double sc[3] = {1.0, iL, iL * iL};
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double f = wt * rad[c];
        const float fs[3] = {(float)f, (float)(f * sc[1]), (float)(f * sc[2])};
#pragma unroll
        for (int t = 0; t < NQ; ++t) cvec[c * NQ + t] = (CT)(fs[t == 0 ? 0 : (t < 4 ? 1 : 2)] * q32[t]);
      }
      return true;
    }
  }
#endif
  double F, gF[D], HF[D * (D + 1) / 2];
  bool ok;
  if constexpr (D == 3) ok = ff_triangle(rv[0], rv[1], rv[2], F, gF, HF);
  else ok = ff_segment(rv[0], rv[1], F, gF, HF);
  if (!ok) return false;
  double w[D], q[NQ];
#pragma unroll
  for (int a = 0; a < D; ++a) w[a] = -(rep == 0 ? rv[0][a] : (rep == 1 || D == 2 ? rv[1][a] : rv[D - 1][a]));
  element_q<D>(w, rep == 0 ? dist[0] : (rep == 1 || D == 2 ? dist[1] : dist[D - 1]), S.sigma_t, F, gF, HF, q);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double f = wt * rad[c];
#pragma unroll
    for (int t = 0; t < NQ; ++t) cvec[c * NQ + t] = (CT)(f * q[t]);
  }
  return true;
}

// Warp transpose-reduction: every lane holds 32 values v[0..31]; afterwards lane l holds
// Σ_lanes v[l] in v[0] (31 double shuffles; no per-lane persistent accumulators).
template <class T>
__device__ __forceinline__ void warp_transpose_sum(T (&v)[32], int lane) {
#pragma unroll
  for (int h = 16; h >= 1; h >>= 1) {
    const bool up = lane & h;
#pragma unroll
    for (int k = 0; k < h; ++k) {
      T send = up ? v[k] : v[k + h];
      T keep = up ? v[k + h] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, h);
    }
  }
}

#ifndef VC_ASM_EVAL_MINB
#define VC_ASM_EVAL_MINB VC_ASM_MINB
#endif
#ifndef VC_ASM_SCAN_MINB
#define VC_ASM_SCAN_MINB 24  // the scan alone: ≤ 40 registers, 48 warps per SM
#endif

// EMIT = false: scan + evaluate (fused; records whose item lists overflowed).
// EMIT = true: scan only — every warp copies its ballot-ordered item batches into its own
// segment of W.asm_items for k_asm_eval (a light kernel at high occupancy, so the dependent
// element → vertex → live-mask loads overlap).
template <int D, bool EMIT>
__global__ void __launch_bounds__(kAsmBS, EMIT ? VC_ASM_SCAN_MINB : VC_ASM_MINB)
    k_assemble_t(DevScene S, BuildParams P, Wave W) {
  constexpr int NQ = 1 + D + D * (D + 1) / 2;
  constexpr int NW = kAsmBS / 32;
  static_assert(3 * NQ <= 32, "contribution vector must fit one warp");
  __shared__ uint2 queue[NW][kQCap];
  const int rec = blockIdx.y, part = blockIdx.x;  // kAsmSplit CTAs share one record
  const int n = P.n_angular;
  const int E = (D == 2) ? n : P.n_tris;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // every warp writes its own partial sums (no block barrier: warps finish independently)
  const size_t slot = (size_t)rec * kAsmParts + (size_t)part * NW + wid;
  double* out_part = W.partial + slot * 64;
  long long* out_cnt = (long long*)(W.partial + (size_t)W.B * kAsmParts * 64) + slot * 5;
  if (D == 3 && W.tri_status[rec] != 0) return;  // k_asm_final reports the failure
  if (!EMIT && W.asm_items && !W.asm_fb[rec]) return;  // evaluated by k_asm_eval
  const AsmCtx<D> ring_ctx = asm_ctx<D>(P, W, rec);
  // EMIT: this warp's segment [seg, seg + seg_cap) and its fill
  const long long seg_cap = W.item_cap / kAsmParts;
  uint2* seg = EMIT ? W.asm_items + (size_t)slot * seg_cap : nullptr;
  int fill = 0;
  const DirInfo* info = W.info + (size_t)rec * n;
  const size_t rb = (size_t)rec * n;
  const int* idx = W.idx + rb;
  const int* cnt = W.cnt + rb;
  const double fbar = S.sigma_s / (D == 2 ? 2.0 * kPi : 4.0 * kPi);
  const double step = P.march_step;
  const bool media_on = S.sigma_s > 0.0;  // σs = 0: media rings carry zero radiance
  long long n_eval = 0, n_drop = 0, ev_kind[2] = {0, 0};

  for (int kind = 0; kind < 2; ++kind) {
    const double wt = fbar * (kind == 0 ? 1.0 : step);
    double acc = 0.0;  // lane l accumulates contribution component l (c·NQ + t)
    int qn = 0;        // warp-uniform queue length

    // contribution of one queued item (element e at ring `ring`, representative slot rep)
    auto eval_item = [&](uint2 it, AsmT<D> (&cvec)[32]) {
      int v[D];
      elem_vertices<D>(W, P, rec, (int)it.x, v);
      const bool ok = asm_item<D, AsmT<D>>(S, ring_ctx, kind, wt, v, (int)(it.y >> 2), (int)(it.y & 3u), cvec);
      ++n_eval;
      ++ev_kind[kind];
      if (!ok) ++n_drop;
    };
    // evaluate one item per lane (all lanes take part) and fold the 3·NQ components:
    // lane l accumulates component l, no per-lane 3·NQ accumulator array
    auto evaluate = [&](uint2 it, bool valid) {
      if constexpr (EMIT) {
        const int m = __popc(__ballot_sync(0xffffffffu, valid));
        if (fill + m > seg_cap) {
          if (lane == 0) W.asm_fb[rec] = 1;  // segment full: the fused kernel takes the record
        } else if (valid) {
          seg[fill + lane] = it;
        }
        fill += m;
        return;
      }
      AsmT<D> cvec[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) cvec[t] = 0.0;
      if (valid) eval_item(it, cvec);
      warp_transpose_sum(cvec, lane);
      acc += cvec[0];
    };

    // lane cursor over (element, ring); liveness of media samples comes from the per-direction
    // bit masks, so the scan itself touches memory once per element (and per 64 rings)
    const unsigned long long* live = W.live + (size_t)rec * W.live_words * n;
    const int kStride = kAsmBS * (int)gridDim.x;  // elements interleaved across the record's CTAs
    int e = part * kAsmBS + threadIdx.x;
    int ring = 0;
    int vv[D];
    int cv[D];
    double sd[D];
    int sl[D];
    unsigned long long mk[D];
    int word = -1;
    int maxc_e = 0;
    // rings [0, minc_e) have every vertex live: the representative is vertex 0 (equal
    // distances, first argmax) and the element is live exactly on vertex 0's mask bits,
    // which are popped directly; rings [minc_e, maxc_e) are resolved one by one
    int minc_e = 0, bw = 0;
    unsigned long long bits = 0;
    bool fresh = true;
    while (true) {
      bool has = e < E;
      bool flag = false;
      uint2 item = make_uint2(0, 0);
      if (has) {
        if (fresh) {
          elem_vertices<D>(W, P, rec, e, vv);
          maxc_e = 0;
          minc_e = 1 << 30;
#pragma unroll
          for (int j = 0; j < D; ++j) {
            const DirInfo di = info[vv[j]];
            cv[j] = di.cnt;
            sd[j] = di.s;
            sl[j] = di.surf_live;
            maxc_e = max(maxc_e, cv[j]);
            minc_e = min(minc_e, cv[j]);
          }
          fresh = false;
          word = -1;
          if (kind == 1) {
            bw = 0;
            bits = 0;
            if (!media_on) {
              minc_e = 0;
              ring = maxc_e;  // media rings carry no radiance
            } else {
              ring = minc_e;
              if (minc_e > 0) {
                const unsigned long long m0 = live[vv[0]];
                bits = (minc_e >= 64) ? m0 : (m0 & ((1ULL << minc_e) - 1ULL));
              }
            }
          }
        }
        if (kind == 0) {
          int rep = 0;
#pragma unroll
          for (int j = 1; j < D; ++j)
            if (sd[j] > sd[rep]) rep = j;
          flag = sl[rep] != 0;
          item = make_uint2((unsigned)e, (unsigned)rep);
          e += kStride;
          fresh = true;
        } else if (bits) {
          const int b = __ffsll((long long)bits) - 1;
          bits &= bits - 1ULL;
          flag = true;
          item = make_uint2((unsigned)e, ((unsigned)(bw * 64 + b) << 2));
          if (!bits && !((bw + 1) * 64 < minc_e) && ring >= maxc_e) {
            e += kStride;
            fresh = true;
          }
        } else if ((bw + 1) * 64 < minc_e) {
          ++bw;
          const int hi = minc_e - bw * 64;
          const unsigned long long m0 = live[(size_t)bw * n + vv[0]];
          bits = (hi >= 64) ? m0 : (m0 & ((1ULL << hi) - 1ULL));
        } else {
          if (ring < maxc_e) {
            double ri = ring_radius(ring, step);
            int rep = 0;
            double best = (ring < cv[0]) ? ri : sd[0];
            bool lrep = ring < cv[0];
#pragma unroll
            for (int j = 1; j < D; ++j) {
              bool lj = ring < cv[j];
              double dj = lj ? ri : sd[j];
              if (dj > best) {
                best = dj;
                rep = j;
                lrep = lj;
              }
            }
            if (lrep && media_on) {
              if ((ring >> 6) != word) {
                word = ring >> 6;
#pragma unroll
                for (int jj = 0; jj < D; ++jj) mk[jj] = live[(size_t)word * n + vv[jj]];
              }
              flag = (mk[rep] >> (ring & 63)) & 1ULL;
            }
            item = make_uint2((unsigned)e, ((unsigned)ring << 2) | (unsigned)rep);
            ++ring;
          }
          if (ring >= maxc_e) {
            e += kStride;
            ring = 0;
            fresh = true;
          }
        }
      }
      unsigned bal = __ballot_sync(0xffffffffu, flag);
      if (flag) queue[wid][qn + __popc(bal & ((1u << lane) - 1u))] = item;
      qn += __popc(bal);
      __syncwarp();
      if (qn >= 32) {
        evaluate(queue[wid][lane], true);
        __syncwarp();
        int rest = qn - 32;
        if (lane < rest) queue[wid][lane] = queue[wid][32 + lane];
        __syncwarp();
        qn = rest;
      }
      if (!__any_sync(0xffffffffu, e < E)) break;
    }
    if (qn > 0) evaluate(queue[wid][lane], lane < qn);
    __syncwarp();

    // lane l holds component l (order c·NQ + t) of this warp's sum
    if constexpr (EMIT) {
      if (lane == 0) W.item_n[slot * 2 + kind] = fill;  // end of this kind's items
    } else {
      out_part[kind * 32 + lane] = acc;
    }
  }
  if constexpr (EMIT) return;

  // counters: evaluated / dropped / per-kind evaluated
  // star vertices: Σ_k [idx_k ≥ 0] · deg_k · (maxc − cnt_k)  (src/subdivision.py:205-207)
  const int maxc = W.rec_maxc[rec];
  long long stars = 0;
  for (int k = part * kAsmBS + threadIdx.x; k < n; k += kAsmBS * (int)gridDim.x) {
    if (idx[k] >= 0) {
      int dg = (D == 2) ? 2 : W.deg[rb + k];
      stars += (long long)dg * (maxc - cnt[k]);
    }
  }
  // counters: evaluated / dropped / per-kind evaluated / stars
  long long cs[5] = {n_eval, n_drop, ev_kind[0], ev_kind[1], stars};
#pragma unroll
  for (int k = 0; k < 5; ++k)
#pragma unroll
    for (int o = 16; o; o >>= 1) cs[k] += __shfl_xor_sync(0xffffffffu, cs[k], o);
  if (lane == 0)
    for (int k = 0; k < 5; ++k) out_cnt[k] = cs[k];
}

// Evaluation of the item segments written by k_assemble_t<D, true>: warp w of a record
// evaluates producer warp w's segment in order (a fixed summation order per record).
template <int D>
__global__ void __launch_bounds__(kAsmBS, VC_ASM_EVAL_MINB) k_asm_eval(DevScene S, BuildParams P, Wave W) {
  constexpr int NW = kAsmBS / 32;
  const int rec = blockIdx.y, part = blockIdx.x;
  const int n = P.n_angular;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const size_t slot = (size_t)rec * kAsmParts + (size_t)part * NW + wid;
  double* out_part = W.partial + slot * 64;
  long long* out_cnt = (long long*)(W.partial + (size_t)W.B * kAsmParts * 64) + slot * 5;
  if (D == 3 && W.tri_status[rec] != 0) return;
  if (W.asm_fb[rec]) return;  // a segment overflowed: the fused kernel takes the record
  const AsmCtx<D> C = asm_ctx<D>(P, W, rec);
  const long long seg_cap = W.item_cap / kAsmParts;
  const uint2* seg = W.asm_items + (size_t)slot * seg_cap;
  const int end0 = W.item_n[slot * 2], end1 = W.item_n[slot * 2 + 1];
  const double fbar = S.sigma_s / (D == 2 ? 2.0 * kPi : 4.0 * kPi);
  long long n_eval = 0, n_drop = 0, ev_kind[2] = {0, 0};
  for (int kind = 0; kind < 2; ++kind) {
    const double wt = fbar * (kind == 0 ? 1.0 : P.march_step);
    const int a = kind ? end0 : 0, b = kind ? end1 : end0;
    double acc = 0.0;
    // the next round's item and vertex indices are fetched while this round evaluates
    uint2 q = make_uint2(0, 0);
    int v[D];
    auto fetch = [&](int t) {
      if (t < b) {
        q = seg[t];
        elem_vertices<D>(W, P, rec, (int)q.x, v);
      }
    };
    fetch(a + lane);
    for (int t0 = a; t0 < b; t0 += 32) {
      const int t = t0 + lane;
      const bool valid = t < b;
      const uint2 qc = q;
      int vc[D];
#pragma unroll
      for (int j = 0; j < D; ++j) vc[j] = v[j];
      fetch(t + 32);
      AsmT<D> cvec[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) cvec[c] = 0.0;
      if (valid) {
        if (!asm_item<D, AsmT<D>>(S, C, kind, wt, vc, (int)(qc.y >> 2), (int)(qc.y & 3u), cvec)) ++n_drop;
        ++n_eval;
        ++ev_kind[kind];
      }
      warp_transpose_sum(cvec, lane);
      acc += cvec[0];
    }
    out_part[kind * 32 + lane] = acc;
  }
  // star vertices: Σ_k [idx_k ≥ 0] · deg_k · (maxc − cnt_k)  (src/subdivision.py:205-207)
  const size_t rb = (size_t)rec * n;
  const int maxc = W.rec_maxc[rec];
  long long stars = 0;
  for (int k = part * kAsmBS + threadIdx.x; k < n; k += kAsmBS * (int)gridDim.x) {
    if (W.idx[rb + k] >= 0) {
      const int dg = (D == 2) ? 2 : W.deg[rb + k];
      stars += (long long)dg * (maxc - W.cnt[rb + k]);
    }
  }
  long long cs[5] = {n_eval, n_drop, ev_kind[0], ev_kind[1], stars};
#pragma unroll
  for (int k = 0; k < 5; ++k)
#pragma unroll
    for (int o = 16; o; o >>= 1) cs[k] += __shfl_xor_sync(0xffffffffu, cs[k], o);
  if (lane == 0)
    for (int k = 0; k < 5; ++k) out_cnt[k] = cs[k];
}

// Fixed-order sum of the kAsmSplit partials per record (deterministic), scattered into
// the reference layout L(3), grad(3, D), hess(3, D, D); stats.
template <int D>
__global__ void k_asm_final(BuildParams P, Wave W, int parts) {  // parts: per-warp partials written per record
  constexpr int NQ = 1 + D + D * (D + 1) / 2;
  const int rec = blockIdx.x;
  const int tid = threadIdx.x;  // 64 threads: kind · 32 + component
  const bool failed = (D == 3) && W.tri_status[rec] != 0;
  const int kind = tid >> 5, comp = tid & 31;
  if (comp < 3 * NQ) {
    double v = 0.0;
    if (!failed)
      for (int p = 0; p < parts; ++p) v += W.partial[((size_t)rec * kAsmParts + p) * 64 + kind * 32 + comp];
    const int c = comp / NQ, t = comp - c * NQ;
    double* M = W.moments + ((size_t)rec * 2 + kind) * moment_size(D);
    if (t == 0) {
      M[c] = v;
    } else if (t <= D) {
      M[3 + c * D + (t - 1)] = v;
    } else {
      int e2 = t - 1 - D, a = 0;
      while (e2 >= D - a) { e2 -= D - a; ++a; }
      const int b = a + e2;
      M[3 + 3 * D + c * D * D + a * D + b] = v;
      M[3 + 3 * D + c * D * D + b * D + a] = v;
    }
  }
  if (tid == 0) {
    const long long* cnt = (const long long*)(W.partial + (size_t)W.B * kAsmParts * 64);
    long long t[5] = {0, 0, 0, 0, 0};
    if (!failed)
      for (int p = 0; p < parts; ++p)
        for (int k = 0; k < 5; ++k) t[k] += cnt[((size_t)rec * kAsmParts + p) * 5 + k];
    long long* o = W.stats + (size_t)rec * kStats;
    o[0] = t[0];
    o[1] = t[1];
    o[2] = t[4];
    o[3] = W.rec_base[rec + 1] - W.rec_base[rec];
    o[4] = W.rec_R[rec];
    o[5] = (D == 3) ? W.tri_status[rec] : 0;
    o[6] = t[2];
    o[7] = t[3];
    (void)P;
  }
}

// ---------------------------------------------------------------------------
// make_record (src/cache.py:146-189)
// ---------------------------------------------------------------------------

template <int D>
__global__ void k_make_record(DevScene S, BuildParams P, Wave W) {
  int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= W.B * 2) return;
  int rec = gid >> 1, kind = gid & 1;
  const double* M = W.moments + (size_t)gid * moment_size(D);
  double* R = W.records + (size_t)gid * record_size(D);
  const double lw[3] = {0.2126, 0.7152, 0.0722};
  double lum = add(add(mul(M[0], lw[0]), mul(M[1], lw[1])), mul(M[2], lw[2]));
  double Hl[9];
  for (int e = 0; e < D * D; ++e) {
    double h = 0.0;
    for (int c = 0; c < 3; ++c) h += M[3 + 3 * D + c * D * D + e] * lw[c];
    Hl[e] = h;
  }
  lum = fmax(lum, 1e-6 * S.max_emission);
  double vals[3], V[9], radii[3];
  const double rmax = 0.25 * S.scale;
  if (lum <= 0.0) {
    for (int e = 0; e < D * D; ++e) V[e] = (e % (D + 1) == 0) ? 1.0 : 0.0;
    for (int a = 0; a < D; ++a) radii[a] = rmax;
  } else {
    eigen_sym<D>(Hl, vals, V);
    if (!P.anisotropic) {
      double mx = 0.0;
      for (int a = 0; a < D; ++a) mx = fmax(mx, fabs(vals[a]));
      for (int a = 0; a < D; ++a) vals[a] = mx;
    }
    const double floor_ = 1e-12 * lum / (S.scale * S.scale);
    for (int a = 0; a < D; ++a) {
      double lam = fabs(vals[a]);
      double r = rmax;
      if (lam > floor_) {
        r = (D == 2) ? pow(4.0 * lum * P.epsilon / (kPi * lam), 0.25)
                     : pow(15.0 * lum * P.epsilon / (4.0 * kPi * lam), 0.2);
      }
      radii[a] = fmin(r, rmax);
    }
  }
  int o = 0;
  for (int a = 0; a < D; ++a) R[o++] = W.x[rec * D + a];
  for (int c = 0; c < 3; ++c) R[o++] = M[c];
  for (int c = 0; c < 3 * D; ++c) R[o++] = M[3 + c];
  for (int e = 0; e < D * D; ++e) R[o++] = V[e];
  for (int a = 0; a < D; ++a) R[o++] = radii[a];
}

// ---------------------------------------------------------------------------
// Seeds: SeedSequence(entropy words) → PCG64 states on device
// ---------------------------------------------------------------------------

__global__ void k_seedseq(int n, const uint32_t* words, int nw, uint64_t* states) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t w[16];
  for (int k = 0; k < nw && k < 16; ++k) w[k] = words[(size_t)i * nw + k];
  uint64_t st[4];
  seedseq_pcg64(w, nw < 16 ? nw : 16, st);
  for (int k = 0; k < 4; ++k) states[(size_t)i * 4 + k] = st[k];
}

static int grid_for(long long threads, int bs) { return (int)((threads + bs - 1) / bs); }

// Raw nearest-hit queries (src/scene.py:271-315): trace (misses → inf, −1) or
// trace_or_bounds (misses → bounds exit distance).
template <int D>
__global__ void k_trace(DevScene S, int m, const double* org, const double* dir, double* t_out, int* idx_out,
                        int with_bounds) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double o[3], d[3];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    o[a] = org[(size_t)i * D + a];
    d[a] = dir[(size_t)i * D + a];
  }
  double t;
  int id;
  if (with_bounds) trace_or_bounds<D>(S, o, d, t, id);
  else trace_closest<D>(S, o, d, t, id);
  t_out[i] = t;
  idx_out[i] = id;
}

// surface_radiance_batch (src/transport.py:240-254) per hit: emission + albedo · direct
// lighting with shadow rays, float64 in the reference's order (surface_radiance).
template <int D>
__global__ void __launch_bounds__(128) k_surface_radiance(DevScene S, int m, const double* pts, const double* dirs,
                                                          const int* idx, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double p[3] = {0.0, 0.0, 0.0}, d[3] = {0.0, 0.0, 0.0}, L[3];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    p[a] = pts[(size_t)i * D + a];
    d[a] = dirs[(size_t)i * D + a];
  }
  surface_radiance<D>(S, idx[i], p, d, L);
#pragma unroll
  for (int c = 0; c < 3; ++c) out[(size_t)i * 3 + c] = L[c];
}

void launch_surface_radiance(const DevScene& S, int m, const double* pts, const double* dirs, const int* idx,
                             double* out, cudaStream_t st) {
  if (S.dim == 2) k_surface_radiance<2><<<grid_for(m, 128), 128, 0, st>>>(S, m, pts, dirs, idx, out);
  else k_surface_radiance<3><<<grid_for(m, 128), 128, 0, st>>>(S, m, pts, dirs, idx, out);
}

void launch_trace(const DevScene& S, int m, const double* o, const double* d, double* t, int* idx, int with_bounds,
                  cudaStream_t st) {
  if (S.dim == 2) k_trace<2><<<grid_for(m, 128), 128, 0, st>>>(S, m, o, d, t, idx, with_bounds);
  else k_trace<3><<<grid_for(m, 128), 128, 0, st>>>(S, m, o, d, t, idx, with_bounds);
}

// ---------------------------------------------------------------------------
// Host launch sequence for one wave
// ---------------------------------------------------------------------------

// Dynamic shared memory of a 256-thread ray kernel: one traversal stack column per thread.
template <class K>
static size_t stack_smem(K kernel, const DevBvh& H) {
  if (!VC_SMEM_STACK) return 0;
  const size_t bytes = (size_t)(H.n_nodes ? H.stack_need : 0) * 256 * sizeof(uint2);
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  return bytes;
}

// Off: forking the triangulation beside the gather chain gave 36.25 ms (side stream at the
// greatest priority) vs 36.56 ms per 2048 records — both chains fill the SMs on their own —
// and overlapped kernels make the per-class event times (the roofline's denominators)
// meaningless.
#ifndef VC_WAVE_FORK
#define VC_WAVE_FORK 0
#endif
#ifndef VC_FORK_PRIO
#define VC_FORK_PRIO 0  // side-stream priority: 0 default, 1 the greatest
#endif
// One side stream per device, created on first use; fork/join events are per call, so
// concurrent callers (on their own streams) cannot pick up each other's fork points.
static cudaStream_t side_stream() {
  static cudaStream_t per_dev[64] = {};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  cudaStream_t& s = per_dev[dev & 63];
  if (!s) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, VC_FORK_PRIO ? hi : lo);
  }
  return s;
}

// a waits for everything enqueued on b so far
static void stream_after(cudaStream_t a, cudaStream_t b) {
  cudaEvent_t e;
  cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  cudaEventRecord(e, b);
  cudaStreamWaitEvent(a, e, 0);
  cudaEventDestroy(e);  // released once recorded work completes
}

template <int D>
static void launch_wave_t(const DevScene& S, const BuildParams& P, const Wave& W, const JumpTables& jt,
                          int* own, int* own_cnt, int sm_count, cudaStream_t st, KernelCounter* kc) {
  const long long nt = (long long)W.B * P.n_angular;
  prof_begin(KC_PRIMARY, st);
  if (S.reflective) {
    k_primary<D, true><<<grid_for(nt, VC_PRIMARY_BS), VC_PRIMARY_BS, stack_smem(k_primary<D, true>, S.geo), st>>>(
        S, P, W, jt);
  } else if (VC_PRIMARY_PT && D == 3 && S.geo.n_nodes > 0 && W.ray_cursor) {
    k_directions<D><<<grid_for(nt, 256), 256, 0, st>>>(P, W, jt);
    cudaMemsetAsync(W.ray_cursor, 0, sizeof(unsigned long long), st);
    k_primary_pt<D><<<sm_count * 8, 256, 0, st>>>(S, P, W, W.ray_cursor);
    if (kc) kc->launches += 1;
  } else {
    k_primary<D, false><<<grid_for(nt, VC_PRIMARY_BS), VC_PRIMARY_BS, stack_smem(k_primary<D, false>, S.geo), st>>>(
        S, P, W, jt);
  }
  prof_end(st);
  int nl = 3;
  // Spherical Delaunay (depends only on the directions): on a forked side stream it runs
  // beside the rings + gather chain (VC_WAVE_FORK).
  auto triangulate = [&](cudaStream_t ts) {
  if constexpr (D == 3) {
    cudaMemsetAsync(W.tri_status, 0, sizeof(int) * W.B, ts);
    if (!P.host_adjacency) {
      static bool smem_attr = false;
      if (!smem_attr) {
        cudaFuncSetAttribute(k_delaunay_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDelSmem);
        cudaFuncSetAttribute(k_delaunay_list, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDelSmem);
        cudaFuncSetAttribute(k_delaunay_hull, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kHullBS * (kHullSlots * sizeof(float2) + kHullH)));
        cudaFuncSetAttribute(k_delaunay_cap, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCapSmem);
        cudaFuncSetAttribute(k_delaunay_capg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCapSmem);
        cudaFuncSetAttribute(k_delaunay_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWarpSmem);
        smem_attr = true;
      }
      prof_begin(KC_DELAUNAY, ts);
      cudaMemsetAsync(W.del_retry_count, 0, sizeof(unsigned int), ts);
      if (P.del_kmax > 0) {
        // stratum-window hulls for most cells, the cap kernel for the polar rows, clipping
        // for the cells either hands back
        cudaMemsetAsync(W.del_fb_count, 0, sizeof(unsigned int), ts);
        for (int k = 0; k < 3; ++k) {
          const int nr = P.del_cls[k + 1] - P.del_cls[k];
          if (!nr) continue;
          const size_t smem = (size_t)kHullBS * ((P.del_cls_k[k] + 1) * sizeof(float2) + kHullH);
          k_delaunay_hull<<<grid_for((long long)W.B * nr * P.cols, kHullBS), kHullBS, smem, ts>>>(P, W, own,
                                                                                                 own_cnt, k);
          ++nl;
        }
        if (P.del_cls[3] + (P.del_cap ? 2 : 0) < P.rows) {
          k_delaunay_rest<<<grid_for(nt, 256), 256, 0, ts>>>(P, W);
          ++nl;
        }
        if (P.del_cap) {
          CapGrid cg;
          if (cap_grid(P, cg)) {
            k_cap_bin<<<2 * W.B, kCapGBS, kCapBinSmem, ts>>>(P, W, cg);
            k_delaunay_capg<<<grid_for(2LL * W.B * P.cols, kHullBS), kHullBS, kCapSmem, ts>>>(P, W, own, own_cnt, cg);
            ++nl;
          } else {
            k_delaunay_cap<<<grid_for(2LL * W.B * P.cols, kHullBS), kHullBS, kCapSmem, ts>>>(P, W, own, own_cnt);
          }
          ++nl;
        }
        if (getenv("VOLCACHE_DEL_STATS")) {  // debug: cells handed to the clipping kernel
          unsigned c = 0;
          cudaMemcpyAsync(&c, W.del_fb_count, 4, cudaMemcpyDeviceToHost, ts);
          cudaStreamSynchronize(ts);
          fprintf(stderr, "[volcache] hull fallback cells: %u of %lld\n", c, nt);
          if (getenv("VOLCACHE_DEL_STATS")[0] == '3') {  // handed-back cells per stratum row
            std::vector<int> l(c), hist(P.rows, 0);
            cudaMemcpy(l.data(), W.del_fb, (size_t)c * 4, cudaMemcpyDeviceToHost);
            for (int g : l) ++hist[(g % P.n_angular) / P.cols];
            for (int r = 0; r < P.rows; ++r) fprintf(stderr, "%d:%d ", r, hist[r]);
            fprintf(stderr, "\n");
          }
          if (getenv("VOLCACHE_DEL_STATS")[0] >= '2') {
            k_delaunay_warp<<<sm_count * 4, kWarpBS, kWarpSmem, ts>>>(P, W, own, own_cnt);
            cudaMemcpyAsync(&c, W.del_fb2_count, 4, cudaMemcpyDeviceToHost, ts);
            cudaStreamSynchronize(ts);
            fprintf(stderr, "[volcache] after the float64 wrap: %u\n", c);
            std::vector<int> l(c), hist(P.rows, 0);
            cudaMemcpy(l.data(), W.del_fb2, (size_t)c * 4, cudaMemcpyDeviceToHost);
            for (int g : l) ++hist[(g % P.n_angular) / P.cols];
            for (int r = 0; r < P.rows; ++r) fprintf(stderr, "%d:%d ", r, hist[r]);
            fprintf(stderr, "\n");
            for (unsigned t = 0; t < c && t < 8; ++t)
              fprintf(stderr, "[volcache] clipping cell: record %d direction %d\n", l[t] / P.n_angular, l[t] % P.n_angular);
          }
        }
        cudaMemsetAsync(W.del_fb2_count, 0, sizeof(unsigned int), ts);
        k_delaunay_warp<<<sm_count * 4, kWarpBS, kWarpSmem, ts>>>(P, W, own, own_cnt);
        k_delaunay_list<<<sm_count * VC_LB_DEL2, kDelBS, kDelSmem, ts>>>(P, W, own, own_cnt);
        nl += 2;
      } else {
        k_delaunay_smem<<<grid_for(nt, kDelBS), kDelBS, kDelSmem, ts>>>(P, W, own, own_cnt);
        ++nl;
      }
      k_delaunay_retry<<<sm_count * 2, 128, 0, ts>>>(P, W, own, own_cnt, W.del_scratch);
      ++nl;
      prof_end(ts);
      prof_begin(KC_COMPACT, ts);
  // W.del_fb (B × n ints) is free once the Delaunay kernels are done: the offsets
  k_own_scan<<<W.B, kCompactBS, 0, ts>>>(P, W, own_cnt, W.del_fb);
  k_tri_scatter<<<grid_for(nt, 256), 256, 0, ts>>>(P, W, own, own_cnt, W.del_fb);
  ++nl;
  prof_end(ts);
      nl += 2;
    } else {
      cudaMemsetAsync(W.deg, 0, sizeof(int) * nt, ts);
      prof_begin(KC_DEGREE, ts);
  k_degree<<<grid_for((long long)W.B * P.n_tris, 256), 256, 0, ts>>>(P, W);
  prof_end(ts);
      ++nl;
    }
  }
  };
  const bool fork = VC_WAVE_FORK && D == 3;
  cudaStream_t side = nullptr;
  if (fork) {
    side = side_stream();
    stream_after(side, st);
    triangulate(side);
  }
  prof_begin(KC_RINGS, st);
  k_rings<<<W.B, kRingBS, 0, st>>>(P, W);
  prof_end(st);
  prof_begin(KC_WAVESCAN, st);
  k_wave_scan<<<1, 1024, 0, st>>>(W, S.sigma_s > 0.0 ? 1 : 0);
  prof_end(st);
  // live-sample masks are set by the gather itself (mark_live)
  cudaMemsetAsync(W.live, 0, sizeof(unsigned long long) * (size_t)W.live_words * nt, st);
  if (S.sigma_s > 0.0) {
    // (the HG extension with one media event only weighs the emitter hits: still two passes)
    const bool two_pass = !S.reflective && 2 * S.emit.K <= S.geo.K && P.n_inner == 1 && W.gather_q_cap > 0 &&
                          P.media_bounces <= 1;
    // nothing emits and nothing reflects: every gather path carries zero radiance (only the
    // delta lights, extension, light the media — k_gather_delta below, or inside k_gather's
    // bounce loop when further media events are on)
    const bool dark = S.emit.K == 0 && !S.reflective && (P.media_bounces <= 1 || S.n_lights == 0);
    prof_begin(KC_GATHER, st);
    if (dark) {
      if (W.dense_media) cudaMemsetAsync(W.media, 0, sizeof(float) * 3 * (size_t)W.media_cap, st);
    } else if (two_pass) {
      cudaMemsetAsync(W.gather_q_count, 0, 2 * sizeof(unsigned long long), st);
      if (VC_GATHER_SPLIT && !W.dense_media) {  // filter → survivor evaluation → redo pass
        cudaMemsetAsync(W.surv_cnt, 0, sizeof(int) * 2 * (size_t)W.B, st);  // surv_cnt and redo
        k_gather_emit<D, 1><<<dim3(VC_EMIT_CTAS * 256 / VC_EMIT_BS, W.B), VC_EMIT_BS, 0, st>>>(S, P, W, jt, (GatherItem*)W.gather_q, W.gather_q_count,
                                                           W.gather_q_cap);
        k_gather_eval<D><<<dim3(VC_EVAL_CTAS * 256 / VC_EVAL_BS, W.B), VC_EVAL_BS, 0, st>>>(S, P, W, jt, (GatherItem*)W.gather_q, W.gather_q_count,
                                                      W.gather_q_cap);
        k_gather_emit<D, 2><<<dim3(VC_EMIT_CTAS * 256 / VC_EMIT_BS, W.B), VC_EMIT_BS, 0, st>>>(S, P, W, jt, (GatherItem*)W.gather_q, W.gather_q_count,
                                                           W.gather_q_cap);
        nl += 2;
      } else {
        k_gather_emit<D, 0><<<dim3(VC_EMIT_CTAS * 256 / VC_EMIT_BS, W.B), VC_EMIT_BS, 0, st>>>(S, P, W, jt, (GatherItem*)W.gather_q, W.gather_q_count,
                                                           W.gather_q_cap);
      }
      const bool hg_on = D == 3 && P.hg_g != 0.0;
      if (VC_OCCL_PT && S.geo.n_nodes > 0) {
        auto kern = hg_on ? k_gather_occl_pt<D, true> : k_gather_occl_pt<D, false>;
        kern<<<sm_count * 8, 256, 0, st>>>(S, W, P.n_angular, (const GatherItem*)W.gather_q, W.gather_q_count,
                                           W.gather_q_cap, W.media, P.hg_g);
      } else {
        auto kern = hg_on ? k_gather_occl<D, true> : k_gather_occl<D, false>;
        kern<<<sm_count * 8, 256, stack_smem(k_gather_occl<D, false>, S.geo), st>>>(
            S, W, P.n_angular, (const GatherItem*)W.gather_q, W.gather_q_count, W.gather_q_cap, W.media, P.hg_g);
      }
      nl += 2;
    } else {
      k_gather<D><<<sm_count * 8, 256, 0, st>>>(S, P, W, jt);
      ++nl;
    }
    if (S.n_lights > 0) {  // extension: delta lights lit the media samples too
      if (VC_DELTA_PT && S.geo.n_nodes > 0 && W.ray_cursor) {
        cudaMemsetAsync(W.ray_cursor, 0, sizeof(unsigned long long), st);
        k_gather_delta_pt<D><<<sm_count * 6, 256, 0, st>>>(S, P, W, W.ray_cursor);
      } else {
        k_gather_delta<D><<<sm_count * 8, 256, 0, st>>>(S, P, W);
      }
      ++nl;
    }
    prof_end(st);
  }
  if (fork) {  // join: the assembly needs both the media and the triangles
    stream_after(st, side);
  } else {
    triangulate(st);
  }
  prof_begin(KC_ASSEMBLE, st);

  // CTAs per record: kAsmSplit for the 3D sizes (n ≥ 8192), fewer for short element lists — the
  // small 2D records pay for idle CTAs otherwise (cfg1: 4.5 M records/s at 16, 3.0 M at 32)
  int split = kAsmSplit;
  {
    const int E = (D == 2) ? P.n_angular : P.n_tris;
    while (split > 2 && (long long)split * kAsmBS * 8 > E) split >>= 1;
    if (const char* es = getenv("VOLCACHE_ASM_SPLIT")) split = std::max(1, std::min(kAsmSplit, atoi(es)));
  }
  if (W.asm_items) {
    cudaMemsetAsync(W.asm_fb, 0, sizeof(int) * W.B, st);
    k_assemble_t<D, true><<<dim3(split, W.B), kAsmBS, 0, st>>>(S, P, W);
    k_asm_eval<D><<<dim3(split, W.B), kAsmBS, 0, st>>>(S, P, W);
    nl += 2;
  }
  k_assemble_t<D, false><<<dim3(split, W.B), kAsmBS, 0, st>>>(S, P, W);  // overflowed records
  k_asm_final<D><<<W.B, 64, 0, st>>>(P, W, split * (kAsmBS / 32));
  ++nl;
  if (S.n_lights > 0 && S.sigma_s > 0.0) {
    k_delta_single<D><<<grid_for(W.B, 128), 128, 0, st>>>(S, W);
    ++nl;
  }
  prof_end(st);
  ++nl;
  if (P.make_records) {
    prof_begin(KC_RECORD, st);
    k_make_record<D><<<grid_for(2LL * W.B, 128), 128, 0, st>>>(S, P, W);
    prof_end(st);
    ++nl;
  }
  if (kc) kc->launches += nl;
}

void launch_wave(const DevScene& S, const BuildParams& P, const Wave& W, const JumpTables& jt, int* own,
                 int* own_cnt, int sm_count, cudaStream_t st, KernelCounter* kc) {
  if (S.dim == 2) launch_wave_t<2>(S, P, W, jt, own, own_cnt, sm_count, st, kc);
  else launch_wave_t<3>(S, P, W, jt, own, own_cnt, sm_count, st, kc);
}

void launch_make_records(const DevScene& S, const BuildParams& P, const Wave& W, cudaStream_t st) {
  if (S.dim == 2) k_make_record<2><<<grid_for(2LL * W.B, 128), 128, 0, st>>>(S, P, W);
  else k_make_record<3><<<grid_for(2LL * W.B, 128), 128, 0, st>>>(S, P, W);
}

void launch_seedseq(int n, const uint32_t* words, int nw, uint64_t* states, cudaStream_t st) {
  prof_begin(KC_SEED, st);
  k_seedseq<<<grid_for(n, 128), 128, 0, st>>>(n, words, nw, states);
  prof_end(st);
}

}  // namespace vc
