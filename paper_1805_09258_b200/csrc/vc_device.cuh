// Device building blocks of the cache-record path.
//
// Exactness rules (SURVEY.md §7 hard parts 3-4, Appendix A):
//  * PCG64 streams are bit-exact with numpy (128-bit LCG, XSL-RR, double = (x>>11)·2⁻⁵³).
//  * Ray–primitive tests run in float64 in the reference's operation order with FMA
//    contraction disabled (__d*_rn), nearest hit with first-min (lowest index) tie break.
//  * BVH boxes are float32, padded so culling is conservative; hits are decided in float64.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdint>

#include "vc_internal.h"

namespace vc {

typedef unsigned __int128 u128;

// ---------------------------------------------------------------------------
// PCG64 (numpy's default bit generator) — src/renderer.py:278-279 seeds it via SeedSequence
// ---------------------------------------------------------------------------

__host__ __device__ inline u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;
}

struct Pcg64 {
  u128 s, inc;
  __device__ inline uint64_t next64() {
    s = s * pcg_mult() + inc;
    uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
    uint64_t x = hi ^ lo;
    unsigned rot = (unsigned)(s >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  __device__ inline double next_double() {
    return (double)(next64() >> 11) * (1.0 / 9007199254740992.0);
  }
};

__device__ inline u128 ld128(const unsigned long long* p) {
  return ((u128)p[0] << 64) | (u128)p[1];
}

// Advance by delta draws with the precomputed 3-level table (delta < 2^30),
// falling back to square-and-multiply beyond it.
__device__ inline void pcg_advance(Pcg64& g, unsigned long long delta, const JumpTables& jt) {
  if (delta < (1ULL << 30)) {
#pragma unroll
    for (int lv = 0; lv < 3; ++lv) {
      unsigned k = (unsigned)(delta >> (10 * lv)) & 1023u;
      if (k) {
        const unsigned long long* e = jt.tab + ((size_t)lv * 1024 + k) * 4;
        u128 A = ld128(e), G = ld128(e + 2);
        g.s = A * g.s + G * g.inc;
      }
    }
    return;
  }
  u128 am = 1, ap = 0, cm = pcg_mult(), cp = g.inc;
  while (delta) {
    if (delta & 1) {
      am *= cm;
      ap = ap * cm + cp;
    }
    cp = (cm + 1) * cp;
    cm *= cm;
    delta >>= 1;
  }
  g.s = am * g.s + ap;
}

__device__ inline Pcg64 pcg_load(const uint64_t* st) {
  Pcg64 g;
  g.s = ((u128)st[0] << 64) | (u128)st[1];
  g.inc = ((u128)st[2] << 64) | (u128)st[3];
  return g;
}

// numpy SeedSequence(entropy words) → PCG64 (state, inc).  Pool size 4, 32-bit hashes.
__host__ __device__ inline void seedseq_pcg64(const uint32_t* w, int nw, uint64_t out[4]) {
  const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu,
                 MULT_B = 0x58f38dedu, MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
  uint32_t pool[4];
  uint32_t hc = INIT_A;
  auto hashmix = [&](uint32_t v) {
    v ^= hc;
    hc *= MULT_A;
    v *= hc;
    v ^= v >> 16;
    return v;
  };
  auto mix = [](uint32_t x, uint32_t y) {
    uint32_t r = MIX_L * x - MIX_R * y;
    r ^= r >> 16;
    return r;
  };
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < nw ? w[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (int s = 4; s < nw; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(w[s]));
  uint32_t st[8];
  uint32_t hb = INIT_B;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= MULT_B;
    v *= hb;
    v ^= v >> 16;
    st[i] = v;
  }
  uint64_t q[4];
  for (int i = 0; i < 4; ++i) q[i] = (uint64_t)st[2 * i] | ((uint64_t)st[2 * i + 1] << 32);
  u128 seed = ((u128)q[0] << 64) | q[1];
  u128 inc = ((((u128)q[2] << 64) | q[3]) << 1) | 1;
  u128 s = 0;
  s = s * pcg_mult() + inc;
  s += seed;
  s = s * pcg_mult() + inc;
  out[0] = (uint64_t)(s >> 64);
  out[1] = (uint64_t)s;
  out[2] = (uint64_t)(inc >> 64);
  out[3] = (uint64_t)inc;
}

// ---------------------------------------------------------------------------
// numpy-faithful float64 helpers (no FMA contraction)
// ---------------------------------------------------------------------------

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dot3(const double* a, const double* b) {
  return add(add(mul(a[0], b[0]), mul(a[1], b[1])), mul(a[2], b[2]));
}
__device__ __forceinline__ void cross3(const double* a, const double* b, double* c) {
  c[0] = sub(mul(a[1], b[2]), mul(a[2], b[1]));
  c[1] = sub(mul(a[2], b[0]), mul(a[0], b[2]));
  c[2] = sub(mul(a[0], b[1]), mul(a[1], b[0]));
}
// np.maximum / np.minimum propagate NaN
__device__ __forceinline__ double np_max(double a, double b) {
  return (isnan(a) || isnan(b)) ? __longlong_as_double(0x7ff8000000000000LL) : (a >= b ? a : b);
}
__device__ __forceinline__ double np_min(double a, double b) {
  return (isnan(a) || isnan(b)) ? __longlong_as_double(0x7ff8000000000000LL) : (a <= b ? a : b);
}

// ---------------------------------------------------------------------------
// Ray–primitive tests (src/scene.py:227-268)
// ---------------------------------------------------------------------------

// 3D Möller–Trumbore on (v0, e1, e2); returns t or +inf when invalid.
__device__ inline double hit_tri(const double* P, const double* o, const double* d, double t_eps) {
  const double* v0 = P;
  const double* e1 = P + 3;
  const double* e2 = P + 6;
  double pv[3], tv[3], qv[3];
  cross3(d, e2, pv);
  double det = dot3(e1, pv);
  tv[0] = sub(o[0], v0[0]);
  tv[1] = sub(o[1], v0[1]);
  tv[2] = sub(o[2], v0[2]);
  double inv = __ddiv_rn(1.0, det);
  double u = mul(dot3(tv, pv), inv);
  cross3(tv, e1, qv);
  double v = mul(dot3(d, qv), inv);
  double t = mul(dot3(e2, qv), inv);
  bool ok = isfinite(t) && (fabs(det) > 0.0) && (u >= 0.0) && (v >= 0.0) && (add(u, v) <= 1.0) &&
            (t > t_eps);
  return ok ? t : INFINITY;
}

// 2D segment (a, e) cross-product test; returns t or +inf.
__device__ inline double hit_seg(const double* P, const double* o, const double* d, double t_eps) {
  double ax = sub(P[0], o[0]), ay = sub(P[1], o[1]);
  double ex = P[2], ey = P[3];
  double den = sub(mul(d[0], ey), mul(d[1], ex));
  double t = __ddiv_rn(sub(mul(ax, ey), mul(ay, ex)), den);
  double u = __ddiv_rn(sub(mul(ax, d[1]), mul(ay, d[0])), den);
  bool ok = (fabs(den) > 0.0) && (u >= 0.0) && (u <= 1.0) && (t > t_eps);
  return ok ? t : INFINITY;
}

template <int D>
__device__ __forceinline__ double hit_prim(const double* P, const double* o, const double* d, double t_eps) {
  if constexpr (D == 3) return hit_tri(P, o, d, t_eps);
  else return hit_seg(P, o, d, t_eps);
}

// Packed float32 FMA on (left, right) pairs (sm_100a FFMA2): one instruction per slab plane
// for both children of a node.  Same rounding as two fmaf.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&r);
}

// Conservative float32 slab tests of both children of a node (layout: vc_bvh.cpp):
// t = lo·inv − of·inv as one packed FMA per plane (the rounding it adds is far inside the
// 1e-5·scale box padding; an exactly zero direction component gives NaN slabs, which
// fminf/fmaxf drop — that axis then never culls).
template <int D>
__device__ __forceinline__ void box_hit2(const float4& A, const float4& B, const float4& C, const float2* inv2,
                                         const float2* noi2, float t_best, bool& hl, bool& hr, float& tl, float& tr) {
  const float2 lx = ffma2(make_float2(A.x, A.y), inv2[0], noi2[0]);
  const float2 ly = ffma2(make_float2(A.z, A.w), inv2[1], noi2[1]);
  const float2 hx = ffma2(make_float2(B.z, B.w), inv2[0], noi2[0]);
  const float2 hy = ffma2(make_float2(C.x, C.y), inv2[1], noi2[1]);
  float nl = fmaxf(fminf(lx.x, hx.x), fminf(ly.x, hy.x)), fl = fminf(fmaxf(lx.x, hx.x), fmaxf(ly.x, hy.x));
  float nr = fmaxf(fminf(lx.y, hx.y), fminf(ly.y, hy.y)), fr = fminf(fmaxf(lx.y, hx.y), fmaxf(ly.y, hy.y));
  if constexpr (D == 3) {
    const float2 lz = ffma2(make_float2(B.x, B.y), inv2[2], noi2[2]);
    const float2 hz = ffma2(make_float2(C.z, C.w), inv2[2], noi2[2]);
    nl = fmaxf(nl, fminf(lz.x, hz.x));
    fl = fminf(fl, fmaxf(lz.x, hz.x));
    nr = fmaxf(nr, fminf(lz.y, hz.y));
    fr = fminf(fr, fmaxf(lz.y, hz.y));
  }
  tl = nl;
  tr = nr;
  hl = nl <= fl && fl >= 0.0f && nl <= t_best;
  hr = nr <= fr && fr >= 0.0f && nr <= t_best;
}

// Certified float32 Möller–Trumbore pre-test: true only when the float64 test of
// hit_tri (src/scene.py:242-268) certainly rejects the triangle, or certainly puts its hit
// beyond tmax (a float32 upper bound of the current best / threshold distance).
// With u = 2⁻²⁴, |d|∞ ≤ 1, E ≥ |e1|∞, |e2|∞ and Tb ≥ |o − v0|∞ (origin and vertex both
// relative to the bounds centre, each rounded once), the float32 values of
// det = e1·(d×e2), U = (o−v0)·(d×e2), V = d·((o−v0)×e1), T = e2·((o−v0)×e1) are within
// 48u·E², 54u·Tb·E, 54u·Tb·E and 54u·Tb·E² of the exact ones (input roundings and every
// product and sum); the margins below are 128u·(…), so a decision taken here also holds
// for the float64 values (errors ~1e-16 relative).  NaN never rejects.
__device__ __forceinline__ bool tri_rejects32(const float4& f0, const float4& f1, const float4& f2, const float* orl,
                                              float Ob, const float* df, float teps, float tmax) {
  const float E = f1.w;
  if (!(E > 0.0f)) return false;
  constexpr float c = 128.0f * 5.9604645e-8f;
  const float tv0 = orl[0] - f0.x, tv1 = orl[1] - f0.y, tv2 = orl[2] - f0.z;
  const float pv0 = df[1] * f2.z - df[2] * f2.y;
  const float pv1 = df[2] * f2.x - df[0] * f2.z;
  const float pv2 = df[0] * f2.y - df[1] * f2.x;
  const float det = f1.x * pv0 + f1.y * pv1 + f1.z * pv2;
  const float eD = c * E * E;
  const float ad = fabsf(det);
  if (!(ad > eD)) return false;  // sign of det (or det = 0) not decided here
  const float sg = det > 0.0f ? 1.0f : -1.0f;
  const float eU = c * (Ob + f0.w) * E;
  const float su = sg * (tv0 * pv0 + tv1 * pv1 + tv2 * pv2);
  if (su < -eU) return true;  // u < 0
  const float qv0 = tv1 * f1.z - tv2 * f1.y;
  const float qv1 = tv2 * f1.x - tv0 * f1.z;
  const float qv2 = tv0 * f1.y - tv1 * f1.x;
  const float sv = sg * (df[0] * qv0 + df[1] * qv1 + df[2] * qv2);
  if (sv < -eU) return true;  // v < 0
  constexpr float r4 = 4.0f * 5.9604645e-8f;
  if (su + sv - ad > 2.0f * eU + eD + r4 * (fabsf(su) + fabsf(sv) + ad)) return true;  // u + v > 1
  const float eT = eU * E;
  const float st = sg * (f2.x * qv0 + f2.y * qv1 + f2.z * qv2);
  if (st + eT < teps * (ad - eD) * (1.0f - r4)) return true;  // t ≤ t_eps
  if (st - eT > tmax * (ad + eD) * (1.0f + r4)) return true;  // t beyond the current bound
  return false;
}

// Traversal stacks: entry = (child reference, entry distance bits).  LocalStack is a
// per-thread array; SharedStack a per-thread column of a CTA's shared-memory block
// ([entry][thread], conflict-free), sized from DevBvh::stack_need at launch.
struct LocalStack {
  uint2 e[kBvhMaxDepth];
  __device__ __forceinline__ void put(int i, uint2 v) { e[i] = v; }
  __device__ __forceinline__ uint2 get(int i) const { return e[i]; }
};
template <int BS>
struct SharedStack {
  uint2* col;  // this thread's column: smem + threadIdx.x
  __device__ __forceinline__ void put(int i, uint2 v) { col[i * BS] = v; }
  __device__ __forceinline__ uint2 get(int i) const { return col[i * BS]; }
};

// Float32 pre-test in the leaf loop: measured r2 per 2048-record wave, primary 6.34 vs 6.15 ms
// and gather 13.87 vs 13.45 ms with it on — traversal (box tests, stack) dominates, the
// float64 leaf tests are ~15% of the primary kernel's instructions — so it is off by default.
#ifndef VC_PRETEST32
#define VC_PRETEST32 0
#endif

// Ordered BVH traversal.  mode 0: nearest hit (t_best/id_best out).  mode 1: any hit
// that precedes (thr, id_thr) in (t, index) order — returns true on the first one.
// Node layout (vc_bvh.cpp): per interior node the two children's boxes and references
// (bit 31: leaf, walked up to the primitive flagged last-in-leaf in prim32).
// while-while: descend interior nodes until a leaf, then test it — the lanes of a warp
// run the leaf tests together instead of interleaving them with box tests.
template <int D, int MODE, class Stack>
__device__ bool bvh_query(const DevBvh& H, double t_eps, float slack, const double* o, const double* d,
                          double& t_best, int& id_best, Stack& stk) {
  float orl[3] = {0.f, 0.f, 0.f}, df[3] = {0.f, 0.f, 0.f};
  float2 inv2[3], noi2[3];  // (inv, inv) and (−of·inv, −of·inv) per axis, for the packed slabs
  float Ob = 0.0f;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    float inv = 0.0f, noi = 0.0f;
    if (a < D) {
      orl[a] = (float)(o[a] - H.ctr[a]);
      df[a] = (float)d[a];
      // approximate reciprocal (≤ 1 ulp; ±0 → ±inf): inside the box padding
      asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(df[a]));
      noi = -orl[a] * inv;
      Ob = fmaxf(Ob, fabsf(orl[a]));
    }
    inv2[a] = make_float2(inv, inv);
    noi2[a] = make_float2(noi, noi);
  }
  Ob *= 1.0000005f;
  const float teps = (float)t_eps;
  // slack: float32 t limit strictly above the float64 one
  auto tlim = [&](double t) { return isfinite(t) ? __double2float_ru(t) * 1.0001f + slack : INFINITY; };
  float tbf = tlim(t_best);
  int sp = 0;
  unsigned cur = 0;  // interior node 0 (the root)
  while (true) {
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
      } else {
        bool got = false;
        while (sp > 0) {  // pop, skipping entries whose entry distance is beyond the best
          const uint2 e = stk.get(--sp);
          if (__uint_as_float(e.y) <= tbf) {
            cur = e.x;
            got = true;
            break;
          }
        }
        if (!got) return false;
      }
    }
    for (int k = (int)(cur & 0x7fffffffu);; ++k) {
      const float4* Q = H.prim32 + 3 * (size_t)k;
      const float4 f0 = __ldg(Q), f1 = __ldg(Q + 1), f2 = __ldg(Q + 2);
      const int idf = __float_as_int(f2.w);
      bool maybe = true;
#if VC_PRETEST32
      if constexpr (D == 3) maybe = !tri_rejects32(f0, f1, f2, orl, Ob, df, teps, tbf);
#endif
      if (maybe) {
        const double t = hit_prim<D>(H.prim + (size_t)k * prim_stride(D), o, d, t_eps);
        if (t != INFINITY) {
          const int id = idf & 0x7fffffff;
          if (t < t_best || (t == t_best && id < id_best)) {
            if (MODE == 1) return true;
            t_best = t;
            id_best = id;
            tbf = tlim(t_best);
          }
        }
      }
      if (idf < 0) break;
    }
    bool got = false;
    while (sp > 0) {
      const uint2 e = stk.get(--sp);
      if (__uint_as_float(e.y) <= tbf) {
        cur = e.x;
        got = true;
        break;
      }
    }
    if (!got) return false;
  }
}

template <int D, int MODE>
__device__ __forceinline__ bool bvh_query(const DevBvh& H, double t_eps, float slack, const double* o,
                                          const double* d, double& t_best, int& id_best) {
  LocalStack stk;
  return bvh_query<D, MODE>(H, t_eps, slack, o, d, t_best, id_best, stk);
}

// Nearest hit in a primitive set; `id_best` is the original surface index.
template <int D, class Stack = LocalStack>
__device__ void bvh_closest(const DevBvh& H, double t_eps, float slack, const double* o, const double* d,
                            double& t_best, int& id_best, Stack* stk = nullptr) {
  t_best = INFINITY;
  id_best = -1;
  if (H.K == 0) return;
  if (H.n_nodes == 0) {
    for (int k = 0; k < H.K; ++k) {
      double t = hit_prim<D>(H.prim + (size_t)k * prim_stride(D), o, d, t_eps);
      if (t < t_best) {  // primitives in original order: strict < keeps the first minimum
        t_best = t;
        id_best = H.prim_id[k];
      }
    }
    return;
  }
  if (stk) bvh_query<D, 0>(H, t_eps, slack, o, d, t_best, id_best, *stk);
  else bvh_query<D, 0>(H, t_eps, slack, o, d, t_best, id_best);
}

// Nearest hit over the scene (src/scene.py:271-292).
template <int D, class Stack = LocalStack>
__device__ __forceinline__ void trace_closest(const DevScene& S, const double* o, const double* d, double& t_best,
                                              int& id_best, Stack* stk = nullptr) {
  bvh_closest<D, Stack>(S.geo, S.t_eps, 1e-5f * (float)S.scale, o, d, t_best, id_best, stk);
}

// Is there a valid hit preceding (thr, id_thr) in (t, index) order?  Shadow rays use
// id_thr = −1 (visible iff nearest t ≥ thr, src/transport.py:213-214).
template <int D, class Stack = LocalStack>
__device__ bool occluded(const DevScene& S, const double* o, const double* d, double thr, int id_thr = -1,
                         Stack* stk = nullptr) {
  const DevBvh& H = S.geo;
  if (H.K == 0) return false;
  if (H.n_nodes == 0) {
    for (int k = 0; k < H.K; ++k) {
      double t = hit_prim<D>(H.prim + (size_t)k * prim_stride(D), o, d, S.t_eps);
      if (t < thr || (t == thr && H.prim_id[k] < id_thr)) return true;
    }
    return false;
  }
  double t = thr;
  int id = id_thr;
  if (stk) return bvh_query<D, 1>(H, S.t_eps, 1e-5f * (float)S.scale, o, d, t, id, *stk);
  return bvh_query<D, 1>(H, S.t_eps, 1e-5f * (float)S.scale, o, d, t, id);
}

// Nearest emitter hit (lowest original index wins ties), through the emitter BVH.
template <int D>
__device__ __forceinline__ void nearest_emitter(const DevScene& S, const double* o, const double* d, double& te,
                                                int& ie) {
  if constexpr (D == 3) {
    if (S.ep.ng > 0) {
      // plane grids: the float64 hit test on the triangles of the cell the ray lands in,
      // (t, index) minimum as the BVH; rays within 1e-3 of grazing a plane take the BVH
      const EmitPlanes& E = S.ep;
      te = INFINITY;
      ie = -1;
      bool ok = true;
      for (int g = 0; g < E.ng && ok; ++g) {
        const double dn = E.n[g][0] * d[0] + E.n[g][1] * d[1] + E.n[g][2] * d[2];
        if (fabs(dn) < 1e-3) {
          ok = false;
          break;
        }
        // the landing distance only picks the grid cell: a float32 reciprocal (≤ 1e-7
        // relative) keeps it within ~1e-7·scale for the distances that matter (|tp| ≤ 1.01·scale:
        // the planes are built only for emitters inside the bounds, so a hit from a point of
        // the medium is nearer), far inside the cells' 1e-5·scale padding
        float rdn;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rdn) : "f"((float)dn));
        const double tp = (E.c[g] - (E.n[g][0] * o[0] + E.n[g][1] * o[1] + E.n[g][2] * o[2])) * (double)rdn;
        if (tp < -1e-5 * S.scale || tp > 1.01 * S.scale) continue;
        const double X[3] = {o[0] + tp * d[0], o[1] + tp * d[1], o[2] + tp * d[2]};
        const double px = E.a1[g][0] * X[0] + E.a1[g][1] * X[1] + E.a1[g][2] * X[2];
        const double py = E.a2[g][0] * X[0] + E.a2[g][1] * X[1] + E.a2[g][2] * X[2];
        const double fx = (px - E.lo[g][0]) * E.inv[g][0], fy = (py - E.lo[g][1]) * E.inv[g][1];
        if (!(fx >= 0.0 && fy >= 0.0 && fx < E.gx[g] && fy < E.gy[g])) continue;
        const int cell = E.cell0[g] + (int)fy * E.gx[g] + (int)fx;
        for (int q = E.cell_start[cell]; q < E.cell_start[cell + 1]; ++q) {
          const int k = E.cell_tri[q];
          const double t = hit_tri(S.emit.prim + (size_t)k * 9, o, d, S.t_eps);
          if (t == INFINITY) continue;
          const int id = S.emit.prim_id[k];
          if (t < te || (t == te && id < ie)) {
            te = t;
            ie = id;
          }
        }
      }
      if (ok) return;
    }
  }
  bvh_closest<D>(S.emit, S.t_eps, 1e-5f * (float)S.scale, o, d, te, ie);
}

// Distance to the bounds box exit (src/scene.py:295-303), NaN semantics of numpy.
template <int D>
__device__ inline double bounds_exit(const DevScene& S, const double* o, const double* d) {
  double res = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double t1 = __ddiv_rn(sub(S.bmin[a], o[a]), d[a]);
    double t2 = __ddiv_rn(sub(S.bmax[a], o[a]), d[a]);
    double far = isnan(t1) ? INFINITY : np_max(t1, t2);
    res = (a == 0) ? far : np_min(res, far);
  }
  return res;
}

// ---------------------------------------------------------------------------
// Surface shading (src/transport.py:127-254)
// ---------------------------------------------------------------------------

// Extension (oracle delta_incident): one delta light seen from o — the unit direction d
// toward it and its attenuated geometric term, 0 when occluded.  Point light: e^{−σt r} /
// max(r, 1e-6·scale)^{D−1}, visible iff the nearest hit lies at t ≥ r(1 − 1e-6) (the
// reference's shadow-ray rule); directional light: the ray must leave the scene without a
// hit, e^{−σt s_b} over the distance s_b to the bounds exit.
template <int D, class Stack = LocalStack>
__device__ inline double delta_term(const DevScene& S, const double* L8, const double* o, double* d,
                                    Stack* stk = nullptr) {
  const double off = 1e-6 * S.scale;
  d[0] = d[1] = d[2] = 0.0;
  if (L8[0] == 0.0) {
    double to[3], r2 = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      to[a] = sub(L8[1 + a], o[a]);
      r2 = add(r2, mul(to[a], to[a]));
    }
    const double r = sqrt(r2);
    if (!(r > off)) return 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) d[a] = __ddiv_rn(to[a], r);
    if (occluded<D, Stack>(S, o, d, mul(r, 1.0 - 1e-6), -1, stk)) return 0.0;
    const double rm = fmax(r, off);
    return __ddiv_rn(exp(-S.sigma_t * r), D == 3 ? mul(rm, rm) : rm);
  }
#pragma unroll
  for (int a = 0; a < D; ++a) d[a] = L8[1 + a];
  if (occluded<D, Stack>(S, o, d, INFINITY, -1, stk)) return 0.0;
  return exp(-S.sigma_t * bounds_exit<D>(S, o, d));
}

template <int D, class Stack = LocalStack>
__device__ void direct_light(const DevScene& S, const double* p, const double* n, double acc[3],
                             Stack* stk = nullptr) {
  acc[0] = acc[1] = acc[2] = 0.0;
  const double off = 1e-6 * S.scale;
  double org[3];
#pragma unroll
  for (int a = 0; a < D; ++a) org[a] = add(p[a], mul(off, n[a]));
  for (int l = 0; l < S.n_lights; ++l) {  // extension: delta lights, same cosine and ÷π / ÷2
    const double* L8 = S.lights + 8 * (size_t)l;
    double dd[3];
    const double val = delta_term<D, Stack>(S, L8, org, dd, stk);
    if (!(val > 0.0)) continue;
    double cp = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) cp = add(cp, mul(n[a], dd[a]));
    cp = mul(fmax(cp, 0.0), val);
    acc[0] = add(acc[0], mul(cp, L8[4]));
    acc[1] = add(acc[1], mul(cp, L8[5]));
    acc[2] = add(acc[2], mul(cp, L8[6]));
  }
  for (int j = 0; j < S.n_es; ++j) {
    const double* P = S.es_pos + (size_t)j * D;
    double to[3], dd[3] = {0.0, 0.0, 0.0};
    double r2 = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      to[a] = sub(P[a], org[a]);
      r2 = add(r2, mul(to[a], to[a]));
    }
    double r = sqrt(r2);
    bool ok = r > off;
    if (!ok) continue;
#pragma unroll
    for (int a = 0; a < D; ++a) dd[a] = __ddiv_rn(to[a], r);
    int e = S.es_surf[j];
    const double* N = S.normal + (size_t)e * D;
    double cp = 0.0, cq = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      cp = add(cp, mul(n[a], dd[a]));
      cq = add(cq, mul(dd[a], N[a]));
    }
    cp = fmax(cp, 0.0);
    cq = fabs(cq);
    if (!(cp > 0.0 && cq > 0.0)) continue;
    if (occluded<D, Stack>(S, org, dd, mul(r, 1.0 - 1e-6), -1, stk)) continue;
    double rm = fmax(r, off);
    double g = __ddiv_rn(mul(cp, cq), D == 3 ? mul(rm, rm) : rm);
    g = mul(mul(g, exp(-S.sigma_t * r)), S.es_w[j]);
    const double* E = S.emission + (size_t)e * 3;
    acc[0] = add(acc[0], mul(g, E[0]));
    acc[1] = add(acc[1], mul(g, E[1]));
    acc[2] = add(acc[2], mul(g, E[2]));
  }
  const double norm = (D == 3) ? 3.141592653589793 : 2.0;
  acc[0] = __ddiv_rn(acc[0], norm);
  acc[1] = __ddiv_rn(acc[1], norm);
  acc[2] = __ddiv_rn(acc[2], norm);
}

// Outgoing radiance at a hit: emission + albedo·direct; idx < 0 → 0.
template <int D, class Stack = LocalStack>
__device__ void surface_radiance(const DevScene& S, int idx, const double* hit, const double* dir,
                                 double out[3], Stack* stk = nullptr) {
  out[0] = out[1] = out[2] = 0.0;
  if (idx < 0) return;
  const double* E = S.emission + (size_t)idx * 3;
  out[0] = E[0];
  out[1] = E[1];
  out[2] = E[2];
  if (!S.reflective) return;
  const double* A = S.albedo + (size_t)idx * 3;
  if (!(A[0] > 0.0 || A[1] > 0.0 || A[2] > 0.0)) return;
  const double* nn = S.normal + (size_t)idx * D;
  double sd = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) sd = add(sd, mul(nn[a], dir[a]));
  double sg = sd > 0.0 ? 1.0 : (sd < 0.0 ? -1.0 : 1.0);
  double no[3];
#pragma unroll
  for (int a = 0; a < D; ++a) no[a] = -(nn[a] * sg);
  double dl[3];
  direct_light<D, Stack>(S, hit, no, dl, stk);
  out[0] = add(out[0], mul(A[0], dl[0]));
  out[1] = add(out[1], mul(A[1], dl[1]));
  out[2] = add(out[2], mul(A[2], dl[2]));
}

// trace_or_bounds (src/scene.py:306-315)
template <int D, class Stack = LocalStack>
__device__ __forceinline__ void trace_or_bounds(const DevScene& S, const double* o, const double* d,
                                                double& s, int& idx, Stack* stk = nullptr) {
  double t;
  trace_closest<D, Stack>(S, o, d, t, idx, stk);
  s = isfinite(t) ? t : bounds_exit<D>(S, o, d);
}

// ---------------------------------------------------------------------------
// Form factors with derivatives (src/formfactor.py:85-343), float64 scalar form.
// H is returned symmetrized, packed as xx, xy, (xz), yy, (yz), (zz).
// ---------------------------------------------------------------------------

constexpr double kPi = 3.141592653589793;

__device__ inline bool ff_triangle(const double* r1v, const double* r2v, const double* r3v, double& F,
                                   double g[3], double H[6]) {
  const double* R[3] = {r1v, r2v, r3v};
  double r[3];
  for (int i = 0; i < 3; ++i) r[i] = sqrt(R[i][0] * R[i][0] + R[i][1] * R[i][1] + R[i][2] * R[i][2]);
  if (!(r[0] > 0.0 && r[1] > 0.0 && r[2] > 0.0)) return false;
  double c23[3], c12[3], c31[3];
  cross3(R[1], R[2], c23);
  cross3(R[0], R[1], c12);
  cross3(R[2], R[0], c31);
  double A = R[0][0] * c23[0] + R[0][1] * c23[1] + R[0][2] * c23[2];
  double d12 = R[0][0] * R[1][0] + R[0][1] * R[1][1] + R[0][2] * R[1][2];
  double d23 = R[1][0] * R[2][0] + R[1][1] * R[2][1] + R[1][2] * R[2][2];
  double d13 = R[0][0] * R[2][0] + R[0][1] * R[2][1] + R[0][2] * R[2][2];
  double B = r[0] * r[1] * r[2] + d12 * r[2] + d23 * r[0] + d13 * r[1];
  double aA = fabs(A);
  if (!(aA >= 1e-12 * r[0] * r[1] * r[2])) return false;
  const double k2pi = 1.0 / (2.0 * kPi);
  F = atan2(aA, B) * k2pi;  // 2·atan2 / 4π
  // Closed forms of the reference's term-by-term chain (src/formfactor.py:199-251) with
  // unit vectors n_i = R_i/r_i, σ₂ = r₀r₁ + r₀r₂ + r₁r₂, ρ = r₀ + r₁ + r₂, m = Σn_i,
  // d = (d23, d13, d12):  ∇B = −Σ (σ₂ + d_i) n_i
  //   HB = (Σ c_i/r_i + 2ρ) I − Σ (c_i/r_i + ρ) n_i n_iᵀ + ρ m mᵀ,  c_i = Π_{j≠i} r_j + d_i
  // (the outer(∇r, ·) terms of j_rrr and j_dot_term sum to ρ·(m mᵀ − Σ n_i n_iᵀ)).
  const double sg = A >= 0.0 ? 1.0 : -1.0;
  const double s2 = r[0] * r[1] + r[0] * r[2] + r[1] * r[2];
  const double rho = r[0] + r[1] + r[2];
  const double dk[3] = {d23, d13, d12};
  double n[3][3], cr[3], gU[3], gB[3], m[3];
  double diag = 2.0 * rho;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double inv = 1.0 / r[i];
#pragma unroll
    for (int c = 0; c < 3; ++c) n[i][c] = R[i][c] * inv;
    cr[i] = (r[(i + 1) % 3] * r[(i + 2) % 3] + dk[i]) * inv;  // c_i / r_i
    diag += cr[i];
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    gU[c] = -sg * (c12[c] + c23[c] + c31[c]);
    gB[c] = -((s2 + dk[0]) * n[0][c] + (s2 + dk[1]) * n[1][c] + (s2 + dk[2]) * n[2][c]);
    m[c] = n[0][c] + n[1][c] + n[2][c];
  }
  // one reciprocal of den = A² + B² for the gradient and Hessian (results within a few ulp
  // of the reference's divisions)
  const double iden = 1.0 / (A * A + B * B);
  double num[3], gD[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    num[c] = B * gU[c] - aA * gB[c];
    gD[c] = 2.0 * aA * gU[c] + 2.0 * B * gB[c];
    g[c] = num[c] * iden * k2pi;
  }
  const double ia = -aA * iden, id2 = -0.5 * iden * iden;
  int e = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int b = a; b < 3; ++b) {
      double hb = (a == b ? diag : 0.0) + rho * m[a] * m[b];
#pragma unroll
      for (int i = 0; i < 3; ++i) hb -= (cr[i] + rho) * n[i][a] * n[i][b];
      H[e++] = (ia * hb + id2 * (num[a] * gD[b] + num[b] * gD[a])) * k2pi;
    }
  }
  return true;
}

// The ok-mask of ff_triangle in float64 (r_i > 0 and |A| ≥ 1e-12·r₁r₂r₃ with the same
// operations), so the element counts stay exact whatever precision evaluates the element.
__device__ __forceinline__ bool ff_triangle_ok(const double* r1v, const double* r2v, const double* r3v) {
  const double r0 = sqrt(r1v[0] * r1v[0] + r1v[1] * r1v[1] + r1v[2] * r1v[2]);
  const double r1 = sqrt(r2v[0] * r2v[0] + r2v[1] * r2v[1] + r2v[2] * r2v[2]);
  const double r2 = sqrt(r3v[0] * r3v[0] + r3v[1] * r3v[1] + r3v[2] * r3v[2]);
  if (!(r0 > 0.0 && r1 > 0.0 && r2 > 0.0)) return false;
  double c23[3];
  cross3(r2v, r3v, c23);
  const double A = r1v[0] * c23[0] + r1v[1] * c23[1] + r1v[2] * c23[2];
  return fabs(A) >= 1e-12 * r0 * r1 * r2;
}

// float32 evaluation of ff_triangle's closed forms for an element whose ok-mask was decided
// in float64 (ff_triangle_ok); inputs are the float-rounded offsets y_i − x.  The 3D form is
// well conditioned (worst record H 2.8e-5 relative in float32).
__device__ inline void ff_triangle_f32(const float* r1v, const float* r2v, const float* r3v, float& F, float g[3],
                                       float H[6]) {
  const float* R[3] = {r1v, r2v, r3v};
  float r[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) r[i] = sqrtf(R[i][0] * R[i][0] + R[i][1] * R[i][1] + R[i][2] * R[i][2]);
  float c23[3], c12[3], c31[3];
  c23[0] = R[1][1] * R[2][2] - R[1][2] * R[2][1];
  c23[1] = R[1][2] * R[2][0] - R[1][0] * R[2][2];
  c23[2] = R[1][0] * R[2][1] - R[1][1] * R[2][0];
  c12[0] = R[0][1] * R[1][2] - R[0][2] * R[1][1];
  c12[1] = R[0][2] * R[1][0] - R[0][0] * R[1][2];
  c12[2] = R[0][0] * R[1][1] - R[0][1] * R[1][0];
  c31[0] = R[2][1] * R[0][2] - R[2][2] * R[0][1];
  c31[1] = R[2][2] * R[0][0] - R[2][0] * R[0][2];
  c31[2] = R[2][0] * R[0][1] - R[2][1] * R[0][0];
  const float A = R[0][0] * c23[0] + R[0][1] * c23[1] + R[0][2] * c23[2];
  const float d12 = R[0][0] * R[1][0] + R[0][1] * R[1][1] + R[0][2] * R[1][2];
  const float d23 = R[1][0] * R[2][0] + R[1][1] * R[2][1] + R[1][2] * R[2][2];
  const float d13 = R[0][0] * R[2][0] + R[0][1] * R[2][1] + R[0][2] * R[2][2];
  const float B = r[0] * r[1] * r[2] + d12 * r[2] + d23 * r[0] + d13 * r[1];
  const float aA = fabsf(A);
  const float k2pi = (float)(1.0 / (2.0 * kPi));
  F = atan2f(aA, B) * k2pi;
  const float sg = A >= 0.0f ? 1.0f : -1.0f;
  const float s2 = r[0] * r[1] + r[0] * r[2] + r[1] * r[2];
  const float rho = r[0] + r[1] + r[2];
  const float dk[3] = {d23, d13, d12};
  float n[3][3], cr[3], gU[3], gB[3], m[3];
  float diag = 2.0f * rho;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const float inv = 1.0f / r[i];
#pragma unroll
    for (int c = 0; c < 3; ++c) n[i][c] = R[i][c] * inv;
    cr[i] = (r[(i + 1) % 3] * r[(i + 2) % 3] + dk[i]) * inv;
    diag += cr[i];
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    gU[c] = -sg * (c12[c] + c23[c] + c31[c]);
    gB[c] = -((s2 + dk[0]) * n[0][c] + (s2 + dk[1]) * n[1][c] + (s2 + dk[2]) * n[2][c]);
    m[c] = n[0][c] + n[1][c] + n[2][c];
  }
  const float iden = 1.0f / (A * A + B * B);
  float num[3], gD[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    num[c] = B * gU[c] - aA * gB[c];
    gD[c] = 2.0f * aA * gU[c] + 2.0f * B * gB[c];
    g[c] = num[c] * iden * k2pi;
  }
  const float ia = -aA * iden, id2 = -0.5f * iden * iden;
  int e = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int b = a; b < 3; ++b) {
      float hb = (a == b ? diag : 0.0f) + rho * m[a] * m[b];
#pragma unroll
      for (int i = 0; i < 3; ++i) hb -= (cr[i] + rho) * n[i][a] * n[i][b];
      H[e++] = (ia * hb + id2 * (num[a] * gD[b] + num[b] * gD[a])) * k2pi;
    }
  }
}

__device__ inline bool ff_segment(const double* u, const double* v, double& F, double g[2], double H[3]) {
  double r0 = sqrt(u[0] * u[0] + u[1] * u[1]);
  double r1 = sqrt(v[0] * v[0] + v[1] * v[1]);
  if (!(r0 > 0.0 && r1 > 0.0)) return false;
  double dt = u[0] * v[0] + u[1] * v[1];
  double cr = u[0] * v[1] - u[1] * v[0];
  double gam = atan2(fabs(cr), dt);
  if (!(gam > 1e-5 && gam < kPi - 1e-5)) return false;
  F = gam / (2.0 * kPi);
  double ab = r0 * r1;
  double c = fmin(fmax(dt / ab, -1.0), 1.0);
  double sn = fabs(cr) / ab;
  double a2 = r0 * r0, b2 = r1 * r1;
  double gc[2];
  for (int k = 0; k < 2; ++k) gc[k] = (c / a2) * u[k] + (c / b2) * v[k] - (u[k] + v[k]) / ab;
  for (int k = 0; k < 2; ++k) g[k] = -(gc[k] / sn) / (2.0 * kPi);
  const int pij[3][2] = {{0, 0}, {0, 1}, {1, 1}};
  double w0[2], s[2];
  for (int k = 0; k < 2; ++k) {
    w0[k] = u[k] / (a2 * r0 * r1) + v[k] / (r0 * b2 * r1);
    s[k] = u[k] + v[k];
  }
  for (int e = 0; e < 3; ++e) {
    int a = pij[e][0], b = pij[e][1];
    double I = (a == b) ? 1.0 : 0.0;
    double jc = 0.5 * (u[a] * gc[b] + u[b] * gc[a]) / a2 + 2.0 * (c / (a2 * a2)) * u[a] * u[b] -
                (c / a2) * I + 0.5 * (v[a] * gc[b] + v[b] * gc[a]) / b2 +
                2.0 * (c / (b2 * b2)) * v[a] * v[b] - (c / b2) * I + 2.0 * I / ab -
                0.5 * (s[a] * w0[b] + s[b] * w0[a]);
    H[e] = -(jc / sn + (c / (sn * sn * sn)) * gc[a] * gc[b]) / (2.0 * kPi);
  }
  return true;
}

// float32 form of element_q (3D), for unit-scaled inputs (every length divided by L, σt
// multiplied by L): the gradient part then carries 1/L and the Hessian part 1/L², which the
// caller restores in float64.
__device__ __forceinline__ void element_q_f32(const float* w, float dr, float sigma_t, float F, const float* gF,
                                              const float* HF, float* q /* 10 */) {
  const float T = __expf(-sigma_t * dr);
  const float idr = 1.0f / dr, idr2 = idr * idr;
  float gT[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) gT[a] = (-sigma_t * w[a]) * idr * T;
  q[0] = T * F;
#pragma unroll
  for (int a = 0; a < 3; ++a) q[1 + a] = T * gF[a] + gT[a] * F;
  int e = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int b = a; b < 3; ++b) {
      const float ww = w[a] * w[b];
      const float I = (a == b) ? 1.0f : 0.0f;
      const float HT = -sigma_t * (I * idr - ww * idr2 * idr - sigma_t * ww * idr2) * T;
      q[4 + e] = T * HF[e] + gT[a] * gF[b] + gF[a] * gT[b] + HT * F;
      ++e;
    }
  }
}

// Element contribution q = (T·F, ∇(T·F), H(T·F)) for representative offset w = x − y_rep
// at stored distance dr (src/subdivision.py:320-340, src/transport.py:108-119).
template <int D>
__device__ inline void element_q(const double* w, double dr, double sigma_t, double F, const double* gF,
                                 const double* HF, double* q /* 1 + D + D(D+1)/2 */) {
  constexpr int NH = D * (D + 1) / 2;
  double T = exp(-sigma_t * dr);
  // one reciprocal of dr for ∇T and HT (within a few ulp of the reference's divisions)
  const double idr = 1.0 / dr, idr2 = idr * idr;
  double gT[D];
#pragma unroll
  for (int a = 0; a < D; ++a) gT[a] = (-sigma_t * w[a]) * idr * T;
  q[0] = T * F;
#pragma unroll
  for (int a = 0; a < D; ++a) q[1 + a] = T * gF[a] + gT[a] * F;
  int e = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
#pragma unroll
    for (int b = a; b < D; ++b) {
      double ww = w[a] * w[b];
      double I = (a == b) ? 1.0 : 0.0;
      double HT = -sigma_t * (I * idr - ww * idr2 * idr - sigma_t * ww * idr2) * T;
      q[1 + D + e] = T * HF[e] + gT[a] * gF[b] + gF[a] * gT[b] + HT * F;
      ++e;
    }
  }
  (void)NH;
}

// ---------------------------------------------------------------------------
// Stratified directions (src/scene.py:401-434)
// ---------------------------------------------------------------------------

template <int D>
__device__ inline void stratum_direction(int k, const BuildParams& P, Pcg64 g0, const JumpTables& jt,
                                         double* out) {
  if constexpr (D == 2) {
    // θ = (k + ξ)·2π/n  (src/scene.py:415-418)
    Pcg64 g = g0;
    pcg_advance(g, (unsigned long long)k, jt);
    double xi = g.next_double();
    double th = mul(add((double)k, xi), __ddiv_rn(2.0 * kPi, (double)P.n_angular));
    out[0] = cos(th);
    out[1] = sin(th);
  } else {
    // z = 1 − 2(r+u)/rows, φ = (c+v)·2π/cols (src/scene.py:420-431); u block then v block
    int r = k / P.cols, c = k - r * P.cols;
    Pcg64 g = g0;
    pcg_advance(g, (unsigned long long)k, jt);
    double u = g.next_double();
    Pcg64 h = g0;
    pcg_advance(h, (unsigned long long)P.rows * P.cols + k, jt);
    double v = h.next_double();
    double z = sub(1.0, __ddiv_rn(mul(2.0, add((double)r, u)), (double)P.rows));
    double phi = mul(add((double)c, v), __ddiv_rn(2.0 * kPi, (double)P.cols));
    double sq = sqrt(fmax(sub(1.0, mul(z, z)), 0.0));
    double sp, cp;
    sincos(phi, &sp, &cp);
    out[0] = mul(sq, cp);
    out[1] = mul(sq, sp);
    out[2] = z;
  }
}

}  // namespace vc
