// Occlusion-unaware baseline estimator on the device:
// baseline_estimate (src/subdivision.py:416-521) + make_baseline_record
// (src/cache.py:190-226).
//
// Thread per (record, direction): the stratified primary direction from the record's
// PCG64 stream (same draws as the subdivision build), trace_or_bounds, surface radiance
// and oriented normal at the hit, the rigid-path value/gradient of the final segment,
// then max_media_bounces − 1 transmittance-sampled collisions with uniform secondary
// directions.  Draw offsets follow the reference's batch order: after the 2n (3D) or
// n (2D) direction draws, bounce b consumes rng.random(n) for the collision distances
// and then rng.random(n) (2D) / rng.random((n, 2)) (3D) for the new directions — drawn
// for every sample, colliding or not — so sample i jumps straight to its draws.
// Per-record sums are block-reduced in a fixed order (deterministic) and finalized
// into (value, grad) means and the sphere record of log_gradient_radius.
#include <algorithm>
#include <cmath>
#include <vector>

#include "vc_api_internal.h"
#include "vc_build.h"
#include "vc_device.cuh"

namespace vc {

constexpr int kBlBS = 128;
__constant__ double kLuma[3] = {0.2126, 0.7152, 0.0722};  // LUMINANCE_WEIGHTS (src/scene.py:24)
constexpr double kBaselineCosMin = 1e-4;              // BASELINE_COS_MIN (src/subdivision.py:53)

struct BaselineParams {
  BuildParams P;  // n_angular, rows, cols
  int n_bounce;   // max(0, max_media_bounces − 1)
  double fb;      // f̄ = σs / full_angle
};

// per_sample (src/subdivision.py:448-471) for one final segment points → hit
template <int D>
__device__ inline void baseline_segment(const DevScene& S, const double* p, const double* h, const double* lo,
                                        const double* nrm, double weight, double val[3], double grad[3][D]) {
  double w[D];
  double r2 = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    w[a] = sub(p[a], h[a]);
    r2 = add(r2, mul(w[a], w[a]));
  }
  double r = sqrt(r2);
  if (!(r > 0.0)) r = 1.0;
  const double tr = exp(mul(-S.sigma_t, r));
  const double wt = mul(weight, tr);
#pragma unroll
  for (int c = 0; c < 3; ++c) val[c] = mul(wt, lo[c]);
  double ndw = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) ndw = add(ndw, mul(nrm[a], w[a]));
  const bool safe = ndw > mul(kBaselineCosMin, r);
  const double inv_ndw = safe ? __ddiv_rn(1.0, ndw) : 0.0;
  const double rr = mul(r, r);
  double vec[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const double gtr = mul(__ddiv_rn(mul(-S.sigma_t, w[a]), r), tr);  // ∇T_r (src/transport.py:108-110)
    double g = sub(mul(nrm[a], inv_ndw), __ddiv_rn(mul((double)D, w[a]), rr));
    g = safe ? g : 0.0;
    vec[a] = add(gtr, mul(tr, g));
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double wl = mul(weight, lo[c]);
#pragma unroll
    for (int a = 0; a < D; ++a) grad[c][a] = mul(wl, vec[a]);
  }
}

template <int D>
__device__ inline void oriented_normal(const DevScene& S, int idx, const double* dir, double* out) {
#pragma unroll
  for (int a = 0; a < D; ++a) out[a] = 0.0;
  if (idx < 0) return;
  const double* nn = S.normal + (size_t)idx * D;
  double sd = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) sd = add(sd, mul(nn[a], dir[a]));
  const double sg = sd > 0.0 ? 1.0 : (sd < 0.0 ? -1.0 : 1.0);
#pragma unroll
  for (int a = 0; a < D; ++a) out[a] = -(nn[a] * sg);
}

// components per sample and kind: value(3), grad(3D), luminance, |∇luminance|
template <int D>
__host__ __device__ constexpr int bl_comps() {
  return 2 * (3 + 3 * D + 2);
}

template <int D>
__global__ void __launch_bounds__(kBlBS) k_baseline(DevScene S, BaselineParams BP, const double* X,
                                                   const uint64_t* rng, JumpTables jt, double* partial,
                                                   double* samples, int* max_coll) {
  constexpr int NC = bl_comps<D>();
  __shared__ double sm[NC][kBlBS + 1];
  const int rec = blockIdx.y;
  const int n = BP.P.n_angular;
  const int i = blockIdx.x * kBlBS + threadIdx.x;
  double acc[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) acc[k] = 0.0;
  if (i < n) {
    const Pcg64 g0 = pcg_load(rng + (size_t)rec * 4);
    double x[D], d[D];
#pragma unroll
    for (int a = 0; a < D; ++a) x[a] = X[(size_t)rec * D + a];
    stratum_direction<D>(i, BP.P, g0, jt, d);
    double s;
    int idx;
    trace_or_bounds<D>(S, x, d, s, idx);
    double hit[D], lo[3], nrm[D];
#pragma unroll
    for (int a = 0; a < D; ++a) hit[a] = add(x[a], mul(s, d[a]));
    surface_radiance<D>(S, idx, hit, d, lo);
    oriented_normal<D>(S, idx, d, nrm);
    double v[3], gr[3][D];
    baseline_segment<D>(S, x, hit, lo, nrm, BP.fb, v, gr);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      acc[c] = v[c];
#pragma unroll
      for (int a = 0; a < D; ++a) acc[3 + c * D + a] = gr[c][a];
    }
    // multiple scattering: collisions along the current segment (src/subdivision.py:480-509)
    if (S.sigma_t > 0.0 && S.sigma_s > 0.0 && BP.n_bounce > 0) {
      const unsigned long long n_dir_draws = (D == 3) ? 2ULL * n : (unsigned long long)n;
      const unsigned long long per_bounce = (unsigned long long)n * (D == 3 ? 3 : 2);
      const double ratio = __ddiv_rn(S.sigma_s, S.sigma_t);
      double weight = BP.fb, pos[D], cur_d[D], cur_s = s;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        pos[a] = x[a];
        cur_d[a] = d[a];
      }
      int b = 0;
      for (; b < BP.n_bounce; ++b) {
        const unsigned long long base = n_dir_draws + (unsigned long long)b * per_bounce;
        Pcg64 gt = g0;
        pcg_advance(gt, base + (unsigned long long)i, jt);
        const double u = gt.next_double();
        const double t = __ddiv_rn(-log1p(-u), S.sigma_t);
        if (!(t < cur_s)) break;  // no collision: this sample stays dead
#pragma unroll
        for (int a = 0; a < D; ++a) pos[a] = add(pos[a], mul(t, cur_d[a]));
        weight = mul(weight, ratio);
        double nd[D];
        Pcg64 gu = g0;
        if (D == 2) {
          pcg_advance(gu, base + (unsigned long long)n + (unsigned long long)i, jt);
          const double th = mul(2.0 * kPi, gu.next_double());
          nd[0] = cos(th);
          nd[D - 1] = sin(th);
        } else {
          pcg_advance(gu, base + (unsigned long long)n + 2ULL * i, jt);
          const double u0 = gu.next_double(), u1 = gu.next_double();
          const double z = sub(1.0, mul(2.0, u0));
          const double phi = mul(2.0 * kPi, u1);
          const double sq = sqrt(fmax(sub(1.0, mul(z, z)), 0.0));
          double sp, cp;
          sincos(phi, &sp, &cp);
          nd[0] = mul(sq, cp);
          nd[1] = mul(sq, sp);
          nd[D - 1] = z;
        }
        double s2;
        int idx2;
        trace_or_bounds<D>(S, pos, nd, s2, idx2);
        double h2[D], lo2[3], n2[D];
#pragma unroll
        for (int a = 0; a < D; ++a) h2[a] = add(pos[a], mul(s2, nd[a]));
        surface_radiance<D>(S, idx2, h2, nd, lo2);
        oriented_normal<D>(S, idx2, nd, n2);
        baseline_segment<D>(S, pos, h2, lo2, n2, weight, v, gr);
        constexpr int M0 = 3 + 3 * D + 2;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          acc[M0 + c] = add(acc[M0 + c], v[c]);
#pragma unroll
          for (int a = 0; a < D; ++a) acc[M0 + 3 + c * D + a] = add(acc[M0 + 3 + c * D + a], gr[c][a]);
        }
#pragma unroll
        for (int a = 0; a < D; ++a) cur_d[a] = nd[a];
        cur_s = s2;
      }
      if (b > 0) atomicMax(max_coll + rec, b);  // collisions along this path
    }
    // luminance value and gradient norm per kind (src/subdivision.py:512-521)
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int o = k * (3 + 3 * D + 2);
      double lv = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) lv = add(lv, mul(acc[o + c], kLuma[c]));
      double q = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        double lg = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) lg = add(lg, mul(acc[o + 3 + c * D + a], kLuma[c]));
        q = add(q, mul(lg, lg));
      }
      acc[o + 3 + 3 * D] = lv;
      acc[o + 3 + 3 * D + 1] = sqrt(q);
      if (samples) {
        double* sp = samples + (((size_t)rec * 2 + k) * 2) * n;
        sp[i] = lv;
        sp[(size_t)n + i] = acc[o + 3 + 3 * D + 1];
      }
    }
  }
  // fixed-order block reduction of every component
#pragma unroll
  for (int k = 0; k < NC; ++k) sm[k][threadIdx.x] = acc[k];
  __syncthreads();
  for (int w = kBlBS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int k = 0; k < NC; ++k) sm[k][threadIdx.x] = add(sm[k][threadIdx.x], sm[k][threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x < NC) partial[((size_t)rec * gridDim.x + blockIdx.x) * NC + threadIdx.x] = sm[threadIdx.x][0];
}

// means, record rows (position, value, grad, I, radius·1) per kind
template <int D>
__global__ void k_baseline_final(DevScene S, BaselineParams BP, const double* X, const double* partial, int nblk,
                                 int B, double alpha, double* est, double* records, const int* max_coll,
                                 long long* draws) {
  constexpr int NC = bl_comps<D>();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 2 * B) return;
  const int rec = t >> 1, k = t & 1;
  const int o = k * (3 + 3 * D + 2);
  if (draws && k == 0) {
    // the reference draws n collision distances per bounce it enters and n·(d − 1) direction
    // doubles per bounce with a collision; it leaves the loop at the first bounce without one
    const long long n = BP.P.n_angular;
    long long c = n * (D == 3 ? 2 : 1);
    if (S.sigma_t > 0.0 && S.sigma_s > 0.0 && BP.n_bounce > 0) {
      const int m = max_coll[rec];
      c += (long long)m * n * (D == 3 ? 3 : 2) + (m < BP.n_bounce ? n : 0);
    }
    draws[rec] = c;
  }
  double sum[3 + 3 * D + 2];
  for (int c = 0; c < 3 + 3 * D + 2; ++c) sum[c] = 0.0;
  for (int b = 0; b < nblk; ++b)
    for (int c = 0; c < 3 + 3 * D + 2; ++c) sum[c] = add(sum[c], partial[((size_t)rec * nblk + b) * NC + o + c]);
  const double nn = (double)BP.P.n_angular;
  constexpr int ES = 3 + 3 * D;
  if (est)
    for (int c = 0; c < ES; ++c) est[((size_t)rec * 2 + k) * ES + c] = __ddiv_rn(sum[c], nn);
  if (records) {
    // log_gradient_radius (src/cache.py:190-209)
    const double num = sum[ES], den = sum[ES + 1];
    const double r_max = mul(0.25, S.scale), r_min = mul(1e-3, S.scale);
    double r = r_max;
    if (den > 0.0) r = fmin(fmax(__ddiv_rn(mul(alpha, num), den), r_min), r_max);
    constexpr int RS = record_size(D);
    double* R = records + ((size_t)rec * 2 + k) * RS;
    for (int a = 0; a < D; ++a) R[a] = X[(size_t)rec * D + a];
    for (int c = 0; c < ES; ++c) R[D + c] = __ddiv_rn(sum[c], nn);
    for (int a = 0; a < D; ++a)
      for (int b = 0; b < D; ++b) R[D + ES + a * D + b] = (a == b) ? 1.0 : 0.0;
    for (int a = 0; a < D; ++a) R[D + ES + D * D + a] = r;
  }
}

int baseline_impl(vc_scene* sc, int N, const double* x, const void* rng, const vc_baseline_params* prm,
                  double* est, double* records, double* samples, cudaStream_t st) {
  if (!sc || !prm) return fail(VC_EINVAL, "null scene or params");
  if (N < 0) return fail(VC_EINVAL, "n_records must be non-negative");
  if (sc->n_lights > 0)  // the extension covers the record build and its callers only
    return fail(VC_EINVAL, "delta lights (vc_scene_set_lights) are not supported by the baseline estimator");
  if (N == 0) return VC_OK;
  const int D = sc->dim;
  const int n = prm->n_angular;
  const bool host = prm->flags & VC_MEM_HOST;
  const bool words = prm->flags & VC_SEED_WORDS;
  if (prm->n_light_samples < 1) return fail(VC_EINVAL, "n_light_samples must be >= 1");
  BaselineParams BP{};
  BP.P.n_angular = n;
  if (D == 2) {
    if (n < 3) return fail(VC_EINVAL, "2D stratification needs n >= 3");
    BP.P.rows = 1;
    BP.P.cols = n;
  } else if (!grid_shape_3d(n, &BP.P.rows, &BP.P.cols)) {
    return fail(VC_EINVAL, "n=" + std::to_string(n) + " is not expressible as rows x cols with rows >= 2 and cols >= 3");
  }
  BP.n_bounce = std::max(0, prm->max_media_bounces - 1);
  BP.fb = sc->sigma_s * (1.0 / (D == 2 ? 2.0 * 3.141592653589793 : 4.0 * 3.141592653589793));
  {
    const int rc = check_inside(sc, N, x, host, "estimate center lies outside the medium bounds", st);
    if (rc) return rc;
  }
  int rc = ensure_emitters(sc, prm->n_light_samples);
  if (rc) return rc;
  cudaError_t err = cudaSuccess;
  JumpTables jt{jump_tables(&err)};
  if (!jt.tab) return cuda_fail(err, "jump tables");
  DevScene S = dev_scene(sc);
  const int nblk = (n + kBlBS - 1) / kBlBS;
  const int NC = D == 2 ? bl_comps<2>() : bl_comps<3>();
  const int ES = 3 + 3 * D, RS = record_size(D);
  const int B = std::min(N, 4096);
  Workspace ws;
  double* dx = (double*)ws.get(0, (size_t)B * D * 8, &err);
  uint64_t* drng = (uint64_t*)ws.get(1, (size_t)B * 32, &err);
  uint32_t* dw = (uint32_t*)ws.get(2, words ? (size_t)B * prm->seed_words * 4 + 4 : 16, &err);
  double* part = (double*)ws.get(3, (size_t)B * nblk * NC * 8, &err);
  double* dest = (double*)ws.get(4, (size_t)B * 2 * ES * 8, &err);
  double* drec = (double*)ws.get(5, (size_t)B * 2 * RS * 8, &err);
  double* dsmp = (double*)ws.get(6, samples ? (size_t)B * 4 * n * 8 : 16, &err);
  int* dmaxc = (int*)ws.get(7, (size_t)B * 4, &err);
  long long* ddraws = (long long*)ws.get(8, (size_t)B * 8, &err);
  if (err != cudaSuccess) return cuda_fail(err, "baseline workspace");
  long long launches = 0;
  for (int w0 = 0; w0 < N; w0 += B) {
    const int b = std::min(B, N - w0);
    const double* xin = x + (size_t)w0 * D;
    if (host) {
      err = cudaMemcpyAsync(dx, xin, (size_t)b * D * 8, cudaMemcpyHostToDevice, st);
      xin = dx;
    }
    const uint64_t* rin;
    if (words) {
      const uint32_t* wsrc = (const uint32_t*)rng + (size_t)w0 * prm->seed_words;
      if (host) {
        err = cudaMemcpyAsync(dw, wsrc, (size_t)b * prm->seed_words * 4, cudaMemcpyHostToDevice, st);
        wsrc = dw;
      }
      launch_seedseq(b, wsrc, prm->seed_words, drng, st);
      ++launches;
      rin = drng;
    } else if (host) {
      err = cudaMemcpyAsync(drng, (const uint64_t*)rng + (size_t)w0 * 4, (size_t)b * 32, cudaMemcpyHostToDevice, st);
      rin = drng;
    } else {
      rin = (const uint64_t*)rng + (size_t)w0 * 4;
    }
    if (err != cudaSuccess) return cuda_fail(err, "baseline upload");
    double* e_out = (host || !est) ? dest : est + (size_t)w0 * 2 * ES;
    double* r_out = (host || !records) ? drec : records + (size_t)w0 * 2 * RS;
    double* s_out = !samples ? nullptr : (host ? dsmp : samples + (size_t)w0 * 4 * n);
    long long* d_out = !prm->draws ? nullptr : (host ? ddraws : (long long*)prm->draws + w0);
    dim3 grid(nblk, b);
    err = cudaMemsetAsync(dmaxc, 0, (size_t)b * 4, st);
    if (err != cudaSuccess) return cuda_fail(err, "baseline memset");
    if (D == 2) {
      k_baseline<2><<<grid, kBlBS, 0, st>>>(S, BP, xin, rin, jt, part, s_out, dmaxc);
      k_baseline_final<2><<<(2 * b + 127) / 128, 128, 0, st>>>(S, BP, xin, part, nblk, b, prm->alpha, e_out, r_out,
                                                              dmaxc, d_out);
    } else {
      k_baseline<3><<<grid, kBlBS, 0, st>>>(S, BP, xin, rin, jt, part, s_out, dmaxc);
      k_baseline_final<3><<<(2 * b + 127) / 128, 128, 0, st>>>(S, BP, xin, part, nblk, b, prm->alpha, e_out, r_out,
                                                              dmaxc, d_out);
    }
    launches += 2;
    err = cudaGetLastError();
    if (err != cudaSuccess) return cuda_fail(err, "baseline launch");
    if (host) {
      if (est) err = cudaMemcpyAsync(est + (size_t)w0 * 2 * ES, dest, (size_t)b * 2 * ES * 8, cudaMemcpyDeviceToHost, st);
      if (err == cudaSuccess && records)
        err = cudaMemcpyAsync(records + (size_t)w0 * 2 * RS, drec, (size_t)b * 2 * RS * 8, cudaMemcpyDeviceToHost, st);
      if (err == cudaSuccess && samples)
        err = cudaMemcpyAsync(samples + (size_t)w0 * 4 * n, dsmp, (size_t)b * 4 * n * 8, cudaMemcpyDeviceToHost, st);
      if (err == cudaSuccess && prm->draws)
        err = cudaMemcpyAsync((long long*)prm->draws + w0, ddraws, (size_t)b * 8, cudaMemcpyDeviceToHost, st);
      if (err == cudaSuccess) err = cudaStreamSynchronize(st);
      if (err != cudaSuccess) return cuda_fail(err, "baseline download");
    }
  }
  count_launches(launches);
  if (!host) {  // scratch is freed with the workspace: finish before returning
    err = cudaStreamSynchronize(st);
    if (err != cudaSuccess) return cuda_fail(err, "baseline");
  }
  return VC_OK;
}

}  // namespace vc

using namespace vc;

extern "C" {

int vc_baseline_records(vc_scene* scene, int n_records, const double* x, const void* rng,
                        const vc_baseline_params* params, double* estimates, double* records, double* samples,
                        void* stream) {
  return baseline_impl(scene, n_records, x, rng, params, estimates, records, samples, (cudaStream_t)stream);
}

}  // extern "C"
