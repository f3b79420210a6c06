// Path-traced reference estimator on the device:
// path_trace_radiance (src/transport.py:318-391), the derivative oracle's inner loop
// (fd_derivatives, src/renderer.py:590-643) and the "path" render mode.
//
// Thread per (query point, sample).  The reference draws its variates per chunk of
// 2^16 samples in a fixed order — primary directions, then per bounce the collision
// distances, then the secondary directions — so sample i of chunk k finds its draws
// at fixed offsets of the point's PCG64 stream and jumps there directly (common random
// numbers across finite-difference offsets come for free: every offset point reuses
// the same stream).  Sums are block-reduced in a fixed order (deterministic).
#include <algorithm>
#include <cmath>

#include "vc_api_internal.h"
#include "vc_build.h"
#include "vc_device.cuh"

namespace vc {

constexpr int kPtBS = 128;
constexpr long long kPtChunk = 1LL << 16;  // _CHUNK (src/transport.py:34)

struct PathParams {
  long long n_samples;
  int n_bounce;  // max(0, max_media_bounces − 1)
  double fb;     // f̄
};

template <int D>
__device__ __forceinline__ void uniform_dir(Pcg64 g, double* d) {  // src/transport.py:274-285
  if (D == 2) {
    const double th = mul(2.0 * kPi, g.next_double());
    d[0] = cos(th);
    d[D - 1] = sin(th);
  } else {
    const double u0 = g.next_double(), u1 = g.next_double();
    const double z = sub(1.0, mul(2.0, u0));
    const double phi = mul(2.0 * kPi, u1);
    const double sq = sqrt(fmax(sub(1.0, mul(z, z)), 0.0));
    double sp, cp;
    sincos(phi, &sp, &cp);
    d[0] = mul(sq, cp);
    d[1] = mul(sq, sp);
    d[D - 1] = z;
  }
}

template <int D>
__global__ void __launch_bounds__(kPtBS) k_path(DevScene S, PathParams PP, const double* X, const uint64_t* rng,
                                               JumpTables jt, double* partial) {
  __shared__ double sm[6][kPtBS + 1];
  const int q = blockIdx.y;
  const long long i = (long long)blockIdx.x * kPtBS + threadIdx.x;
  double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  if (i < PP.n_samples) {
    constexpr int pd = (D == 2) ? 1 : 2;
    const long long k = i / kPtChunk, il = i - k * kPtChunk;
    const long long c = min(kPtChunk, PP.n_samples - k * kPtChunk);
    const long long per = pd + (long long)PP.n_bounce * (1 + pd);
    const unsigned long long base = (unsigned long long)(k * kPtChunk * per);
    const Pcg64 g0 = pcg_load(rng + (size_t)q * 4);
    double x[D], d[D];
#pragma unroll
    for (int a = 0; a < D; ++a) x[a] = X[(size_t)q * D + a];
    Pcg64 g = g0;
    pcg_advance(g, base + (unsigned long long)(il * pd), jt);
    uniform_dir<D>(g, d);
    double s;
    int idx;
    trace_or_bounds<D>(S, x, d, s, idx);
    double hit[D], lo[3];
#pragma unroll
    for (int a = 0; a < D; ++a) hit[a] = add(x[a], mul(s, d[a]));
    surface_radiance<D>(S, idx, hit, d, lo);
    const double T = exp(mul(-S.sigma_t, s));
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) acc[ch] = mul(T, lo[ch]);  // f̄ applied to the sum
    if (S.sigma_t > 0.0 && S.sigma_s > 0.0) {
      const double ratio = __ddiv_rn(S.sigma_s, S.sigma_t);
      double weight = PP.fb, pos[D], cur_d[D], cur_s = s;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        pos[a] = x[a];
        cur_d[a] = d[a];
      }
      const unsigned long long dist0 = base + (unsigned long long)(c * pd);
      const unsigned long long sec0 = dist0 + (unsigned long long)(PP.n_bounce * c);
      for (int b = 0; b < PP.n_bounce; ++b) {
        Pcg64 gt = g0;
        pcg_advance(gt, dist0 + (unsigned long long)(b * c + il), jt);
        const double t = __ddiv_rn(-log1p(-gt.next_double()), S.sigma_t);
        if (!(t < cur_s)) break;
#pragma unroll
        for (int a = 0; a < D; ++a) pos[a] = add(pos[a], mul(t, cur_d[a]));
        weight = mul(weight, ratio);
        Pcg64 gu = g0;
        pcg_advance(gu, sec0 + (unsigned long long)((b * c + il) * pd), jt);
        double nd[D];
        uniform_dir<D>(gu, nd);
        double s2;
        int idx2;
        trace_or_bounds<D>(S, pos, nd, s2, idx2);
        double h2[D], lo2[3];
#pragma unroll
        for (int a = 0; a < D; ++a) h2[a] = add(pos[a], mul(s2, nd[a]));
        surface_radiance<D>(S, idx2, h2, nd, lo2);
        const double wt = mul(weight, exp(mul(-S.sigma_t, s2)));
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) acc[3 + ch] = add(acc[3 + ch], mul(wt, lo2[ch]));
#pragma unroll
        for (int a = 0; a < D; ++a) cur_d[a] = nd[a];
        cur_s = s2;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 6; ++k) sm[k][threadIdx.x] = acc[k];
  __syncthreads();
  for (int w = kPtBS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
#pragma unroll
      for (int k = 0; k < 6; ++k) sm[k][threadIdx.x] = add(sm[k][threadIdx.x], sm[k][threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x < 6) partial[((size_t)q * gridDim.x + blockIdx.x) * 6 + threadIdx.x] = sm[threadIdx.x][0];
}

// (single, multiple) per point: (f̄·Σ T·L_o, Σ w·T·L_o) / n (src/transport.py:356, :385-391)
__global__ void k_path_final(PathParams PP, const double* partial, int nblk, int m, double* out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m * 6) return;
  const int q = t / 6, k = t % 6;
  double s = 0.0;
  for (int b = 0; b < nblk; ++b) s = add(s, partial[((size_t)q * nblk + b) * 6 + k]);
  if (k < 3) s = mul(PP.fb, s);
  out[(size_t)q * 6 + k] = __ddiv_rn(s, (double)PP.n_samples);
}

int path_impl(vc_scene* sc, int m, const double* x, const void* rng, long long n_samples, int max_media_bounces,
              int n_light_samples, int flags, int seed_words, double* out, cudaStream_t st) {
  if (!sc) return fail(VC_EINVAL, "null scene");
  if (m < 0) return fail(VC_EINVAL, "negative point count");
  if (n_samples < 1) return fail(VC_EINVAL, "n_samples must be positive");
  if (n_light_samples < 1) return fail(VC_EINVAL, "n_light_samples must be >= 1");
  if (sc->n_lights > 0)  // the extension covers the record build and its callers only
    return fail(VC_EINVAL, "delta lights (vc_scene_set_lights) are not supported by the path tracer");
  if (m == 0) return VC_OK;
  const int D = sc->dim;
  const bool host = flags & VC_MEM_HOST;
  const bool words = flags & VC_SEED_WORDS;
  {  // scene.contains (src/transport.py:337-338, src/scene.py:212-219)
    const int rc = check_inside(sc, m, x, host, "query point lies outside the medium bounds", st);
    if (rc) return rc;
  }
  int rc = ensure_emitters(sc, n_light_samples);
  if (rc) return rc;
  cudaError_t err = cudaSuccess;
  JumpTables jt{jump_tables(&err)};
  if (!jt.tab) return cuda_fail(err, "jump tables");
  DevScene S = dev_scene(sc);
  PathParams PP{};
  PP.n_samples = n_samples;
  PP.n_bounce = std::max(0, max_media_bounces - 1);
  PP.fb = sc->sigma_s * (1.0 / (D == 2 ? 2.0 * 3.141592653589793 : 4.0 * 3.141592653589793));
  const long long nblk_ll = (n_samples + kPtBS - 1) / kPtBS;
  if (nblk_ll > (1LL << 31) - 1) return fail(VC_EINVAL, "n_samples too large");
  const int nblk = (int)nblk_ll;
  const int B = std::max(1, std::min(m, (int)std::min<long long>(65535, (1LL << 26) / nblk_ll + 1)));
  Workspace ws;
  double* dx = (double*)ws.get(0, (size_t)B * D * 8, &err);
  uint64_t* drng = (uint64_t*)ws.get(1, (size_t)B * 32, &err);
  uint32_t* dw = (uint32_t*)ws.get(2, words ? (size_t)B * seed_words * 4 + 4 : 16, &err);
  double* part = (double*)ws.get(3, (size_t)B * nblk * 6 * 8, &err);
  double* dout = (double*)ws.get(4, (size_t)B * 6 * 8, &err);
  if (err != cudaSuccess) return cuda_fail(err, "path workspace");
  long long launches = 0;
  for (int w0 = 0; w0 < m; w0 += B) {
    const int b = std::min(B, m - w0);
    const double* xin = x + (size_t)w0 * D;
    if (host) {
      err = cudaMemcpyAsync(dx, xin, (size_t)b * D * 8, cudaMemcpyHostToDevice, st);
      xin = dx;
    }
    const uint64_t* rin;
    if (words) {
      const uint32_t* wsrc = (const uint32_t*)rng + (size_t)w0 * seed_words;
      if (host) {
        err = cudaMemcpyAsync(dw, wsrc, (size_t)b * seed_words * 4, cudaMemcpyHostToDevice, st);
        wsrc = dw;
      }
      launch_seedseq(b, wsrc, seed_words, drng, st);
      ++launches;
      rin = drng;
    } else if (host) {
      err = cudaMemcpyAsync(drng, (const uint64_t*)rng + (size_t)w0 * 4, (size_t)b * 32, cudaMemcpyHostToDevice, st);
      rin = drng;
    } else {
      rin = (const uint64_t*)rng + (size_t)w0 * 4;
    }
    if (err != cudaSuccess) return cuda_fail(err, "path upload");
    double* o = host ? dout : out + (size_t)w0 * 6;
    dim3 grid(nblk, b);
    if (D == 2) k_path<2><<<grid, kPtBS, 0, st>>>(S, PP, xin, rin, jt, part);
    else k_path<3><<<grid, kPtBS, 0, st>>>(S, PP, xin, rin, jt, part);
    k_path_final<<<(b * 6 + 127) / 128, 128, 0, st>>>(PP, part, nblk, b, o);
    launches += 2;
    err = cudaGetLastError();
    if (err != cudaSuccess) return cuda_fail(err, "path launch");
    if (host) {
      err = cudaMemcpyAsync(out + (size_t)w0 * 6, dout, (size_t)b * 48, cudaMemcpyDeviceToHost, st);
      if (err == cudaSuccess) err = cudaStreamSynchronize(st);
      if (err != cudaSuccess) return cuda_fail(err, "path download");
    }
  }
  count_launches(launches);
  err = cudaStreamSynchronize(st);
  if (err != cudaSuccess) return cuda_fail(err, "path trace");
  return VC_OK;
}

}  // namespace vc

using namespace vc;

extern "C" {

int vc_path_trace(vc_scene* scene, int m, const double* x, const void* rng, int64_t n_samples,
                  int max_media_bounces, int n_light_samples, int flags, int seed_words, double* out, void* stream) {
  return path_impl(scene, m, x, rng, (long long)n_samples, max_media_bounces, n_light_samples, flags, seed_words,
                   out, (cudaStream_t)stream);
}

}  // extern "C"
