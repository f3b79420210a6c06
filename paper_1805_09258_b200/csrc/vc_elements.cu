// Per-element form factors with derivatives on the device: ff_segment_derivs_batch /
// ff_triangle_derivs_batch (src/formfactor.py:85-158, :298-343) as a batch entry point.
//
// The record build evaluates the same device functions inside the assembly kernels
// (vc_build.cu); this entry point exposes them element by element so the ok-mask, the
// values and the derivatives can be checked against the reference's own batch outputs,
// including its degenerate rows (γ outside (1e-5, π − 1e-5), vertex on x, |A| below
// 1e-12·r₁r₂r₃ → not ok, zeros), src/formfactor.py:23-30, :99-106, :306.
//
// precision: 0 = the float64 functions the build uses (ff_segment / ff_triangle);
//            1 = the float32 element path of the 3D assembly (ff_triangle_f32).
#include <cmath>

#include "vc_api_internal.h"
#include "vc_build.h"
#include "vc_device.cuh"

namespace vc {

template <int D>
__global__ void k_form_factors(int m, const double* x, const double* verts, int precision, unsigned char* ok,
                               double* val, double* grad, double* hess) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  constexpr int NH = D * (D + 1) / 2;
  double r[D][D];
#pragma unroll
  for (int k = 0; k < D; ++k)
#pragma unroll
    for (int a = 0; a < D; ++a) r[k][a] = verts[((size_t)i * D + k) * D + a] - x[(size_t)i * D + a];
  double F = 0.0, g[D], H[NH];
#pragma unroll
  for (int a = 0; a < D; ++a) g[a] = 0.0;
#pragma unroll
  for (int e = 0; e < NH; ++e) H[e] = 0.0;
  bool good;
  if constexpr (D == 2) {
    good = ff_segment(r[0], r[1], F, g, H);
  } else if (precision == 1) {
    float rf[3][3], Ff = 0.0f, gf[3] = {0.0f, 0.0f, 0.0f}, Hf[6] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int a = 0; a < 3; ++a) rf[k][a] = (float)r[k][a];
    good = ff_triangle_ok(r[0], r[1], r[2]);
    if (good) ff_triangle_f32(rf[0], rf[1], rf[2], Ff, gf, Hf);
    F = Ff;
#pragma unroll
    for (int a = 0; a < 3; ++a) g[a] = gf[a];
#pragma unroll
    for (int e = 0; e < 6; ++e) H[e] = Hf[e];
  } else {
    good = ff_triangle(r[0], r[1], r[2], F, g, H);
  }
  if (!good) {  // invalid elements: zeros (src/formfactor.py:142-158, :332-343)
    F = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) g[a] = 0.0;
#pragma unroll
    for (int e = 0; e < NH; ++e) H[e] = 0.0;
  }
  ok[i] = good ? 1 : 0;
  val[i] = F;
#pragma unroll
  for (int a = 0; a < D; ++a) grad[(size_t)i * D + a] = g[a];
  int e = 0;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = a; b < D; ++b) {
      hess[((size_t)i * D + a) * D + b] = H[e];
      hess[((size_t)i * D + b) * D + a] = H[e];
      ++e;
    }
}

}  // namespace vc

using namespace vc;

extern "C" {

int vc_form_factors(int dim, int m, const double* x, const double* verts, int precision, int flags,
                    uint8_t* ok, double* value, double* grad, double* hess, void* stream) {
  if (dim != 2 && dim != 3) return fail(VC_EINVAL, "dimensionality must be 2 or 3");
  if (m < 0) return fail(VC_EINVAL, "negative element count");
  if (precision != 0 && !(precision == 1 && dim == 3)) return fail(VC_EINVAL, "precision 1 is the 3D float32 path");
  if (m == 0) return VC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const bool host = flags & VC_MEM_HOST;
  const size_t nx = (size_t)m * dim, nv = (size_t)m * dim * dim;
  const double *dx = x, *dv = verts;
  unsigned char* dok = ok;
  double *dval = value, *dgrad = grad, *dhess = hess;
  void* buf = nullptr;
  cudaError_t e = cudaSuccess;
  if (host) {
    const size_t bytes = (nx + nv + m + nx + nv) * 8 + m;
    e = cudaMalloc(&buf, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "form-factor buffers");
    double* p = (double*)buf;
    dx = p;
    dv = p + nx;
    dval = p + nx + nv;
    dgrad = dval + m;
    dhess = dgrad + nx;
    dok = (unsigned char*)(dhess + nv);
    e = cudaMemcpyAsync((void*)dx, x, nx * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync((void*)dv, verts, nv * 8, cudaMemcpyHostToDevice, st);
  }
  if (e == cudaSuccess) {
    if (dim == 2) k_form_factors<2><<<(m + 127) / 128, 128, 0, st>>>(m, dx, dv, precision, dok, dval, dgrad, dhess);
    else k_form_factors<3><<<(m + 127) / 128, 128, 0, st>>>(m, dx, dv, precision, dok, dval, dgrad, dhess);
    count_launches(1);
    e = cudaGetLastError();
  }
  if (host && e == cudaSuccess) {
    e = cudaMemcpyAsync(ok, dok, m, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(value, dval, (size_t)m * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(grad, dgrad, nx * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hess, dhess, nv * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  if (buf) cudaFree(buf);
  return e == cudaSuccess ? VC_OK : cuda_fail(e, "form factors");
}

}  // extern "C"
