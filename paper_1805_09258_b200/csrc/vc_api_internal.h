// Host-side handle types behind the C ABI (not part of the public header).
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/volcache_b200.h"
#include "vc_internal.h"

namespace vc {

struct Workspace {
  static constexpr int kSlots = 56;
  void* ptr[kSlots] = {nullptr};
  size_t cap[kSlots] = {0};
  void* get(int slot, size_t bytes, cudaError_t* err);
  ~Workspace();
};

struct Inspect {
  double* dirs;
  double* s;
  int32_t* idx;
  int32_t* counts;
  int32_t* tris;
  float* media;
  int64_t media_cap;
  int64_t* P;
};

int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);
bool grid_shape_3d(int n, int* rows, int* cols);
void count_launches(long long n);
const unsigned long long* jump_tables(cudaError_t* err);
// scene.contains for every point (src/scene.py:212-219): host arrays are checked on the
// host; device arrays by one flag kernel and a 4-byte readback (synchronises `st`).
// Returns VC_OK or VC_EOUTSIDE (with `what` as the message) / a CUDA error.
int check_inside(const vc_scene* sc, long long N, const double* x, bool host, const char* what,
                 cudaStream_t st);

// Split form: check_begin tests host arrays at once; for device arrays it enqueues the flag
// kernel (flag also left in ck->dflag for kernels to read) and check_end waits for it.
struct InsideCheck {
  bool pending = false;
  int* dflag = nullptr;
  int* hflag = nullptr;
  cudaEvent_t ev = nullptr;
  const char* what = nullptr;
};
int check_begin(const vc_scene* sc, long long N, const double* x, bool host, const char* what, cudaStream_t st,
                InsideCheck* ck);
int check_end(InsideCheck* ck);
int check_defer(InsideCheck* ck, cudaStream_t st);
int check_deferred_read(cudaStream_t st);

}  // namespace vc

// Device copy of one primitive set (all surfaces, or the emitters) with its BVH.
struct GpuBvh {
  int K = 0, n_nodes = 0, stack_need = 0;
  double* prim = nullptr;
  int* prim_id = nullptr;
  float4* nodes = nullptr;
  float4* prim32 = nullptr;
  double ctr[3] = {0, 0, 0};
  vc::DevBvh dev() const {
    return vc::DevBvh{K, n_nodes, nodes, prim, prim_id, prim32, {ctr[0], ctr[1], ctr[2]}, stack_need};
  }
  ~GpuBvh() {
    cudaFree(prim);
    cudaFree(prim_id);
    cudaFree(nodes);
    cudaFree(prim32);
  }
};

struct vc_scene {
  int dim = 0, K = 0;
  std::vector<double> verts, emission, albedo;
  double bmin[3] = {0, 0, 0}, bmax[3] = {0, 0, 0};
  double scale = 0.0, sigma_s = 0.0, sigma_a = 0.0, max_emission = 0.0;
  int reflective = 0;
  int sm_count = 148;
  GpuBvh geo, emit;
  vc::EmitPlanes ep{};   // device pointers owned here
  int* d_ep_start = nullptr;
  int* d_ep_tri = nullptr;
  unsigned* d_ep_occ = nullptr;
  double* d_normal = nullptr;
  double* d_emission = nullptr;
  double* d_albedo = nullptr;
  int es_nlight = -1, n_es = 0;
  double* d_es_pos = nullptr;
  double* d_es_w = nullptr;
  int* d_es_surf = nullptr;
  int n_lights = 0;            // extension: delta lights (vc_scene_set_lights)
  double* d_lights = nullptr;  // n_lights × 8
  long long budget = 0;  // 0: a third of the device memory, capped at 64 GiB
  vc::Workspace ws;
  ~vc_scene() {
    cudaFree(d_normal);
    cudaFree(d_emission);
    cudaFree(d_albedo);
    cudaFree(d_es_pos);
    cudaFree(d_es_w);
    cudaFree(d_es_surf);
    cudaFree(d_ep_start);
    cudaFree(d_ep_tri);
    cudaFree(d_ep_occ);
    cudaFree(d_lights);
  }
};

namespace vc {
int ensure_emitters(vc_scene* sc, int n_light);
DevScene dev_scene(const vc_scene* sc);
int baseline_impl(vc_scene* sc, int N, const double* x, const void* rng, const vc_baseline_params* prm,
                  double* est, double* records, double* samples, cudaStream_t st);
int path_impl(vc_scene* sc, int m, const double* x, const void* rng, long long n_samples, int max_media_bounces,
              int n_light_samples, int flags, int seed_words, double* out, cudaStream_t st);
int build_impl(vc_scene* sc, int N, const double* x, const void* rng, const int32_t* adjacency,
               const vc_build_params* prm, double* moments, int64_t* stats, double* records,
               cudaStream_t st, Inspect* insp);
}  // namespace vc
