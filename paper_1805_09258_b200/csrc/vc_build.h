// Host-side declarations of the record-build launchers and runtime helpers.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "vc_internal.h"

namespace vc {

struct KernelCounter {
  long long launches = 0;
};

// Kernel classes for the optional per-kernel CUDA-event profile (vc_profile_*).
enum KernelClass {
  KC_PRIMARY, KC_RINGS, KC_WAVESCAN, KC_GATHER, KC_DELAUNAY, KC_COMPACT, KC_DEGREE, KC_ASSEMBLE,
  KC_RECORD, KC_SEED, KC_INTERP, KC_MARCH, KC_COUNT
};
void prof_begin(int kc, cudaStream_t st);
void prof_end(cudaStream_t st);

void launch_wave(const DevScene& S, const BuildParams& P, const Wave& W, const JumpTables& jt, int* own,
                 int* own_cnt, int sm_count, cudaStream_t st, KernelCounter* kc);
void launch_surface_radiance(const DevScene& S, int m, const double* pts, const double* dirs, const int* idx,
                             double* out, cudaStream_t st);
void launch_trace(const DevScene& S, int m, const double* o, const double* d, double* t, int* idx, int with_bounds,
                  cudaStream_t st);
void launch_make_records(const DevScene& S, const BuildParams& P, const Wave& W, cudaStream_t st);
void launch_seedseq(int n, const uint32_t* words, int nw, uint64_t* states, cudaStream_t st);

// Host BVH build (binned SAH) over primitive bounds; returns nodes (2 float4 each)
// and the leaf order of primitives.
struct HostBVH {
  int n_nodes = 0;
  float4* nodes = nullptr;  // host array, 2*n_nodes
  int* order = nullptr;     // leaf order → original primitive
  unsigned char* leaf_last = nullptr;  // leaf order: 1 on the last primitive of each leaf
  int max_depth = 0;        // deepest leaf (bounds the traversal stack)
};
void build_bvh(int dim, int K, const double* verts, double pad, HostBVH* out, int leaf_max = 0);
void free_bvh(HostBVH* b);

}  // namespace vc
