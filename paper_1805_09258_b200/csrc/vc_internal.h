// Internal types shared by the host runtime and the device kernels of libvolcache_b200.
//
// Layout in HBM (all device arrays are structure-of-arrays unless noted):
//   scene   : primitives in BVH-leaf order as float64 (3D: v0,e1,e2 = 9 doubles;
//             2D: a,e = 4 doubles), original-order normals/emission/albedo, fp32
//             BVH nodes (2×float4 each), emitter quadrature samples (float64).
//   wave    : per-record scratch for B records processed together — directions,
//             primary hits, ring counts/prefixes, surface radiance (float64),
//             media-sample radiance (float32×3, one entry per live (dir, ring)),
//             canonical spherical-Delaunay triangles (int32×3).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace vc {

constexpr int kMaxDim = 3;
constexpr int kBvhMaxDepth = 32;
constexpr int kCapGMax = 32;     // binned cap kernel: bins per axis
constexpr int kCapGCols = 1024;  // binned cap kernel: largest stratum row  // BVH depth cap = device traversal stack size
#ifndef VC_ASM_SPLIT
#define VC_ASM_SPLIT 32
#endif
#ifndef VC_ASM_BS
#define VC_ASM_BS 64
#endif
constexpr int kAsmSplit = VC_ASM_SPLIT;  // CTAs per record in the moment assembly (32: 5.21 ms per 2048 cfg3
                                         // records; 16: 5.62, 48: 5.29, 64: 5.34, 8: 6.33)
constexpr int kAsmBS = VC_ASM_BS;        // threads per assembly CTA
constexpr int kAsmParts = kAsmSplit * (kAsmBS / 32);  // per-warp partial sums per record

// A BVH over a primitive set: float32 nodes, float64 primitives in leaf order.
struct DevBvh {
  int K;                 // primitives
  int n_nodes;           // nodes (0 → brute force over K in original order)
  const float4* nodes;   // 4 float4 per interior node, children interleaved (vc_bvh.cpp); boxes relative to ctr
  const double* prim;    // leaf order, prim_stride(dim) doubles each
  const int* prim_id;    // leaf order → original surface index
  // leaf order, 3 float4 per primitive (relative to ctr): (v0, |v0|∞), (e1, E), (e2, id | last);
  // E = max(|e1|∞, |e2|∞) rounded up (−1: no float32 pre-test), last = bit 31 on the final
  // primitive of a leaf (2D: (a, 0, 0), (e, 0, −1), (0, 0, 0, id | last))
  const float4* prim32;
  double ctr[3];         // bounds centre: node boxes and prim32 are relative to it
  int stack_need;        // deepest leaf: traversal stack entries needed
};

// Emitters grouped by plane (3D, ≤ kEmitPlanes planes), each with a 2D grid of the
// triangles overlapping its cells: a gather ray meets each plane once and tests only the
// triangles of the cell it lands in (vc_api.cu: build_emit_planes).
constexpr int kEmitPlanes = 4;
struct EmitPlanes {
  int ng;                        // planes (0: the emitter BVH answers every query)
  double n[kEmitPlanes][3], c[kEmitPlanes];          // unit normal, offset (n·x = c)
  double a1[kEmitPlanes][3], a2[kEmitPlanes][3];     // in-plane frame about c·n
  double lo[kEmitPlanes][2], inv[kEmitPlanes][2];    // grid origin and 1 / cell size
  int gx[kEmitPlanes], gy[kEmitPlanes], cell0[kEmitPlanes];
  int axis[kEmitPlanes];         // n = ±e_axis exactly (−1: not axis-aligned)
  int axis_only;                 // every plane axis-aligned (the gather's draw-only test)
  const int* cell_start;         // CSR over every plane's cells
  const int* cell_tri;           // leaf-order indices into the emitter set
  // coarse occupancy per plane (≤ 32 × 32 blocks of cells; row j = one 32-bit word, bit i
  // set when a cell of block (i, j) lists a triangle): the gather's float32 pre-filter
  const unsigned* occ;           // kEmitPlanes × 32 words (nullptr: no pre-filter)
  double occ_inv[kEmitPlanes][2];
  int occ_w[kEmitPlanes], occ_h[kEmitPlanes];
};

// Scene as seen by kernels (passed by value).
struct DevScene {
  int dim;
  int K;                 // primitives
  int n_es;              // emitter quadrature samples (all emitters)
  int reflective;        // any albedo > 0
  double bmin[3], bmax[3];
  double scale, t_eps;   // bounds diagonal; 1e-6·scale self-hit guard (src/scene.py:22)
  double sigma_s, sigma_a, sigma_t;
  double max_emission;
  DevBvh geo;            // every surface
  DevBvh emit;           // emitting surfaces only (emitter-first gather when !reflective)
  EmitPlanes ep;         // plane grids over the emitters (gather queries)
  const double* normal;  // original order, dim doubles each
  const double* emission;// original order, 3 doubles
  const double* albedo;  // original order, 3 doubles
  const double* es_pos;  // n_es × dim
  const double* es_w;    // n_es
  const int* es_surf;    // n_es → original surface index of the emitter
  // extension (not in the reference): delta lights, 8 doubles each — kind (0 point, 1
  // directional), v[3] (position, or the unit vector toward the light), rgb, 0
  int n_lights;
  const double* lights;
};

__host__ __device__ constexpr int prim_stride(int dim) { return dim == 3 ? 9 : 4; }

// Triangulation search radius α and its trigonometry, per retry level (host-computed).
struct DelAngle {
  double alpha, sin_a, cos_a, tan_half;
};
constexpr int kDelLevels = 10;
// Stratum-window triangulation (k_delaunay_hull): candidates per window and rows covered.
constexpr int kHullK = 64;
constexpr int kDelRowsMax = 512;

// Per-call record-build parameters (mirrors estimate_moments' arguments).
struct BuildParams {
  DelAngle del[kDelLevels];  // α_k = min(2.8 · spacing · 1.5^k, 1.5)
  int n_angular;
  double march_step;
  int n_inner;
  int media_bounces;     // media events per gather path (1: the reference; extension > 1)
  double hg_g;           // extension: Henyey–Greenstein g of the media (0: the reference)
  int rows, cols;        // 3D stratum grid (src/scene.py:370-385); 2D: rows = 1, cols = n
  int n_tris;            // elements per ring: n (2D) or 2n-4 (3D)
  int r_ub;              // upper bound on rings per record (allocation)
  int host_adjacency;    // 1 → triangles supplied by the caller
  double epsilon;        // record error budget (make_record)
  int anisotropic;
  int make_records;
  // per stratum row: (h << 6) | w — the hull kernel's candidate window is rows r ± h,
  // columns c ± w; 0 = the row goes to the clipping kernel (polar caps, wide rows)
  unsigned char del_hw[kDelRowsMax];
  int del_kmax;  // largest window in del_hw (0: no row uses the hull kernel)
  // hull rows grouped by window size (classes ≤ 34, ≤ 44, ≤ 64 candidates: 6, 4, 3 CTAs
  // per SM by shared memory): rows del_rows[del_cls[k] .. del_cls[k+1]) of class k, whose
  // largest window is del_cls_k[k]
  unsigned short del_rows[kDelRowsMax];
  int del_cls[4];
  int del_cls_k[3];
  double del_zstep;  // 2 / rows: stratum height in z
  int del_cap;       // 1: the polar rows go to the cap kernel
  float del_cap_cos, del_cap_sin;  // cos δ, sin δ: the cap kernel's candidate radius
  double del_cap_c2, del_cap_s2;  // cos²(δ/2), sin²(δ/2)
  double del_warp_delta;          // first candidate radius of the one-warp fallback
  int del_dbg_cell;               // VOLCACHE_DEL_DEBUG_CELL: warp_cell reports why it gives up
};

// Per-direction data read by the assembly scan, one 16-byte load per vertex.
struct alignas(16) DirInfo {
  double s;        // primary hit distance (or bounds exit)
  int cnt;         // live rings
  int surf_live;   // surface radiance > 0 in any channel
};

// Per-record scratch for one wave (device pointers).
struct Wave {
  const int* outside;    // device bounds-check flag (nullptr: host-checked); set → no rings
  int* surv_cnt;         // B: survivors of the gather filter per record; redo = surv_cnt + B
  int* redo;             // B: 1 → the record's survivor evaluation found the queue full
  unsigned long long* ray_cursor;  // persistent-lane primary pass: next ray index
  DirInfo* info;         // B × n
  double* partial;       // B × kAsmParts × 2 × 32 assembly partial sums (+ counters)
  int B;                 // records in this wave
  const double* x;       // B × dim
  const uint64_t* rng;   // B × 4: state_hi, state_lo, inc_hi, inc_lo (PCG64, numpy layout)
  double* dirs;          // B × n × dim
  float4* dirs32;        // B × n float32 copy (3D triangulation pre-tests)
  double* s;             // B × n primary hit distance (or bounds exit)
  int* idx;              // B × n primary hit surface (−1: bounds)
  int* cnt;              // B × n live rings per direction (after clamp to R)
  int* pre;              // B × n exclusive prefix of cnt within the record
  int* run_dir;          // B × run_stride: direction of media sample 16·m (gather runs)
  int run_stride;
  double* lo;            // B × n × 3 surface radiance (reflective scenes)
  const double* emit_tab;  // non-reflective scenes: L_o = emission[idx] (DevScene::emission), lo is not
                           // written or read (nullptr: read lo)
  int* rec_R;            // B rings per record
  int* rec_P;            // B live media samples per record
  int* rec_maxc;         // B max cnt (rings that carry any live sample)
  long long* rec_base;   // B+1 exclusive prefix of rec_P across the wave (+ total)
  float* media;          // Σ P × 3 media radiance (positive values floored at FLT_TRUE_MIN)
  long long media_cap;   // capacity in samples
  int* tris;             // B × n_tris × 3 (3D) canonical or injected triangles
  int* deg;              // B × n vertex valence (3D)
  int* tri_status;       // B: 0 ok, else triangulation failure code
  double* moments;       // B × 2 × M (M = 3 + 3d + 3d²)
  long long* stats;      // B × kStats
  double* records;       // B × 2 × RecordSize(d) (optional)
  unsigned long long* live;  // B × live_words × n: bit i of word w = media sample (k, 64w+i) has rad > 0
  int live_words;            // ⌈r_ub / 64⌉
  int dense_media;           // 1: write zero radiance for dead samples too (inspection)
  int* del_retry;        // triangulation cells that outgrew the shared-memory polygon
  unsigned int* del_retry_count;
  int del_retry_cap;
  double* del_scratch;   // del_retry_cap × 48 × 3 doubles of global-memory polygons
  int* del_fb;           // B × n: cells the float32 hull kernels hand back
  unsigned int* del_fb_count;
  int* del_fb2;          // B × n: cells the float64 wrap hands to the clipping kernel
  unsigned int* del_fb2_count;
  long long own_stride;  // cells per slot row of the owned-triangle array (wave capacity × n)
  int* cap_bins;         // B × 2 × cap_bin_stride: binned cap rows (k_cap_bin → k_delaunay_capg)
  int cap_bin_stride;
  uint2* asm_items;      // B × item_cap assembly items (element, ring·4 + rep) in
                         // kAsmParts per-warp segments (null: fused assembly only)
  int* item_n;           // B × kAsmParts × 2: segment end of the surface / media items
  int* asm_fb;           // B: 1 = a segment overflowed, the fused kernel takes the record
  long long item_cap;    // items per record
  void* gather_q;        // two-pass gather: queued emitter-hit rays (GatherItem)
  unsigned long long* gather_q_count;
  long long gather_q_cap;
};

constexpr int kStats = 8;  // evaluated, dropped, stars, P, R, tri_status, eval_single, eval_multiple

__host__ __device__ constexpr int moment_size(int d) { return 3 + 3 * d + 3 * d * d; }
__host__ __device__ constexpr int record_size(int d) { return d + 3 + 3 * d + d * d + d; }

// PCG64 jump tables (3 levels × 1024 entries): A = MULT^delta, G = Σ_{j<delta} MULT^j.
struct JumpTables {
  const unsigned long long* tab;  // [level][1024][4]: A_hi, A_lo, G_hi, G_lo
};

}  // namespace vc
