// Host BVH builder: binned SAH over primitive boxes, built once per scene.
//
// The reference traces by brute force over every primitive (src/scene.py:227-268);
// the BVH only culls, so the nearest hit (float64 decision, lowest-index tie break)
// is unchanged.  Boxes are float32 rounded outward and padded by `pad`, which keeps
// float32 slab culling conservative for float64 rays.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "vc_build.h"

namespace vc {

namespace {

struct Box {
  float lo[3], hi[3];
  void reset() {
    for (int a = 0; a < 3; ++a) {
      lo[a] = FLT_MAX;
      hi[a] = -FLT_MAX;
    }
  }
  void grow(const Box& b) {
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], b.lo[a]);
      hi[a] = std::max(hi[a], b.hi[a]);
    }
  }
  float area() const {
    float d[3];
    for (int a = 0; a < 3; ++a) d[a] = std::max(0.0f, hi[a] - lo[a]);
    return 2.0f * (d[0] * d[1] + d[1] * d[2] + d[0] * d[2]);
  }
};

struct Node {
  Box b;
  int first, count;  // interior: first = left child, count = 0
};

constexpr int kBins = 16;
constexpr int kLeafDefault = 4;

}  // namespace

void build_bvh(int dim, int K, const double* verts, double pad, HostBVH* out, int leaf_max) {
  const int kLeafMax = leaf_max > 0 ? leaf_max : kLeafDefault;
  std::vector<Box> pb(K);
  std::vector<float> cen(3 * (size_t)K);
  const int nv = dim;  // vertices per primitive
  for (int k = 0; k < K; ++k) {
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int a = 0; a < dim; ++a) {
      lo[a] = hi[a] = verts[((size_t)k * nv) * dim + a];
      for (int v = 1; v < nv; ++v) {
        double x = verts[((size_t)k * nv + v) * dim + a];
        lo[a] = std::min(lo[a], x);
        hi[a] = std::max(hi[a], x);
      }
    }
    for (int a = 0; a < 3; ++a) {
      float fl = std::nextafter((float)(lo[a] - pad), -FLT_MAX);
      float fh = std::nextafter((float)(hi[a] + pad), FLT_MAX);
      pb[k].lo[a] = fl;
      pb[k].hi[a] = fh;
      cen[3 * (size_t)k + a] = 0.5f * (fl + fh);
    }
  }
  std::vector<int> order(K);
  for (int k = 0; k < K; ++k) order[k] = k;
  std::vector<Node> nodes;
  nodes.reserve(2 * (size_t)K + 1);
  nodes.push_back(Node{});  // root
  nodes.push_back(Node{});  // pad: child pairs start at even indices → 64-byte aligned
  struct Task {
    int node, begin, end, depth;
  };
  std::vector<Task> stack;
  stack.push_back({0, 0, K, 0});
  while (!stack.empty()) {
    Task t = stack.back();
    stack.pop_back();
    Box nb, cb;
    nb.reset();
    cb.reset();
    for (int i = t.begin; i < t.end; ++i) {
      int k = order[i];
      nb.grow(pb[k]);
      Box c;
      for (int a = 0; a < 3; ++a) c.lo[a] = c.hi[a] = cen[3 * (size_t)k + a];
      cb.grow(c);
    }
    const int cnt = t.end - t.begin;
    nodes[t.node].b = nb;
    // the device traversal stack holds kBvhMaxDepth entries: cap the depth with a large leaf
    if (cnt <= kLeafMax || t.depth >= kBvhMaxDepth - 1) {
      nodes[t.node].first = t.begin;
      nodes[t.node].count = cnt;
      continue;
    }
    // binned SAH over all axes
    float best_cost = FLT_MAX;
    int best_axis = -1, best_split = -1;
    for (int a = 0; a < dim; ++a) {
      float ext = cb.hi[a] - cb.lo[a];
      if (!(ext > 0.0f)) continue;
      Box bb[kBins];
      int bc[kBins] = {0};
      for (int i = 0; i < kBins; ++i) bb[i].reset();
      for (int i = t.begin; i < t.end; ++i) {
        int k = order[i];
        int bi = (int)((cen[3 * (size_t)k + a] - cb.lo[a]) / ext * kBins);
        bi = std::min(std::max(bi, 0), kBins - 1);
        bc[bi]++;
        bb[bi].grow(pb[k]);
      }
      float la[kBins], ra[kBins];
      int lc[kBins], rc[kBins];
      Box acc;
      acc.reset();
      int c = 0;
      for (int i = 0; i < kBins; ++i) {
        acc.grow(bb[i]);
        c += bc[i];
        la[i] = acc.area();
        lc[i] = c;
      }
      acc.reset();
      c = 0;
      for (int i = kBins - 1; i >= 0; --i) {
        acc.grow(bb[i]);
        c += bc[i];
        ra[i] = acc.area();
        rc[i] = c;
      }
      for (int s = 0; s < kBins - 1; ++s) {
        if (lc[s] == 0 || rc[s + 1] == 0) continue;
        float cost = la[s] * lc[s] + ra[s + 1] * rc[s + 1];
        if (cost < best_cost) {
          best_cost = cost;
          best_axis = a;
          best_split = s;
        }
      }
    }
    int mid;
    if (best_axis >= 0) {
      float ext = cb.hi[best_axis] - cb.lo[best_axis];
      auto it = std::partition(order.begin() + t.begin, order.begin() + t.end, [&](int k) {
        int bi = (int)((cen[3 * (size_t)k + best_axis] - cb.lo[best_axis]) / ext * kBins);
        bi = std::min(std::max(bi, 0), kBins - 1);
        return bi <= best_split;
      });
      mid = (int)(it - order.begin());
      if (mid == t.begin || mid == t.end) mid = (t.begin + t.end) / 2;
    } else {
      mid = (t.begin + t.end) / 2;  // coincident centroids: split by index
    }
    int left = (int)nodes.size();
    nodes.push_back(Node{});
    nodes.push_back(Node{});
    nodes[t.node].first = left;
    nodes[t.node].count = 0;
    stack.push_back({left + 1, mid, t.end, t.depth + 1});
    stack.push_back({left, t.begin, mid, t.depth + 1});
  }
  // Device layout: one 64-byte record per interior node holding its two children's boxes
  // and references, the boxes interleaved by child so every float4 half is a (left, right)
  // pair for the packed FFMA2 slab tests: (lo.x l r, lo.y l r), (lo.z l r, hi.x l r),
  // (hi.y l r, hi.z l r), (ref l, count l, ref r, count r); ref = first primitive of a leaf
  // with bit 31 set (the traversal walks it to the primitive flagged last-in-leaf), or the
  // child's interior-node index.  A visit loads one cache line and tests both children.
  std::vector<int> inner(nodes.size(), -1);
  int n_inner = 0;
  for (size_t i = 0; i < nodes.size(); ++i)
    if (i != 1 && nodes[i].count == 0) inner[i] = n_inner++;
  const bool root_leaf = nodes[0].count > 0;
  if (root_leaf) n_inner = 1;  // a single leaf: wrap it
  out->n_nodes = n_inner;
  out->nodes = (float4*)malloc(sizeof(float4) * 4 * (size_t)n_inner);
  out->order = (int*)malloc(sizeof(int) * (size_t)std::max(K, 1));
  auto bits = [](int v) {
    float f;
    std::memcpy(&f, &v, 4);
    return f;
  };
  auto pair = [&](float4* dst, int cl, int cr) {
    const Node& l = nodes[cl];
    const Node& r = nodes[cr];
    const int rl = l.count > 0 ? (int)((unsigned)l.first | 0x80000000u) : inner[cl];
    const int rr = r.count > 0 ? (int)((unsigned)r.first | 0x80000000u) : inner[cr];
    dst[0] = make_float4(l.b.lo[0], r.b.lo[0], l.b.lo[1], r.b.lo[1]);
    dst[1] = make_float4(l.b.lo[2], r.b.lo[2], l.b.hi[0], r.b.hi[0]);
    dst[2] = make_float4(l.b.hi[1], r.b.hi[1], l.b.hi[2], r.b.hi[2]);
    dst[3] = make_float4(bits(rl), bits(l.count), bits(rr), bits(r.count));
  };
  if (root_leaf) {  // both children the same leaf (tested twice: same result)
    pair(out->nodes, 0, 0);
  } else {
    for (size_t i = 0; i < nodes.size(); ++i) {
      if (inner[i] < 0) continue;
      pair(out->nodes + 4 * (size_t)inner[i], nodes[i].first, nodes[i].first + 1);
    }
  }
  std::memcpy(out->order, order.data(), sizeof(int) * K);
  // leaf extents (leaf order) and the traversal stack bound: a push happens only below an
  // interior node, so the stack never holds more entries than the deepest interior level
  out->leaf_last = (unsigned char*)calloc((size_t)std::max(K, 1), 1);
  int depth_max = 0;
  std::vector<std::pair<int, int>> todo;  // (node, depth)
  todo.push_back({0, 0});
  while (!todo.empty()) {
    auto [i, dep] = todo.back();
    todo.pop_back();
    const Node& n = nodes[i];
    if (n.count > 0) {
      out->leaf_last[n.first + n.count - 1] = 1;
      depth_max = std::max(depth_max, dep);
      continue;
    }
    todo.push_back({n.first, dep + 1});
    todo.push_back({n.first + 1, dep + 1});
  }
  out->max_depth = depth_max;
}

void free_bvh(HostBVH* b) {
  free(b->nodes);
  free(b->order);
  free(b->leaf_last);
  b->nodes = nullptr;
  b->order = nullptr;
  b->leaf_last = nullptr;
  b->n_nodes = 0;
}

}  // namespace vc
