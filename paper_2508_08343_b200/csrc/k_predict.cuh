// Placement-model training on the device: the CART
// regression trees of train_tree / train_forest / train_placement_model
// (predictor.cpp:67-269), bit-identical to the reference's.
//
// A tree job is one train_tree call: rows are the tree's positions p (the
// bootstrap resample's p-th draw, or the row itself), the target one of the
// y rows. Trees are grown in steps over a set of active nodes (host-driven,
// host_predict.h); per step:
//   node_begin_kernel  per node: the ordered sum / sum of squares of its
//                      targets in its row order (grow, predictor.cpp:97-103),
//                      the leaf test, the candidate features (all, or the
//                      {kFeatureSubset, tree_tag, node} shuffle, :138-147);
//   per candidate k:   split_keys_kernel + two stable radix sorts (by the
//                      feature, then by the node): each node's order
//                      re-sorted stably by feature f_k, exactly the
//                      reference's chain of std::stable_sort calls on one
//                      `order` vector (:156-159) -- ties keep the previous
//                      feature's order, then row order;
//                      split_eval_kernel: the sequential prefix sums (:160-
//                      163), every split point between distinct values
//                      (:164-180) and the strict-< first optimum;
//   node_finish_kernel the parent-SSE test (:182) and the stable partition
//                      of the node's rows into left / right (:112-118).
// The sums are sequential FP64 chains in the reference's order (one lane);
// everything else is parallel.
#pragma once

#include <cstdint>

#include "k_workload.cuh"  // mt64_twist_block, mt64_temper
#include "lt_rng.h"

namespace lt {

constexpr int kNumFeatures = 16;  // placement.hpp:43

// One train_tree call.
struct DTreeJob {
  int32_t y_index;    // row of the target matrix
  int32_t bootstrap;  // resample with replacement (train_forest, :227-233)
  uint64_t boot_tag;  // RngStream(seed, {kBootstrap, boot_tag, boot_index})
  uint64_t boot_index;
  uint64_t tree_tag;  // feature-subset substream key (:142)
};

// An active node of a step.
struct DNode {
  int32_t job;
  int32_t begin;  // first position of its rows in perm[job]
  int32_t len;
  int32_t depth;
  int32_t node_id;  // preorder id (the feature-subset stream key)
  int32_t off;      // first row of its segment in the step's work arrays
};

// Per-node results of a step.
struct DNodeOut {
  double mean;
  double sse;
  double best_sse;
  double threshold;
  int32_t leaf;  // 1: grow stops here (depth, size or sse)
  int32_t feature;  // best split feature, -1: none
  int32_t found;    // split kept after the parent-SSE test
  int32_t left_len;
  int32_t cand[kNumFeatures];
};

__device__ __forceinline__ uint64_t orderable(double x) {
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(x == 0.0 ? 0.0 : x));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}

// Bootstrap draws (or the identity) and the root order of every job
// (train_forest, :227-233): j = uniform_below(n) per row from the tree's
// {kBootstrap, target, tree} stream. One warp per job: lane 0 seeds the
// stream, the warp twists 312 state words at a time and every lane tempers
// and reduces its own words. uniform_below rejects draws >= 2^64 - 2^64 mod n
// (a shift of every later draw); a block holding one (probability ~n / 2^64)
// sends the job to lane 0's sequential replay of the reference's loop.
__global__ void __launch_bounds__(128) tree_rows_kernel(const DTreeJob* jobs, int n_jobs, int32_t n, uint64_t seed,
                                                        int32_t* src, int32_t* perm) {
  __shared__ uint64_t st_all[4][kMtN];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * 4 + warp;
  if (j >= n_jobs) return;
  int32_t* sj = src + static_cast<int64_t>(j) * n;
  int32_t* p = perm + static_cast<int64_t>(j) * n;
  for (int32_t i = lane; i < n; i += 32) p[i] = i;
  if (!jobs[j].bootstrap) {
    for (int32_t i = lane; i < n; i += 32) sj[i] = i;
    return;
  }
  uint64_t* st = st_all[warp];
  const uint64_t bound = static_cast<uint64_t>(n);
  const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
  if (lane == 0) {
    Mt64 e;
    rng_stream_init3(e, seed, 3 /* stream_id::kBootstrap */, jobs[j].boot_tag, jobs[j].boot_index);
    for (int w = 0; w < kMtN; ++w) st[w] = e.x[w];
  }
  __syncwarp();
  bool replay = false;
  for (int32_t i0 = 0; i0 < n && !replay; i0 += kMtN) {
    mt64_twist_block(st, lane);
    bool rej = false;
    for (int w = lane; w < kMtN && i0 + w < n; w += 32) {
      const uint64_t z = mt64_temper(st[w]);
      rej |= z >= limit;
      sj[i0 + w] = static_cast<int32_t>(z % bound);
    }
    replay = __any_sync(0xffffffffu, rej);
  }
  if (replay && lane == 0) {
    Mt64 e;
    rng_stream_init3(e, seed, 3, jobs[j].boot_tag, jobs[j].boot_index);
    for (int32_t i = 0; i < n; ++i) sj[i] = static_cast<int32_t>(uniform_below(e, bound));
  }
}

// grow() up to best_split (predictor.cpp:93-107, :138-147). One warp per node.
__global__ void node_begin_kernel(const DNode* nodes, int n_nodes, const DTreeJob* jobs, int32_t n, const double* y,
                                  const int32_t* src, const int32_t* perm, int max_depth, int min_leaf, int subset,
                                  uint64_t seed, int32_t* ord, int32_t* seg_end, DNodeOut* out) {
  const int a = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (a >= n_nodes) return;
  const DNode nd = nodes[a];
  const DTreeJob jb = jobs[nd.job];
  const int32_t* s = src + static_cast<int64_t>(nd.job) * n;
  const int32_t* p = perm + static_cast<int64_t>(nd.job) * n + nd.begin;
  const double* yy = y + static_cast<int64_t>(jb.y_index) * n;
  // the ordered sums of grow() (:97-103) over the node's row order: 32
  // targets per round gathered by the lanes, broadcast by shuffles into one
  // chain (every lane runs it; lane 0's result is kept)
  double sum = 0.0, sumsq = 0.0;
  for (int32_t base = 0; base < nd.len; base += 32) {
    const int32_t i = base + lane;
    double v = 0.0;
    if (i < nd.len) {
      const int32_t pi = p[i];
      ord[nd.off + i] = pi;  // the node's order starts as its row order (`order(idx)`, :153)
      v = yy[s[pi]];
    }
    const int32_t lim = nd.len - base;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const double w = __shfl_sync(0xffffffffu, v, k);
      if (k < lim) {
        sum += w;
        sumsq += w * w;
      }
    }
  }
  if (lane != 0) return;
  const double cnt = static_cast<double>(nd.len);
  DNodeOut o;
  o.mean = sum / cnt;
  o.sse = sumsq - sum * sum / cnt;
  o.leaf = (nd.depth >= max_depth || nd.len < 2 * min_leaf || o.sse <= 1e-12) ? 1 : 0;
  o.best_sse = INFINITY;
  o.threshold = 0.0;
  o.feature = -1;
  o.found = 0;
  o.left_len = 0;
  for (int f = 0; f < kNumFeatures; ++f) o.cand[f] = f;
  if (!o.leaf && subset < kNumFeatures) {  // candidate_features (:138-147)
    Mt64 e;
    rng_stream_init3(e, seed, 4 /* stream_id::kFeatureSubset */, jb.tree_tag, static_cast<uint64_t>(nd.node_id));
    for (int i = kNumFeatures; i > 1; --i) {
      const int j = static_cast<int>(uniform_below(e, static_cast<uint64_t>(i)));
      const int t = o.cand[i - 1];
      o.cand[i - 1] = o.cand[j];
      o.cand[j] = t;
    }
    for (int i = 1; i < subset; ++i) {  // std::sort of the kept prefix
      const int v = o.cand[i];
      int k = i - 1;
      while (k >= 0 && o.cand[k] > v) {
        o.cand[k + 1] = o.cand[k];
        --k;
      }
      o.cand[k + 1] = v;
    }
  }
  out[a] = o;
  seg_end[a] = o.leaf ? nd.off : nd.off + nd.len;
}

__device__ __forceinline__ int node_of_row(const DNode* nodes, int n_nodes, int64_t r) {
  int lo = 0, hi = n_nodes - 1;  // last node with off <= r
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (nodes[mid].off <= r) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Sort keys of candidate k for every row of the step's nodes: the feature
// value (orderable bits) and, as the value, {node, position}. A stable radix
// sort by the feature, then a stable one by the node (node_keys_kernel),
// leaves every node's rows contiguous, in feature order, ties in the
// previous order -- the reference's std::stable_sort of the node's `order`.
// Leaf nodes' rows ride along (their order is never read).
__global__ void split_keys_kernel(const DNode* nodes, int n_nodes, const DNodeOut* out, int k, int32_t n,
                                  const double* x, const int32_t* src, const int32_t* ord, int64_t rows,
                                  uint64_t* keys, uint64_t* node_pos) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  const int a = node_of_row(nodes, n_nodes, r);
  const int32_t pos = ord[r];
  node_pos[r] = (static_cast<uint64_t>(a) << 32) | static_cast<uint32_t>(pos);
  if (out[a].leaf) {
    keys[r] = 0;
    return;
  }
  const DNode nd = nodes[a];
  const int f = out[a].cand[k];
  const int32_t row = src[static_cast<int64_t>(nd.job) * n + pos];
  keys[r] = orderable(x[static_cast<int64_t>(row) * kNumFeatures + f]);
}

// After the sort by feature: the node of each row as the key of the second
// (stable) sort, the position as its value.
__global__ void node_keys_kernel(const uint64_t* node_pos, int64_t rows, uint32_t* node_key, int32_t* pos) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  const uint64_t v = node_pos[r];
  node_key[r] = static_cast<uint32_t>(v >> 32);
  pos[r] = static_cast<int32_t>(static_cast<uint32_t>(v));
}

// best_split's scan of candidate k (predictor.cpp:160-180), one warp per node:
// lane 0 runs the two prefix-sum chains in the sorted order, then the lanes
// price every split point between distinct values; the first minimum (lowest
// split index) is compared to the node's running best with strict <, in
// candidate order, as the reference's nested loops do.
__global__ void split_eval_kernel(const DNode* nodes, int n_nodes, DNodeOut* out, int k, int32_t n, int min_leaf,
                                  const double* x, const double* y, const DTreeJob* jobs, const int32_t* src,
                                  const int32_t* ord, double* xbuf, double* psum, double* psumsq) {
  const int a = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (a >= n_nodes) return;
  const DNode nd = nodes[a];
  DNodeOut& o = out[a];
  if (o.leaf) return;
  const int f = o.cand[k];
  const int32_t* s = src + static_cast<int64_t>(nd.job) * n;
  const double* yy = y + static_cast<int64_t>(jobs[nd.job].y_index) * n;
  const int32_t* od = ord + nd.off;
  double* ps = psum + nd.off + a;  // len + 1 entries per node
  double* pq = psumsq + nd.off + a;
  double* xb = xbuf + nd.off;
  // The two prefix-sum chains in the sorted order (:160-163): 32 values per
  // round, one per lane (independent gathers, the next round's in flight),
  // broadcast by shuffles; every lane runs the same chain and keeps its own
  // element's prefixes for a coalesced store.
  const int32_t len = nd.len;
  auto gather = [&](int32_t i, double& v, double& xv) {
    if (i < len) {
      const int64_t row = s[od[i]];
      v = yy[row];
      xv = x[row * kNumFeatures + f];
    }
  };
  double nv = 0.0, nx = 0.0;
  gather(lane, nv, nx);
  double s1 = 0.0, s2 = 0.0;
  if (lane == 0) {
    ps[0] = 0.0;
    pq[0] = 0.0;
  }
  for (int32_t base = 0; base < len; base += 32) {
    const double v = nv;
    const int32_t i = base + lane;
    if (i < len) xb[i] = nx;
    gather(i + 32, nv, nx);
    double m1 = 0.0, m2 = 0.0;
    const int32_t lim = len - base;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const double w = __shfl_sync(0xffffffffu, v, k);
      if (k < lim) {
        s1 = s1 + w;
        s2 = s2 + w * w;
      }
      if (k == lane) {
        m1 = s1;
        m2 = s2;
      }
    }
    if (i < len) {
      ps[i + 1] = m1;
      pq[i + 1] = m2;
    }
  }
  __syncwarp();
  double best = INFINITY;
  int32_t best_s = INT32_MAX;
  for (int32_t sp = min_leaf + lane; sp + min_leaf <= len; sp += 32) {
    const double lo = xb[sp - 1];
    const double hi = xb[sp];
    if (!(lo < hi)) continue;
    const double ls = static_cast<double>(sp), rs = static_cast<double>(len - sp);
    const double left_sse = pq[sp] - ps[sp] * ps[sp] / ls;
    const double dr = ps[len] - ps[sp];
    const double right_sse = (pq[len] - pq[sp]) - dr * dr / rs;
    const double total = left_sse + right_sse;
    if (total < best) {  // per lane: ascending split index, strict <
      best = total;
      best_s = sp;
    }
  }
  // warp argmin: smallest total, then smallest split index (NaN never wins)
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const double ob = __shfl_down_sync(0xffffffffu, best, d);
    const int32_t os = __shfl_down_sync(0xffffffffu, best_s, d);
    if (ob < best || (ob == best && os < best_s)) {
      best = ob;
      best_s = os;
    }
  }
  if (lane == 0 && best_s != INT32_MAX && best < o.best_sse) {
    const double lo = xb[best_s - 1];
    const double hi = xb[best_s];
    o.best_sse = best;
    o.feature = f;
    o.threshold = lo + (hi - lo) / 2.0;
  }
}

// The parent-SSE test (:182) and the stable partition of the node's rows, in
// its row order, into left (x <= threshold) then right (:112-118). One warp
// per node; tmp holds the right part while the left one is compacted.
__global__ void node_finish_kernel(const DNode* nodes, int n_nodes, DNodeOut* out, int32_t n, const double* x,
                                   const int32_t* src, int32_t* perm, int32_t* tmp) {
  const int a = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (a >= n_nodes) return;
  const DNode nd = nodes[a];
  DNodeOut& o = out[a];
  const bool found = !o.leaf && o.feature >= 0 && !(o.best_sse >= o.sse - 1e-12);
  if (!found) {
    if (lane == 0) o.found = 0;
    return;
  }
  const int32_t* s = src + static_cast<int64_t>(nd.job) * n;
  int32_t* p = perm + static_cast<int64_t>(nd.job) * n + nd.begin;
  int32_t* t = tmp + nd.off;
  int32_t nl = 0, nr = 0;
  for (int32_t base = 0; base < nd.len; base += 32) {
    const int32_t i = base + lane;
    int32_t v = 0;
    bool left = false;
    if (i < nd.len) {
      v = p[i];
      left = x[static_cast<int64_t>(s[v]) * kNumFeatures + o.feature] <= o.threshold;
    }
    const unsigned lm = __ballot_sync(0xffffffffu, i < nd.len && left);
    const unsigned rm = __ballot_sync(0xffffffffu, i < nd.len && !left);
    const unsigned lt = (1u << lane) - 1u;
    __syncwarp();  // every lane read its slot before the left part is written back in place
    if (i < nd.len) {
      if (left)
        p[nl + __popc(lm & lt)] = v;
      else
        t[nr + __popc(rm & lt)] = v;
    }
    nl += __popc(lm);
    nr += __popc(rm);
    __syncwarp();
  }
  for (int32_t i = lane; i < nr; i += 32) p[nl + i] = t[i];
  if (lane == 0) {
    o.found = 1;
    o.left_len = nl;
  }
}

// ForestModel::predict (predictor.cpp:205-216) for every (row, target): the
// trees' predictions summed in tree order, divided by the tree count, then
// clamped (throughput) or rounded and clamped (n*, g*). One thread each.
struct DTreeNode {
  int32_t feature_index;
  int32_t left;
  int32_t right;
  int32_t _pad;
  double threshold;
  double value;
  int64_t coverage;
};

__global__ void forest_predict_kernel(const DTreeNode* nodes, const int64_t* node_off, int n_trees,
                                      const int32_t* target_tags, int n_targets, const double* x, int64_t n_rows,
                                      double* out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n_rows * n_targets) return;
  const int tg = static_cast<int>(i / n_rows);
  const int64_t row = i % n_rows;
  const double* xr = x + row * kNumFeatures;
  double sum = 0.0;
  for (int t = 0; t < n_trees; ++t) {
    const DTreeNode* tree = nodes + node_off[tg * n_trees + t];
    int k = 0;
    while (tree[k].feature_index >= 0) k = xr[tree[k].feature_index] <= tree[k].threshold ? tree[k].left : tree[k].right;
    sum += tree[k].value;
  }
  const double raw = sum / static_cast<double>(n_trees);
  const int tag = target_tags[tg];  // < 0: predict_raw (no target transform)
  out[i] = tag < 0 ? raw : tag == 0 ? (raw < 0.0 ? 0.0 : raw) : fmax(1.0, round(raw));
}

}  // namespace lt
