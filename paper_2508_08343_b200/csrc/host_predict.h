// Placement-model training and inference on the device: lt_train_tree /
// lt_train_forests / lt_predict_forests (include/loratwin_gpu.h), replacing
// train_tree, train_forest, train_placement_model and ForestModel::predict
// (predictor.cpp:202-269). Included by capi.cu (C-ABI section).
//
// Every tree of the call (all targets x n_trees) grows at once. Steps are
// host-driven: the host keeps each tree's pending nodes, the device does the
// row work of a step's active nodes (k_predict.cuh). Without a feature
// subset a step takes every pending node (level by level; the preorder ids
// of the reference's node vector are assigned once the shape is known).
// With a subset the candidate features are drawn from a stream keyed by the
// node's preorder id (predictor.cpp:142), so each step takes the next node
// of every tree in preorder, as grow() recurses (left subtree first).

namespace {

struct HostTreeNode {
  int32_t feature = -1;
  double threshold = 0.0;
  double value = 0.0;
  int64_t coverage = 0;
  int32_t left = -1, right = -1;  // creation indices
};

struct PendingNode {
  int32_t begin, len, depth;
  int32_t parent;  // creation index of the parent, -1 for the root
  bool is_left;
};

void preorder(const std::vector<HostTreeNode>& t, int32_t k, std::vector<int32_t>& order) {
  order.push_back(k);
  if (t[k].feature >= 0) {
    preorder(t, t[k].left, order);
    preorder(t, t[k].right, order);
  }
}

bool validate_tree_params(const lt_tree_params& p, HostErr* e) {
  if (p.max_depth < 0) return e->set(LT_ERR_VALIDATION, "tree.max_depth: must be >= 0");
  if (p.min_leaf < 1) return e->set(LT_ERR_VALIDATION, "tree.min_leaf: must be >= 1");
  if (p.feature_subset < 1 || p.feature_subset > kNumFeatures)
    return e->set(LT_ERR_VALIDATION, "tree.feature_subset: must be in [1, " + std::to_string(kNumFeatures) + "]");
  return true;
}

// Grows jobs.size() trees over the n rows of x (n x 16) with targets y
// (rows of n). out[j] = job j's nodes in the reference's preorder.
void grow_trees(lt_ctx* ctx, const double* x, int32_t n, const double* y, int32_t n_y,
                const std::vector<DTreeJob>& jobs, const lt_tree_params& prm, uint64_t seed,
                std::vector<std::vector<HostTreeNode>>& out, lt_timing* tm) {
  cudaSetDevice(ctx->device);
  cudaStream_t st = ctx->stream;
  const int J = static_cast<int>(jobs.size());
  const int64_t total = static_cast<int64_t>(J) * n;
  DBuf<double> d_x, d_y;
  DBuf<DTreeJob> d_jobs;
  DBuf<int32_t> src, perm, ord, tmp, seg_end;
  DBuf<uint64_t> keys, keys2, np1, np2;
  DBuf<uint32_t> nkey, nkey2;
  DBuf<double> psum, psumsq, xbuf;
  DBuf<DNode> d_nodes;
  DBuf<DNodeOut> d_out;
  DBuf<char> sort_tmp;
  cudaEventRecord(ctx->ev[0], st);
  d_x.upload(x, static_cast<size_t>(n) * kNumFeatures, st);
  d_y.upload(y, static_cast<size_t>(n) * n_y, st);
  d_jobs.upload(jobs, st);
  src.alloc(std::max<int64_t>(total, 1));
  perm.alloc(std::max<int64_t>(total, 1));
  ord.alloc(std::max<int64_t>(total, 1));
  tmp.alloc(std::max<int64_t>(total, 1));
  keys.alloc(std::max<int64_t>(total, 1));
  keys2.alloc(std::max<int64_t>(total, 1));
  np1.alloc(std::max<int64_t>(total, 1));
  np2.alloc(std::max<int64_t>(total, 1));
  nkey.alloc(std::max<int64_t>(total, 1));
  nkey2.alloc(std::max<int64_t>(total, 1));
  xbuf.alloc(std::max<int64_t>(total, 1));
  psum.alloc(std::max<int64_t>(2 * total, 1));  // a step's rows + one entry per node (<= rows)
  psumsq.alloc(std::max<int64_t>(2 * total, 1));
  tree_rows_kernel<<<(J + 3) / 4, 128, 0, st>>>(d_jobs.p, J, n, seed, src.p, perm.p);
  after_launch("tree_rows_kernel", st);
  int64_t launches = 1;
  const bool dfs = prm.feature_subset < kNumFeatures;
  const int m = prm.feature_subset;
  out.assign(J, std::vector<HostTreeNode>());
  std::vector<std::vector<PendingNode>> pending(J);  // BFS: queue of the next level; DFS: stack
  for (int j = 0; j < J; ++j) pending[j].push_back({0, n, 0, -1, false});
  std::vector<DNode> act;
  std::vector<std::pair<int, PendingNode>> act_src;
  std::vector<DNodeOut> res;
  for (;;) {
    act.clear();
    act_src.clear();
    int64_t rows = 0;
    for (int j = 0; j < J; ++j) {
      if (pending[j].empty()) continue;
      auto take = [&](const PendingNode& pn) {
        // the node's index in the tree's node vector: in DFS order it is the
        // preorder id (grow() pushes a node before recursing)
        const int32_t id = static_cast<int32_t>(out[j].size());
        act.push_back(DNode{j, pn.begin, pn.len, pn.depth, id, static_cast<int32_t>(rows)});
        act_src.push_back({j, pn});
        out[j].push_back(HostTreeNode{});
        rows += pn.len;
      };
      if (dfs) {
        take(pending[j].back());
        pending[j].pop_back();
      } else {
        for (const PendingNode& pn : pending[j]) take(pn);
        pending[j].clear();
      }
    }
    if (act.empty()) break;
    if (rows >= (int64_t(1) << 31)) throw CudaError{"lt_train: step too large"};
    const int A = static_cast<int>(act.size());
    d_nodes.upload(act, st);
    d_out.alloc(A);
    seg_end.alloc(A);
    node_begin_kernel<<<(A + 7) / 8, 256, 0, st>>>(d_nodes.p, A, d_jobs.p, n, d_y.p, src.p, perm.p, prm.max_depth,
                                                   prm.min_leaf, prm.feature_subset, seed, ord.p, seg_end.p, d_out.p);
    after_launch("node_begin_kernel", st);
    ++launches;
    int node_bits = 1;
    while ((1 << node_bits) < A) ++node_bits;
    const int R = static_cast<int>(rows);
    size_t need1 = 0, need2 = 0;
    LT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, need1, keys.p, keys2.p, np1.p, np2.p, R, 0, 64, st));
    LT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, need2, nkey.p, nkey2.p, tmp.p, ord.p, R, 0, node_bits, st));
    sort_tmp.alloc(std::max<size_t>(std::max(need1, need2), 1));
    const unsigned rg = static_cast<unsigned>((rows + 255) / 256);
    for (int k = 0; k < m; ++k) {
      split_keys_kernel<<<rg, 256, 0, st>>>(d_nodes.p, A, d_out.p, k, n, d_x.p, src.p, ord.p, rows, keys.p, np1.p);
      after_launch("split_keys_kernel", st);
      size_t b1 = need1, b2 = need2;
      LT_CUDA(cub::DeviceRadixSort::SortPairs(sort_tmp.p, b1, keys.p, keys2.p, np1.p, np2.p, R, 0, 64, st));
      node_keys_kernel<<<rg, 256, 0, st>>>(np2.p, rows, nkey.p, tmp.p);
      after_launch("node_keys_kernel", st);
      LT_CUDA(cub::DeviceRadixSort::SortPairs(sort_tmp.p, b2, nkey.p, nkey2.p, tmp.p, ord.p, R, 0, node_bits, st));
      split_eval_kernel<<<(A + 7) / 8, 256, 0, st>>>(d_nodes.p, A, d_out.p, k, n, prm.min_leaf, d_x.p, d_y.p,
                                                     d_jobs.p, src.p, ord.p, xbuf.p, psum.p, psumsq.p);
      after_launch("split_eval_kernel", st);
      launches += 5;
    }
    node_finish_kernel<<<(A + 7) / 8, 256, 0, st>>>(d_nodes.p, A, d_out.p, n, d_x.p, src.p, perm.p, tmp.p);
    after_launch("node_finish_kernel", st);
    ++launches;
    res.resize(A);
    LT_CUDA(cudaMemcpyAsync(res.data(), d_out.p, A * sizeof(DNodeOut), cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaStreamSynchronize(st));
    // record the nodes; children become pending (DFS: right below left on the stack)
    std::vector<std::vector<PendingNode>> next(J);
    for (int a = 0; a < A; ++a) {
      const int j = act_src[a].first;
      const PendingNode& pn = act_src[a].second;
      const int32_t me = act[a].node_id;
      HostTreeNode& hn = out[j][me];
      hn.value = res[a].mean;
      hn.coverage = pn.len;
      if (pn.parent >= 0) (pn.is_left ? out[j][pn.parent].left : out[j][pn.parent].right) = me;
      if (!res[a].found) continue;
      hn.feature = res[a].feature;
      hn.threshold = res[a].threshold;
      const PendingNode l{pn.begin, res[a].left_len, pn.depth + 1, me, true};
      const PendingNode r{pn.begin + res[a].left_len, pn.len - res[a].left_len, pn.depth + 1, me, false};
      if (dfs) {
        pending[j].push_back(r);
        pending[j].push_back(l);
      } else {
        next[j].push_back(l);
        next[j].push_back(r);
      }
    }
    if (!dfs)
      for (int j = 0; j < J; ++j) pending[j] = std::move(next[j]);
  }
  // the reference's node vector order: preorder, left first (grow(), :93-125)
  for (int j = 0; j < J; ++j) {
    std::vector<int32_t> order;
    preorder(out[j], 0, order);
    std::vector<int32_t> pos(out[j].size());
    for (size_t i = 0; i < order.size(); ++i) pos[order[i]] = static_cast<int32_t>(i);
    std::vector<HostTreeNode> t(order.size());
    for (size_t i = 0; i < order.size(); ++i) {
      t[i] = out[j][order[i]];
      if (t[i].feature >= 0) {
        t[i].left = pos[t[i].left];
        t[i].right = pos[t[i].right];
      }
    }
    out[j] = std::move(t);
  }
  cudaEventRecord(ctx->ev[1], st);
  LT_CUDA(cudaStreamSynchronize(st));
  if (tm) {
    *tm = lt_timing{};
    tm->engine_ms = elapsed(ctx->ev[0], ctx->ev[1]);
    tm->run_ms = tm->engine_ms;
    tm->engine_launches = launches;
  }
}

int32_t write_trees(const std::vector<std::vector<HostTreeNode>>& trees, lt_tree_node* nodes, int64_t capacity,
                    int64_t* node_offset, int32_t* node_count, lt_status* status) {
  int64_t off = 0;
  for (size_t t = 0; t < trees.size(); ++t) {
    if (node_offset) node_offset[t] = off;
    if (node_count) node_count[t] = static_cast<int32_t>(trees[t].size());
    for (const HostTreeNode& h : trees[t]) {
      if (off < capacity && nodes) {
        lt_tree_node& o = nodes[off];
        o.feature_index = h.feature;
        o.left = h.feature >= 0 ? h.left : -1;
        o.right = h.feature >= 0 ? h.right : -1;
        o._pad = 0;
        o.threshold = h.feature >= 0 ? h.threshold : 0.0;
        o.value = h.value;
        o.coverage = h.coverage;
      }
      ++off;
    }
  }
  if (off > capacity) {
    set_status(status, LT_ERR_VALIDATION, LT_K_MESSAGE, -1, off, capacity,
               "lt_train: node capacity " + std::to_string(capacity) + " < " + std::to_string(off) + " nodes");
    return LT_ERR_VALIDATION;
  }
  return LT_OK;
}

bool validate_training(int64_t n_rows, HostErr* e) {
  if (n_rows <= 0) return e->set(LT_ERR_VALIDATION, "training set is empty");
  if (n_rows >= (int64_t(1) << 31)) return e->set(LT_ERR_UNSUPPORTED, "training set larger than 2^31 rows");
  return true;
}

}  // namespace

extern "C" {

int32_t lt_train_tree(lt_ctx* ctx, const double* x, int64_t n_rows, const double* y, const lt_tree_params* params,
                      uint64_t seed, uint64_t tree_tag, lt_tree_node* nodes, int64_t node_capacity,
                      int32_t* node_count, lt_status* status) {
  ok_status(status);
  if (!ctx->members.empty()) ctx = ctx->members[0];
  HostErr e;
  if (!validate_training(n_rows, &e) || !validate_tree_params(*params, &e)) {
    set_status(status, e.code, e.kind, -1, 0, 0, e.msg);
    return e.code;
  }
  try {
    std::vector<DTreeJob> jobs{DTreeJob{0, 0, 0, 0, tree_tag}};
    std::vector<std::vector<HostTreeNode>> trees;
    grow_trees(ctx, x, static_cast<int32_t>(n_rows), y, 1, jobs, *params, seed, trees, &ctx->timing);
    int64_t off = 0;
    return write_trees(trees, nodes, node_capacity, &off, node_count, status);
  } catch (const CudaError& err) {
    set_status(status, LT_ERR_DEVICE, LT_K_MESSAGE, -1, 0, 0, err.what);
    return LT_ERR_DEVICE;
  }
}

int32_t lt_train_forests(lt_ctx* ctx, const double* x, int64_t n_rows, const double* y, const int32_t* target_tags,
                         int32_t n_targets, const lt_forest_params* params, uint64_t seed, lt_tree_node* nodes,
                         int64_t node_capacity, int64_t* node_offset, int32_t* node_count, lt_status* status) {
  ok_status(status);
  if (!ctx->members.empty()) ctx = ctx->members[0];
  HostErr e;
  if (!validate_training(n_rows, &e)) {
    set_status(status, e.code, e.kind, -1, 0, 0, e.msg);
    return e.code;
  }
  if (params->n_trees < 1) {
    set_status(status, LT_ERR_VALIDATION, LT_K_VALIDATION_MSG, -1, 0, 0, "forest.n_trees: must be >= 1");
    return LT_ERR_VALIDATION;
  }
  if (!validate_tree_params(params->tree, &e)) {
    set_status(status, e.code, e.kind, -1, 0, 0, e.msg);
    return e.code;
  }
  try {
    // train_forest (predictor.cpp:213-245): tree t of target g is keyed
    // {kBootstrap, g, t} for its resample and g * 1000003 + t for its
    // feature subsets; train_placement_model (:250-269) is three of them.
    std::vector<DTreeJob> jobs;
    for (int32_t g = 0; g < n_targets; ++g)
      for (int32_t t = 0; t < params->n_trees; ++t) {
        const uint64_t tag = static_cast<uint64_t>(target_tags[g]);
        jobs.push_back(DTreeJob{g, params->bootstrap ? 1 : 0, tag, static_cast<uint64_t>(t),
                                tag * 1000003ull + static_cast<uint64_t>(t)});
      }
    std::vector<std::vector<HostTreeNode>> trees;
    grow_trees(ctx, x, static_cast<int32_t>(n_rows), y, n_targets, jobs, params->tree, seed, trees, &ctx->timing);
    return write_trees(trees, nodes, node_capacity, node_offset, node_count, status);
  } catch (const CudaError& err) {
    set_status(status, LT_ERR_DEVICE, LT_K_MESSAGE, -1, 0, 0, err.what);
    return LT_ERR_DEVICE;
  }
}

int32_t lt_predict_forests(lt_ctx* ctx, const lt_tree_node* nodes, int64_t n_nodes, const int64_t* node_offset,
                           int32_t n_trees, const int32_t* target_tags, int32_t n_targets, const double* x,
                           int64_t n_rows, double* out, lt_status* status) {
  ok_status(status);
  if (!ctx->members.empty()) ctx = ctx->members[0];
  if (n_trees < 1 || n_targets < 1) {
    set_status(status, LT_ERR_INTERNAL, LT_K_MESSAGE, -1, 0, 0, "forest has no trees");
    return LT_ERR_INTERNAL;
  }
  try {
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    static_assert(sizeof(DTreeNode) == sizeof(lt_tree_node), "layout");
    DBuf<DTreeNode> d_nodes;
    DBuf<int64_t> d_off;
    DBuf<int32_t> d_tags;
    DBuf<double> d_x, d_out;
    d_nodes.upload(reinterpret_cast<const DTreeNode*>(nodes), static_cast<size_t>(n_nodes), st);
    d_off.upload(node_offset, static_cast<size_t>(n_trees) * n_targets, st);
    d_tags.upload(target_tags, static_cast<size_t>(n_targets), st);
    d_x.upload(x, static_cast<size_t>(n_rows) * kNumFeatures, st);
    const int64_t total = n_rows * n_targets;
    d_out.alloc(std::max<int64_t>(total, 1));
    cudaEventRecord(ctx->ev[0], st);
    if (total > 0)
      forest_predict_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(
          d_nodes.p, d_off.p, n_trees, d_tags.p, n_targets, d_x.p, n_rows, d_out.p);
    after_launch("forest_predict_kernel", st);
    cudaEventRecord(ctx->ev[1], st);
    if (total > 0) LT_CUDA(cudaMemcpyAsync(out, d_out.p, total * sizeof(double), cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaStreamSynchronize(st));
    ctx->timing = lt_timing{};
    ctx->timing.engine_ms = elapsed(ctx->ev[0], ctx->ev[1]);
    ctx->timing.engine_launches = 1;
    return LT_OK;
  } catch (const CudaError& err) {
    set_status(status, LT_ERR_DEVICE, LT_K_MESSAGE, -1, 0, 0, err.what);
    return LT_ERR_DEVICE;
  }
}

}  // extern "C"
