// Multi-device contexts (`lt_create(device_mask)`; 8e: scenarios
// sharded across the GPUs of one box, one gather of the per-workload optima).
// Included by capi.cu after host_sweep.h.
//
// A group context owns one member context per device entry, each with its own
// streams and block cache partition. A batch call:
//   * shards the scenarios / conditions by estimated cost (LPT greedy: the
//     largest remaining item goes to the least loaded member), since every
//     (condition, N, G) engine is independent (placement.cpp:209-217, :492-522);
//     all grid points of a condition stay on one member so K3's reduction is
//     local;
//   * runs the members on one host thread each (cudaSetDevice per thread);
//   * sweeps: gathers every member's fixed-size placement and frontier rows
//     to the first member's device -- over NCCL (ncclSend / ncclRecv in one
//     group, single process, ncclCommInitAll) when the members are distinct
//     devices, else with peer copies -- and copies them back once;
//   * simulations: each member returns its summaries (and per-request states)
//     to host memory directly and the host scatters them to batch order (the
//     per-scenario records are the caller's output, not an exchange).
// Statuses and messages are those of the single-device call, and the
// call-level status is the lowest failing index (placement.cpp:93-95).
//
// NCCL is opened at run time (dlopen "libnccl.so.2"): a process that already
// loaded one (PyTorch's) shares it, and single-device use never needs it.

#include <dlfcn.h>
#include <nccl.h>  // types and enums only; entry points come from dlsym

namespace {

struct NcclApi {
  bool ok = false;
  std::string error;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;

  static NcclApi& get() {
    static NcclApi* api = [] {
      auto* a = new NcclApi();
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
      if (!h) {
        const char* e = dlerror();
        a->error = std::string("libnccl.so.2 not loadable: ") + (e ? e : "?");
        return a;
      }
      auto sym = [&](auto& fn, const char* name) {
        fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
        if (!fn && a->error.empty()) a->error = std::string("libnccl.so.2 lacks ") + name;
      };
      sym(a->CommInitAll, "ncclCommInitAll");
      sym(a->CommDestroy, "ncclCommDestroy");
      sym(a->GroupStart, "ncclGroupStart");
      sym(a->GroupEnd, "ncclGroupEnd");
      sym(a->Send, "ncclSend");
      sym(a->Recv, "ncclRecv");
      sym(a->GetErrorString, "ncclGetErrorString");
      a->ok = a->error.empty();
      return a;
    }();
    return *api;
  }
  void check(ncclResult_t r, const char* what) const {
    if (r != ncclSuccess) throw CudaError{std::string(what) + ": " + (GetErrorString ? GetErrorString(r) : "nccl error")};
  }
};

// LPT greedy: item costs -> member of each item. Equal costs keep index
// order, so the partition is deterministic.
std::vector<int> lpt_assign(const std::vector<double>& cost, int members) {
  std::vector<int64_t> order(cost.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int64_t>(i);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return cost[a] > cost[b]; });
  std::vector<double> load(members, 0.0);
  std::vector<int> who(cost.size(), 0);
  for (int64_t i : order) {
    int m = 0;
    for (int k = 1; k < members; ++k)
      if (load[k] < load[m]) m = k;
    who[i] = m;
    load[m] += cost[i];
  }
  return who;
}

// Estimated engine work of a condition's whole grid: per row, its G
// candidates x the row's offered tokens (instantiate_condition's
// round-robin mix, placement.cpp:148-155: leg i % m for i in [0, N)).
double condition_cost(const lt_condition_batch* b, int64_t c, const lt_sweep_grid* grid, double duration) {
  const lt_condition& cd = b->conditions[c];
  const int m = std::max(cd.mix_count, 1);
  double out_mean = 1.0;
  if (cd.length_index >= 0 && cd.length_index < b->n_lengths)
    out_mean = std::max(output_mean(b->lengths[cd.length_index], b->full_lengths), 0.0) + 1.0;
  double cost = 0.0;
  for (int r = 0; r < grid->n_count; ++r) {
    const int n = grid->n_values[r];
    double rate = 0.0;
    for (int j = 0; j < cd.mix_count; ++j) {
      const double cnt = static_cast<double>(n / m + (j < n % m ? 1 : 0));
      rate += cnt * std::max(b->templates[cd.mix_offset + j].rate, 0.0);
    }
    const int g_count = grid->g_mode == LT_G_EXPLICIT ? std::max(grid->g_count, 1) : 4;
    cost += g_count * (rate * std::max(duration, 0.0) * out_mean + 64.0);
  }
  return cost;
}

// Runs fn(member index) on one host thread per member; CUDA errors are
// carried back and the lowest member's is rethrown.
template <typename F>
void on_members(lt_ctx* g, F&& fn) {
  const int k = static_cast<int>(g->members.size());
  std::vector<std::string> err(k);
  std::vector<std::thread> pool;
  for (int m = 0; m < k; ++m) {
    pool.emplace_back([&, m] {
      try {
        cudaSetDevice(g->members[m]->device);
        fn(m);
      } catch (const CudaError& e) {
        err[m] = e.what.empty() ? "device error" : e.what;
      } catch (const std::exception& e) {
        err[m] = e.what();
      }
    });
  }
  for (auto& t : pool) t.join();
  for (int m = 0; m < k; ++m)
    if (!err[m].empty()) throw CudaError{"device " + std::to_string(g->members[m]->device) + ": " + err[m]};
}

void add_member_timing(lt_timing& sum, const lt_timing& t) {
  // device phases overlap across members: the call takes the slowest one
  sum.tables_ms = std::max(sum.tables_ms, t.tables_ms);
  sum.merge_ms = std::max(sum.merge_ms, t.merge_ms);
  sum.engine_ms = std::max(sum.engine_ms, t.engine_ms);
  sum.reduce_ms = std::max(sum.reduce_ms, t.reduce_ms);
  sum.run_ms = std::max(sum.run_ms, t.run_ms);
  sum.plan_ms = std::max(sum.plan_ms, t.plan_ms);
  sum.h2d_ms = std::max(sum.h2d_ms, t.h2d_ms);
  sum.d2h_ms = std::max(sum.d2h_ms, t.d2h_ms);
  sum.h2d_bytes += t.h2d_bytes;
  sum.d2h_bytes += t.d2h_bytes;
  sum.engine_launches += t.engine_launches;
  sum.algorithmic_bytes += t.algorithmic_bytes;
}

// Gathers `bytes[m]` bytes at src[m] (on member m's device) into dst (on
// member 0's device) at byte offset off[m], in stream order after each
// member's work (the callers have synchronised the members).
void gather_to_first(lt_ctx* g, const std::vector<const void*>& src, const std::vector<size_t>& bytes,
                     const std::vector<size_t>& off, char* dst) {
  const int k = static_cast<int>(g->members.size());
  lt_ctx* m0 = g->members[0];
  cudaSetDevice(m0->device);
  if (bytes[0]) LT_CUDA(cudaMemcpyAsync(dst + off[0], src[0], bytes[0], cudaMemcpyDeviceToDevice, m0->stream));
  if (g->transport == LT_GATHER_NCCL) {
    const NcclApi& nc = NcclApi::get();
    nc.check(nc.GroupStart(), "ncclGroupStart");
    for (int m = 1; m < k; ++m) {
      if (!bytes[m]) continue;
      nc.check(nc.Send(src[m], bytes[m], ncclInt8, 0, static_cast<ncclComm_t>(g->comms[m]), g->members[m]->stream),
               "ncclSend");
      nc.check(nc.Recv(dst + off[m], bytes[m], ncclInt8, m, static_cast<ncclComm_t>(g->comms[0]), m0->stream),
               "ncclRecv");
    }
    nc.check(nc.GroupEnd(), "ncclGroupEnd");
  } else {
    for (int m = 1; m < k; ++m)
      if (bytes[m])
        LT_CUDA(cudaMemcpyPeerAsync(dst + off[m], m0->device, src[m], g->members[m]->device, bytes[m], m0->stream));
  }
  for (int m = 1; m < k; ++m) {
    cudaSetDevice(g->members[m]->device);
    LT_CUDA(cudaStreamSynchronize(g->members[m]->stream));
  }
  cudaSetDevice(m0->device);
}

int32_t group_sweep(lt_ctx* g, const lt_condition_batch* batch, const lt_server_config* config,
                    const lt_sweep_grid* grid, double duration_s, uint64_t seed, const lt_sweep_options* options,
                    const lt_sim_options* sim_options, lt_placement* out, lt_frontier_point* frontier,
                    int32_t max_frontier, lt_status* status) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  const int64_t n = batch->n_conditions;
  const int k = static_cast<int>(g->members.size());
  g->messages.assign(n, std::string());
  try {
    std::vector<double> cost(n);
    for (int64_t c = 0; c < n; ++c) cost[c] = condition_cost(batch, c, grid, duration_s);
    const std::vector<int> who = lpt_assign(cost, k);
    std::vector<std::vector<int64_t>> idx(k);
    for (int64_t c = 0; c < n; ++c) idx[who[c]].push_back(c);
    std::vector<std::vector<lt_condition>> conds(k);
    std::vector<SweepRun> runs(k);
    on_members(g, [&](int m) {
      for (int64_t c : idx[m]) conds[m].push_back(batch->conditions[c]);
      lt_condition_batch sub = *batch;
      sub.conditions = conds[m].data();
      sub.n_conditions = static_cast<int64_t>(conds[m].size());
      sweep_run(g->members[m], &sub, config, grid, duration_s, seed, options, sim_options, max_frontier, runs[m]);
    });
    // one gather of the fixed-size rows to the first device, one copy back
    const auto tg = clk::now();
    std::vector<const void*> src_p(k), src_f(k);
    std::vector<size_t> bytes_p(k), bytes_f(k), off_p(k), off_f(k);
    size_t tot_p = 0, tot_f = 0;
    for (int m = 0; m < k; ++m) {
      const size_t nm = idx[m].size();
      src_p[m] = runs[m].d_out.p;
      src_f[m] = runs[m].d_front.p;
      bytes_p[m] = nm * sizeof(lt_placement);
      bytes_f[m] = nm * static_cast<size_t>(max_frontier) * sizeof(lt_frontier_point);
      off_p[m] = tot_p;
      off_f[m] = tot_f;
      tot_p += bytes_p[m];
      tot_f += bytes_f[m];
    }
    lt_ctx* m0 = g->members[0];
    cudaSetDevice(m0->device);
    DBuf<char> d_p, d_f;
    d_p.alloc(std::max<size_t>(tot_p, 1));
    d_f.alloc(std::max<size_t>(tot_f, 1));
    gather_to_first(g, src_p, bytes_p, off_p, d_p.p);
    gather_to_first(g, src_f, bytes_f, off_f, d_f.p);
    std::vector<lt_placement> h_p(n);
    std::vector<lt_frontier_point> h_f(static_cast<size_t>(n) * max_frontier);
    if (tot_p) LT_CUDA(cudaMemcpyAsync(h_p.data(), d_p.p, tot_p, cudaMemcpyDeviceToHost, m0->stream));
    if (tot_f) LT_CUDA(cudaMemcpyAsync(h_f.data(), d_f.p, tot_f, cudaMemcpyDeviceToHost, m0->stream));
    LT_CUDA(cudaStreamSynchronize(m0->stream));
    const double gather_ms = std::chrono::duration<double, std::milli>(clk::now() - tg).count();
    // scatter to batch order, statuses and messages per member
    lt_timing t{};
    int64_t pos = 0;
    for (int m = 0; m < k; ++m) {
      const int64_t nm = static_cast<int64_t>(idx[m].size());
      std::vector<lt_placement*> rows(nm);
      std::vector<std::string> msgs(nm);
      for (int64_t j = 0; j < nm; ++j) {
        const int64_t c = idx[m][j];
        out[c] = h_p[pos + j];
        if (max_frontier > 0)
          std::memcpy(frontier + c * max_frontier, h_f.data() + (pos + j) * max_frontier,
                      max_frontier * sizeof(lt_frontier_point));
        rows[j] = out + c;
      }
      sweep_statuses(runs[m], rows.data(), msgs.data());
      for (int64_t j = 0; j < nm; ++j) g->messages[idx[m][j]] = std::move(msgs[j]);
      lt_timing tm{};
      tm.tables_ms = runs[m].tm.tables_ms;
      tm.merge_ms = runs[m].tm.merge_ms;
      tm.engine_ms = runs[m].tm.engine_ms;
      tm.reduce_ms = runs[m].reduce_ms;
      tm.run_ms = runs[m].tm.run_ms;
      tm.engine_launches = runs[m].tm.launches;
      tm.algorithmic_bytes = runs[m].tm.algo;
      add_member_timing(t, tm);
      pos += nm;
    }
    for (auto& r : runs) {  // release each member's rows on its own device's stream order
      cudaSetDevice(r.d_out.dev);
      r.d_out.release();
      r.d_front.release();
    }
    cudaSetDevice(m0->device);
    t.gather_ms = gather_ms;
    t.gather_bytes = static_cast<int64_t>(tot_p + tot_f - bytes_p[0] - bytes_f[0]);
    t.d2h_bytes = static_cast<int64_t>(tot_p + tot_f);
    t.devices = k;
    t.total_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
    g->timing = t;
    return first_condition_error(g, out, n, status);
  } catch (const CudaError& e) {
    set_status(status, LT_ERR_DEVICE, LT_K_MESSAGE, -1, 0, 0, e.what);
    return LT_ERR_DEVICE;
  }
}

int32_t group_simulate(lt_ctx* g, const lt_workload_batch* batch, const lt_server_config* config,
                       const lt_sim_options* options, lt_sim_summary* out, lt_request_states* states,
                       lt_status* status) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  const int64_t n = batch->n_scenarios;
  const int k = static_cast<int>(g->members.size());
  g->messages.assign(n, std::string());
  std::vector<double> est(n);
  for (int64_t i = 0; i < n; ++i) est[i] = est_requests(batch, i);
  const std::vector<int> who = lpt_assign(est, k);
  std::vector<std::vector<int64_t>> idx(k);
  for (int64_t i = 0; i < n; ++i) idx[who[i]].push_back(i);
  // per-member outputs; request rows are bounded by the same estimate that
  // sizes the RNG tables (a scenario cannot generate more)
  struct Part {
    std::vector<lt_scenario> scen;
    std::vector<lt_sim_summary> sum;
    std::vector<std::string> msg;
    lt_timing timing{};
    int32_t rc = LT_OK;
    std::vector<int64_t> off;
    std::vector<int8_t> phase;
    std::vector<int32_t> gen, pre, adp, in, outv;
    std::vector<double> first, last, arr;
  };
  std::vector<Part> parts(k);
  try {
    on_members(g, [&](int m) {
      Part& P = parts[m];
      for (int64_t i : idx[m]) P.scen.push_back(batch->scenarios[i]);
      lt_workload_batch sub = *batch;
      sub.scenarios = P.scen.data();
      sub.n_scenarios = static_cast<int64_t>(P.scen.size());
      P.sum.assign(std::max<size_t>(P.scen.size(), 1), lt_sim_summary{});
      lt_request_states rs{};
      if (states) {
        double cap = 0.0;
        for (int64_t i : idx[m]) cap += std::ceil(est[i]);
        const size_t c = static_cast<size_t>(cap);
        P.off.resize(P.scen.size() + 1);
        P.phase.resize(c);
        P.gen.resize(c);
        P.pre.resize(c);
        P.adp.resize(c);
        P.in.resize(c);
        P.outv.resize(c);
        P.first.resize(c);
        P.last.resize(c);
        P.arr.resize(c);
        rs.capacity = static_cast<int64_t>(c);
        rs.req_offset = P.off.data();
        rs.phase = P.phase.data();
        rs.tokens_generated = P.gen.data();
        rs.first_token_time_s = P.first.data();
        rs.completion_time_s = P.last.data();
        rs.preemption_count = P.pre.data();
        rs.adapter_id = P.adp.data();
        rs.input_tokens = P.in.data();
        rs.output_tokens = P.outv.data();
        rs.arrival_time_s = P.arr.data();
      }
      lt_ctx* mc = g->members[m];
      lt_status st{};
      P.rc = sub.n_scenarios ? lt_simulate_batch(mc, &sub, config, options, P.sum.data(), states ? &rs : nullptr, &st)
                             : LT_OK;
      if (P.rc == LT_ERR_DEVICE) throw CudaError{st.message};
      P.msg = mc->messages;
      P.timing = mc->timing;
    });
  } catch (const CudaError& e) {
    set_status(status, LT_ERR_DEVICE, LT_K_MESSAGE, -1, 0, 0, e.what);
    return LT_ERR_DEVICE;
  }
  lt_timing t{};
  for (int m = 0; m < k; ++m) {
    const Part& P = parts[m];
    for (size_t j = 0; j < idx[m].size(); ++j) {
      out[idx[m][j]] = P.sum[j];
      g->messages[idx[m][j]] = j < P.msg.size() ? P.msg[j] : std::string();
    }
    add_member_timing(t, P.timing);
  }
  if (states) {  // request rows in batch order, as the single-device call lays them out
    std::vector<int64_t> member_row(n, -1);
    for (int m = 0; m < k; ++m)
      for (size_t j = 0; j < idx[m].size(); ++j) member_row[idx[m][j]] = static_cast<int64_t>(j);
    int64_t off = 0;
    for (int64_t i = 0; i < n; ++i) {
      const Part& P = parts[who[i]];
      const int64_t j = member_row[i];
      if (states->req_offset) states->req_offset[i] = off;
      const int64_t src = P.off[j];
      for (int64_t r = 0; r < out[i].n_requests; ++r, ++off) {
        if (off >= states->capacity) continue;
        const int64_t s = src + r;
        if (states->phase) states->phase[off] = P.phase[s];
        if (states->tokens_generated) states->tokens_generated[off] = P.gen[s];
        if (states->first_token_time_s) states->first_token_time_s[off] = P.first[s];
        if (states->completion_time_s) states->completion_time_s[off] = P.last[s];
        if (states->preemption_count) states->preemption_count[off] = P.pre[s];
        if (states->adapter_id) states->adapter_id[off] = P.adp[s];
        if (states->input_tokens) states->input_tokens[off] = P.in[s];
        if (states->output_tokens) states->output_tokens[off] = P.outv[s];
        if (states->arrival_time_s) states->arrival_time_s[off] = P.arr[s];
      }
    }
  }
  t.devices = k;
  t.total_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
  g->timing = t;
  return first_error(g, out, n, status);
}

}  // namespace
