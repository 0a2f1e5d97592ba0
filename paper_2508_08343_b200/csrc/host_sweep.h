// lt_sweep_batch's grid points: sweep_optimal (placement.cpp:185-264) over
// many conditions at once. Included by capi.cu (anonymous namespace).
//
// Rows are simulated in waves, as sweep_optimal consumes them
// (placement.cpp:204-245): wave r holds row r (one N, its G candidates) of
// every condition that has neither stopped early nor failed, so the device
// simulates exactly the grid points the reference simulates.
//
// Device waves (Mean mode, the sweep's normal case):
//   * conditions are instantiated on the device from their mix templates
//     (cond_adapters_kernel), one adapter block per condition, shared by
//     all its grid points; the RNG tables of ids 1..N_max (one seed per
//     sweep) are drawn once per call (K0), not per wave;
//   * per wave the host writes only the row's scenario records (a few
//     scalars per point, from per-(condition, row) values computed once) and
//     sizes the request arrays from the device's arrival counts; pairs,
//     merge, engine, metrics run on the device and the summaries are
//     scattered into a device point table;
//   * the early-exit decision (best non-starved throughput, stall counter,
//     errors) is taken on the device (wave_decide_kernel), and the next
//     wave's conditions are a stable device compaction of the survivors;
//   * K3 reduces the point table on the device; one copy of the placements
//     and frontiers comes back.
// Batches outside that case (Full-mode sweeps, templates or configs that
// fail validation, which need the reference's exact per-adapter messages)
// take the host waves: each wave a regular plan built from lt_scenario
// records, as lt_simulate_batch would.

struct SweepSetup {
  const lt_condition_batch* batch = nullptr;
  std::vector<SweepRow> rows;
  std::vector<int32_t> g_list;
  int32_t per_cond = 0;
  int n_max = 1;
  int64_t n_points = 0;
  std::vector<int64_t> cond_base;  // first point of condition c, -1: failed validation
  double duration = 0.0;
  uint64_t seed = 0;
  const lt_sweep_options* options = nullptr;
};

struct SweepTiming {
  double engine_ms = 0, tables_ms = 0, merge_ms = 0, run_ms = 0;
  int64_t launches = 0, algo = 0;
  void add(const lt_timing& t) {
    engine_ms += t.engine_ms;
    tables_ms += t.tables_ms;
    merge_ms += t.merge_ms;
    run_ms += t.run_ms;
    launches += t.engine_launches;
    algo += t.algorithmic_bytes;
  }
};

// estimated requests per device batch: a whole row in one batch lets its
// longest engines run side by side (memory stays bounded)
constexpr double kSweepWaveRequests = 5.0e8;

// Host waves: every wave is a plan over lt_scenario records.
void sweep_waves_host(lt_ctx* ctx, const SweepSetup& S, const lt_server_config* config, const lt_sim_options& so,
                      DBuf<lt_sim_summary>& d_pts, std::unordered_map<int64_t, std::string>& point_msg,
                      SweepTiming& tm) {
  const lt_condition_batch* batch = S.batch;
  const int64_t n_cond = batch->n_conditions;
  std::vector<lt_adapter> adapters;
  std::vector<int64_t> cond_ab(n_cond, -1);
  for (int64_t c = 0; c < n_cond; ++c) {
    if (S.cond_base[c] < 0) continue;
    const lt_condition& cd = batch->conditions[c];
    cond_ab[c] = static_cast<int64_t>(adapters.size());
    for (int i = 0; i < S.n_max; ++i) {
      const lt_template& t = batch->templates[cd.mix_offset + (i % cd.mix_count)];
      lt_adapter a{};
      a.adapter_id = i + 1;
      a.rank = t.rank;
      a.rate = t.rate;
      a.length_index = -1;
      adapters.push_back(a);
    }
  }
  std::vector<lt_sim_summary> pts(std::max<int64_t>(S.n_points, 1));
  std::vector<char> active(n_cond, 0);
  std::vector<double> best(n_cond, -1.0);
  std::vector<int> stall(n_cond, 0);
  for (int64_t c = 0; c < n_cond; ++c) active[c] = S.cond_base[c] >= 0;
  for (size_t ni = 0; ni < S.rows.size(); ++ni) {
    const SweepRow& r = S.rows[ni];
    std::vector<int64_t> conds;
    for (int64_t c = 0; c < n_cond; ++c)
      if (active[c]) conds.push_back(c);
    size_t ci = 0;
    while (ci < conds.size()) {
      std::vector<lt_scenario> scen;
      std::vector<int64_t> pidx;
      double est = 0.0;
      while (ci < conds.size() && (scen.empty() || est < kSweepWaveRequests)) {
        const int64_t c = conds[ci++];
        const lt_condition& cd = batch->conditions[c];
        double rate_sum = 0.0;
        for (int i = 0; i < r.n; ++i) rate_sum += batch->templates[cd.mix_offset + (i % cd.mix_count)].rate;
        for (int gi = 0; gi < r.g_count; ++gi) {
          lt_scenario s{};
          s.adapter_offset = cond_ab[c];
          s.n_adapters = r.n;
          s.length_index = cd.length_index;
          s.duration_s = S.duration;
          s.seed = S.seed;
          s.slots = S.g_list[r.g_offset + gi];
          s.mode = S.options->mode;
          s.n_requests = -1;
          scen.push_back(s);
          pidx.push_back(S.cond_base[c] + r.point_offset + gi);
          est += rate_sum * S.duration;
        }
      }
      lt_workload_batch wb{};
      wb.scenarios = scen.data();
      wb.n_scenarios = static_cast<int64_t>(scen.size());
      wb.adapters = adapters.data();
      wb.n_adapters = static_cast<int64_t>(adapters.size());
      wb.lengths = batch->lengths;
      wb.n_lengths = batch->n_lengths;
      wb.full_lengths = batch->full_lengths;
      wb.n_full_pairs = batch->n_full_pairs;
      std::unique_ptr<lt_plan> plan(build_plan(ctx, &wb, config, &so));
      run_plan(*plan);
      std::vector<lt_sim_summary> part(scen.size());
      fetch_results(*plan, part.data(), nullptr);
      for (size_t k = 0; k < scen.size(); ++k) {
        pts[pidx[k]] = part[k];
        if (part[k].status != LT_OK) point_msg[pidx[k]] = ctx->messages[k];
      }
      tm.add(ctx->timing);
    }
    // which conditions continue (sweep_optimal's control flow)
    for (int64_t c : conds) {
      bool improved = false, err = false;
      for (int gi = 0; gi < r.g_count; ++gi) {
        const lt_sim_summary& p = pts[S.cond_base[c] + r.point_offset + gi];
        if (p.status != LT_OK) err = true;
        if (!p.starved && p.throughput_tok_s > best[c]) {
          best[c] = p.throughput_tok_s;
          improved = true;
        }
      }
      if (err) {
        active[c] = 0;
        continue;
      }
      if (S.options->early_exit) {
        stall[c] = improved ? 0 : stall[c] + 1;
        if (stall[c] >= S.options->early_exit_k && ni + 1 < S.rows.size()) active[c] = 0;
      }
    }
  }
  d_pts.upload(pts, ctx->stream);
}

// Whether every valid condition can be instantiated on the device: Mean-mode
// sweep, a valid config, positive duration, and templates that pass
// WorkloadSpec::validate (rank >= 0, rate > 0), at most kMaxAdapters adapters.
bool sweep_device_eligible(const SweepSetup& S, const Config& cfg) {
  if (S.options->mode != LT_MODE_MEAN || !cfg.body_ok || !(S.duration > 0.0) || S.n_max > kMaxAdapters) return false;
  if (std::getenv("LT_SWEEP_HOST")) return false;  // (test hook: the host waves)
  const lt_condition_batch* b = S.batch;
  for (int64_t c = 0; c < b->n_conditions; ++c) {
    if (S.cond_base[c] < 0) continue;
    const lt_condition& cd = b->conditions[c];
    for (int j = 0; j < cd.mix_count; ++j) {
      const lt_template& t = b->templates[cd.mix_offset + j];
      if (t.rank < 0 || !(t.rate > 0.0)) return false;
    }
  }
  return true;
}

// Device waves (see the top of this file).
void sweep_waves_device(lt_ctx* ctx, const SweepSetup& S, const lt_server_config* config, const lt_sim_options& so,
                        DBuf<lt_sim_summary>& d_pts, std::unordered_map<int64_t, std::string>& point_msg,
                        SweepTiming& tm) {
  const auto t_setup = std::chrono::steady_clock::now();
  const lt_condition_batch* batch = S.batch;
  const int64_t n_cond = batch->n_conditions;
  const int n_rows = static_cast<int>(S.rows.size());
  auto plan = std::make_unique<lt_plan>();
  lt_plan& W = *plan;
  W.ctx = ctx;
  W.st = ctx->stream;
  cudaStream_t st = W.st;
  for (cudaEvent_t& e : W.ev) LT_CUDA(cudaEventCreate(&e));
  load_config(W.cfg, config, &so);
  W.want_digest = 0;
  W.fresh = true;
  const int64_t iter_cap = W.cfg.raw.iteration_cap;
  const int64_t budget = W.cfg.raw.total_kv_budget;
  // conditions: templates with their load latencies, length parameters
  std::vector<DTemplate> tmpl(std::max<int64_t>(batch->n_templates, 1));
  for (int64_t j = 0; j < batch->n_templates; ++j) {
    tmpl[j].rank = batch->templates[j].rank;
    tmpl[j]._pad = 0;
    tmpl[j].rate = batch->templates[j].rate;
    tmpl[j].load_lat = load_latency_cached(W.cfg, batch->templates[j].rank);
  }
  std::vector<int32_t> mix_off(std::max<int64_t>(n_cond, 1), 0), mix_cnt(std::max<int64_t>(n_cond, 1), 0);
  std::vector<DLen> lens;
  std::map<std::string, int32_t> len_index;
  std::vector<int32_t> cond_len(n_cond, 0);
  // per (condition, row): ideal throughput and engine cost (sequential sums in
  // adapter order, as prepare_scenario forms them), the slot cost of the
  // points' max rank (or its ConfigError)
  std::vector<double> row_ideal(static_cast<size_t>(n_cond) * n_rows, 0.0), row_cost(row_ideal.size(), 0.0);
  std::vector<int64_t> row_slot(row_ideal.size(), 0);
  std::vector<HostErr> row_err(row_ideal.size());
  std::vector<char> row_bad(row_ideal.size(), 0);
  double rate_max = 0.0;
  for (int64_t c = 0; c < n_cond; ++c) {
    if (S.cond_base[c] < 0) continue;
    const lt_condition& cd = batch->conditions[c];
    mix_off[c] = static_cast<int32_t>(cd.mix_offset);
    mix_cnt[c] = cd.mix_count;
    const lt_length_spec& l = batch->lengths[cd.length_index];
    const DLen dl = as_dlen(l, batch->full_lengths);
    const std::string key(reinterpret_cast<const char*>(&dl), sizeof(dl));
    auto it = len_index.find(key);
    if (it == len_index.end()) {
      it = len_index.emplace(key, static_cast<int32_t>(lens.size())).first;
      lens.push_back(dl);
    }
    cond_len[c] = it->second;
    double tokens = output_mean(l, batch->full_lengths);
    if (W.cfg.raw.ideal_includes_input) tokens += input_mean(l, batch->full_lengths);
    const double out_mean1 = output_mean(l, batch->full_lengths) + 1.0;
    double ideal = 0.0, cost = 0.0;
    int max_rank = 0, i = 0;
    for (int ri = 0; ri < n_rows; ++ri) {
      const int N = S.rows[ri].n;
      for (; i < N; ++i) {
        const lt_template& t = batch->templates[cd.mix_offset + (i % cd.mix_count)];
        ideal += t.rate * tokens;
        cost += t.rate * S.duration * out_mean1;
        max_rank = std::max(max_rank, t.rank);
        rate_max = std::max(rate_max, t.rate);
      }
      const size_t q = static_cast<size_t>(c) * n_rows + ri;
      row_ideal[q] = ideal;
      row_cost[q] = cost;
      int64_t cs = 0;
      if (!slot_cost(W.cfg, max_rank, &cs, &row_err[q])) row_bad[q] = 1;
      row_slot[q] = cs;
    }
  }
  // device condition blocks (instantiate_condition at N_max)
  const int n_max = S.n_max;
  DBuf<DTemplate> d_tmpl;
  DBuf<int32_t> d_mix_off, d_mix_cnt;
  d_tmpl.upload(tmpl, st);
  d_mix_off.upload(mix_off, st);
  d_mix_cnt.upload(mix_cnt, st);
  W.adapters.alloc(std::max<int64_t>(n_cond * n_max, 1));
  if (n_cond > 0) {
    const int64_t nt = n_cond * n_max;
    cond_adapters_kernel<<<static_cast<unsigned>((nt + 255) / 256), 256, 0, st>>>(
        static_cast<int>(n_cond), n_max, d_mix_off.p, d_mix_cnt.p, d_tmpl.p, W.adapters.p);
    after_launch("cond_adapters_kernel", st);
    ++tm.launches;
  }
  if (lens.empty()) lens.push_back(DLen{1, 0, 1, 0});
  W.lens.upload(lens, st);
  // K0 once: keys (seed, 1..N_max) at the batch's largest rate
  PinnedVec<DKeyNI> keys(n_max);
  for (int i = 0; i < n_max; ++i) {
    DKey k{};
    k.seed = S.seed;
    k.id = i + 1;
    k.rate_max = rate_max;
    k.dur_max = S.duration;
    keys[i] = k;
  }
  int64_t e_total = size_keys(keys);
  W.n_keys = n_max;
  W.seed_state.alloc(std::min<int64_t>(n_max, kSeedChunk) * 2 * kMtN);
  W.tab_overflow.alloc(1);
  cudaEventRecord(W.ev[0], st);
  for (int attempt = 0;; ++attempt) {
    LT_CUDA(cudaMemsetAsync(W.tab_overflow.p, 0, sizeof(int32_t), st));
    W.keys.upload(keys.data(), keys.size(), st);
    W.E.alloc(std::max<int64_t>(e_total, 1));
    W.Z.alloc(std::max<int64_t>(e_total, 1));
    tm.launches += launch_tables(W, n_max, st);
    int32_t any = 0;
    LT_CUDA(cudaMemcpyAsync(&any, W.tab_overflow.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaStreamSynchronize(st));
    if (!any) break;
    if (attempt > 4) throw CudaError{"RNG table sizing failed"};
    std::vector<DKey> back(keys.size());
    LT_CUDA(cudaMemcpy(back.data(), W.keys.p, back.size() * sizeof(DKey), cudaMemcpyDeviceToHost));
    e_total = 0;
    for (size_t k = 0; k < keys.size(); ++k) {
      if (back[k].overflow) keys[k].cap = static_cast<int32_t>(std::min<int64_t>(int64_t(keys[k].cap) * 4, 2000000000));
      keys[k].e_off = keys[k].z_off = e_total;
      e_total += keys[k].cap;
    }
  }
  cudaEventRecord(W.ev[1], st);
  bool tables_timed = false;  // read once the first wave has synchronised the stream
  // point table and the per-condition early-exit state
  d_pts.alloc(std::max<int64_t>(S.n_points, 1));
  DBuf<int64_t> d_base;
  DBuf<double> d_best;
  DBuf<int32_t> d_stall, d_act, d_num;
  DBuf<uint8_t> d_alive;
  DBuf<int64_t> d_pidx;
  DBuf<char> sel_tmp;
  d_base.upload(S.cond_base, st);
  d_best.upload(std::vector<double>(std::max<int64_t>(n_cond, 1), -1.0), st);
  d_stall.upload(std::vector<int32_t>(std::max<int64_t>(n_cond, 1), 0), st);
  std::vector<uint8_t> alive0(std::max<int64_t>(n_cond, 1), 0);
  std::vector<int32_t> act;
  for (int64_t c = 0; c < n_cond; ++c)
    if (S.cond_base[c] >= 0) {
      alive0[c] = 1;
      act.push_back(static_cast<int32_t>(c));
    }
  d_alive.upload(alive0, st);
  d_act.upload(act.empty() ? std::vector<int32_t>{0} : act, st);
  d_num.alloc(1);
  size_t sel_bytes = 0;
  LT_CUDA(cub::DeviceSelect::Flagged(nullptr, sel_bytes, cub::CountingInputIterator<int32_t>(0), d_alive.p, d_act.p,
                                     d_num.p, static_cast<int>(std::max<int64_t>(n_cond, 1)), st));
  sel_tmp.alloc(std::max<size_t>(sel_bytes, 1));
  if (std::getenv("LT_HOST_TIMING"))
    std::fprintf(stderr, "[lt] sweep setup (conditions, rows, K0): %.1f ms\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_setup).count());
  for (int ni = 0; ni < n_rows && !act.empty(); ++ni) {
    const SweepRow& r = S.rows[ni];
    size_t ci = 0;
    while (ci < act.size()) {
      // the wave (or a budget-bounded part of it): the row's points of act[ci..)
      const auto tw = std::chrono::steady_clock::now();
      W.h_scen.clear();
      std::vector<int64_t> pidx;
      std::vector<double> cost;
      double est = 0.0;
      double rate_sum = 0.0;
      while (ci < act.size() && (W.h_scen.empty() || est < kSweepWaveRequests)) {
        const int32_t c = act[ci++];
        const size_t q = static_cast<size_t>(c) * n_rows + ni;
        const lt_condition& cd = batch->conditions[c];
        rate_sum = 0.0;
        for (int i = 0; i < r.n; ++i) rate_sum += batch->templates[cd.mix_offset + (i % cd.mix_count)].rate;
        for (int gi = 0; gi < r.g_count; ++gi) {
          const int G = S.g_list[r.g_offset + gi];
          DScen d;
          std::memset(&d, 0, sizeof(d));
          d.n_adapters = r.n;
          d.adapter_begin = static_cast<int64_t>(c) * n_max;
          d.G = G;
          d.generated = 1;
          d.ids_sorted = 1;
          d.duration = S.duration;
          d.iter_cap = iter_cap;
          d.length_param = cond_len[c];
          const int64_t point = S.cond_base[c] + r.point_offset + gi;
          if (row_bad[q]) {  // the Engine ctor's slot-cost ConfigError (engine.cpp:48-54)
            const HostErr& e = row_err[q];
            d.status = e.code;
            d.status_kind = e.kind;
            d.status_a = e.a;
            d.status_b = e.b;
            d.n_adapters = 0;
            point_msg[point] = e.msg;
          } else {
            const int64_t capacity = std::max<int64_t>(budget - static_cast<int64_t>(G) * row_slot[q], 0);
            if (capacity <= 0) {
              d.status = LT_ERR_CONFIG;
              d.status_kind = LT_K_INFEASIBLE_SLOTS;
              d.status_a = G;
              d.n_adapters = 0;
            }
            d.capacity = capacity;
            d.ideal = row_ideal[q];
          }
          W.h_scen.push_back(d);
          pidx.push_back(point);
          cost.push_back(d.status == LT_OK ? row_cost[q] : 0.0);
          est += rate_sum * S.duration;
        }
      }
      // scenario records up; (scenario, adapter) pairs and arrival counts on the device
      W.n_scen = static_cast<int64_t>(W.h_scen.size());
      W.scen.upload(W.h_scen, st);
      d_pidx.upload(pidx, st);
      W.n_pairs = W.n_scen * r.n;
      W.pair_scen.alloc(W.n_pairs);
      W.pair_adp.alloc(W.n_pairs);
      W.pair_begin.alloc(W.n_scen);
      W.adp_count.alloc(W.n_pairs);
      W.scen_count.alloc(W.n_scen);
      W.overflow.alloc(1);
      cudaEventRecord(W.ev[2], st);
      wave_pairs_kernel<<<static_cast<unsigned>((W.n_pairs + 255) / 256), 256, 0, st>>>(
          W.n_pairs, r.n, W.pair_scen.p, W.pair_adp.p, W.pair_begin.p);
      after_launch("wave_pairs_kernel", st);
      LT_CUDA(cudaMemsetAsync(W.scen_count.p, 0, W.n_scen * sizeof(unsigned long long), st));
      LT_CUDA(cudaMemsetAsync(W.overflow.p, 0, sizeof(int32_t), st));
      W.pair_g = pair_group(W.n_pairs ? est / static_cast<double>(W.n_pairs) : 1e9);
      launch_count(W, st);
      tm.launches += 2;
      std::vector<unsigned long long> counts(W.n_scen);
      int32_t ovf = 0;
      LT_CUDA(cudaMemcpyAsync(counts.data(), W.scen_count.p, W.n_scen * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(&ovf, W.overflow.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaStreamSynchronize(st));
      if (ovf) throw CudaError{"internal: RNG table shorter than an arrival stream"};
      int64_t off = 0;
      W.max_req = 0;
      for (int64_t i = 0; i < W.n_scen; ++i) {
        DScen& d = W.h_scen[i];
        d.n_req = d.status == LT_OK ? static_cast<int32_t>(counts[i]) : 0;
        d.req_begin = off;
        off += counts[i];  // (a failed point's arrivals are counted but never gathered)
        W.max_req = std::max<int64_t>(W.max_req, d.n_req);
      }
      W.total_req = off;
      W.scen.upload(W.h_scen, st);
      // merge, engine + metrics, scatter into the point table
      W.max_adapters = std::max(32, (r.n + 31) / 32 * 32);
      W.warps_per_block = 8;
      alloc_requests(W);
      tm.launches += merge_requests(W, false);  // (sized after the merge)
      cudaEventRecord(W.ev[3], st);
      size_engine(W, cost, 1024, false);  // (waves keep 8-warp blocks)
      size_workspace(W);
      reset_state(W);
      const EngineParams E = engine_params(W);
      cudaEventRecord(W.ev[4], st);
      launch_engine(W, E, st);
      after_launch("metrics_kernel", st);
      cudaEventRecord(W.ev[5], st);
      wave_scatter_kernel<<<static_cast<unsigned>((W.n_scen + 255) / 256), 256, 0, st>>>(
          static_cast<int>(W.n_scen), W.out.p, d_pidx.p, d_pts.p);
      after_launch("wave_scatter_kernel", st);
      tm.launches += 3 + (W.engine_variant == kEngineLatency);  // (links), engine, metrics, scatter
      LT_CUDA(cudaStreamSynchronize(st));
      if (!tables_timed) {
        tm.tables_ms += elapsed(W.ev[0], W.ev[1]);
        tables_timed = true;
      }
      tm.engine_ms += elapsed(W.ev[4], W.ev[5]);
      tm.merge_ms += elapsed(W.ev[2], W.ev[3]);
      tm.run_ms += elapsed(W.ev[2], W.ev[5]);
      if (std::getenv("LT_HOST_TIMING"))
        std::fprintf(stderr, "[lt] sweep wave N=%d: %lld points, %lld requests (max %lld), count+merge %.1f ms, "
                     "engine %.1f ms, variant %d, wall %.1f ms\n", r.n, static_cast<long long>(W.n_scen),
                     static_cast<long long>(W.total_req), static_cast<long long>(W.max_req), elapsed(W.ev[2], W.ev[3]),
                     elapsed(W.ev[4], W.ev[5]), W.engine_variant,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tw).count());
    }
    // the row's early-exit decisions, then the surviving conditions in order
    d_act.upload(act, st);
    wave_decide_kernel<<<static_cast<unsigned>((act.size() + 127) / 128), 128, 0, st>>>(
        static_cast<int>(act.size()), d_act.p, r, ni, n_rows, d_base.p, d_pts.p, S.options->early_exit,
        S.options->early_exit_k, d_best.p, d_stall.p, d_alive.p);
    after_launch("wave_decide_kernel", st);
    ++tm.launches;
    size_t sb = sel_bytes;
    LT_CUDA(cub::DeviceSelect::Flagged(sel_tmp.p, sb, cub::CountingInputIterator<int32_t>(0), d_alive.p, d_act.p,
                                       d_num.p, static_cast<int>(n_cond), st));
    int32_t n_act = 0;
    LT_CUDA(cudaMemcpyAsync(&n_act, d_num.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaStreamSynchronize(st));
    act.resize(n_act);
    if (n_act > 0)
      LT_CUDA(cudaMemcpyAsync(act.data(), d_act.p, n_act * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaStreamSynchronize(st));
  }
  // engine work and messages of the points that failed on the device: K3 reads the table
  (void)point_msg;
}

// One lt_sweep_batch call up to K3, with the placements and frontiers left on
// ctx's device (d_out, d_front): the single-device call copies them back, a
// multi-device context gathers every member's rows to its first device first.
struct SweepRun {
  int64_t n_cond = 0;
  std::vector<HostErr> cond_err;   // validation failures (cond_base < 0)
  std::vector<int64_t> cond_base;  // first grid point of condition c, -1: failed validation
  std::unordered_map<int64_t, std::string> point_msg;
  DBuf<lt_placement> d_out;
  DBuf<lt_frontier_point> d_front;
  SweepTiming tm;
  double reduce_ms = 0.0;
};

void sweep_run(lt_ctx* ctx, const lt_condition_batch* batch, const lt_server_config* config,
               const lt_sweep_grid* grid, double duration_s, uint64_t seed, const lt_sweep_options* options,
               const lt_sim_options* sim_options, int32_t max_frontier, SweepRun& R) {
  const int64_t n_cond = batch->n_conditions;
  R.n_cond = n_cond;
  cudaSetDevice(ctx->device);
  cudaStream_t st = ctx->stream;
  // SweepGrid::validate (placement.cpp:169-183)
  HostErr grid_err;
  bool grid_ok = true;
  if (grid->n_count <= 0) {
    grid_ok = grid_err.set(LT_ERR_VALIDATION, "grid.n_values: must be non-empty");
  } else {
    for (int i = 0; i < grid->n_count && grid_ok; ++i) {
      if (grid->n_values[i] < 1)
        grid_ok = grid_err.set(LT_ERR_VALIDATION, "grid.n_values: entries must be >= 1");
      else if (i > 0 && grid->n_values[i] <= grid->n_values[i - 1])
        grid_ok = grid_err.set(LT_ERR_VALIDATION, "grid.n_values: must be strictly ascending");
    }
    if (grid_ok && grid->g_mode == LT_G_EXPLICIT) {
      if (grid->g_count <= 0)
        grid_ok = grid_err.set(LT_ERR_VALIDATION, "grid.g_values: must be non-empty in explicit mode");
      for (int i = 0; i < grid->g_count && grid_ok; ++i)
        if (grid->g_values[i] < 1) grid_ok = grid_err.set(LT_ERR_VALIDATION, "grid.g_values: entries must be >= 1");
    }
  }
  // rows: SweepGrid::g_candidates (placement.cpp:159-167)
  std::vector<SweepRow> rows;
  std::vector<int32_t> g_list;
  int32_t per_cond = 0;
  int n_max = 1;
  if (grid_ok) {
    for (int i = 0; i < grid->n_count; ++i) {
      const int n = grid->n_values[i];
      n_max = std::max(n_max, n);
      std::set<int> gs;
      if (grid->g_mode == LT_G_GEOMETRIC) {
        for (int g : {8, n / 4, n / 2, n}) gs.insert(std::clamp(g, 1, n));
      } else {
        for (int k = 0; k < grid->g_count; ++k) gs.insert(std::clamp(grid->g_values[k], 1, n));
      }
      SweepRow r{n, static_cast<int32_t>(gs.size()), static_cast<int32_t>(g_list.size()), per_cond};
      for (int g : gs) g_list.push_back(g);
      per_cond += r.g_count;
      rows.push_back(r);
    }
  }
  // Condition validation (sweep_optimal, placement.cpp:186-188); grid
  // points of valid conditions are numbered row-major per condition.
  SweepSetup S;
  S.batch = batch;
  S.rows = rows;
  S.g_list = g_list;
  S.per_cond = per_cond;
  S.n_max = n_max;
  S.duration = duration_s;
  S.seed = seed;
  S.options = options;
  S.cond_base.assign(n_cond, -1);
  R.cond_err.assign(n_cond, HostErr());
  for (int64_t c = 0; c < n_cond; ++c) {
    const lt_condition& cd = batch->conditions[c];
    HostErr& e = R.cond_err[c];
    if (!grid_ok) {
      e = grid_err;
      continue;
    }
    if (!validate_lengths(batch->lengths[cd.length_index], batch->full_lengths, "condition.lengths", &e)) continue;
    if (cd.mix_count <= 0) {
      e.set(LT_ERR_VALIDATION, "condition.mix: must be non-empty");
      continue;
    }
    S.cond_base[c] = S.n_points;
    S.n_points += per_cond;
  }
  R.cond_base = S.cond_base;
  lt_sim_options so{};
  if (sim_options) so = *sim_options;
  so.want_digest = 0;
  Config probe;
  load_config(probe, config, &so);
  DBuf<lt_sim_summary> d_pts;
  if (grid_ok && sweep_device_eligible(S, probe))
    sweep_waves_device(ctx, S, config, so, d_pts, R.point_msg, R.tm);
  else
    sweep_waves_host(ctx, S, config, so, d_pts, R.point_msg, R.tm);
  DBuf<SweepRow> d_rows;
  DBuf<int32_t> d_g;
  DBuf<int64_t> d_base;
  d_rows.upload(rows, st);
  d_g.upload(g_list, st);
  d_base.upload(R.cond_base, st);
  R.d_out.alloc(std::max<int64_t>(n_cond, 1));
  R.d_front.alloc(std::max<int64_t>(n_cond * max_frontier, 1));
  // rows past a condition's frontier_count read as zeros, not stale cache blocks
  LT_CUDA(cudaMemsetAsync(R.d_front.p, 0, R.d_front.n * sizeof(lt_frontier_point), st));
  cudaEventRecord(ctx->ev[5], st);
  if (n_cond > 0 && !rows.empty()) {
    sweep_reduce_kernel<<<static_cast<unsigned>((n_cond + 127) / 128), 128, 0, st>>>(
        static_cast<int>(n_cond), d_rows.p, static_cast<int>(rows.size()), d_g.p, per_cond, d_base.p, d_pts.p,
        options->early_exit, options->early_exit_k, max_frontier, R.d_out.p, R.d_front.p);
    after_launch("sweep_reduce_kernel", st);
    ++R.tm.launches;
  }
  cudaEventRecord(ctx->ev[6], st);
  LT_CUDA(cudaStreamSynchronize(st));  // K3's inputs are released on return
  R.reduce_ms = elapsed(ctx->ev[5], ctx->ev[6]);
}

// Status and reference message of every condition of R from its placement
// row as copied back (rows[c] = condition c of R's batch; messages[c] gets
// the text).
void sweep_statuses(const SweepRun& R, lt_placement* const* rows, std::string* messages) {
  for (int64_t c = 0; c < R.n_cond; ++c) {
    lt_placement& p = *rows[c];
    std::string msg;
    if (R.cond_base[c] < 0) {
      std::memset(&p, 0, sizeof(p));
      p.status_point = -1;
      p.status = R.cond_err[c].code;
      p.status_kind = R.cond_err[c].kind;
      p.status_a = R.cond_err[c].a;
      p.status_b = R.cond_err[c].b;
      msg = R.cond_err[c].msg;
    } else if (p.status != LT_OK) {
      auto it = R.point_msg.find(p.status_point);
      msg = it != R.point_msg.end() ? it->second : render(p.status, p.status_kind, p.status_a, p.status_b);
    }
    messages[c] = std::move(msg);
  }
}

void sweep_timing(lt_ctx* ctx, const SweepRun& R, double d2h_ms) {
  lt_timing& t = ctx->timing;
  t.tables_ms = R.tm.tables_ms;
  t.merge_ms = R.tm.merge_ms;
  t.engine_ms = R.tm.engine_ms;
  t.reduce_ms = R.reduce_ms;
  t.d2h_ms = d2h_ms;
  t.run_ms = R.tm.run_ms;
  t.engine_launches = R.tm.launches;
  t.algorithmic_bytes = R.tm.algo;
}

// The call-level status of a sweep: the lowest failing condition
// (placement.cpp:93-95).
int32_t first_condition_error(lt_ctx* ctx, const lt_placement* out, int64_t n, lt_status* status) {
  for (int64_t c = 0; c < n; ++c) {
    if (out[c].status != LT_OK) {
      set_status(status, out[c].status, out[c].status_kind, c, out[c].status_a, out[c].status_b, ctx->messages[c]);
      return out[c].status;
    }
  }
  return LT_OK;
}
