// Running a built plan (capi.cu includes this after host_plan.h): the
// transient buffers between runs, K0 + merge per run, the engine builds'
// launches, the percentile and report passes, result collection.
#pragma once

namespace {

// Buffers a run regenerates from the plan's inputs (K0 tables, request
// arrays, merge scratch, engine workspace): what lt_plan_trim releases.
template <typename F>
void for_transient(lt_plan& P, F&& f) {
  f(P.seed_state);
  f(P.E);
  f(P.Z);
  f(P.r_arr);
  f(P.r_first);
  f(P.r_last);
  f(P.r_in);
  f(P.r_out);
  f(P.r_adp);
  f(P.r_gen);
  f(P.r_pre);
  f(P.r_phase);
  f(P.ws_run);
  f(P.ws_pq);
  f(P.ws_node);
  f(P.r_link);
  f(P.ws_ov);
  f(P.ws_link);
  f(P.pair_excl);
  f(P.st_in);
  f(P.st_out);
  f(P.sv_in);
  f(P.sv_out);
  f(P.pos_a);
  f(P.pos_b);
  f(P.skey_a);
  f(P.skey_b);
  f(P.sort_tmp);
}

void trim_plan(lt_plan& P) {
  if (P.trimmed || P.has_scripted) return;
  P.trimmed_sizes.clear();
  for_transient(P, [&](auto& b) {
    P.trimmed_sizes.push_back(b.n);
    b.release();
  });
  P.trimmed = true;
  P.fresh = false;  // the next run regenerates the tables
}

void untrim_plan(lt_plan& P) {
  if (!P.trimmed) return;
  size_t k = 0;
  for_transient(P, [&](auto& b) { b.alloc(P.trimmed_sizes[k++]); });
  P.trimmed = false;
}

int64_t merge_requests(lt_plan& P, bool sized = true);

// K0 + merge: (re)generates every request of every generated scenario.
void prepare_requests(lt_plan& P) {
  cudaStream_t st = P.st;
  P.run_fresh = P.fresh;  // (a fresh run's tables were timed while the plan was built)
  cudaEventRecord(P.ev[0], st);
  // K0: RNG tables, arrival counts and request offsets are recomputed on
  // device every run (the first run after lt_plan_simulate reuses the ones
  // computed while sizing the buffers).
  int64_t launches = 0;
  if (!P.fresh && P.n_keys > 0) launches += launch_tables(P, P.n_keys, st);
  cudaEventRecord(P.ev[1], st);
  if (!P.fresh && P.n_scen > 0) {
    LT_CUDA(cudaMemcpyAsync(P.scen_count.p, P.base_count.p, P.n_scen * sizeof(unsigned long long),
                            cudaMemcpyDeviceToDevice, st));
    if (P.n_pairs > 0) {
      launch_count(P, st);
      ++launches;
    }
    size_t tb = P.scan_tmp_bytes;
    LT_CUDA(cub::DeviceScan::ExclusiveSum(P.scan_tmp.p, tb, P.scen_count.p, P.scen_off.p,
                                          static_cast<int>(P.n_scen), st));
    set_offsets_kernel<<<static_cast<unsigned>((P.n_scen + 255) / 256), 256, 0, st>>>(
        P.scen.p, static_cast<int>(P.n_scen), P.scen_count.p, P.scen_off.p);
    after_launch("set_offsets_kernel", st);
    launches += 2;
  }
  cudaEventRecord(P.ev[2], st);
  launches += merge_requests(P);
  cudaEventRecord(P.ev[3], st);
  P.fresh = false;
  P.launches_run = launches + 2 + (P.engine_variant == kEngineLatency);  // + (links), engine, metrics
}

// Arrival merge of the counted streams: per-pair times (expand), stable sort
// by time per scenario, gather into the request arrays. Returns own launches.
int64_t merge_requests(lt_plan& P, bool sized) {
  cudaStream_t st = P.st;
  int64_t launches = 0;
  if (P.n_pairs > 0) {
    // sort-based merge: unsorted times per (scenario, adapter), stable
    // segmented sort by time, gather into request arrays
    size_t tb = P.pscan_tmp_bytes;
    LT_CUDA(cub::DeviceScan::ExclusiveSum(P.pscan_tmp.p, tb, P.adp_count.p, P.pair_excl.p,
                                          static_cast<int>(P.n_pairs), st));
    launch_expand(P, st);
    size_t sb = P.sort_tmp_bytes;
    const int nr = static_cast<int>(std::max<int64_t>(P.total_req, 1));
    const unsigned gr = static_cast<unsigned>((nr + 255) / 256);
    const int32_t* perm = nullptr;
    if (P.pos_a.p) {  // two global stable radix sorts (see scen_key_kernel)
      iota_kernel<<<gr, 256, 0, st>>>(P.pos_a.p, nr);
      after_launch("iota_kernel", st);
      LT_CUDA(cub::DeviceRadixSort::SortPairs(P.sort_tmp.p, sb, P.st_in.p, P.st_out.p, P.pos_a.p, P.pos_b.p, nr, 0,
                                              64, st));
      scen_key_kernel<<<gr, 256, 0, st>>>(P.scen.p, static_cast<int>(P.n_scen), nr, P.pos_b.p, P.skey_a.p);
      after_launch("scen_key_kernel", st);
      sb = P.sort_tmp_bytes;
      LT_CUDA(cub::DeviceRadixSort::SortPairs(P.sort_tmp.p, sb, P.skey_a.p, P.skey_b.p, P.pos_b.p, P.pos_a.p, nr, 0,
                                              P.scen_bits, st));
      perm = P.pos_a.p;
      launches += 2;  // iota, scen_key
    } else if (merge_mode() == 2) {  // the per-scenario stable segmented sort (CUB)
      segments_kernel<<<static_cast<unsigned>((P.n_scen + 255) / 256), 256, 0, st>>>(
          P.scen.p, static_cast<int>(P.n_scen), P.seg_begin.p, P.seg_end.p);
      after_launch("segments_kernel", st);
      LT_CUDA(cub::DeviceSegmentedSort::StableSortPairs(P.sort_tmp.p, sb, P.st_in.p, P.st_out.p, P.sv_in.p,
                                                        P.sv_out.p, nr, static_cast<int>(P.n_scen), P.seg_begin.p,
                                                        P.seg_end.p, st));
      launches += 1;  // segments
    } else {  // merge tree of the per-adapter lists, one block per scenario
      // A sized latency-bound plan merges in its cost order (on the device
      // by now): the longest merges start in the first wave of blocks (C2
      // -0.08 ms; throughput plans measured +0.1 ms with it and keep theirs)
      const int32_t* order = sized && P.engine_variant == kEngineLatency && P.order.n == static_cast<size_t>(P.n_scen)
                                 ? P.order.p
                                 : nullptr;
      merge_kernel<<<static_cast<unsigned>(P.n_scen), 512, 0, st>>>(P.scen.p, P.pair_begin.p, P.pair_excl.p,
                                                                    P.st_in.p, P.sv_in.p, P.st_out.p, P.sv_out.p,
                                                                    order);
      after_launch("merge_kernel", st);
      launches += 1;
    }
    gather_kernel<<<gr, 256, 0, st>>>(P.scen.p, static_cast<int>(P.n_scen), P.total_req, P.adapters.p, P.keys.p,
                                      P.lens.p, P.Z.p, perm ? P.st_in.p : P.st_out.p, perm ? P.sv_in.p : P.sv_out.p,
                                      P.r_arr.p, P.r_in.p, P.r_out.p, P.r_adp.p, P.decks.p, P.deck_tab.p, P.full.p,
                                      perm);
    after_launch("gather_kernel", st);
    launches += 2;  // expand, gather (own kernels; CUB's scan and sorts not counted)
  }
  return launches;
}

// The report / checked engine build (engine_kernel<256,1,true>) on the plan's
// warp layout, at most 8 warps per block.
// The fresh-queue chain links of the plan's requests (link_kernel), before
// each pass of a linked engine build (latency, report, recording).
void launch_links(lt_plan& P, cudaStream_t st) {
  if (P.n_scen <= 0 || P.total_req <= 0) return;
  P.r_link.alloc(P.total_req);  // (on first use: the throughput builds never read it)
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((P.n_scen + 7) / 8, int64_t(P.ctx->sm_count) * 8));
  link_launch(grid, 8 * P.max_adapters * sizeof(int32_t), st, P.scen.p, static_cast<int>(P.n_scen), P.max_adapters,
              P.r_in.p, P.r_adp.p, P.r_link.p);
  after_launch("link_kernel", st);
}

void launch_engine_checked(lt_plan& P, const EngineParams& E, cudaStream_t st, int build = kEngineChecked) {
  launch_links(P, st);
  const int warps = std::min(P.block / 32, 8);
  LT_CUDA(cudaFuncSetAttribute(engine_kernel_fn(build), cudaFuncAttributeMaxDynamicSharedMemorySize,
                               P.ctx->smem_optin));
  EngineParams EL = E;
  EL.r_link = P.r_link.p;
  launch_engine_build(build, static_cast<unsigned>(P.grid), static_cast<unsigned>(warps * 32),
                      static_cast<size_t>(P.smem_per_warp) * warps, st, EL);
}

// K1 (the engine kernel) then K2 (metrics_kernel) over the plan's scenarios.
void launch_engine(lt_plan& P, const EngineParams& E, cudaStream_t st) {
  if (E.check_invariants) {
    launch_engine_checked(P, E, st);
  } else {
    EngineParams EL = E;
    if (P.engine_variant == kEngineLatency) {  // (the throughput builds append at ingest)
      launch_links(P, st);
      EL.r_link = P.r_link.p;
    }
    launch_engine_build(P.engine_variant, static_cast<unsigned>(P.grid), static_cast<unsigned>(P.block), P.smem, st,
                        EL);
  }
  after_launch("engine_kernel", st);
  metrics_kernel<<<static_cast<unsigned>((P.n_scen + 7) / 8), 256, 0, st>>>(
      E.scen, E.n_scen, E.r_phase, E.r_first, E.r_arr, E.r_last, E.r_out, E.r_gen, E.out);
}

// Per-request engine state before an engine pass.
void reset_state(lt_plan& P) {
  cudaStream_t st = P.st;
  const int64_t nr = std::max<int64_t>(P.total_req, 1);
  LT_CUDA(cudaMemsetAsync(P.r_phase.p, 0, nr, st));
  LT_CUDA(cudaMemsetAsync(P.r_gen.p, 0, nr * sizeof(int32_t), st));
  LT_CUDA(cudaMemsetAsync(P.r_pre.p, 0, nr * sizeof(int32_t), st));
  LT_CUDA(cudaMemsetAsync(P.r_first.p, 0xff, nr * sizeof(double), st));  // NaN: no first token
  LT_CUDA(cudaMemsetAsync(P.r_last.p, 0, nr * sizeof(double), st));
  LT_CUDA(cudaMemsetAsync(P.counter.p, 0, sizeof(int32_t), st));
}

// Kernel parameters of a plan's engine pass.
EngineParams engine_params(const lt_plan& P) {
  EngineParams E{};
  E.scen = P.scen.p;
  E.order = P.order.p;
  E.n_scen = static_cast<int32_t>(P.n_scen);
  E.max_adapters = P.max_adapters;
  E.run_cap = P.run_cap;
  E.smem_per_warp = P.smem_per_warp;
  E.counter = P.counter.p;
  E.adapters = P.adapters.p;
  E.r_arr = P.r_arr.p;
  E.r_in = P.r_in.p;
  E.r_out = P.r_out.p;
  E.r_adp = P.r_adp.p;
  E.r_phase = P.r_phase.p;
  E.r_gen = P.r_gen.p;
  E.r_first = P.r_first.p;
  E.r_last = P.r_last.p;
  E.r_pre = P.r_pre.p;
  E.ws_run = P.ws_run.p;
  E.ws_pq = P.ws_pq.p;
  E.ws_node = P.ws_node.p;
  E.ws_link = P.ws_link.p;
  E.ws_ov = P.ws_ov.p;
  E.ws_stride = P.ws_stride;
  E.ws_per_scenario = P.ws_per_scenario;
  E.k1 = P.cfg.raw.k1;
  E.k2 = P.cfg.raw.k2;
  E.k3 = P.cfg.raw.k3;
  E.k4 = P.cfg.raw.k4;
  E.k5 = P.cfg.raw.k5;
  E.k6 = P.cfg.raw.k6;
  E.k7 = P.cfg.raw.k7;
  E.priority = P.cfg.raw.loaded_adapter_priority;
  E.want_digest = P.want_digest;
  E.out = P.out.p;
  E.check_invariants = P.want_check;
  const char* inject = std::getenv("LT_INVARIANT_INJECT");  // test hook: a ledger fault at this iteration
  E.inject_iteration = inject ? std::atoll(inject) : -1;
  return E;
}

void run_percentiles(lt_plan& P, EngineParams E);

bool run_percentiles_single(lt_plan& P);

void run_plan(lt_plan& P) {
  cudaStream_t st = P.st;
  untrim_plan(P);
  prepare_requests(P);
  // percentiles in one recording engine pass when its record pool holds
  // them (else the engine pass, then a second one sized by its counts)
  if (P.want_pct && P.n_scen > 0 && !std::getenv("LT_PCT_TWO_PASS") && run_percentiles_single(P)) return;
  reset_state(P);
  const EngineParams E = engine_params(P);
  cudaEventRecord(P.ev[4], st);
  if (P.n_scen > 0) {
    launch_engine(P, E, st);
    after_launch("metrics_kernel", st);
  }
  cudaEventRecord(P.ev[5], st);
  if (P.want_pct && P.n_scen > 0) run_percentiles(P, E);
}

// TTFT/ITL p50/p99 from one engine pass of the recording build: the ITL
// records go to a chunked pool (sized from the records per request the
// context has seen, 8 before), are compacted per scenario and sorted. False
// when the pool ran out (the caller falls back to two passes).
bool run_percentiles_single(lt_plan& P) {
  cudaStream_t st = P.st;
  lt_ctx* ctx = P.ctx;
  const int64_t n = P.n_scen, nr = std::max<int64_t>(P.total_req, 1);
  const double per_req = ctx->rec_per_req > 0.0 ? 1.25 * ctx->rec_per_req : 8.0;
  const double est = per_req * static_cast<double>(P.total_req) + static_cast<double>(n);
  const int64_t max_chunks = (int64_t(8) << 30) / (12 * kRecChunk);  // an 8 GB pool at most
  const int64_t chunks = std::min<int64_t>(max_chunks, 2 * n + static_cast<int64_t>(est / kRecChunk) + 1);
  if (chunks <= n || chunks >= (int64_t(1) << 31)) return false;
  const int64_t pool = chunks * kRecChunk;
  P.pool_d.alloc(pool);
  P.pool_c.alloc(pool);
  P.chunk_next.alloc(chunks);
  P.rec_total.alloc(std::max<int64_t>(n, 1));
  P.pool_next.alloc(2);  // {next chunk, overflow}
  LT_CUDA(cudaMemsetAsync(P.chunk_next.p, 0xff, chunks * sizeof(int32_t), st));
  LT_CUDA(cudaMemsetAsync(P.rec_total.p, 0, P.rec_total.n * sizeof(int64_t), st));
  const int32_t init[2] = {static_cast<int32_t>(n), 0};
  LT_CUDA(cudaMemcpyAsync(P.pool_next.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
  reset_state(P);
  EngineParams E = engine_params(P);
  E.rec_chunked = 1;
  E.rec_pool_chunks = static_cast<int32_t>(chunks);
  E.rec_pool_next = P.pool_next.p;
  E.rec_overflow = P.pool_next.p + 1;
  E.rec_chunk_next = P.chunk_next.p;
  E.rec_total = P.rec_total.p;
  E.rec_d = P.pool_d.p;
  E.rec_c = P.pool_c.p;
  cudaEventRecord(P.ev[4], st);
  // the recording build (no report / check code) unless invariants are checked too
  launch_engine_checked(P, E, st, E.check_invariants ? kEngineChecked : kEngineRecord);
  after_launch("engine_kernel(recording)", st);
  metrics_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, 0, st>>>(E.scen, E.n_scen, E.r_phase, E.r_first, E.r_arr,
                                                                     E.r_last, E.r_out, E.r_gen, E.out);
  after_launch("metrics_kernel", st);
  cudaEventRecord(P.ev[5], st);
  int32_t ovf = 0;
  LT_CUDA(cudaMemcpyAsync(&ovf, P.pool_next.p + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  // the records' segments: exclusive scan of the counts
  P.rec_off.alloc(std::max<int64_t>(n, 1));
  size_t sb = 0;
  LT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, sb, P.rec_total.p, P.rec_off.p, static_cast<int>(n), st));
  P.pct_tmp.alloc(static_cast<int64_t>(std::max<size_t>(sb, 1)));
  LT_CUDA(cub::DeviceScan::ExclusiveSum(P.pct_tmp.p, sb, P.rec_total.p, P.rec_off.p, static_cast<int>(n), st));
  int64_t last_off = 0, last_len = 0;
  LT_CUDA(cudaMemcpyAsync(&last_off, P.rec_off.p + n - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  LT_CUDA(cudaMemcpyAsync(&last_len, P.rec_total.p + n - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  LT_CUDA(cudaStreamSynchronize(st));
  if (ovf) return false;
  const int64_t tot = last_off + last_len;
  if (tot >= (int64_t(1) << 31)) throw CudaError{"percentiles: more than 2^31 ITL records in one plan"};
  ctx->rec_per_req = std::max(ctx->rec_per_req, static_cast<double>(tot) / static_cast<double>(nr));
  const int64_t nt = std::max<int64_t>(tot, 1);
  P.rec_d.alloc(nt);
  P.rec_c.alloc(nt);
  P.rec_d_sorted.alloc(nt);
  P.rec_c_sorted.alloc(nt);
  P.pct_rseg_b.alloc(std::max<int64_t>(n, 1));
  P.pct_rseg_e.alloc(std::max<int64_t>(n, 1));
  rec_compact_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, 0, st>>>(
      static_cast<int>(n), P.chunk_next.p, P.rec_total.p, P.rec_off.p, P.pool_d.p, P.pool_c.p, P.rec_d.p, P.rec_c.p,
      P.pct_rseg_b.p, P.pct_rseg_e.p);
  after_launch("rec_compact_kernel", st);
  std::vector<int32_t> tb(n), te(n);
  for (int64_t i = 0; i < n; ++i) {
    tb[i] = static_cast<int32_t>(P.h_scen[i].req_begin);
    te[i] = static_cast<int32_t>(P.h_scen[i].req_begin + P.h_scen[i].n_req);
  }
  P.pct_seg_b.upload(tb, st);
  P.pct_seg_e.upload(te, st);
  P.ttft_keys.alloc(nr);
  P.ttft_sorted.alloc(nr);
  ttft_keys_kernel<<<static_cast<unsigned>((nr + 255) / 256), 256, 0, st>>>(P.r_arr.p, P.r_first.p, nr,
                                                                            P.ttft_keys.p);
  after_launch("ttft_keys_kernel", st);
  size_t b1 = 0, b2 = 0;
  LT_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, b1, P.ttft_keys.p, P.ttft_sorted.p, static_cast<int>(nr),
                                             static_cast<int>(n), P.pct_seg_b.p, P.pct_seg_e.p, st));
  LT_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, b2, P.rec_d.p, P.rec_d_sorted.p, P.rec_c.p,
                                              P.rec_c_sorted.p, static_cast<int>(nt), static_cast<int>(n),
                                              P.pct_rseg_b.p, P.pct_rseg_e.p, st));
  P.pct_tmp.alloc(static_cast<int64_t>(std::max<size_t>(std::max(b1, b2), 1)));
  LT_CUDA(cub::DeviceSegmentedSort::SortKeys(P.pct_tmp.p, b1, P.ttft_keys.p, P.ttft_sorted.p, static_cast<int>(nr),
                                             static_cast<int>(n), P.pct_seg_b.p, P.pct_seg_e.p, st));
  LT_CUDA(cub::DeviceSegmentedSort::SortPairs(P.pct_tmp.p, b2, P.rec_d.p, P.rec_d_sorted.p, P.rec_c.p,
                                              P.rec_c_sorted.p, static_cast<int>(nt), static_cast<int>(n),
                                              P.pct_rseg_b.p, P.pct_rseg_e.p, st));
  percentile_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, 0, st>>>(
      P.scen.p, static_cast<int>(n), P.ttft_sorted.p, P.rec_off.p, P.rec_total.p, P.rec_d_sorted.p,
      P.rec_c_sorted.p, P.out.p);
  after_launch("percentile_kernel", st);
  P.launches_run += 6;  // links, the recording engine, compaction, ttft keys, percentiles (metrics counted by the caller)
  return true;
}

// TTFT/ITL p50/p99 (metrics.cpp:47-54): a second, recording engine pass sized
// by the first pass's iteration and preemption counts, then segmented sorts
// and a weighted rank select (k_metrics.cuh).
void run_percentiles(lt_plan& P, EngineParams E) {
  cudaStream_t st = P.st;
  const int64_t n = P.n_scen;
  std::vector<lt_sim_summary> h(n);
  LT_CUDA(cudaMemcpyAsync(h.data(), P.out.p, n * sizeof(lt_sim_summary), cudaMemcpyDeviceToHost, st));
  LT_CUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> off(n), len(n);
  std::vector<int32_t> rb(n), re(n), tb(n), te(n);
  int64_t tot = 0;
  for (int64_t i = 0; i < n; ++i) {
    len[i] = (h[i].status == LT_OK) ? h[i].iterations + h[i].preemptions : 0;
    off[i] = tot;
    tot += len[i];
    tb[i] = static_cast<int32_t>(P.h_scen[i].req_begin);
    te[i] = static_cast<int32_t>(P.h_scen[i].req_begin + P.h_scen[i].n_req);
  }
  if (tot >= (int64_t(1) << 31)) throw CudaError{"percentiles: more than 2^31 ITL records in one plan"};
  for (int64_t i = 0; i < n; ++i) {
    rb[i] = static_cast<int32_t>(off[i]);
    re[i] = static_cast<int32_t>(off[i] + len[i]);
  }
  const int64_t nt = std::max<int64_t>(tot, 1), nr = std::max<int64_t>(P.total_req, 1);
  P.rec_off.upload(off, st);
  P.rec_len.upload(len, st);
  P.pct_rseg_b.upload(rb, st);
  P.pct_rseg_e.upload(re, st);
  P.pct_seg_b.upload(tb, st);
  P.pct_seg_e.upload(te, st);
  P.rec_d.alloc(nt);
  P.rec_c.alloc(nt);
  P.rec_d_sorted.alloc(nt);
  P.rec_c_sorted.alloc(nt);
  P.ttft_keys.alloc(nr);
  P.ttft_sorted.alloc(nr);
  LT_CUDA(cudaMemsetAsync(P.rec_c.p, 0, nt * sizeof(int32_t), st));
  reset_state(P);
  E.record = 1;
  E.rec_off = P.rec_off.p;
  E.rec_d = P.rec_d.p;
  E.rec_c = P.rec_c.p;
  launch_engine(P, E, st);
  after_launch("metrics_kernel(record)", st);
  ttft_keys_kernel<<<static_cast<unsigned>((nr + 255) / 256), 256, 0, st>>>(P.r_arr.p, P.r_first.p, nr,
                                                                            P.ttft_keys.p);
  after_launch("ttft_keys_kernel", st);
  size_t b1 = 0, b2 = 0;
  LT_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, b1, P.ttft_keys.p, P.ttft_sorted.p, static_cast<int>(nr),
                                             static_cast<int>(n), P.pct_seg_b.p, P.pct_seg_e.p, st));
  LT_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, b2, P.rec_d.p, P.rec_d_sorted.p, P.rec_c.p,
                                              P.rec_c_sorted.p, static_cast<int>(nt), static_cast<int>(n),
                                              P.pct_rseg_b.p, P.pct_rseg_e.p, st));
  P.pct_tmp.alloc(static_cast<int64_t>(std::max<size_t>(std::max(b1, b2), 1)));
  LT_CUDA(cub::DeviceSegmentedSort::SortKeys(P.pct_tmp.p, b1, P.ttft_keys.p, P.ttft_sorted.p, static_cast<int>(nr),
                                             static_cast<int>(n), P.pct_seg_b.p, P.pct_seg_e.p, st));
  LT_CUDA(cub::DeviceSegmentedSort::SortPairs(P.pct_tmp.p, b2, P.rec_d.p, P.rec_d_sorted.p, P.rec_c.p,
                                              P.rec_c_sorted.p, static_cast<int>(nt), static_cast<int>(n),
                                              P.pct_rseg_b.p, P.pct_rseg_e.p, st));
  percentile_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, 0, st>>>(
      P.scen.p, static_cast<int>(n), P.ttft_sorted.p, P.rec_off.p, P.rec_len.p, P.rec_d_sorted.p,
      P.rec_c_sorted.p, P.out.p);
  after_launch("percentile_kernel", st);
  P.launches_run += 6;  // links + engine + metrics (recording pass), ttft keys, percentiles
}

// lt_simulate_report's second engine pass (engine_kernel<256, 1, true>),
// sized by the first pass's counts, and the emit-time expansion
// (k_report.cuh). The rows stay on the device in R until copied out.
struct ReportRun {
  std::vector<int64_t> tr_off, ld_off, ld_len;
  int64_t n_tr = 0, n_ld = 0, n_log = 0, n_emit = 0;
  DBuf<int64_t> d_tr_off, d_ld_off, d_sl_off, tokens, emit_off;
  DBuf<double> tr_time, tr_lat, emit;
  DBuf<int4> tr_rwal;
  DBuf<lt_trace_row> trace;
  DBuf<DLoadEvent> ld;
  DBuf<int2> sl_log;
  DBuf<int32_t> sl_cnt, iters, iters_sorted;
  DBuf<uint32_t> keys, keys_sorted;
  DBuf<char> tmp;
};

void run_report(lt_plan& P, ReportRun& R) {
  cudaStream_t st = P.st;
  const int64_t n = P.n_scen;
  const int64_t nr = std::max<int64_t>(P.total_req, 1);
  std::vector<lt_sim_summary> h(n);
  LT_CUDA(cudaMemcpyAsync(h.data(), P.out.p, n * sizeof(lt_sim_summary), cudaMemcpyDeviceToHost, st));
  LT_CUDA(cudaStreamSynchronize(st));
  // rows per scenario: a trace row per iteration, the load events, and at
  // most one stint-log entry per first admission, re-admission and
  // preemption. A scenario that fails in the engine still writes the rows of
  // its completed iterations, plus the loads of the failing call (<= N).
  R.tr_off.resize(n);
  R.ld_off.resize(n);
  R.ld_len.resize(n);
  std::vector<int64_t> sl_off(n);
  int64_t n_sl = 0;
  for (int64_t i = 0; i < n; ++i) {
    R.tr_off[i] = R.n_tr;
    R.ld_off[i] = R.n_ld;
    sl_off[i] = n_sl;
    R.ld_len[i] = h[i].load_events;
    R.n_tr += h[i].iterations;
    R.n_ld += h[i].load_events + (h[i].status != LT_OK ? h[i].served_adapters : 0);
    n_sl += P.h_scen[i].n_req + 2 * h[i].preemptions;
  }
  if (n_sl >= (int64_t(1) << 31) || P.total_req >= (int64_t(1) << 32) - 1)
    throw CudaError{"lt_simulate_report: batch too large for one report (2^31 stint entries)"};
  R.n_log = n_sl;
  R.d_tr_off.upload(R.tr_off, st);
  R.d_ld_off.upload(R.ld_off, st);
  R.d_sl_off.upload(sl_off, st);
  R.tr_time.alloc(std::max<int64_t>(R.n_tr, 1));
  R.tr_lat.alloc(std::max<int64_t>(R.n_tr, 1));
  R.tr_rwal.alloc(std::max<int64_t>(R.n_tr, 1));
  R.ld.alloc(std::max<int64_t>(R.n_ld, 1));
  R.sl_log.alloc(std::max<int64_t>(n_sl, 1));
  R.sl_cnt.alloc(std::max<int64_t>(n, 1));
  LT_CUDA(cudaMemsetAsync(R.sl_cnt.p, 0, R.sl_cnt.n * sizeof(int32_t), st));
  reset_state(P);
  EngineParams E = engine_params(P);
  E.tr_off = R.d_tr_off.p;
  E.tr_time = R.tr_time.p;
  E.tr_lat = R.tr_lat.p;
  E.tr_rwal = R.tr_rwal.p;
  E.ld_off = R.d_ld_off.p;
  E.ld = R.ld.p;
  E.sl_off = R.d_sl_off.p;
  E.sl_log = R.sl_log.p;
  E.sl_cnt = R.sl_cnt.p;
  E.report = 1;
  launch_engine_checked(P, E, st);
  after_launch("engine_kernel(report)", st);
  metrics_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, 0, st>>>(E.scen, E.n_scen, E.r_phase, E.r_first, E.r_arr,
                                                                     E.r_last, E.r_out, E.r_gen, E.out);
  after_launch("metrics_kernel(report)", st);
  // trace rows as lt_trace_row
  R.trace.alloc(std::max<int64_t>(R.n_tr, 1));
  if (R.n_tr > 0) {
    trace_pack_kernel<<<static_cast<unsigned>((R.n_tr + 255) / 256), 256, 0, st>>>(
        R.d_tr_off.p, static_cast<int>(n), R.n_tr, R.tr_time.p, R.tr_lat.p, R.tr_rwal.p, R.trace.p);
    after_launch("trace_pack_kernel", st);
  }
  // emit times: stint log grouped by request (stable), then expanded
  R.keys.alloc(std::max<int64_t>(n_sl, 1));
  R.keys_sorted.alloc(std::max<int64_t>(n_sl, 1));
  R.iters.alloc(std::max<int64_t>(n_sl, 1));
  R.iters_sorted.alloc(std::max<int64_t>(n_sl, 1));
  LT_CUDA(cudaMemsetAsync(R.keys.p, 0xff, R.keys.n * sizeof(uint32_t), st));
  stint_keys_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, 0, st>>>(P.scen.p, static_cast<int>(n), R.d_sl_off.p,
                                                                        R.sl_cnt.p, R.sl_log.p, R.keys.p, R.iters.p);
  after_launch("stint_keys_kernel", st);
  R.tokens.alloc(nr);
  R.emit_off.alloc(nr);
  request_tokens_kernel<<<static_cast<unsigned>((nr + 255) / 256), 256, 0, st>>>(
      P.scen.p, static_cast<int>(n), P.out.p, P.r_phase.p, P.r_gen.p, P.r_out.p, P.total_req, R.tokens.p);
  after_launch("request_tokens_kernel", st);
  size_t b1 = 0, b2 = 0;
  LT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b1, R.keys.p, R.keys_sorted.p, R.iters.p, R.iters_sorted.p,
                                          static_cast<int>(std::max<int64_t>(n_sl, 1)), 0, 32, st));
  LT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b2, R.tokens.p, R.emit_off.p, static_cast<int>(nr), st));
  R.tmp.alloc(std::max<size_t>(std::max(b1, b2), 1));
  LT_CUDA(cub::DeviceRadixSort::SortPairs(R.tmp.p, b1, R.keys.p, R.keys_sorted.p, R.iters.p, R.iters_sorted.p,
                                          static_cast<int>(std::max<int64_t>(n_sl, 1)), 0, 32, st));
  LT_CUDA(cub::DeviceScan::ExclusiveSum(R.tmp.p, b2, R.tokens.p, R.emit_off.p, static_cast<int>(nr), st));
  int64_t last_off = 0, last_tok = 0;
  if (P.total_req > 0) {
    LT_CUDA(cudaMemcpyAsync(&last_off, R.emit_off.p + P.total_req - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaMemcpyAsync(&last_tok, R.tokens.p + P.total_req - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  }
  LT_CUDA(cudaStreamSynchronize(st));
  R.n_emit = last_off + last_tok;
  R.emit.alloc(std::max<int64_t>(R.n_emit, 1));
  if (P.total_req > 0) {
    emit_times_kernel<<<static_cast<unsigned>((P.total_req + 255) / 256), 256, 0, st>>>(
        P.scen.p, static_cast<int>(n), P.total_req, R.keys_sorted.p, R.iters_sorted.p, n_sl, R.tokens.p,
        R.emit_off.p, R.d_tr_off.p, R.tr_time.p, R.tr_lat.p, R.emit.p);
    after_launch("emit_times_kernel", st);
  }
  P.launches_run += 8;  // (with the chain links)
}

void fetch_results(lt_plan& P, lt_sim_summary* out, lt_request_states* states) {
  lt_ctx* ctx = P.ctx;
  cudaStream_t st = P.st;
  if (P.n_scen > 0)
    LT_CUDA(cudaMemcpyAsync(out, P.out.p, P.n_scen * sizeof(lt_sim_summary), cudaMemcpyDeviceToHost, st));
  int64_t d2h = P.n_scen * sizeof(lt_sim_summary);
  std::vector<int8_t> phase;
  std::vector<int32_t> gen, pre, in, outv, adp;
  std::vector<double> first, last, arr;
  if (states && P.trimmed) throw CudaError{"lt_plan_results: per-request states were released by lt_plan_trim"};
  if (states) {
    const int64_t n = P.total_req;
    phase.resize(n);
    gen.resize(n);
    pre.resize(n);
    in.resize(n);
    outv.resize(n);
    adp.resize(n);
    first.resize(n);
    last.resize(n);
    arr.resize(n);
    if (n) {
      LT_CUDA(cudaMemcpyAsync(phase.data(), P.r_phase.p, n, cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(gen.data(), P.r_gen.p, n * 4, cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(pre.data(), P.r_pre.p, n * 4, cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(in.data(), P.r_in.p, n * 4, cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(outv.data(), P.r_out.p, n * 4, cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(adp.data(), P.r_adp.p, n * 4, cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(first.data(), P.r_first.p, n * 8, cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(last.data(), P.r_last.p, n * 8, cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(arr.data(), P.r_arr.p, n * 8, cudaMemcpyDeviceToHost, st));
    }
    d2h += n * 45;
  }
  cudaEventRecord(P.ev[6], st);
  LT_CUDA(cudaStreamSynchronize(st));
  ctx->messages.assign(P.n_scen, std::string());
  for (int64_t i = 0; i < P.n_scen; ++i) {
    const HostErr& e = P.errs[i];
    if (e.code != LT_OK) {
      out[i].status = e.code;
      out[i].status_kind = e.kind;
      out[i].status_a = e.a;
      out[i].status_b = e.b;
      ctx->messages[i] = e.msg;
    } else if (out[i].status != LT_OK) {
      ctx->messages[i] = render(out[i].status, out[i].status_kind, out[i].status_a, out[i].status_b);
    }
  }
  if (states) {
    int64_t off = 0;
    for (int64_t i = 0; i < P.n_scen; ++i) {
      if (states->req_offset) states->req_offset[i] = off;
      const DScen& d = P.h_scen[i];
      for (int64_t r = 0; r < d.n_req; ++r, ++off) {
        if (off >= states->capacity) continue;
        const int64_t g = d.req_begin + r;
        const int8_t ph = phase[g];
        int32_t tg = gen[g];
        if (ph == kFinished) tg = outv[g];
        if (states->phase) states->phase[off] = ph;
        if (states->tokens_generated) states->tokens_generated[off] = tg;
        if (states->first_token_time_s) states->first_token_time_s[off] = first[g];
        if (states->completion_time_s)
          states->completion_time_s[off] =
              (ph == kFinished || (ph == kRunning && tg == outv[g])) ? last[g] : 0.0;
        if (states->preemption_count) states->preemption_count[off] = pre[g];
        if (states->adapter_id) states->adapter_id[off] = P.adapter_ids[d.adapter_begin + adp[g]];
        if (states->input_tokens) states->input_tokens[off] = in[g];
        if (states->output_tokens) states->output_tokens[off] = outv[g];
        if (states->arrival_time_s) states->arrival_time_s[off] = arr[g];
      }
    }
  }
  lt_timing& t = ctx->timing;
  t.tables_ms = P.run_fresh ? P.tables_ms : elapsed(P.ev[0], P.ev[1]);
  t.merge_ms = elapsed(P.ev[1], P.ev[3]);
  t.engine_ms = elapsed(P.ev[4], P.ev[5]);
  t.d2h_ms = elapsed(P.ev[5], P.ev[6]);
  t.run_ms = elapsed(P.ev[0], P.ev[5]);
  t.d2h_bytes = d2h;
  t.h2d_bytes = P.h2d_bytes;
  t.engine_launches = P.launches_run;
  int64_t bytes = 0;
  for (int64_t i = 0; i < P.n_scen; ++i) {
    const lt_sim_summary& o = out[i];
    bytes += 20 * o.sum_running + 16 * o.sum_visited + 24 * o.sum_arrivals + 16 * o.sum_moves + 64 * o.iterations;
  }
  t.algorithmic_bytes = bytes;
}

int32_t first_error(lt_ctx* ctx, const lt_sim_summary* out, int64_t n, lt_status* st) {
  for (int64_t i = 0; i < n; ++i) {
    if (out[i].status != LT_OK) {
      set_status(st, out[i].status, out[i].status_kind, i, out[i].status_a, out[i].status_b,
                 ctx->messages[i]);
      return out[i].status;
    }
  }
  return LT_OK;
}

// Requests a scenario can generate: the Poisson mean of every adapter plus
// 8 sigma and slack (the same bound that sizes the RNG tables), or the
// scripted list.
double est_requests(const lt_workload_batch* b, int64_t i) {
  const lt_scenario& s = b->scenarios[i];
  if (s.n_requests >= 0) return static_cast<double>(s.n_requests);
  double e = 0.0;
  for (int32_t k = 0; k < s.n_adapters; ++k) {
    const double lam = std::max(b->adapters[s.adapter_offset + k].rate, 0.0) * std::max(s.duration_s, 0.0);
    e += lam + 8.0 * std::sqrt(lam) + 32.0;
  }
  return e;
}

}  // namespace
