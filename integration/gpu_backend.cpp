// See gpu_backend.hpp. Converts the reference's types to the POD mirrors of
// include/loratwin_gpu.h, calls one batched entry point and rebuilds the
// reference's results, or rethrows the reference's own exception type with
// the library's verbatim what() text (errors.hpp:25-54).
#include "gpu_backend.hpp"

#include <cmath>
#include <memory>
#include <string>

#include "loratwin/errors.hpp"
#include "loratwin_gpu.h"

namespace loratwin::gpu {
namespace {

[[noreturn]] void rethrow(const lt_status& st) {
  switch (st.code) {
    case LT_ERR_VALIDATION: throw ValidationError(st.message);
    case LT_ERR_CONFIG: throw ConfigError(st.message);
    case LT_ERR_SIMULATION: throw SimulationError(st.message);
    default: throw InternalError(st.message);
  }
}

std::uint64_t g_mask = 1;

struct Ctx {  // one per host thread (the library's contexts are not shared)
  lt_ctx* p = nullptr;
  Ctx() {
    lt_status st{};
    p = lt_create_mask(g_mask, &st);
    if (!p) rethrow(st);
  }
  ~Ctx() { lt_destroy(p); }
};

lt_ctx* ctx() {
  thread_local std::unique_ptr<Ctx> c;
  if (!c) c = std::make_unique<Ctx>();
  return c->p;
}

// ServerConfig (server_config.hpp:26-43) -> lt_server_config; the tables are
// flattened into vectors kept alive for the call.
struct PackedConfig {
  lt_server_config c{};
  std::vector<int32_t> cost_rank, load_rank;
  std::vector<int64_t> cost_tokens;
  std::vector<double> load_seconds;
  explicit PackedConfig(const ServerConfig& s) {
    c.slots = s.slots;
    c.loaded_adapter_priority = s.loaded_adapter_priority;
    c.iteration_cap = s.iteration_cap;
    c.ideal_includes_input = s.ideal_includes_input;
    c.load_source = s.load.default_source == LoadSource::Disk ? LT_SOURCE_DISK : LT_SOURCE_CPU;
    const LatencyCoefficients& k = s.latency;
    c.k1 = k.k1;
    c.k2 = k.k2;
    c.k3 = k.k3;
    c.k4 = k.k4;
    c.k5 = k.k5;
    c.k6 = k.k6;
    c.k7 = k.k7;
    c.total_kv_budget = s.memory.total_kv_budget;
    c.kv_bytes_per_token = s.memory.kv_bytes_per_token;
    if (s.memory.slot_cost_base_rank8) {
      c.has_slot_cost_base_rank8 = 1;
      c.slot_cost_base_rank8 = *s.memory.slot_cost_base_rank8;
    }
    for (const auto& [r, t] : s.memory.slot_cost_table) {
      cost_rank.push_back(r);
      cost_tokens.push_back(t);
    }
    for (const auto& [r, x] : s.load.cpu_load_seconds) {
      load_rank.push_back(r);
      load_seconds.push_back(x);
    }
    c.n_slot_cost = static_cast<int32_t>(cost_rank.size());
    c.slot_cost_rank = cost_rank.data();
    c.slot_cost_tokens = cost_tokens.data();
    c.n_load = static_cast<int32_t>(load_rank.size());
    c.load_rank = load_rank.data();
    c.load_seconds = load_seconds.data();
    c.disk_multiplier = s.load.disk_multiplier;
  }
};

// LengthSpecs and Full-mode pairs of a batch.
struct PackedLengths {
  std::vector<lt_length_spec> specs;
  std::vector<int32_t> pairs;
  int32_t add(const LengthSpec& l) {
    lt_length_spec p{};
    p.mode = l.mode == LengthMode::Full ? LT_MODE_FULL : LT_MODE_MEAN;
    p.mean_input = l.mean_input;
    p.std_input = l.std_input;
    p.mean_output = l.mean_output;
    p.std_output = l.std_output;
    p.full_offset = static_cast<int64_t>(pairs.size() / 2);
    p.full_count = static_cast<int64_t>(l.full_lengths.size());
    for (const auto& [in, out] : l.full_lengths) {
      pairs.push_back(in);
      pairs.push_back(out);
    }
    specs.push_back(p);
    return static_cast<int32_t>(specs.size() - 1);
  }
};

Phase phase_of(int8_t p) {
  switch (p) {
    case 1: return Phase::Running;
    case 2: return Phase::Preempted;
    case 3: return Phase::Finished;
    case 4: return Phase::Rejected;
    default: return Phase::Waiting;
  }
}

// One scenario through lt_simulate_report: the full SimulationResult.
SimulationResult simulate_one(const WorkloadSpec& w, const std::vector<Request>* scripted, LengthMode mode,
                              const ServerConfig& config, const SimOptions& options, MetricsSummary* metrics) {
  PackedConfig pc(config);
  PackedLengths pl;
  std::vector<lt_adapter> ads;
  const int32_t wl = pl.add(w.lengths);
  for (const AdapterSpec& a : w.adapters)
    ads.push_back({a.adapter_id, a.rank, a.rate, a.lengths ? pl.add(*a.lengths) : -1, 0});
  std::vector<lt_request> reqs;
  if (scripted)
    for (const Request& r : *scripted)
      reqs.push_back({r.request_id, r.adapter_id, r.input_tokens, r.output_tokens, 0, r.arrival_time_s});
  lt_scenario sc{};
  sc.adapter_offset = 0;
  sc.n_adapters = static_cast<int32_t>(ads.size());
  sc.length_index = wl;
  sc.duration_s = w.duration_s;
  sc.seed = w.seed;
  sc.slots = 0;
  sc.mode = mode == LengthMode::Full ? LT_MODE_FULL : LT_MODE_MEAN;
  sc.request_offset = 0;
  sc.n_requests = scripted ? static_cast<int64_t>(reqs.size()) : -1;
  lt_workload_batch b{&sc, 1, ads.data(), static_cast<int64_t>(ads.size()), pl.specs.data(),
                      static_cast<int64_t>(pl.specs.size()), pl.pairs.data(),
                      static_cast<int64_t>(pl.pairs.size() / 2), reqs.data(), static_cast<int64_t>(reqs.size())};
  lt_sim_options so{};
  so.check_invariants = options.check_invariants;
  so.iteration_cap_override = options.iteration_cap_override ? std::max<int64_t>(*options.iteration_cap_override, 1) : 0;
  so.libm_variant = -1;
  so.want_percentiles = 1;
  lt_status st{};
  // first call: the counts that size the report buffers
  lt_sim_summary s{};
  if (lt_simulate_batch(ctx(), &b, &pc.c, &so, &s, nullptr, &st) != LT_OK) rethrow(st);
  const int64_t nr = s.n_requests;
  std::vector<int64_t> roff(1);
  std::vector<int8_t> phase(nr);
  std::vector<int32_t> gen(nr), pre(nr), adp(nr), in(nr), outv(nr);
  std::vector<double> first(nr), last(nr), arr(nr);
  lt_request_states rs{nr,         roff.data(), phase.data(), gen.data(), first.data(), last.data(),
                       pre.data(), adp.data(),  in.data(),    outv.data(), arr.data()};
  std::vector<lt_trace_row> trace(s.iterations);
  std::vector<lt_load_event> loads(s.load_events);
  std::vector<double> emit(s.tokens_total);
  int64_t toff = 0, loff = 0;
  std::vector<int64_t> eoff(nr);
  lt_report rep{trace.data(), s.iterations, &toff, loads.data(), s.load_events, &loff,
                emit.data(),  s.tokens_total, eoff.data()};
  if (lt_simulate_report(ctx(), &b, &pc.c, &so, &s, &rs, &rep, &st) != LT_OK) rethrow(st);
  SimulationResult r;
  r.iterations = s.iterations;
  r.final_clock_s = s.final_clock_s;
  r.duration_s = s.duration_s;
  r.truncated = s.truncated;
  r.slots = s.slots;
  r.served_adapters = s.served_adapters;
  r.kv_capacity_tokens = s.kv_capacity_tokens;
  r.requests.resize(nr);
  for (int64_t j = 0; j < nr; ++j) {
    RequestState& q = r.requests[j];
    q.request.request_id = j;
    q.request.adapter_id = adp[j];
    q.request.arrival_time_s = arr[j];
    q.request.input_tokens = in[j];
    q.request.output_tokens = outv[j];
    q.phase = phase_of(phase[j]);
    q.tokens_generated = gen[j];
    if (!std::isnan(first[j])) q.first_token_time_s = first[j];
    q.completion_time_s = last[j];
    q.preemption_count = pre[j];
    q.token_emit_times_s.assign(emit.begin() + eoff[j], emit.begin() + eoff[j] + gen[j]);
  }
  for (const lt_load_event& e : loads)
    r.load_events.push_back(LoadEvent{e.time_s, e.adapter_id, e.rank,
                                      e.source == LT_SOURCE_DISK ? LoadSource::Disk : LoadSource::Cpu,
                                      e.latency_s});
  if (options.record_iteration_trace)
    for (const lt_trace_row& t : trace)
      r.iteration_trace.push_back(
          IterationTraceRow{t.time_s, t.iteration, t.r_running, t.r_waiting, t.a_running, t.lat_step_s, t.loads});
  if (metrics) {
    MetricsSummary& m = *metrics;
    m.throughput_tok_s = s.throughput_tok_s;
    m.itl_mean_s = s.itl_mean_s;
    m.itl_p50_s = s.itl_p50_s;
    m.itl_p99_s = s.itl_p99_s;
    m.ttft_mean_s = s.ttft_mean_s;
    m.ttft_p50_s = s.ttft_p50_s;
    m.ttft_p99_s = s.ttft_p99_s;
    m.ideal_throughput_tok_s = s.ideal_throughput_tok_s;
    m.starved = s.starved;
    m.finished_count = s.finished_count;
    m.rejected_count = s.rejected_count;
    m.degenerate = s.degenerate;
  }
  return r;
}

}  // namespace

void set_device_mask(std::uint64_t mask) { g_mask = mask ? mask : 1; }

SimulationResult run_simulation(const WorkloadSpec& workload, const ServerConfig& config, LengthMode mode,
                                const SimOptions& options, MetricsSummary* metrics) {
  return simulate_one(workload, nullptr, mode, config, options, metrics);
}

SimulationResult run_scripted(const std::vector<Request>& requests, const std::vector<AdapterSpec>& adapters,
                              double duration_s, const ServerConfig& config, const SimOptions& options,
                              MetricsSummary* metrics) {
  WorkloadSpec w;
  w.adapters = adapters;
  w.duration_s = duration_s;
  w.lengths = LengthSpec::mean(1.0, 0.0, 1.0, 0.0);  // unused by scripted runs
  return simulate_one(w, &requests, LengthMode::Mean, config, options, metrics);
}

std::vector<PlacementResult> sweep_optimal_batch(const std::vector<Condition>& conds, const ServerConfig& config,
                                                 const SweepGrid& grid, double duration_s, std::uint64_t seed,
                                                 const SweepOptions& opt) {
  PackedConfig pc(config);
  PackedLengths pl;
  std::vector<lt_condition> lc;
  std::vector<lt_template> tm;
  for (const Condition& c : conds) {
    lc.push_back({static_cast<int64_t>(tm.size()), static_cast<int32_t>(c.mix.size()), pl.add(c.lengths)});
    for (const AdapterTemplate& t : c.mix) tm.push_back({t.rank, 0, t.rate});
  }
  lt_condition_batch b{lc.data(),        static_cast<int64_t>(lc.size()),       tm.data(),
                       static_cast<int64_t>(tm.size()), pl.specs.data(), static_cast<int64_t>(pl.specs.size()),
                       pl.pairs.data(),   static_cast<int64_t>(pl.pairs.size() / 2)};
  lt_sweep_grid g{grid.n_values.data(), static_cast<int32_t>(grid.n_values.size()),
                  grid.g_mode == SweepGrid::GMode::Explicit ? LT_G_EXPLICIT : LT_G_GEOMETRIC,
                  grid.g_values.data(), static_cast<int32_t>(grid.g_values.size()), 0};
  lt_sweep_options o{opt.early_exit, opt.early_exit_k, opt.jobs,
                     opt.mode == LengthMode::Full ? LT_MODE_FULL : LT_MODE_MEAN};
  const int32_t F = lt_sweep_frontier_capacity(&g);
  std::vector<lt_placement> out(conds.size());
  std::vector<lt_frontier_point> fr(conds.size() * F);
  lt_status st{};
  if (lt_sweep_batch(ctx(), &b, &pc.c, &g, duration_s, seed, &o, nullptr, out.data(), fr.data(), F, &st) != LT_OK)
    rethrow(st);
  std::vector<PlacementResult> res(conds.size());
  for (size_t i = 0; i < conds.size(); ++i) {
    res[i].n_star = out[i].n_star;
    res[i].g_star = out[i].g_star;
    res[i].max_throughput_tok_s = out[i].max_throughput_tok_s;
    res[i].all_starved = out[i].all_starved;
    res[i].frontier_open = out[i].frontier_open;
    for (int k = 0; k < out[i].frontier_count; ++k) {
      const lt_frontier_point& p = fr[i * F + k];
      res[i].frontier.push_back({p.n, p.g, p.throughput_tok_s, p.starved != 0, p.skipped != 0});
    }
  }
  return res;
}

}  // namespace loratwin::gpu
