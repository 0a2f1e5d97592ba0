// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// The loratwin_gpu.h C-ABI implemented on top of the UNMODIFIED reference
// (compiled from /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libloratwin_ref.so; symbols carry the `ltref_` prefix). It lets
// the parity tests and bench.py's reference arm drive the reference's own
// public API -- run_simulation / run_scripted + compute_metrics
// (engine.cpp:198-211, metrics.cpp:70-113), generate_arrivals
// (workload.cpp:170-211), sweep_optimal (placement.cpp:185-264) -- with the
// same POD inputs the GPU library takes. Parallelism follows the reference's
// run_parallel pattern (placement.cpp:65-96): an atomic work counter over a
// std::thread pool, per-task error capture.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <thread>
#include <vector>

#include "loratwin/engine.hpp"
#include "loratwin/errors.hpp"
#include "loratwin/json_io.hpp"
#include "loratwin/metrics.hpp"
#include "loratwin/placement.hpp"
#include "loratwin/workload.hpp"
#include "loratwin_gpu.h"

using namespace loratwin;

namespace {

int g_threads = 1;
std::vector<std::string> g_messages;  // per-scenario / per-condition what() of the last call

void set_status(lt_status* st, int32_t code, int64_t index, const std::string& msg) {
  if (!st) return;
  st->code = code;
  st->kind = LT_K_MESSAGE;
  st->index = index;
  st->detail_a = st->detail_b = 0;
  std::snprintf(st->message, sizeof(st->message), "%s", msg.c_str());
}

int32_t classify(const std::exception_ptr& e, std::string* msg) {
  try {
    std::rethrow_exception(e);
  } catch (const ValidationError& x) {
    *msg = x.what();
    return LT_ERR_VALIDATION;
  } catch (const ConfigError& x) {
    *msg = x.what();
    return LT_ERR_CONFIG;
  } catch (const SimulationError& x) {
    *msg = x.what();
    return LT_ERR_SIMULATION;
  } catch (const InternalError& x) {
    *msg = x.what();
    return LT_ERR_INTERNAL;
  } catch (const std::exception& x) {
    *msg = x.what();
    return LT_ERR_INTERNAL;
  }
}

void run_pool(std::size_t count, const std::function<void(std::size_t)>& task) {
  const int workers = std::max(1, std::min<int>(g_threads, static_cast<int>(count)));
  if (workers == 1) {
    for (std::size_t i = 0; i < count; ++i) task(i);
    return;
  }
  std::atomic<std::size_t> next{0};
  std::vector<std::thread> pool;
  for (int w = 0; w < workers; ++w)
    pool.emplace_back([&] {
      for (std::size_t i; (i = next.fetch_add(1)) < count;) task(i);
    });
  for (auto& t : pool) t.join();
}

ServerConfig to_config(const lt_server_config& c) {
  ServerConfig s;
  s.slots = c.slots;
  s.loaded_adapter_priority = c.loaded_adapter_priority != 0;
  s.iteration_cap = c.iteration_cap;
  s.ideal_includes_input = c.ideal_includes_input != 0;
  s.latency.k1 = c.k1;
  s.latency.k2 = c.k2;
  s.latency.k3 = c.k3;
  s.latency.k4 = c.k4;
  s.latency.k5 = c.k5;
  s.latency.k6 = c.k6;
  s.latency.k7 = c.k7;
  s.memory.total_kv_budget = c.total_kv_budget;
  s.memory.kv_bytes_per_token = c.kv_bytes_per_token;
  for (int i = 0; i < c.n_slot_cost; ++i) s.memory.slot_cost_table[c.slot_cost_rank[i]] = c.slot_cost_tokens[i];
  if (c.has_slot_cost_base_rank8) s.memory.slot_cost_base_rank8 = c.slot_cost_base_rank8;
  for (int i = 0; i < c.n_load; ++i) s.load.cpu_load_seconds[c.load_rank[i]] = c.load_seconds[i];
  s.load.disk_multiplier = c.disk_multiplier;
  s.load.default_source = c.load_source == LT_SOURCE_DISK ? LoadSource::Disk : LoadSource::Cpu;
  return s;
}

LengthSpec to_lengths(const lt_length_spec& l, const int32_t* full) {
  if (l.mode == LT_MODE_FULL) {
    std::vector<std::pair<int, int>> pairs;
    for (int64_t i = 0; i < l.full_count; ++i)
      pairs.emplace_back(full[2 * (l.full_offset + i)], full[2 * (l.full_offset + i) + 1]);
    return LengthSpec::full(std::move(pairs));
  }
  return LengthSpec::mean(l.mean_input, l.std_input, l.mean_output, l.std_output);
}

WorkloadSpec to_workload(const lt_workload_batch& b, const lt_scenario& s) {
  WorkloadSpec w;
  w.lengths = to_lengths(b.lengths[s.length_index], b.full_lengths);
  w.duration_s = s.duration_s;
  w.seed = s.seed;
  for (int32_t i = 0; i < s.n_adapters; ++i) {
    const lt_adapter& a = b.adapters[s.adapter_offset + i];
    AdapterSpec spec;
    spec.adapter_id = a.adapter_id;
    spec.rank = a.rank;
    spec.rate = a.rate;
    if (a.length_index >= 0) spec.lengths = to_lengths(b.lengths[a.length_index], b.full_lengths);
    w.adapters.push_back(spec);
  }
  return w;
}

uint64_t fold(uint64_t h, uint64_t w) {
  h ^= w;
  h *= 0x100000001b3ULL;
  return h;
}

uint64_t digest_of(const SimulationResult& r) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (const IterationTraceRow& t : r.iteration_trace) {
    uint64_t lat;
    std::memcpy(&lat, &t.lat_step_s, 8);
    h = fold(h, static_cast<uint32_t>(t.r_running) | (static_cast<uint64_t>(static_cast<uint32_t>(t.r_waiting)) << 32));
    h = fold(h, static_cast<uint32_t>(t.a_running) | (static_cast<uint64_t>(static_cast<uint32_t>(t.loads)) << 32));
    h = fold(h, lat);
  }
  return h;
}

}  // namespace

extern "C" {

void ltref_set_threads(int32_t n) { g_threads = n < 1 ? 1 : n; }
int32_t ltref_threads(void) { return g_threads; }

int32_t ltref_message(int64_t index, char* buf, size_t len) {
  if (index < 0 || static_cast<std::size_t>(index) >= g_messages.size()) return -1;
  std::snprintf(buf, len, "%s", g_messages[static_cast<std::size_t>(index)].c_str());
  return 0;
}

int32_t ltref_generate_arrivals_batch(void*, const lt_workload_batch* batch, const lt_sim_options*,
                                      lt_request* out, int64_t capacity, int64_t* offsets,
                                      int64_t* counts, lt_status* status) {
  const std::size_t n = static_cast<std::size_t>(batch->n_scenarios);
  std::vector<std::vector<Request>> lists(n);
  std::vector<std::exception_ptr> errors(n);
  g_messages.assign(n, std::string());
  run_pool(n, [&](std::size_t i) {
    try {
      const lt_scenario& s = batch->scenarios[i];
      WorkloadSpec w = to_workload(*batch, s);
      lists[i] = generate_arrivals(w, static_cast<LengthMode>(s.mode));
    } catch (...) {
      errors[i] = std::current_exception();
    }
  });
  int64_t off = 0;
  if (status) status->code = LT_OK;
  for (std::size_t i = 0; i < n; ++i) {
    offsets[i] = off;
    counts[i] = static_cast<int64_t>(lists[i].size());
    if (errors[i]) {
      std::string msg;
      const int32_t code = classify(errors[i], &msg);
      g_messages[i] = msg;
      if (status && status->code == LT_OK) set_status(status, code, static_cast<int64_t>(i), msg);
    }
    for (const Request& r : lists[i]) {
      if (off < capacity) {
        lt_request& o = out[off];
        o.request_id = r.request_id;
        o.adapter_id = r.adapter_id;
        o.input_tokens = r.input_tokens;
        o.output_tokens = r.output_tokens;
        o._pad = 0;
        o.arrival_time_s = r.arrival_time_s;
      }
      ++off;
    }
  }
  return status ? status->code : 0;
}

}  // extern "C"

namespace {

// One scenario through the reference's own run_simulation / run_scripted.
SimulationResult run_one(const lt_workload_batch* batch, std::size_t i, const ServerConfig& base,
                         const lt_sim_options* options, bool trace, WorkloadSpec* w_out, ServerConfig* cfg_out) {
  const lt_scenario& s = batch->scenarios[i];
  ServerConfig cfg = base;
  if (s.slots > 0) cfg.slots = s.slots;
  SimOptions opt;
  opt.record_iteration_trace = trace;
  opt.check_invariants = options && options->check_invariants;
  if (options && options->iteration_cap_override > 0) opt.iteration_cap_override = options->iteration_cap_override;
  WorkloadSpec w = to_workload(*batch, s);
  SimulationResult r;
  if (s.n_requests >= 0) {
    std::vector<Request> rr;
    rr.reserve(static_cast<std::size_t>(s.n_requests));
    for (int64_t k = 0; k < s.n_requests; ++k) {
      const lt_request& q = batch->requests[s.request_offset + k];
      Request x;
      x.request_id = q.request_id;
      x.adapter_id = q.adapter_id;
      x.arrival_time_s = q.arrival_time_s;
      x.input_tokens = q.input_tokens;
      x.output_tokens = q.output_tokens;
      rr.push_back(x);
    }
    r = run_scripted(rr, w.adapters, w.duration_s, cfg, opt);
  } else {
    r = run_simulation(w, cfg, static_cast<LengthMode>(s.mode), opt);
  }
  *w_out = std::move(w);
  *cfg_out = cfg;
  return r;
}

void fill_summary(const SimulationResult& r, const MetricsSummary& m, bool trace, lt_sim_summary& o) {
  o.n_requests = static_cast<int64_t>(r.requests.size());
  o.iterations = r.iterations;
  o.final_clock_s = r.final_clock_s;
  o.duration_s = r.duration_s;
  o.truncated = r.truncated;
  o.slots = r.slots;
  o.served_adapters = r.served_adapters;
  o.kv_capacity_tokens = r.kv_capacity_tokens;
  o.starved = m.starved;
  o.finished_count = m.finished_count;
  o.rejected_count = m.rejected_count;
  o.load_events = static_cast<int64_t>(r.load_events.size());
  o.throughput_tok_s = m.throughput_tok_s;
  o.ideal_throughput_tok_s = m.ideal_throughput_tok_s;
  o.ttft_mean_s = m.ttft_mean_s;
  o.itl_mean_s = m.itl_mean_s;
  o.ttft_p50_s = m.ttft_p50_s;
  o.ttft_p99_s = m.ttft_p99_s;
  o.itl_p50_s = m.itl_p50_s;
  o.itl_p99_s = m.itl_p99_s;
  o.degenerate = m.degenerate;
  // tokens_in_window without another pass over every emit time (the
  // reference already counted them: throughput = tokens / window, and the
  // integer is recovered exactly by rounding the product).
  int64_t pre = 0, tot = 0;
  for (const RequestState& q : r.requests) {
    pre += q.preemption_count;
    tot += q.tokens_generated;
  }
  const int64_t win = r.requests.empty() ? 0 : std::llround(m.throughput_tok_s * r.duration_s);
  o.preemptions = pre;
  o.tokens_total = tot;
  o.tokens_in_window = win;
  if (trace) {
    o.digest = digest_of(r);
    for (const IterationTraceRow& t : r.iteration_trace) o.sum_running += t.r_running;
  }
}

// Runs every scenario on the pool; errors become statuses (lowest index
// first in *status), results are kept when `keep` is non-null.
void simulate_all(const lt_workload_batch* batch, const lt_server_config* config, const lt_sim_options* options,
                  bool trace, lt_sim_summary* out, std::vector<SimulationResult>* keep, lt_status* status) {
  const std::size_t n = static_cast<std::size_t>(batch->n_scenarios);
  const ServerConfig base = to_config(*config);
  std::vector<std::exception_ptr> errors(n);
  if (keep) keep->assign(n, SimulationResult());
  g_messages.assign(n, std::string());
  run_pool(n, [&](std::size_t i) {
    lt_sim_summary& o = out[i];
    std::memset(&o, 0, sizeof(o));
    try {
      WorkloadSpec w;
      ServerConfig cfg;
      SimulationResult r = run_one(batch, i, base, options, trace, &w, &cfg);
      const MetricsSummary m = compute_metrics(r, w, cfg.ideal_includes_input);
      fill_summary(r, m, trace, o);
      if (keep) (*keep)[i] = std::move(r);
    } catch (...) {
      errors[i] = std::current_exception();
    }
  });
  if (status) status->code = LT_OK;
  for (std::size_t i = 0; i < n; ++i) {
    if (!errors[i]) continue;
    std::string msg;
    const int32_t code = classify(errors[i], &msg);
    g_messages[i] = msg;
    out[i].status = code;
    out[i].status_kind = LT_K_MESSAGE;
    if (status && status->code == LT_OK) set_status(status, code, static_cast<int64_t>(i), msg);
  }
}

void write_states(const std::vector<SimulationResult>& keep, lt_request_states* states) {
  int64_t off = 0;
  for (std::size_t i = 0; i < keep.size(); ++i) {
    if (states->req_offset) states->req_offset[i] = off;
    for (const RequestState& q : keep[i].requests) {
      if (off < states->capacity) {
        if (states->phase) states->phase[off] = static_cast<int8_t>(q.phase);
        if (states->tokens_generated) states->tokens_generated[off] = q.tokens_generated;
        if (states->first_token_time_s)
          states->first_token_time_s[off] = q.first_token_time_s ? *q.first_token_time_s : NAN;
        if (states->completion_time_s) states->completion_time_s[off] = q.completion_time_s;
        if (states->preemption_count) states->preemption_count[off] = q.preemption_count;
        if (states->adapter_id) states->adapter_id[off] = q.request.adapter_id;
        if (states->input_tokens) states->input_tokens[off] = q.request.input_tokens;
        if (states->output_tokens) states->output_tokens[off] = q.request.output_tokens;
        if (states->arrival_time_s) states->arrival_time_s[off] = q.request.arrival_time_s;
      }
      ++off;
    }
  }
}

}  // namespace

extern "C" {

int32_t ltref_simulate_batch(void*, const lt_workload_batch* batch, const lt_server_config* config,
                             const lt_sim_options* options, lt_sim_summary* out,
                             lt_request_states* states, lt_status* status) {
  std::vector<SimulationResult> keep;
  simulate_all(batch, config, options, options && options->want_digest, out, states ? &keep : nullptr, status);
  if (states) write_states(keep, states);
  return status ? status->code : 0;
}

// The full SimulationResult (trace rows, load events, token emit times) in
// the lt_report layout of lt_simulate_report.
int32_t ltref_simulate_report(void*, const lt_workload_batch* batch, const lt_server_config* config,
                              const lt_sim_options* options, lt_sim_summary* out, lt_request_states* states,
                              lt_report* report, lt_status* status) {
  std::vector<SimulationResult> keep;
  simulate_all(batch, config, options, true, out, &keep, status);
  if (!(options && options->want_digest))
    for (int64_t i = 0; i < batch->n_scenarios; ++i) out[i].digest = 0, out[i].sum_running = 0;
  write_states(keep, states);
  int64_t to = 0, lo = 0, row = 0, eo = 0;
  for (std::size_t i = 0; i < keep.size(); ++i) {
    const SimulationResult& r = keep[i];
    if (report->trace_offset) report->trace_offset[i] = to;
    if (report->load_offset) report->load_offset[i] = lo;
    for (const IterationTraceRow& t : r.iteration_trace) {
      if (to < report->trace_capacity && report->trace)
        report->trace[to] = lt_trace_row{t.time_s, t.iteration, t.r_running, t.r_waiting, t.a_running, t.loads,
                                         t.lat_step_s};
      ++to;
    }
    for (const LoadEvent& e : r.load_events) {
      if (lo < report->load_capacity && report->loads)
        report->loads[lo] = lt_load_event{e.time_s, e.adapter_id, e.rank, static_cast<int32_t>(e.source), 0,
                                          e.latency_s};
      ++lo;
    }
    for (const RequestState& q : r.requests) {
      if (row < states->capacity && report->emit_offset) report->emit_offset[row] = eo;
      for (double t : q.token_emit_times_s) {
        if (eo < report->emit_capacity && report->emit_times) report->emit_times[eo] = t;
        ++eo;
      }
      ++row;
    }
  }
  return status ? status->code : 0;
}

int32_t ltref_sweep_batch(void*, const lt_condition_batch* batch, const lt_server_config* config,
                          const lt_sweep_grid* grid, double duration_s, uint64_t seed,
                          const lt_sweep_options* options, const lt_sim_options*,
                          lt_placement* out, lt_frontier_point* frontier, int32_t max_frontier,
                          lt_status* status) {
  const std::size_t n = static_cast<std::size_t>(batch->n_conditions);
  const ServerConfig cfg = to_config(*config);
  SweepGrid g;
  g.n_values.assign(grid->n_values, grid->n_values + grid->n_count);
  g.g_mode = grid->g_mode == LT_G_EXPLICIT ? SweepGrid::GMode::Explicit : SweepGrid::GMode::Geometric;
  if (grid->g_values) g.g_values.assign(grid->g_values, grid->g_values + grid->g_count);
  SweepOptions so;
  so.early_exit = options->early_exit != 0;
  so.early_exit_k = options->early_exit_k;
  so.jobs = 1;  // parallelism lives at the condition level, as in generate_dataset
  so.mode = static_cast<LengthMode>(options->mode);
  std::vector<std::exception_ptr> errors(n);
  g_messages.assign(n, std::string());
  run_pool(n, [&](std::size_t i) {
    lt_placement& o = out[i];
    std::memset(&o, 0, sizeof(o));
    o.status_point = -1;
    try {
      const lt_condition& c = batch->conditions[i];
      Condition cond;
      cond.lengths = to_lengths(batch->lengths[c.length_index], batch->full_lengths);
      for (int32_t j = 0; j < c.mix_count; ++j) {
        AdapterTemplate t;
        t.rank = batch->templates[c.mix_offset + j].rank;
        t.rate = batch->templates[c.mix_offset + j].rate;
        cond.mix.push_back(t);
      }
      const PlacementResult p = sweep_optimal(cond, cfg, g, duration_s, seed, so);
      o.max_throughput_tok_s = p.max_throughput_tok_s;
      o.n_star = p.n_star;
      o.g_star = p.g_star;
      o.all_starved = p.all_starved;
      o.frontier_open = p.frontier_open;
      o.frontier_count = static_cast<int32_t>(p.frontier.size());
      for (std::size_t k = 0; k < p.frontier.size() && static_cast<int32_t>(k) < max_frontier; ++k) {
        lt_frontier_point& f = frontier[i * static_cast<std::size_t>(max_frontier) + k];
        f.n = p.frontier[k].n;
        f.g = p.frontier[k].g;
        f.throughput_tok_s = p.frontier[k].throughput_tok_s;
        f.starved = p.frontier[k].starved;
        f.skipped = p.frontier[k].skipped;
        if (!f.skipped) ++o.points_simulated;
      }
    } catch (...) {
      errors[i] = std::current_exception();
    }
  });
  if (status) status->code = LT_OK;
  for (std::size_t i = 0; i < n; ++i) {
    if (!errors[i]) continue;
    std::string msg;
    const int32_t code = classify(errors[i], &msg);
    g_messages[i] = msg;
    out[i].status = code;
    out[i].status_kind = LT_K_MESSAGE;
    if (status && status->code == LT_OK) set_status(status, code, static_cast<int64_t>(i), msg);
  }
  return status ? status->code : 0;
}

}  // extern "C"

// generate_dataset / condition_hash / encode_workload (placement.hpp:104-158)
// of the unmodified reference, for the dataset parity tests.
namespace {
DatasetSpec to_dataset(const lt_dataset_spec& d) {
  DatasetSpec s;
  s.rates.assign(d.rates, d.rates + d.n_rates);
  s.ranks.assign(d.ranks, d.ranks + d.n_ranks);
  s.triple_size = d.triple_size;
  s.condition_stride = d.condition_stride;
  s.lengths = to_lengths(d.lengths, d.full_lengths);
  s.duration_s = d.duration_s;
  s.seed = d.seed;
  s.grid.n_values.assign(d.grid.n_values, d.grid.n_values + d.grid.n_count);
  s.grid.g_mode = d.grid.g_mode == LT_G_EXPLICIT ? SweepGrid::GMode::Explicit : SweepGrid::GMode::Geometric;
  if (d.grid.g_values) s.grid.g_values.assign(d.grid.g_values, d.grid.g_values + d.grid.g_count);
  s.sweep.early_exit = d.sweep.early_exit != 0;
  s.sweep.early_exit_k = d.sweep.early_exit_k;
  s.sweep.jobs = d.sweep.jobs < 1 ? 1 : d.sweep.jobs;
  s.sweep.mode = d.sweep.mode == LT_MODE_FULL ? LengthMode::Full : LengthMode::Mean;
  return s;
}
Condition to_condition(const lt_template* mix, int32_t n_mix, const lt_length_spec* l, const int32_t* full) {
  Condition c;
  for (int32_t i = 0; i < n_mix; ++i) {
    AdapterTemplate t;
    t.rank = mix[i].rank;
    t.rate = mix[i].rate;
    c.mix.push_back(t);
  }
  c.lengths = to_lengths(*l, full);
  return c;
}
}  // namespace

extern "C" {

int32_t ltref_generate_dataset(void*, const lt_dataset_spec* spec, const lt_server_config* config,
                               const char* out_csv, lt_error_fn on_error, void* user,
                               lt_dataset_progress* progress, lt_status* status) {
  if (status) status->code = LT_OK;
  try {
    const DatasetSpec ds = to_dataset(*spec);
    const DatasetProgress p = generate_dataset(ds, to_config(*config), out_csv, [&](const std::string& m) {
      if (on_error) on_error(m.c_str(), user);
    });
    if (progress) {
      progress->total_conditions = static_cast<int64_t>(p.total_conditions);
      progress->completed = static_cast<int64_t>(p.completed);
      progress->failed = static_cast<int64_t>(p.failed);
    }
    return LT_OK;
  } catch (...) {
    std::string msg;
    const int32_t code = classify(std::current_exception(), &msg);
    set_status(status, code, -1, msg);
    return code;
  }
}

uint64_t ltref_condition_hash(const lt_template* mix, int32_t n_mix, const lt_length_spec* lengths,
                              const int32_t* full_lengths, double duration_s, uint64_t seed,
                              const lt_sweep_grid* grid) {
  SweepGrid g;
  g.n_values.assign(grid->n_values, grid->n_values + grid->n_count);
  g.g_mode = grid->g_mode == LT_G_EXPLICIT ? SweepGrid::GMode::Explicit : SweepGrid::GMode::Geometric;
  if (grid->g_values) g.g_values.assign(grid->g_values, grid->g_values + grid->g_count);
  return condition_hash(to_condition(mix, n_mix, lengths, full_lengths), duration_s, seed, g);
}

int32_t ltref_encode_workload(const lt_template* mix, int32_t n_mix, const lt_length_spec* lengths,
                              const int32_t* full_lengths, double* features16, lt_status* status) {
  if (status) status->code = LT_OK;
  try {
    const WorkloadFeatures f = encode_workload(to_condition(mix, n_mix, lengths, full_lengths));
    for (int i = 0; i < 16; ++i) features16[i] = f.values[static_cast<size_t>(i)];
    return LT_OK;
  } catch (...) {
    std::string msg;
    const int32_t code = classify(std::current_exception(), &msg);
    set_status(status, code, -1, msg);
    return code;
  }
}

// The reference's own JSON parser on a server-config file (json_io.cpp:188-235),
// compared with the ABI config `c` through the reference's serializer
// (server_config_to_json): 1 = identical, 0 = different (both texts in
// `diff`), < 0 = the reference rejected the file (status carries what()).
int32_t ltref_config_json_matches(const char* text, const lt_server_config* c, char* diff, size_t len,
                                  lt_status* status) {
  if (status) status->code = LT_OK;
  try {
    ServerConfig parsed = server_config_from_json(text);
    ServerConfig mine = to_config(*c);
    parsed.slots = mine.slots;
    const std::string a = server_config_to_json(parsed), b = server_config_to_json(mine);
    if (a == b) return 1;
    if (diff && len) std::snprintf(diff, len, "reference:\n%s\nabi:\n%s", a.c_str(), b.c_str());
    return 0;
  } catch (...) {
    std::string msg;
    const int32_t code = classify(std::current_exception(), &msg);
    set_status(status, code, -1, msg);
    return -code;
  }
}

}  // extern "C"

// ---- predictor (predictor.cpp:202-269): the reference's own training ------
#include "loratwin/predictor.hpp"

namespace {

std::vector<WorkloadFeatures> to_features(const double* x, int64_t n) {
  std::vector<WorkloadFeatures> v(static_cast<std::size_t>(n));
  for (int64_t i = 0; i < n; ++i)
    for (std::size_t f = 0; f < kNumFeatures; ++f) v[i].values[f] = x[i * kNumFeatures + f];
  return v;
}

TreeParams to_tree_params(const lt_tree_params& p) {
  TreeParams t;
  t.max_depth = p.max_depth;
  t.min_leaf = static_cast<std::size_t>(p.min_leaf < 0 ? 0 : p.min_leaf);
  t.feature_subset = static_cast<std::size_t>(p.feature_subset < 0 ? 0 : p.feature_subset);
  return t;
}

int32_t put_trees(const std::vector<const DecisionTree*>& trees, lt_tree_node* nodes, int64_t cap,
                  int64_t* offset, int32_t* count) {
  int64_t off = 0;
  for (std::size_t t = 0; t < trees.size(); ++t) {
    if (offset) offset[t] = off;
    if (count) count[t] = static_cast<int32_t>(trees[t]->nodes.size());
    for (const TreeNode& n : trees[t]->nodes) {
      if (off < cap && nodes)
        nodes[off] = lt_tree_node{n.feature_index, n.left, n.right, 0, n.threshold, n.value,
                                  static_cast<int64_t>(n.coverage)};
      ++off;
    }
  }
  return off <= cap ? LT_OK : LT_ERR_VALIDATION;
}

int32_t predictor_error(lt_status* st) {
  std::string msg;
  const int32_t code = classify(std::current_exception(), &msg);
  set_status(st, code, -1, msg);
  return code;
}

}  // namespace

extern "C" {

int32_t ltref_train_tree(void*, const double* x, int64_t n_rows, const double* y, const lt_tree_params* params,
                         uint64_t seed, uint64_t tree_tag, lt_tree_node* nodes, int64_t cap, int32_t* count,
                         lt_status* status) {
  if (status) status->code = LT_OK;
  try {
    const DecisionTree t = train_tree(to_features(x, n_rows), std::vector<double>(y, y + n_rows),
                                      to_tree_params(*params), seed, tree_tag);
    return put_trees({&t}, nodes, cap, nullptr, count);
  } catch (...) {
    return predictor_error(status);
  }
}

int32_t ltref_train_forests(void*, const double* x, int64_t n_rows, const double* y, const int32_t* tags,
                            int32_t n_targets, const lt_forest_params* params, uint64_t seed, lt_tree_node* nodes,
                            int64_t cap, int64_t* offset, int32_t* count, lt_status* status) {
  if (status) status->code = LT_OK;
  try {
    ForestParams fp;
    fp.n_trees = params->n_trees;
    fp.bootstrap = params->bootstrap != 0;
    fp.tree = to_tree_params(params->tree);
    const std::vector<WorkloadFeatures> xf = to_features(x, n_rows);
    std::vector<ForestModel> forests;
    for (int32_t g = 0; g < n_targets; ++g)
      forests.push_back(train_forest(xf, std::vector<double>(y + g * n_rows, y + (g + 1) * n_rows),
                                     static_cast<PredictTarget>(tags[g]), fp, seed));
    std::vector<const DecisionTree*> trees;
    for (const ForestModel& f : forests)
      for (const DecisionTree& t : f.trees) trees.push_back(&t);
    return put_trees(trees, nodes, cap, offset, count);
  } catch (...) {
    return predictor_error(status);
  }
}

int32_t ltref_predict_forests(void*, const lt_tree_node* nodes, int64_t, const int64_t* offset, int32_t n_trees,
                              const int32_t* tags, int32_t n_targets, const double* x, int64_t n_rows, double* out,
                              lt_status* status) {
  if (status) status->code = LT_OK;
  try {
    const std::vector<WorkloadFeatures> xf = to_features(x, n_rows);
    for (int32_t g = 0; g < n_targets; ++g) {
      ForestModel m;
      m.target = static_cast<PredictTarget>(tags[g] < 0 ? 0 : tags[g]);
      for (int32_t t = 0; t < n_trees; ++t) {
        const int64_t o = offset[g * n_trees + t];
        DecisionTree d;
        // node count: up to the next tree's offset is not known here; walk the preorder vector
        std::vector<int64_t> stack{0};
        int64_t maxk = 0;
        while (!stack.empty()) {
          const int64_t k = stack.back();
          stack.pop_back();
          maxk = std::max(maxk, k);
          if (nodes[o + k].feature_index >= 0) {
            stack.push_back(nodes[o + k].left);
            stack.push_back(nodes[o + k].right);
          }
        }
        for (int64_t k = 0; k <= maxk; ++k) {
          const lt_tree_node& n = nodes[o + k];
          TreeNode tn;
          tn.feature_index = n.feature_index;
          tn.threshold = n.threshold;
          tn.left = n.left;
          tn.right = n.right;
          tn.value = n.value;
          tn.coverage = static_cast<std::size_t>(n.coverage);
          d.nodes.push_back(tn);
        }
        m.trees.push_back(std::move(d));
      }
      for (int64_t i = 0; i < n_rows; ++i)
        out[g * n_rows + i] = tags[g] < 0 ? m.predict_raw(xf[i]) : m.predict(xf[i]);
    }
    return LT_OK;
  } catch (...) {
    return predictor_error(status);
  }
}

}  // extern "C"
