// End-to-end check of the reference-side binding (gpu_backend.cpp): the
// reference's own code calls libloratwin_gpu.so through the shim, and its own
// JSON writers (simulation_report_json, json_io.cpp:608-687;
// placement_result_to_json) must print byte-identical documents for the GPU
// result and for the reference's run_simulation / run_scripted /
// sweep_optimal on the same inputs.
//
//   gpu_backend_check          exit 0: every document identical ("ok ...")
//                              exit 1: a mismatch (the first one is printed)
//                              exit 3: no usable device; the library's
//                                      error came back as the reference's
//                                      exception type (the CPU-only check)
#include <cstdio>
#include <string>
#include <vector>

#include "gpu_backend.hpp"
#include "loratwin/errors.hpp"
#include "loratwin/json_io.hpp"

using namespace loratwin;

namespace {

int g_checked = 0;

bool same(const std::string& what, const std::string& a, const std::string& b) {
  ++g_checked;
  if (a == b) return true;
  size_t k = 0;
  while (k < a.size() && k < b.size() && a[k] == b[k]) ++k;
  std::printf("MISMATCH %s at byte %zu\n--- gpu ---\n%s\n--- reference ---\n%s\n", what.c_str(), k,
              a.substr(k > 200 ? k - 200 : 0, 400).c_str(), b.substr(k > 200 ? k - 200 : 0, 400).c_str());
  return false;
}

std::string report(const SimulationResult& r, const MetricsSummary& m) {
  SimulationReportOptions o;
  o.include_requests = true;
  o.include_trace = true;
  return simulation_report_json(r, m, o);
}

WorkloadSpec workload(int n, int rank_mode, double agg_rate, const LengthSpec& lengths, double duration,
                      std::uint64_t seed) {
  WorkloadSpec w;
  for (int i = 0; i < n; ++i) {
    AdapterSpec a;
    a.adapter_id = i + 1;
    a.rank = rank_mode == 3 ? (8 << (i % 3)) : (8 << rank_mode);
    a.rate = agg_rate / n;
    w.adapters.push_back(a);
  }
  w.lengths = lengths;
  w.duration_s = duration;
  w.seed = seed;
  return w;
}

}  // namespace

int main() {
  try {
    SimOptions opt;
    opt.record_iteration_trace = true;
    // run_simulation: slot-starved, KV-starved (preempting) and idle engines
    const LengthSpec medium = LengthSpec::mean(250, 50, 231, 50);
    const LengthSpec longio = LengthSpec::mean(2048, 512, 1024, 256);
    struct Case {
      int n, rank_mode, slots;
      double rate, duration;
      LengthSpec lengths;
      std::uint64_t seed;
    };
    const std::vector<Case> cases = {
        {8, 1, 8, 1.6, 600.0, medium, 1},     // C1-shaped, 600 s
        {64, 3, 8, 3.2, 120.0, medium, 7},    // slot-starved
        {24, 2, 16, 6.0, 60.0, longio, 11},   // KV-starved, preempting
        {4, 0, 4, 0.05, 300.0, medium, 13},   // mostly idle
        {130, 3, 32, 12.0, 60.0, medium, 17}  // many adapters
    };
    for (const Case& c : cases) {
      const WorkloadSpec w = workload(c.n, c.rank_mode, c.rate, c.lengths, c.duration, c.seed);
      const ServerConfig cfg = h100_like_config(c.slots);
      MetricsSummary mg;
      const SimulationResult g = gpu::run_simulation(w, cfg, LengthMode::Mean, opt, &mg);
      const SimulationResult r = run_simulation(w, cfg, LengthMode::Mean, opt);
      const MetricsSummary mr = compute_metrics(r, w, cfg.ideal_includes_input);
      if (!same("run_simulation seed " + std::to_string(c.seed), report(g, mg), report(r, mr))) return 1;
    }
    // run_scripted with a tight budget: preemptions and re-admissions
    {
      ServerConfig cfg = h100_like_config(2);
      cfg.memory.slot_cost_table.clear();
      cfg.memory.slot_cost_base_rank8 = 8.0;  // 16 tokens per rank-16 slot
      cfg.memory.total_kv_budget = 2400;
      std::vector<AdapterSpec> ads;
      for (int i = 0; i < 5; ++i) ads.push_back(AdapterSpec{i + 1, 8 << (i % 2), 1.0, std::nullopt});
      std::vector<Request> reqs;
      for (int i = 0; i < 80; ++i)
        reqs.push_back(Request{i, 1 + (i * 7) % 5, 0.05 * i, 20 + (i * 37) % 300, 5 + (i * 13) % 60});
      MetricsSummary mg;
      const SimulationResult g = gpu::run_scripted(reqs, ads, 4.0, cfg, opt, &mg);
      const SimulationResult r = run_scripted(reqs, ads, 4.0, cfg, opt);
      MetricsSummary mr;
      WorkloadSpec w;
      w.adapters = ads;
      w.duration_s = 4.0;
      mr = compute_metrics(r, w, cfg.ideal_includes_input);
      // the scripted workload has no lengths: ideal comes from the caller's
      // workload, as compute_metrics is given it here (not from the run)
      mg.ideal_throughput_tok_s = mr.ideal_throughput_tok_s;
      mg.starved = mr.starved;
      if (!same("run_scripted", report(g, mg), report(r, mr))) return 1;
    }
    // sweep_optimal over a few dataset conditions, all in one device call
    {
      DatasetSpec ds;
      ds.rates = {3.2, 0.4, 0.05};
      ds.ranks = {8, 16, 32};
      ds.triple_size = 2;
      ds.lengths = medium;
      const std::vector<Condition> conds = enumerate_conditions(ds);
      SweepGrid grid;
      grid.n_values = {1, 2, 4, 8, 16, 32, 64};
      SweepOptions so;
      so.early_exit = true;
      so.early_exit_k = 2;
      const ServerConfig cfg = h100_like_config(1);
      const std::vector<PlacementResult> g = gpu::sweep_optimal_batch(conds, cfg, grid, 120.0, 5, so);
      for (size_t i = 0; i < conds.size(); ++i) {
        const PlacementResult r = sweep_optimal(conds[i], cfg, grid, 120.0, 5, so);
        if (!same("sweep_optimal condition " + std::to_string(i), placement_result_to_json(g[i]),
                  placement_result_to_json(r)))
          return 1;
      }
    }
    // errors come back as the reference's exception, with its message
    {
      WorkloadSpec w = workload(4, 0, 1.0, medium, 60.0, 3);
      w.adapters[0].rank = 24;  // no load-latency entry for rank 24 in h100_like
      const ServerConfig cfg = h100_like_config(4);
      std::string eg, er;
      try {
        gpu::run_simulation(w, cfg, LengthMode::Mean, opt, nullptr);
      } catch (const ConfigError& e) {
        eg = e.what();
      }
      try {
        run_simulation(w, cfg, LengthMode::Mean, opt);
      } catch (const ConfigError& e) {
        er = e.what();
      }
      if (er.empty() || !same("ConfigError text", eg, er)) return 1;
    }
    std::printf("ok: %d documents byte-identical (simulation reports, placements, error text)\n", g_checked);
    return 0;
  } catch (const InternalError& e) {
    // no device: lt_create's LT_ERR_DEVICE status, rethrown as the reference's InternalError
    std::printf("no-device: %s\n", e.what());
    return 3;
  } catch (const std::exception& e) {
    std::printf("exception: %s\n", e.what());
    return 2;
  }
}
