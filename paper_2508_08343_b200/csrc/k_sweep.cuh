// K3 placement_reduce: sweep_optimal's reduction (placement.cpp:185-264) on
// device, one thread per condition, over the condition's simulated grid
// points laid out row-major (N rows in grid order, G candidates ascending).
//
// Exact semantics kept:
//   - rows are consumed in N order; an error anywhere in a consumed row is the
//     sweep's error, lowest G index first (run_parallel, placement.cpp:93-95);
//     rows after the early-exit stop are never consumed, so their (speculative)
//     results and errors are ignored (placement.cpp:240-243);
//   - best = strict '>' over non-starved points, ties keep the earlier point;
//   - first_n_best over row 0 includes starved points (placement.cpp:228-231);
//   - stall counter / early exit with k (placement.cpp:234-244);
//   - skipped rows -> {n, 0, 0.0, false, true} (placement.cpp:247-248);
//   - all_starved fallback and frontier_open (placement.cpp:250-263).
#pragma once
#include "lt_device.cuh"

namespace lt {

struct SweepRow {
  int32_t n;
  int32_t g_count;
  int32_t g_offset;  // into the per-row G list
  int32_t point_offset;  // first point of this row within a condition
};

__global__ void sweep_reduce_kernel(int n_cond, const SweepRow* rows, int n_rows, const int32_t* g_list,
                                    int32_t points_per_cond, const int64_t* cond_point_base,
                                    const lt_sim_summary* pts, int early_exit, int early_exit_k,
                                    int max_frontier, lt_placement* out, lt_frontier_point* frontier) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_cond) return;
  lt_placement res;
  memset(&res, 0, sizeof(res));
  res.status_point = -1;
  lt_frontier_point* fr = frontier + static_cast<int64_t>(c) * max_frontier;
  const int64_t base = cond_point_base[c];
  if (base < 0) {  // condition failed host validation; status filled by the host
    out[c] = res;
    return;
  }
  double best_tput = -1.0;
  int best_n = 0, best_g = 0;
  bool any_non_starved = false, any_starved = false;
  int stall = 0;
  int stop = n_rows;
  double first_best = -1.0;
  int first_best_g = 0;
  int nf = 0;
  for (int ni = 0; ni < n_rows; ++ni) {
    const SweepRow row = rows[ni];
    // errors of a consumed row: lowest G index
    for (int gi = 0; gi < row.g_count; ++gi) {
      const lt_sim_summary& p = pts[base + row.point_offset + gi];
      if (p.status != LT_OK) {
        res.status = p.status;
        res.status_kind = p.status_kind;
        res.status_a = p.status_a;
        res.status_b = p.status_b;
        res.status_point = base + row.point_offset + gi;
        res.frontier_count = 0;
        res.points_simulated = 0;  // the reference's sweep throws: no result at all
        res.iterations = 0;
        out[c] = res;
        return;
      }
    }
    bool improved = false;
    for (int gi = 0; gi < row.g_count; ++gi) {
      const lt_sim_summary& p = pts[base + row.point_offset + gi];
      const int g = g_list[row.g_offset + gi];
      const double t = p.throughput_tok_s;
      const bool starved = p.starved != 0;
      if (nf < max_frontier) {
        fr[nf].n = row.n;
        fr[nf].g = g;
        fr[nf].throughput_tok_s = t;
        fr[nf].starved = starved;
        fr[nf].skipped = 0;
      }
      ++nf;
      ++res.points_simulated;
      res.iterations += p.iterations;
      if (starved) any_starved = true;
      if (!starved) {
        any_non_starved = true;
        if (t > best_tput) {
          best_tput = t;
          best_n = row.n;
          best_g = g;
          improved = true;
        }
      }
      if (ni == 0 && t > first_best) {
        first_best = t;
        first_best_g = g;
      }
    }
    if (early_exit) {
      stall = improved ? 0 : stall + 1;
      if (stall >= early_exit_k && ni + 1 < n_rows) {
        stop = ni + 1;
        break;
      }
    }
  }
  for (int ni = stop; ni < n_rows; ++ni) {
    if (nf < max_frontier) {
      fr[nf].n = rows[ni].n;
      fr[nf].g = 0;
      fr[nf].throughput_tok_s = 0.0;
      fr[nf].starved = 0;
      fr[nf].skipped = 1;
    }
    ++nf;
  }
  res.frontier_count = nf;
  if (!any_non_starved) {
    res.all_starved = 1;
    res.n_star = rows[0].n;
    res.g_star = first_best_g;
    res.max_throughput_tok_s = first_best < 0.0 ? 0.0 : first_best;
  } else {
    res.max_throughput_tok_s = best_tput;
    res.n_star = best_n;
    res.g_star = best_g;
    const int last_evaluated = rows[stop - 1].n;
    res.frontier_open = !any_starved && best_n == last_evaluated;
  }
  out[c] = res;
}

// ---------------------------------------------------------------------------
// Device-side sweep waves (lt_sweep_batch, Mean mode): conditions are
// instantiated on the device from their mix templates, every wave simulates
// row r of the still-active conditions, and the early-exit decision that
// keeps a condition in the next wave is taken on the device.

// One mix leg (AdapterTemplate) with its load latency already looked up.
struct DTemplate {
  int32_t rank;
  int32_t _pad;
  double rate;
  double load_lat;  // NaN: rank missing from cpu_load_seconds (lazy ConfigError)
};

// instantiate_condition (placement.cpp:139-157) for every condition at the
// grid's largest N: adapter i has id i + 1 and (rank, rate) = mix[i % |mix|];
// each grid point of the condition reads the prefix of its N adapters. The
// RNG key of adapter id i + 1 is key i (one seed per sweep).
__global__ void cond_adapters_kernel(int n_cond, int n_max, const int32_t* mix_off, const int32_t* mix_cnt,
                                     const DTemplate* tmpl, DAdapter* out) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= static_cast<int64_t>(n_cond) * n_max) return;
  const int c = static_cast<int>(t / n_max), i = static_cast<int>(t % n_max);
  const int cnt = mix_cnt[c];
  if (cnt <= 0) return;
  const DTemplate m = tmpl[mix_off[c] + i % cnt];
  DAdapter a;
  a.id = i + 1;
  a.rank = m.rank;
  a.rate = m.rate;
  a.load_lat = m.load_lat;
  a.key = i;
  a.length_param = -1;
  a.deck = -1;
  a._pad = 0;
  a.list_off = 0;
  out[t] = a;
}

// (scenario, adapter) streams of a wave: every scenario has the row's N adapters.
__global__ void wave_pairs_kernel(int64_t n_pairs, int N, int32_t* pair_scen, int32_t* pair_adp,
                                  int64_t* pair_begin) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= n_pairs) return;
  const int64_t s = p / N;
  const int k = static_cast<int>(p - s * N);
  pair_scen[p] = static_cast<int32_t>(s);
  pair_adp[p] = k;
  if (k == 0) pair_begin[s] = p;
}

// The wave's summaries into the sweep's point table.
__global__ void wave_scatter_kernel(int n, const lt_sim_summary* out, const int64_t* pidx, lt_sim_summary* pts) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) pts[pidx[i]] = out[i];
}

// sweep_optimal's bookkeeping after row ni of every active condition
// (placement.cpp:219-244): best non-starved throughput (strict '>'), the
// stall counter and the early-exit stop; an error in the row ends the
// condition (K3 reports it). alive[c] = 0 takes c out of the next waves.
__global__ void wave_decide_kernel(int n_act, const int32_t* act, SweepRow row, int ni, int n_rows,
                                   const int64_t* cond_point_base, const lt_sim_summary* pts, int early_exit,
                                   int early_exit_k, double* best, int32_t* stall, uint8_t* alive) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_act) return;
  const int c = act[t];
  const int64_t base = cond_point_base[c] + row.point_offset;
  bool improved = false, err = false;
  double b = best[c];
  for (int gi = 0; gi < row.g_count; ++gi) {
    const lt_sim_summary& p = pts[base + gi];
    if (p.status != LT_OK) err = true;
    if (!p.starved && p.throughput_tok_s > b) {
      b = p.throughput_tok_s;
      improved = true;
    }
  }
  best[c] = b;
  if (err) {
    alive[c] = 0;
    return;
  }
  if (early_exit) {
    const int st = improved ? 0 : stall[c] + 1;
    stall[c] = st;
    if (st >= early_exit_k && ni + 1 < n_rows) alive[c] = 0;
  }
}

}  // namespace lt
