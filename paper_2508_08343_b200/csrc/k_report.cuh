// Full simulation report (lt_simulate_report): the per-request token emit
// times of RequestState.token_emit_times_s (engine.cpp:128-135), rebuilt on
// the device from what the report pass of the engine logged:
//   * the emit time of iteration k, tr_time[k] + tr_lat[k] -- the same
//     clock_ + lat add the engine (and the reference) performs;
//   * per scenario, a stint log of {request, iteration} entries, one per
//     admission and one per preemption, in the order they happened. A
//     request's entries alternate admit / preempt (it is admitted first), and
//     it emits one token per iteration in [admit, preempt) (decode_step_alloc
//     evicts before the emit, kv_scheduler.cpp:183-236); its last stint runs
//     until its tokens_generated are all placed.
// The log is regrouped by request with a stable radix sort on the global
// request index (entries of one request stay in time order).
#pragma once

#include <cstdint>

#include "loratwin_gpu.h"
#include "lt_device.cuh"

namespace lt {

// Sort keys of the stint log: entry j of scenario s -> its request's global
// index; unused tail entries keep key UINT32_MAX (sorted last). One warp per
// scenario.
__global__ void __launch_bounds__(256) stint_keys_kernel(const DScen* scen, int n_scen, const int64_t* sl_off,
                                                         const int32_t* sl_cnt, const int2* log, uint32_t* keys,
                                                         int32_t* iters) {
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (s >= n_scen) return;
  const int64_t base = sl_off[s];
  const int32_t n = sl_cnt[s];
  const uint32_t rb = static_cast<uint32_t>(scen[s].req_begin);
  for (int j = lane; j < n; j += 32) {
    const int2 e = log[base + j];
    keys[base + j] = rb + static_cast<uint32_t>(e.x);
    iters[base + j] = e.y;
  }
}

__device__ __forceinline__ int scenario_of(const DScen* scen, int n_scen, int64_t g) {
  int lo = 0, hi = n_scen - 1;  // last scenario with req_begin <= g (req_begin ascending)
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (scen[mid].req_begin <= g) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// RequestState.tokens_generated of every request after the run (a finished
// request's generated count is its output length); 0 for the requests of a
// scenario that failed (the reference throws: there is no report).
__global__ void __launch_bounds__(256) request_tokens_kernel(const DScen* scen, int n_scen, const lt_sim_summary* out,
                                                             const int8_t* phase, const int32_t* gen,
                                                             const int32_t* outv, int64_t n, int64_t* tokens) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int s = scenario_of(scen, n_scen, i);
  tokens[i] = out[s].status != LT_OK ? 0 : (phase[i] == kFinished ? outv[i] : gen[i]);
}

// IterationTraceRow records (lt_trace_row) from the report pass's SoA rows:
// one thread per row; the row's scenario by binary search over tr_off.
__global__ void __launch_bounds__(256) trace_pack_kernel(const int64_t* tr_off, int n_scen, int64_t n_rows,
                                                         const double* tr_time, const double* tr_lat,
                                                         const int4* tr_rwal, lt_trace_row* rows) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n_rows) return;
  int lo = 0, hi = n_scen - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (tr_off[mid] <= i) lo = mid;
    else hi = mid - 1;
  }
  const int4 r = tr_rwal[i];
  lt_trace_row t;
  t.time_s = tr_time[i];
  t.iteration = i - tr_off[lo];
  t.r_running = r.x;
  t.r_waiting = r.y;
  t.a_running = r.z;
  t.loads = r.w;
  t.lat_step_s = tr_lat[i];
  rows[i] = t;
}

// One thread per request: finds its scenario (req_begin ascending), its
// first sorted log entry, and writes its emit times at emit[emit_off[g] ..].
__global__ void __launch_bounds__(256) emit_times_kernel(const DScen* scen, int n_scen, int64_t n_req,
                                                         const uint32_t* keys, const int32_t* iters, int64_t n_log,
                                                         const int64_t* tokens, const int64_t* emit_off,
                                                         const int64_t* tr_off, const double* tr_time,
                                                         const double* tr_lat, double* emit) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= n_req) return;
  int64_t T = tokens[g];
  if (T <= 0) return;
  const int64_t tb = tr_off[scenario_of(scen, n_scen, g)];
  int64_t a = 0, b = n_log;  // first entry with key >= g
  const uint32_t key = static_cast<uint32_t>(g);
  while (a < b) {
    const int64_t m = (a + b) >> 1;
    if (keys[m] < key) a = m + 1;
    else b = m;
  }
  int64_t pos = emit_off[g];
  for (int64_t j = a; j < n_log && keys[j] == key && T > 0; j += 2) {
    const int32_t start = iters[j];
    const bool preempted = j + 1 < n_log && keys[j + 1] == key;
    const int64_t stop = preempted ? static_cast<int64_t>(iters[j + 1]) : static_cast<int64_t>(start) + T;
    for (int64_t k = start; k < stop && T > 0; ++k, --T) emit[pos++] = tr_time[tb + k] + tr_lat[tb + k];
  }
}

// compute_metrics' ITL mean from the materialised emit times, in the
// reference's order: requests in id order, each request's gaps in emit order,
// one sequential sum (std::accumulate over the flattened list, metrics.cpp:
// 29-32, :92-94) -- bit-exact where the engine epilogue's per-request sums
// are within 1e-9. One thread per scenario.
__global__ void __launch_bounds__(128) itl_exact_kernel(const DScen* scen, int n_scen, lt_sim_summary* out,
                                                       const int64_t* tokens, const int64_t* emit_off,
                                                       const double* emit) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_scen || out[s].status != LT_OK || scen[s].n_req == 0) return;
  double sum = 0.0;
  int64_t cnt = 0;
  const int64_t g0 = scen[s].req_begin;
  for (int64_t g = g0; g < g0 + scen[s].n_req; ++g) {
    const double* e = emit + emit_off[g];
    for (int64_t i = 1; i < tokens[g]; ++i) {
      sum += e[i] - e[i - 1];
      ++cnt;
    }
  }
  out[s].itl_mean_s = cnt ? sum / static_cast<double>(cnt) : 0.0;
}

}  // namespace lt
