// K2b: the nearest-rank percentiles of compute_metrics (metrics.cpp:47-54,
// :101-105), filled only when a run asks for them (sweep_optimal reads only
// throughput and the starved verdict, placement.cpp:216).
//
//   TTFT: one value per request with a first token (first - arrival), sorted
//         per scenario (CUB segmented sort); requests without one carry +inf
//         and sort last.
//   ITL:  the reference's list holds every gap between consecutive emits of
//         every request. All running requests emit at the same time, so the
//         list is the multiset {(emit_k - emit_{k-1}) x c_k} over iterations
//         (c_k = requests emitting in both k-1 and k) plus one gap per
//         re-admitted preempted request (first emit after - last emit
//         before). The recording engine pass writes those (value, weight)
//         records; a segmented sort by value and a weighted rank select give
//         the identical order statistic.
#pragma once
#include "lt_device.cuh"

namespace lt {

// K2 compute_metrics (metrics.cpp:70-113) of every engine, after K1: one
// warp per scenario walks its requests in request_id order, 32 at a time
// (coalesced). Counts are ballots; the three FP64 sums (rejected demand
// out/window, TTFT first - arrival, ITL last - first: the telescoped per-
// request sum, SURVEY 7 hard part 8) are the reference's sequential
// accumulate: each block's 32 terms are broadcast by shuffles and added in
// lane order, the three chains interleaved. Unflagged lanes add +0.0, which
// leaves the (non-negative) accumulators unchanged. Finished requests get
// their final token count (gen = out). Kept out of the engine kernel: its
// code would sit in the engine's instruction footprint, and its serial add
// chains at the end of every engine's critical path.
__global__ void __launch_bounds__(256) metrics_kernel(const DScen* scen, int n_scen, const int8_t* r_phase,
                                                     const double* r_first, const double* r_arr,
                                                     const double* r_last, const int32_t* r_out, int32_t* r_gen,
                                                     lt_sim_summary* out) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int s = static_cast<int>((blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5);
  if (s >= n_scen) return;
  if (out[s].status != LT_OK) return;
  const DScen sc = scen[s];
  const int64_t n = sc.n_req;
  if (n == 0) {
    if (lane == 0) out[s].degenerate = 1;
    return;
  }
  const int64_t rb = sc.req_begin;
  const double window = sc.duration;
  // The three ordered sums (rejected demand, TTFT, ITL), one per lane 0..2:
  // each block's 32 terms go through shared memory and the lane adds them in
  // request order (the reference's left-to-right sums, metrics.cpp:84-105).
  __shared__ double terms[8][3][33];  // (33: the three lanes read different banks)
  double (*tw)[33] = terms[(threadIdx.x >> 5) & 7];
  double acc = 0.0;
  long long nrej = 0, nfin = 0, nttft = 0, nitl = 0;
  // the next block's loads are issued before this block's ordered sums (the
  // sums are one dependent add chain; the loads would otherwise wait on it)
  auto load = [&](int64_t i, int8_t& ph, double& first, double& arr, double& last, int& outv, int& gen) {
    ph = kWaiting;
    first = arr = last = 0.0;
    outv = gen = 0;
    if (i < n) {
      ph = r_phase[rb + i];
      first = r_first[rb + i];
      arr = r_arr[rb + i];
      last = r_last[rb + i];
      outv = r_out[rb + i];
      gen = r_gen[rb + i];
    }
  };
  int8_t nph;
  double nfirst, narr, nlast;
  int nout, ngen;
  load(lane, nph, nfirst, narr, nlast, nout, ngen);
  for (int64_t base = 0; base < n; base += 32) {
    const int64_t i = base + lane;
    const bool v = i < n;
    const int8_t ph = nph;
    const double first = nfirst, arr = narr, last = nlast;
    const int outv = nout;
    const int gen = (ph == kFinished) ? outv : ngen;
    if (v && ph == kFinished) r_gen[rb + i] = outv;
    load(i + 32, nph, nfirst, narr, nlast, nout, ngen);
    const bool is_rej = v && ph == kRejected;
    const bool has_first = v && first == first;
    const bool has_itl = v && gen >= 2;
    nrej += __popc(__ballot_sync(full, is_rej));
    nfin += __popc(__ballot_sync(full, v && ph == kFinished));
    nttft += __popc(__ballot_sync(full, has_first));
    long long g1 = has_itl ? gen - 1 : 0;
    for (int o = 16; o > 0; o >>= 1) g1 += __shfl_xor_sync(full, g1, o);
    nitl += g1;
    tw[0][lane] = is_rej ? static_cast<double>(outv) / window : 0.0;
    tw[1][lane] = has_first ? first - arr : 0.0;
    tw[2][lane] = has_itl ? last - first : 0.0;
    __syncwarp();
    if (lane < 3) {
      const double* t = tw[lane];
#pragma unroll
      for (int k = 0; k < 32; ++k) acc = acc + t[k];
    }
    __syncwarp();  // read before the next block's terms overwrite them
  }
  const double rej = __shfl_sync(full, acc, 0), ttft = __shfl_sync(full, acc, 1), itl = __shfl_sync(full, acc, 2);
  if (lane == 0) {
    lt_sim_summary& o = out[s];
    o.rejected_count = nrej;
    o.finished_count = nfin;
    o.ttft_mean_s = nttft ? ttft / static_cast<double>(nttft) : 0.0;
    o.itl_mean_s = nitl ? itl / static_cast<double>(nitl) : 0.0;
    const double eff_raw = sc.ideal - rej;
    const double eff = (eff_raw < 0.0) ? 0.0 : eff_raw;
    o.starved = o.throughput_tok_s < 0.9 * eff;
  }
}

__global__ void ttft_keys_kernel(const double* r_arr, const double* r_first, int64_t n, double* keys) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double f = r_first[i];
  keys[i] = (f == f) ? f - r_arr[i] : INFINITY;
}

// 1-based nearest rank ceil(pct/100 * n) clamped to [1, n] (n >= 1).
__device__ __forceinline__ int64_t nearest_rank(double pct, int64_t n) {
  int64_t r = static_cast<int64_t>(ceil(pct / 100.0 * static_cast<double>(n)));
  return r < 1 ? 1 : (r > n ? n : r);
}

// One warp per scenario.
__global__ void __launch_bounds__(256) percentile_kernel(const DScen* scen, int n_scen, const double* ttft_sorted,
                                                        const int64_t* rec_off, const int64_t* rec_len,
                                                        const double* rec_d, const int32_t* rec_c,
                                                        lt_sim_summary* out) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= n_scen) return;
  lt_sim_summary& o = out[s];
  if (o.status != LT_OK || o.degenerate) return;
  // --- TTFT: count of finite keys by binary search for the first +inf
  const double* t = ttft_sorted + scen[s].req_begin;
  const int64_t nr = scen[s].n_req;
  int64_t lo = 0, hi = nr;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (t[mid] == INFINITY)
      hi = mid;
    else
      lo = mid + 1;
  }
  const int64_t nt = lo;
  if (lane == 0) {
    o.ttft_p50_s = nt ? t[nearest_rank(50.0, nt) - 1] : 0.0;
    o.ttft_p99_s = nt ? t[nearest_rank(99.0, nt) - 1] : 0.0;
  }
  // --- ITL: weighted rank select over (value, weight) records sorted by value
  const int64_t b = rec_off[s], len = rec_len[s];
  long long total = 0;
  for (int64_t i = lane; i < len; i += 32) total += rec_c[b + i];
  for (int off = 16; off > 0; off >>= 1) total += __shfl_xor_sync(full, total, off);
  double p50 = 0.0, p99 = 0.0;
  if (total > 0) {
    const long long r50 = nearest_rank(50.0, total), r99 = nearest_rank(99.0, total);
    long long base = 0;  // weight of the records before this chunk
    bool got50 = false, got99 = false;
    for (int64_t c0 = 0; c0 < len && !got99; c0 += 32) {
      const int64_t i = c0 + lane;
      const long long w = (i < len) ? rec_c[b + i] : 0;
      long long incl = w;  // inclusive prefix within the chunk
      for (int off = 1; off < 32; off <<= 1) {
        const long long y = __shfl_up_sync(full, incl, off);
        if (lane >= off) incl += y;
      }
      const long long cum = base + incl;
      const unsigned h50 = __ballot_sync(full, !got50 && w > 0 && cum >= r50);
      const unsigned h99 = __ballot_sync(full, w > 0 && cum >= r99);
      if (h50) {
        const int src = __ffs(h50) - 1;
        p50 = __shfl_sync(full, (i < len) ? rec_d[b + (c0 + lane)] : 0.0, src);
        got50 = true;
      }
      if (h99) {
        const int src = __ffs(h99) - 1;
        p99 = __shfl_sync(full, (i < len) ? rec_d[b + (c0 + lane)] : 0.0, src);
        got99 = true;
      }
      base += __shfl_sync(full, incl, 31);
    }
  }
  if (lane == 0) {
    o.itl_p50_s = p50;
    o.itl_p99_s = p99;
  }
}

// Single-pass recording: each scenario's chunk list copied into one
// contiguous segment at rec_off[s] (the layout the segmented sort and
// percentile_kernel read), and its segment bounds. One warp per scenario.
__global__ void __launch_bounds__(256) rec_compact_kernel(int n_scen, const int32_t* chunk_next,
                                                          const int64_t* rec_total, const int64_t* rec_off,
                                                          const double* pool_d, const int32_t* pool_c, double* rec_d,
                                                          int32_t* rec_c, int32_t* seg_b, int32_t* seg_e) {
  const int s = static_cast<int>((blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (s >= n_scen) return;
  const int64_t total = rec_total[s], base = rec_off[s];
  if (lane == 0) {
    seg_b[s] = static_cast<int32_t>(base);
    seg_e[s] = static_cast<int32_t>(base + total);
  }
  int chunk = s;
  for (int64_t j0 = 0; j0 < total; j0 += kRecChunk) {
    const int64_t m = total - j0 < kRecChunk ? total - j0 : kRecChunk;
    const int64_t src = static_cast<int64_t>(chunk) * kRecChunk;
    for (int64_t i = lane; i < m; i += 32) {
      rec_d[base + j0 + i] = pool_d[src + i];
      rec_c[base + j0 + i] = pool_c[src + i];
    }
    chunk = chunk_next[chunk];
  }
}

}  // namespace lt
