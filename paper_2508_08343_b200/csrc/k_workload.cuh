// K0 workload generation: generate_arrivals (workload.cpp:170-211) on device.
//
// The reference draws, per adapter, Poisson arrivals from RngStream(seed,
// {1, id}) and Mean-mode lengths from RngStream(seed, {2, id})
// (workload.cpp:143-168, :174-199), then stable-sorts the merged list by
// (time, adapter_id) and numbers it (:204-210). Streams depend only on
// (seed, adapter_id), so they are generated once per key into rate-free
// tables shared by every scenario with that key:
//   E_j = -log1p(-u_j)            arrivals: t_j = t_{j-1} + E_j / rate  (bit-identical)
//   (zc_j, zs_j) Box-Muller pair  lengths:  in = round_clamp(mean_in + std_in*zc_j), out likewise with zs_j
//   tables_kernel  one thread per key (MT19937-64 state in local memory)
//   count_kernel   one thread per (scenario, adapter): arrivals in [0, duration)
//   merge_kernel   one warp per scenario: N-way merge by (time, adapter_id)
#pragma once
#include "lt_device.cuh"
#include "lt_rng.h"

namespace lt {

// Longest a key's tables may need to be: arrivals counted at the key's
// largest rate and duration bound every use (t_j is monotone in the rate:
// division and addition are monotone under round-to-nearest).
template <bool Fma>
__global__ void tables_kernel(DKey* keys, int n_keys, double* E, double2* Z) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_keys) return;
  DKey key = keys[k];
  Mt64 e;
  rng_stream_init(e, key.seed, 1, static_cast<uint64_t>(key.id));
  double t = 0.0;
  int j = 0;
  double* Ek = E + key.e_off;
  for (;;) {
    if (j >= key.cap) {
      key.overflow = 1;
      break;
    }
    const double x = exp_unit<Fma>(e);
    Ek[j++] = x;
    t = t + x / key.rate_max;
    if (t >= key.dur_max) break;
  }
  key.e_len = j;
  const int n = key.overflow ? j : j - 1;  // arrivals strictly inside the window
  rng_stream_init(e, key.seed, 2, static_cast<uint64_t>(key.id));
  double2* Zk = Z + key.z_off;
  for (int i = 0; i < n; ++i) {
    double sp;
    const double c = box_muller<Fma>(e, &sp);
    Zk[i] = make_double2(c, sp);
  }
  key.z_len = n;
  keys[k] = key;
}

// Arrivals of one (scenario, adapter): count t < duration (workload.cpp:179-183).
__global__ void count_kernel(const DScen* scen, const int32_t* pair_scen, const int32_t* pair_adp,
                             int64_t n_pairs, const DAdapter* adapters, const DKey* keys,
                             const double* E, int32_t* adp_count, unsigned long long* scen_count,
                             int32_t* overflow) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= n_pairs) return;
  const DScen& s = scen[pair_scen[p]];
  const DAdapter ad = adapters[s.adapter_begin + pair_adp[p]];
  const DKey& key = keys[ad.key];
  const double* Ek = E + key.e_off;
  double t = 0.0;
  int j = 0;
  for (;;) {
    if (j >= key.e_len) {
      atomicExch(overflow, 1);
      break;
    }
    t = t + Ek[j] / ad.rate;
    if (t >= s.duration) break;
    ++j;
  }
  adp_count[p] = j;
  atomicAdd(&scen_count[pair_scen[p]], static_cast<unsigned long long>(j));
}

// Request offsets of every scenario from the device exclusive scan.
__global__ void set_offsets_kernel(DScen* scen, int n_scen, const unsigned long long* count,
                                   const unsigned long long* off) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_scen) return;
  scen[i].req_begin = static_cast<int64_t>(off[i]);
  if (scen[i].generated && scen[i].status == LT_OK) scen[i].n_req = static_cast<int32_t>(count[i]);
}

// Arrival times of one (scenario, adapter) pair written unsorted at the pair's
// slot of the scenario segment; a stable segmented sort by time then realises
// the reference's stable_sort by (time, adapter_id, sequence)
// (workload.cpp:204-207): pairs are laid out in adapter-id order.
__global__ void expand_kernel(const DScen* scen, const int32_t* pair_scen, const int32_t* pair_adp,
                              int64_t n_pairs, const int64_t* pair_begin, const DAdapter* adapters,
                              const DKey* keys, const double* E, const int32_t* adp_count,
                              const unsigned long long* pair_excl, double* t_out,
                              unsigned long long* v_out) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= n_pairs) return;
  const int si = pair_scen[p];
  const DScen& s = scen[si];
  const int k = pair_adp[p];
  const DAdapter ad = adapters[s.adapter_begin + k];
  const double* Ek = E + keys[ad.key].e_off;
  const int64_t off = s.req_begin + static_cast<int64_t>(pair_excl[p] - pair_excl[pair_begin[si]]);
  const int n = adp_count[p];
  double t = 0.0;
  for (int j = 0; j < n; ++j) {
    t = t + Ek[j] / ad.rate;
    t_out[off + j] = t;
    v_out[off + j] = (static_cast<unsigned long long>(k) << 32) | static_cast<unsigned>(j);
  }
}

// Segment bounds of the generated scenarios (scripted / failed: empty).
__global__ void segments_kernel(const DScen* scen, int n_scen, int* seg_begin, int* seg_end) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_scen) return;
  const DScen& s = scen[i];
  const int b = static_cast<int>(s.req_begin);
  seg_begin[i] = b;
  seg_end[i] = (s.generated && s.status == LT_OK) ? b + s.n_req : b;
}

// Sorted (time, adapter, sequence) -> request arrays; lengths from the Z
// table of the adapter's (seed, id) key (sample_lengths, workload.cpp:162-166).
__global__ void __launch_bounds__(256) gather_kernel(const DScen* scen, int n_scen, const DAdapter* adapters,
                                                    const DKey* keys, const DLen* lens, const double2* Z,
                                                    const double* t_sorted, const unsigned long long* v_sorted,
                                                    double* r_arr, int32_t* r_in, int32_t* r_out,
                                                    int32_t* r_adp) {
  const int lane = threadIdx.x & 31;
  const int si = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (si >= n_scen) return;
  const DScen sc = scen[si];
  if (!sc.generated || sc.status != LT_OK) return;
  const DLen gl = lens[sc.length_param];
  for (int r = lane; r < sc.n_req; r += 32) {
    const int64_t g = sc.req_begin + r;
    const unsigned long long v = v_sorted[g];
    const int a = static_cast<int>(v >> 32);
    const int j = static_cast<int>(v & 0xffffffffULL);
    const DAdapter ad = adapters[sc.adapter_begin + a];
    const double2 z = Z[keys[ad.key].z_off + j];
    const DLen L = ad.length_param >= 0 ? lens[ad.length_param] : gl;
    r_arr[g] = t_sorted[g];
    r_adp[g] = a;
    r_in[g] = round_clamp_token(affine(L.mean_in, L.std_in, z.x));
    r_out[g] = round_clamp_token(affine(L.mean_out, L.std_out, z.y));
  }
}

// N-way merge of one scenario's adapter streams into request_id order.
// Per-lane cache of the lane's best head; one warp argmin per request.
__global__ void __launch_bounds__(256) merge_kernel(const DScen* scen, int n_scen,
                                                   const DAdapter* adapters, const DKey* keys,
                                                   const DLen* lens, const double* E,
                                                   const double2* Z, const int64_t* pair_begin,
                                                   const int32_t* adp_count, double* r_arr,
                                                   int32_t* r_in, int32_t* r_out, int32_t* r_adp,
                                                   int max_adapters) {
  extern __shared__ __align__(16) char smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int s = blockIdx.x * (blockDim.x >> 5) + warp;
  if (s >= n_scen) return;
  const DScen sc = scen[s];
  if (!sc.generated || sc.status != LT_OK) return;
  double* head_t = reinterpret_cast<double*>(smem) + static_cast<size_t>(warp) * max_adapters * 2;
  int32_t* head_j = reinterpret_cast<int32_t*>(head_t + max_adapters);
  const int N = sc.n_adapters;
  const int64_t pb = pair_begin[s];
  for (int a = lane; a < N; a += 32) {
    const DAdapter ad = adapters[sc.adapter_begin + a];
    head_j[a] = 0;
    head_t[a] = (adp_count[pb + a] > 0) ? 0.0 + E[keys[ad.key].e_off] / ad.rate : INFINITY;
  }
  __syncwarp();
  // lane-local best over adapters a = lane + 32 m
  auto local_best = [&](double* bt, int* ba) {
    double b = INFINITY;
    int bi = INT_MAX;
    for (int a = lane; a < N; a += 32) {
      const double t = head_t[a];
      if (t < b) {  // ascending a: strict < keeps the smaller id on ties
        b = t;
        bi = a;
      }
    }
    *bt = b;
    *ba = bi;
  };
  double mt;
  int ma;
  local_best(&mt, &ma);
  const DLen gl = lens[sc.length_param];
  for (int r = 0; r < sc.n_req; ++r) {
    double bt = mt;
    int ba = ma;
    for (int o = 16; o > 0; o >>= 1) {
      const double ot = __shfl_xor_sync(0xffffffffu, bt, o);
      const int oa = __shfl_xor_sync(0xffffffffu, ba, o);
      if (ot < bt || (ot == bt && oa < ba)) {
        bt = ot;
        ba = oa;
      }
    }
    const int owner = ba & 31;
    if (lane == owner) {
      const DAdapter ad = adapters[sc.adapter_begin + ba];
      const DKey& key = keys[ad.key];
      const int j = head_j[ba];
      const double2 z = Z[key.z_off + j];
      const DLen L = ad.length_param >= 0 ? lens[ad.length_param] : gl;
      const int64_t g = sc.req_begin + r;
      r_arr[g] = bt;
      r_adp[g] = ba;
      r_in[g] = round_clamp_token(affine(L.mean_in, L.std_in, z.x));
      r_out[g] = round_clamp_token(affine(L.mean_out, L.std_out, z.y));
      const int nj = j + 1;
      head_j[ba] = nj;
      head_t[ba] = (nj < adp_count[pb + ba]) ? bt + E[key.e_off + nj] / ad.rate : INFINITY;
      local_best(&mt, &ma);
    }
    __syncwarp();
  }
}

}  // namespace lt
