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
//   seed_kernel         one thread per stream: seed_seq -> MT19937-64 state (shared memory)
//   tables_draw_kernel  one warp per key: block twists + E / Box-Muller transforms in parallel
//   count_kernel        one thread per (scenario, adapter): arrivals in [0, duration)
//   expand_kernel + CUB stable segmented sort + gather_kernel: the merge by (time, adapter_id)
#pragma once
#include "lt_device.cuh"
#include "lt_rng.h"

namespace lt {

constexpr int kMtN = 312;  // MT19937-64 state words

// ---- K0a: seeding. RngStream(seed, {a, id}) = std::seed_seq over
// [seed_lo, seed_hi, a_lo, a_hi, id_lo, id_hi] -> mt19937_64::seed
// (rng.hpp:35-46; [rand.util.seedseq]). The generate() recurrence is strictly
// sequential, so it runs one thread per stream (two streams per key) with the
// 624-word array in shared memory (row stride 625: conflict-free both when
// every thread touches its own row and when a row is copied out), then the
// block writes each stream's state contiguously to `state`.
constexpr int kSeedThreads = 90;  // 90 rows x 625 words = 225 KB: three warps' worth of streams per SM
constexpr int kSeedStride = 625;
constexpr size_t kSeedSmem = sizeof(uint32_t) * kSeedThreads * kSeedStride;

// Steps [k0, k1) of one std::seed_seq::generate pass over the row, in a
// range where none of the touched indices wraps: the offsets of b[k+p],
// b[k+q] and of the next step's operands b[k+1], b[k+1+p], b[k+1+q] are
// compile-time constants (OP, OQ, O1, O1P, O1Q: the index minus k, already
// reduced mod n), so every access is one shared-memory op at an immediate
// offset and a step is the dependent chain plus three loads and three
// stores. Step k writes none of b[k+1], b[k+1+p], b[k+1+q] (q - p = 11), so
// the next step's operands are loaded one step ahead and the updates are
// plain stores. kFirst: the first loop (k < m = n); else the second
// (k + m, indices repeat modulo n). kV: steps 0..s, whose add term reads v.
template <bool kFirst, bool kV, int OP, int OQ, int O1, int O1P, int O1Q>
__device__ __forceinline__ void seed_seq_steps(uint32_t* b, int k0, int k1, uint32_t& x0, uint32_t& x1,
                                               uint32_t& x2, uint32_t& prev, const uint32_t* v) {
  constexpr int s = 6;
#pragma unroll 4
  for (int k = k0; k < k1; ++k) {
    uint32_t* bk = b + k;
    uint32_t r, w1, w2;
    if (kFirst) {
      const uint32_t r1 = 1664525u * seedseq_T(x0 ^ x1 ^ prev);
      uint32_t add = static_cast<uint32_t>(k);
      if (kV) add = (k == 0) ? static_cast<uint32_t>(s) : static_cast<uint32_t>(k) + v[k - 1];
      r = r1 + add;
      w1 = x1 + r1;
      w2 = x2 + r;
    } else {
      const uint32_t r3 = 1566083941u * seedseq_T(x0 + x1 + prev);
      r = r3 - static_cast<uint32_t>(k);
      w1 = x1 ^ r3;
      w2 = x2 ^ r;
    }
    x0 = bk[O1];
    x1 = bk[O1P];
    x2 = bk[O1Q];
    bk[OP] = w1;
    bk[OQ] = w2;
    bk[0] = r;
    prev = r;
  }
}

template <bool kFirst>
__device__ __forceinline__ void seed_seq_pass(uint32_t* b, uint32_t& prev, const uint32_t* v) {
  constexpr int n = 624, p = 306, q = 317;
  uint32_t x0 = b[0], x1 = b[p], x2 = b[q];
  // wrap points: k+1+q at k = 306, k+q at 307, k+1+p at 317, k+p at 318, k+1 at 623
  if (kFirst) {
    seed_seq_steps<true, true, p, q, 1, 1 + p, 1 + q>(b, 0, 7, x0, x1, x2, prev, v);  // 0 <= k <= s
    seed_seq_steps<true, false, p, q, 1, 1 + p, 1 + q>(b, 7, 306, x0, x1, x2, prev, v);
  } else {
    seed_seq_steps<false, false, p, q, 1, 1 + p, 1 + q>(b, 0, 306, x0, x1, x2, prev, v);
  }
  seed_seq_steps<kFirst, false, p, q, 1, 1 + p, 1 + q - n>(b, 306, 307, x0, x1, x2, prev, v);
  seed_seq_steps<kFirst, false, p, q - n, 1, 1 + p, 1 + q - n>(b, 307, 317, x0, x1, x2, prev, v);
  seed_seq_steps<kFirst, false, p, q - n, 1, 1 + p - n, 1 + q - n>(b, 317, 318, x0, x1, x2, prev, v);
  seed_seq_steps<kFirst, false, p - n, q - n, 1, 1 + p - n, 1 + q - n>(b, 318, 623, x0, x1, x2, prev, v);
  seed_seq_steps<kFirst, false, p - n, q - n, 1 - n, 1 + p - n, 1 + q - n>(b, 623, 624, x0, x1, x2, prev, v);
}

__device__ __forceinline__ void seed_seq_row(uint32_t* b, const uint32_t* v) {
  constexpr int n = 624;
  for (int k = 0; k < n; ++k) b[k] = 0x8b8b8b8bu;
  uint32_t prev = b[n - 1];
  seed_seq_pass<true>(b, prev, v);   // m = max(s + 1, n) = n
  seed_seq_pass<false>(b, prev, v);  // k + m, m = n: indices repeat modulo n
  // [rand.eng.mers] seed(q): an all-zero state (top w-r bits of x[0]) -> 2^(w-1)
  if ((b[1] == 0u) && ((b[0] & 0x80000000u) == 0u)) {
    bool zero = true;
    for (int k = 2; zero && k < n; ++k) zero = b[k] == 0u;
    if (zero) {
      b[0] = 0u;
      b[1] = 0x80000000u;
    }
  }
}

// keys[k0 .. k0 + nk): stream 2(k-k0) = {1, id}, 2(k-k0)+1 = {2, id}; stream t's
// 312-word state at state[312 t].
__global__ void __launch_bounds__(kSeedThreads) seed_kernel(const DKey* keys, int k0, int nk, uint64_t* state) {
  extern __shared__ uint32_t sb[];
  const int tid = threadIdx.x;
  const int base = blockIdx.x * kSeedThreads;
  const int t = base + tid;
  const int n_streams = 2 * nk;
  if (t < n_streams) {
    const DKey key = keys[k0 + (t >> 1)];
    const uint64_t a = (t & 1) ? 2 : 1;
    const uint64_t id = static_cast<uint64_t>(key.id);
    const uint32_t v[6] = {static_cast<uint32_t>(key.seed), static_cast<uint32_t>(key.seed >> 32),
                           static_cast<uint32_t>(a), static_cast<uint32_t>(a >> 32),
                           static_cast<uint32_t>(id), static_cast<uint32_t>(id >> 32)};
    seed_seq_row(sb + tid * kSeedStride, v);
  }
  __syncthreads();
  // copy-out row by row, the block's threads over a row's words
  // (conflict-free reads, coalesced writes, no per-word index division)
  const int ns = min(kSeedThreads, n_streams - base);
  uint32_t* dst = reinterpret_cast<uint32_t*>(state) + static_cast<size_t>(base) * 2 * kMtN;
  for (int r = 0; r < ns; ++r) {
    const uint32_t* src = sb + r * kSeedStride;
    uint32_t* out = dst + static_cast<size_t>(r) * 2 * kMtN;
#pragma unroll
    for (int j = tid; j < 2 * kMtN; j += kSeedThreads) out[j] = src[j];
  }
}

// One warp replaces st[0..311] by the next MT19937-64 state block: the
// standard's whole-array twist ([rand.eng.mers]) done in two parallel halves
// (i < 156 reads only old words; i >= 156 reads old words and the new
// st[i - 156]), every read before any write of a half.
__device__ __forceinline__ void mt64_twist_block(uint64_t* st, int lane) {
  constexpr uint64_t UM = 0xffffffff80000000ULL, LM = 0x7fffffffULL, MA = 0xb5026f5aa96619e9ULL;
  uint64_t nv[5];
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const int i = lane + 32 * r;
    if (i < 156) {
      const uint64_t y = (st[i] & UM) | (st[i + 1] & LM);
      nv[r] = st[i + 156] ^ (y >> 1) ^ ((y & 1ULL) ? MA : 0ULL);
    }
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const int i = lane + 32 * r;
    if (i < 156) st[i] = nv[r];
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const int i = 156 + lane + 32 * r;
    if (i < kMtN) {
      const uint64_t nx = (i + 1 < kMtN) ? st[i + 1] : st[0];
      const uint64_t y = (st[i] & UM) | (nx & LM);
      nv[r] = st[i - 156] ^ (y >> 1) ^ ((y & 1ULL) ? MA : 0ULL);
    }
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const int i = 156 + lane + 32 * r;
    if (i < kMtN) st[i] = nv[r];
  }
  __syncwarp();
}

__device__ __forceinline__ double mt64_unit(uint64_t w) {
  return static_cast<double>(mt64_temper(w) >> 11) * 0x1.0p-53;  // uniform01 (rng.hpp:51)
}

// ---- K0b: drawing, one warp per key: 312 outputs per block, transformed by all lanes.
// E: -log1p(-u) in parallel; only the stop rule t += E/rate_max >= dur_max
// (workload.cpp:179-183) is a sequential add chain (lane 0). Z: pair q of a
// block is (u[2q], u[2q+1]) exactly as normal() draws them (rng.hpp:57-71)
// unless some u1 == 0 forces a resample; then lane 0 redraws the stream
// sequentially with the reference's loop.
template <bool Fma>
__global__ void __launch_bounds__(128) tables_draw_kernel(DKey* keys, int k0, int nk, const uint64_t* state,
                                                          double* E, double2* Z, int32_t* any_overflow) {
  __shared__ uint64_t st_all[4][kMtN];
  __shared__ double buf_all[4][kMtN];
  __shared__ double q_all[4][kMtN];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int li = blockIdx.x * 4 + warp;
  if (li >= nk) return;
  uint64_t* st = st_all[warp];
  double* buf = buf_all[warp];
  double* qv = q_all[warp];
  const int k = k0 + li;
  DKey key = keys[k];
  key.overflow = 0;
  const uint64_t* src = state + static_cast<size_t>(li) * (2 * kMtN);
  // (unrolled: all of a lane's state loads in flight at once)
#pragma unroll
  for (int r = 0; r < (kMtN + 31) / 32; ++r) {
    const int w = lane + 32 * r;
    if (w < kMtN) st[w] = src[w];
  }
  __syncwarp();
  // ---- E table (arrivals stream {1, id})
  double* Ek = E + key.e_off;
  double t = 0.0;
  int j = 0, overflow = 0;
  for (bool done = false; !done;) {
    mt64_twist_block(st, lane);
    // Transform only the draws the stop rule is expected to reach (the rest of
    // the window at rate_max plus slack); the rest of the block only if the
    // running sum has not stopped by then.
    const double lam = (key.dur_max - __shfl_sync(0xffffffffu, t, 0)) * key.rate_max;
    int hi = kMtN;
    if (lam >= 0.0 && lam < static_cast<double>(kMtN)) hi = min(kMtN, static_cast<int>(lam + 4.0 * sqrt(lam) + 16.0));
    int lo = 0, take = kMtN, stop = 0;
    for (;;) {
      for (int w = lo + lane; w < hi; w += 32) {
        const double x = -glibc_log1p<Fma>(-mt64_unit(st[w]));
        buf[w] = x;
        qv[w] = x / key.rate_max;
      }
      __syncwarp();
      if (lane == 0) {
        for (int w = lo; w < hi; ++w) {
          if (j + w >= key.cap) {
            overflow = 1;
            take = w;
            stop = 1;
            break;
          }
          t = t + qv[w];
          if (t >= key.dur_max) {
            take = w + 1;
            stop = 1;
            break;
          }
        }
      }
      stop = __shfl_sync(0xffffffffu, stop, 0);
      if (stop || hi == kMtN) break;
      lo = hi;
      hi = kMtN;
    }
    take = __shfl_sync(0xffffffffu, take, 0);
    done = stop != 0;
    for (int w = lane; w < take; w += 32) Ek[j + w] = buf[w];
    j += take;
    __syncwarp();
  }
  overflow = __shfl_sync(0xffffffffu, overflow, 0);
  const int n = overflow ? j : j - 1;  // arrivals strictly inside the window
  // ---- Z table (lengths stream {2, id})
#pragma unroll
  for (int r = 0; r < (kMtN + 31) / 32; ++r) {
    const int w = lane + 32 * r;
    if (w < kMtN) st[w] = src[kMtN + w];
  }
  __syncwarp();
  double2* Zk = Z + key.z_off;
  bool slow = false;
  for (int p = 0; p < n; p += kMtN / 2) {
    mt64_twist_block(st, lane);
    bool zero = false;
    for (int q = lane; q < kMtN / 2 && p + q < n; q += 32) zero |= !(mt64_unit(st[2 * q]) > 0.0);
    if (__any_sync(0xffffffffu, zero)) {
      slow = true;
      break;
    }
    for (int q = lane; q < kMtN / 2 && p + q < n; q += 32) {
      const double u1 = mt64_unit(st[2 * q]);
      const double u2 = mt64_unit(st[2 * q + 1]);
      const double radius = sqrt(-2.0 * glibc_log<Fma>(u1));
      const double angle = 6.283185307179586 * u2;
      Zk[p + q] = make_double2(radius * glibc_cos<Fma>(angle), radius * glibc_sin<Fma>(angle));
    }
    __syncwarp();
  }
  if (slow && lane == 0) {
    Mt64 e;
    for (int w = 0; w < kMtN; ++w) e.x[w] = src[kMtN + w];
    e.i = 0;
    for (int i = 0; i < n; ++i) {
      double sp;
      const double c = box_muller<Fma>(e, &sp);
      Zk[i] = make_double2(c, sp);
    }
  }
  if (lane == 0) {
    key.e_len = j;
    key.z_len = n;
    key.overflow = overflow;
    keys[k] = key;
    if (overflow) atomicOr(any_overflow, 1);
  }
}

// ---- K0c: Full-mode decks, one warp per (key, D). Lane 0 runs seed_seq for
// the lengths stream {2, id} (rng.hpp:35-46) and every Fisher-Yates step
// (rng.hpp:86-91) with uniform_below's rejection (rng.hpp:76-82); the warp
// refills 312 tempered outputs at a time. After each shuffle the deck order
// is written as the list indices of the next D arrivals.
constexpr int kDeckSmemMax = 8192;

__global__ void __launch_bounds__(32) deck_kernel(const DKey* keys, const DDeck* decks, int32_t* tab,
                                                  int32_t* big_deck, const int64_t* big_off) {
  extern __shared__ __align__(16) char dsm[];
  uint32_t* sb = reinterpret_cast<uint32_t*>(dsm);                        // 624 words: seed_seq / state
  uint64_t* obuf = reinterpret_cast<uint64_t*>(dsm + 624 * sizeof(uint32_t));  // 312 tempered outputs
  int32_t* sdeck = reinterpret_cast<int32_t*>(obuf + kMtN);
  const int lane = threadIdx.x;
  const DDeck dk = decks[blockIdx.x];
  const DKey key = keys[dk.key];
  const int D = dk.D;
  const int64_t n = key.z_len;  // arrivals at the key's largest rate and window
  if (n <= 0) return;
  int32_t* deck = (D <= kDeckSmemMax) ? sdeck : big_deck + big_off[blockIdx.x];
  if (lane == 0) {
    const uint64_t id = static_cast<uint64_t>(key.id);
    const uint32_t v[6] = {static_cast<uint32_t>(key.seed), static_cast<uint32_t>(key.seed >> 32), 2u, 0u,
                           static_cast<uint32_t>(id), static_cast<uint32_t>(id >> 32)};
    seed_seq_row(sb, v);
  }
  for (int c = lane; c < D; c += 32) deck[c] = c;
  __syncwarp();
  uint64_t* st = reinterpret_cast<uint64_t*>(sb);
  int32_t* out = tab + dk.table_off;
  const int64_t nshuf = 1 + (n - 1) / D;
  int i = D;       // lane 0: Fisher-Yates position of the current shuffle
  int64_t k = 0;   // lane 0: shuffles completed
  for (;;) {
    mt64_twist_block(st, lane);
    for (int w = lane; w < kMtN; w += 32) obuf[w] = mt64_temper(st[w]);
    __syncwarp();
    int stop = 0;
    if (lane == 0) {
      int p = 0;
      while (k < nshuf) {
        if (i > 1) {
          if (p == kMtN) break;  // block exhausted: refill
          const uint64_t bound = static_cast<uint64_t>(i);
          const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
          const uint64_t draw = obuf[p++];
          if (draw >= limit) continue;  // rejected: redraw for the same bound
          const int j = static_cast<int>(draw % bound);
          const int32_t tmp = deck[i - 1];
          deck[i - 1] = deck[j];
          deck[j] = tmp;
          --i;
          continue;
        }
        const int64_t base = k * D;
        const int64_t cnt = (n - base < D) ? n - base : D;
        for (int64_t c = 0; c < cnt; ++c) out[base + c] = deck[c];
        ++k;
        i = D;
      }
      stop = k >= nshuf;
    }
    if (__shfl_sync(0xffffffffu, stop, 0)) break;
  }
}

// Arrivals of every (scenario, adapter) pair: the reference's t += E/rate
// loop (workload.cpp:179-183) with G lanes per pair: G table loads and
// divisions in parallel, the sum one add per draw in draw order, fed by
// shuffles. G = 32 for pairs with many draws (one pair per warp), G = 4 for
// sparse ones (eight pairs per warp: their dependent metadata loads overlap).
template <int G>
__global__ void __launch_bounds__(256) count_kernel(const DScen* scen, const int32_t* pair_scen,
                                                    const int32_t* pair_adp, int64_t n_pairs,
                                                    const DAdapter* adapters, const DKey* keys, const double* E,
                                                    int32_t* adp_count, unsigned long long* scen_count,
                                                    int32_t* overflow) {
  const int lane = threadIdx.x & 31;
  const int g = lane % G;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane - g));
  const int64_t p = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / G;
  if (p >= n_pairs) return;  // whole groups leave together
  const int si = pair_scen[p];
  const double duration = scen[si].duration;
  const DAdapter ad = adapters[scen[si].adapter_begin + pair_adp[p]];
  const DKey& key = keys[ad.key];
  const double* Ek = E + key.e_off;
  const int len = key.e_len;
  double t = 0.0;
  int count = -1;
  for (int j0 = 0; count < 0; j0 += G) {
    if (j0 >= len) {  // table exhausted before the window closed
      if (g == 0) atomicExch(overflow, 1);
      count = len;
      break;
    }
    const int j = j0 + g;
    const double q = (j < len) ? Ek[j] / ad.rate : 0.0;
    int hit = G;
#pragma unroll
    for (int k = 0; k < G; ++k) {
      t = t + __shfl_sync(gmask, q, k, G);
      if (hit == G && t >= duration) hit = k;
    }
    if (hit < G) {
      count = j0 + hit;
    } else if (j0 + G > len) {
      if (g == 0) atomicExch(overflow, 1);
      count = len;
    }
  }
  if (g == 0) {
    adp_count[p] = count;
    atomicAdd(&scen_count[si], static_cast<unsigned long long>(count));
  }
}

// Lanes per pair for a batch: sparse pairs (few expected draws) share warps.
inline int pair_group(double mean_draws) { return mean_draws < 24.0 ? 4 : 32; }

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
// (workload.cpp:204-207): pairs are laid out in adapter-id order. One warp
// group of G lanes per pair, the same sequential sum as count_kernel.
template <int G>
__global__ void __launch_bounds__(256) expand_kernel(const DScen* scen, const int32_t* pair_scen,
                                                     const int32_t* pair_adp, int64_t n_pairs,
                                                     const int64_t* pair_begin, const DAdapter* adapters,
                                                     const DKey* keys, const double* E, const int32_t* adp_count,
                                                     const unsigned long long* pair_excl, double* t_out,
                                                     unsigned long long* v_out) {
  const int lane = threadIdx.x & 31;
  const int g = lane % G;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane - g));
  const int64_t p = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / G;
  if (p >= n_pairs) return;
  const int si = pair_scen[p];
  const DScen& s = scen[si];
  const int k = pair_adp[p];
  const DAdapter ad = adapters[s.adapter_begin + k];
  const double* Ek = E + keys[ad.key].e_off;
  const int64_t off = s.req_begin + static_cast<int64_t>(pair_excl[p] - pair_excl[pair_begin[si]]);
  const int n = adp_count[p];
  double t = 0.0;
  for (int j0 = 0; j0 < n; j0 += G) {
    const int j = j0 + g;
    const double q = (j < n) ? Ek[j] / ad.rate : 0.0;
    double mine = 0.0;
#pragma unroll
    for (int u = 0; u < G; ++u) {
      t = t + __shfl_sync(gmask, q, u, G);
      if (u == g) mine = t;
    }
    if (j < n) {
      t_out[off + j] = mine;
      v_out[off + j] = (static_cast<unsigned long long>(k) << 32) | static_cast<unsigned>(j);
    }
  }
}

// Arrival merge by merge tree (replaces the per-scenario stable segmented
// sort): one block per generated scenario. Its arrivals sit in pair order --
// one list per adapter in ascending id, each list ascending in time (the
// reference's t += E/rate), so the reference's stable_sort by (time,
// adapter_id) (workload.cpp:204-207) is the stable merge of the lists in
// order. Round r merges adjacent runs of 2^r lists; an element of a left run
// lands after the right run's elements with a smaller time, an element of a
// right run after the left run's elements with a time <= its own (ties keep
// the lower adapter id first, within a list the draw order). Each element
// finds its place with one binary search in the partner run, all in
// parallel; the runs ping-pong between (t_a, v_a) and (t_b, v_b), and the
// result ends in (t_b, v_b), the layout gather_kernel reads.
__global__ void __launch_bounds__(512) merge_kernel(const DScen* scen, const int64_t* pair_begin,
                                                    const unsigned long long* pair_excl, double* t_a,
                                                    unsigned long long* v_a, double* t_b, unsigned long long* v_b,
                                                    const int32_t* order) {
  __shared__ int32_t off[kMaxAdapters + 1];
  // (order: the engine's cost-descending scenario order when known, so the
  // longest merges start in the first wave of blocks instead of the last)
  const int s = order ? order[blockIdx.x] : static_cast<int>(blockIdx.x);
  const DScen sc = scen[s];
  if (!sc.generated || sc.status != LT_OK || sc.n_req == 0) return;
  const int n = sc.n_req, np = sc.n_adapters;
  const int64_t rb = sc.req_begin;
  const int64_t p0 = pair_begin[s];
  const unsigned long long e0 = pair_excl[p0];
  for (int k = threadIdx.x; k < np; k += blockDim.x) off[k] = static_cast<int32_t>(pair_excl[p0 + k] - e0);
  if (threadIdx.x == 0) off[np] = n;
  __syncthreads();
  double* st = t_a + rb;
  unsigned long long* sv = v_a + rb;
  double* dt = t_b + rb;
  unsigned long long* dv = v_b + rb;
  for (int w = 1; w < np; w *= 2) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      int lo = 0, hi = np;  // the list holding position i: last k with off[k] <= i
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (off[mid] <= i) lo = mid;
        else hi = mid;
      }
      const int m = lo / w;           // its run this round
      const int a0 = (m & ~1) * w;    // the pair of runs (A, B)
      const int sA = off[a0], sB = off[min(a0 + w, np)], eB = off[min(a0 + 2 * w, np)];
      const double t = st[i];
      int pos;
      if ((m & 1) == 0) {  // in A: after B's elements with a smaller time
        int l = sB, h = eB;
        while (l < h) {
          const int mid = (l + h) >> 1;
          if (st[mid] < t) l = mid + 1;
          else h = mid;
        }
        pos = i + (l - sB);
      } else {  // in B: after A's elements with a time <= its own
        int l = sA, h = sB;
        while (l < h) {
          const int mid = (l + h) >> 1;
          if (st[mid] <= t) l = mid + 1;
          else h = mid;
        }
        pos = sA + (i - sB) + (l - sA);
      }
      dt[pos] = t;
      dv[pos] = sv[i];
    }
    __syncthreads();
    double* tt = st;
    st = dt;
    dt = tt;
    unsigned long long* vv = sv;
    sv = dv;
    dv = vv;
  }
  if (st != t_b + rb) {  // an even number of rounds: the result is still in (t_a, v_a)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      t_b[rb + i] = st[i];
      v_b[rb + i] = sv[i];
    }
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

// Arrival merge as two stable radix sorts over the whole batch: by time
// (values: positions 0..n-1), then by the scenario owning each position. The
// result is each scenario's range ordered by (time, position) -- the stable
// sort by time within the scenario (workload.cpp:204-207), since positions
// within a scenario are in (adapter, draw) order.
__global__ void iota_kernel(int32_t* v, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) v[i] = static_cast<int32_t>(i);
}

__global__ void scen_key_kernel(const DScen* scen, int n_scen, int64_t n, const int32_t* pos, uint32_t* key) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= n) return;
  const int64_t p = pos[g];
  int lo = 0, hi = n_scen - 1;  // last scenario with req_begin <= p
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (scen[mid].req_begin <= p)
      lo = mid;
    else
      hi = mid - 1;
  }
  key[g] = static_cast<uint32_t>(lo);
}

// Sorted (time, adapter, sequence) -> request arrays; lengths from the Z
// table of the adapter's (seed, id) key (sample_lengths, workload.cpp:162-166).
// One thread per request of the whole batch; its scenario is found by binary
// search over the (ascending) request offsets.
__global__ void __launch_bounds__(256) gather_kernel(const DScen* scen, int n_scen, int64_t total_req,
                                                    const DAdapter* adapters, const DKey* keys, const DLen* lens,
                                                    const double2* Z, const double* t_sorted,
                                                    const unsigned long long* v_sorted, double* r_arr,
                                                    int32_t* r_in, int32_t* r_out, int32_t* r_adp,
                                                    const DDeck* decks, const int32_t* deck_tab,
                                                    const int32_t* full, const int32_t* perm) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= total_req) return;
  int lo = 0, hi = n_scen - 1;  // last scenario with req_begin <= g
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (scen[mid].req_begin <= g)
      lo = mid;
    else
      hi = mid - 1;
  }
  const DScen& sc = scen[lo];
  if (!sc.generated || sc.status != LT_OK || g >= sc.req_begin + sc.n_req) return;
  const int64_t src = perm ? perm[g] : g;  // (perm: the radix-sorted positions)
  const unsigned long long v = v_sorted[src];
  const int a = static_cast<int>(v >> 32);
  const int j = static_cast<int>(v & 0xffffffffULL);
  const DAdapter ad = adapters[sc.adapter_begin + a];
  r_arr[g] = t_sorted[src];
  r_adp[g] = a;
  if (ad.deck >= 0) {  // Full mode: the shuffled deck's list entry
    const int64_t q = ad.list_off + deck_tab[decks[ad.deck].table_off + j];
    r_in[g] = full[2 * q];
    r_out[g] = full[2 * q + 1];
    return;
  }
  const double2 z = Z[keys[ad.key].z_off + j];
  const DLen L = lens[ad.length_param >= 0 ? ad.length_param : sc.length_param];
  r_in[g] = round_clamp_token(affine(L.mean_in, L.std_in, z.x));
  r_out[g] = round_clamp_token(affine(L.mean_out, L.std_out, z.y));
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
