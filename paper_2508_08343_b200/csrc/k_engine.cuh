// K1 engine_step + K2 metrics epilogue: one warp simulates one engine.
//
// Reference semantics (Appendix A of SURVEY.md), per iteration of
// Engine::run (engine.cpp:80-150):
//   idle jump (82-85) -> ingest arrivals <= clock (88-92) ->
//   complete_finished (kv_scheduler.cpp:238-259) -> decode_step_alloc
//   (:183-236) -> admit (:170-181, SlotPlan :49-98, scan_queue :109-166) ->
//   SlotCache::ensure_loaded (adapter_cache.cpp:40-78) -> lat_step
//   (estimators.cpp:110-139) -> emit one token per running request
//   (engine.cpp:128-135) -> advance clock, iteration cap (144-149).
//
// Warp mapping: every scalar of the engine is warp-uniform (held by all 32
// lanes); adapter sets (resident, claimed/needed, evicted, blocked, slotful)
// are 1024-bit masks with lane L owning adapters [32L, 32L+32); queues are
// scanned 32 entries per step with ballots, prefix popcounts and
// __match_any_sync; only slot claims/blocks and the memory stop are resolved
// one lane at a time, in queue order.
//
// Event-driven state: a running request never stores its token count. Its
// running entry keeps the iteration at which it retires (admission iteration
// + out - gen), so the per-iteration "+1 KV / +1 token for every running
// request" of the reference is O(1): the ledger grows by R, tokens by R, and
// a request's KV = in + gen is recovered from (fin - iteration) when it
// leaves. LIFO preemption is running.back() because running stays in
// admission order (kv_scheduler.cpp:159, :242-257).
#pragma once
#include <float.h>
#include <limits.h>

#include "lt_device.cuh"

namespace lt {

constexpr unsigned kFull = 0xffffffffu;

// Branch-layout hints: the engine loop is large enough that instruction fetch
// stalls show up (ncu no_instruction); rare paths are kept out of line.
#define LT_UNLIKELY(x) __builtin_expect(!!(x), 0)
#define LT_LIKELY(x) __builtin_expect(!!(x), 1)

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Bit `a` of a lane-distributed 1024-bit mask (a may differ per lane).
__device__ __forceinline__ bool mask_bit(uint32_t w, int a) {
  return (__shfl_sync(kFull, w, (a >> 5) & 31) >> (a & 31)) & 1u;
}
__device__ __forceinline__ void mask_set(uint32_t& w, int a, int lane) {
  if (lane == (a >> 5)) w |= 1u << (a & 31);
}
__device__ __forceinline__ void mask_clear(uint32_t& w, int a, int lane) {
  if (lane == (a >> 5)) w &= ~(1u << (a & 31));
}
// {in, out, next} of a fresh-queue node {in, out, next, adapter}.
__device__ __forceinline__ int3 node_head(const int4* node, int k) {
  const int2 xy = *reinterpret_cast<const int2*>(node + k);
  const int z = reinterpret_cast<const int*>(node + k)[2];
  return make_int3(xy.x, xy.y, z);
}

// Lowest set adapter index of a mask, or -1.
__device__ __forceinline__ int mask_lowest(uint32_t w) {
  const unsigned nz = __ballot_sync(kFull, w != 0);
  if (!nz) return -1;
  const int src = __ffs(nz) - 1;
  const uint32_t ws = __shfl_sync(kFull, w, src);
  return src * 32 + __ffs(ws) - 1;
}

__device__ __forceinline__ int warp_min_i(int v) { return __reduce_min_sync(kFull, v); }
__device__ __forceinline__ long long warp_sum_ll(long long v) {
  // one redux.sync when every lane's value fits in 26 bits (the sum then
  // fits in 32), else a shuffle tree
  if (__all_sync(kFull, v >= 0 && v < (1LL << 26)))
    return static_cast<long long>(__reduce_add_sync(kFull, static_cast<unsigned>(v)));
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// LRU victim: argmin over set bits of `cand` of (last_used, adapter_id);
// dense index order == adapter_id order. Adapters needed by the previous
// ensure_loaded call still carry last_used == prev_now (lazy refresh).
static __device__ __noinline__ int lru_victim(uint32_t cand, uint32_t prev_needed, double prev_now,
                                          const double* last_used, int lane) {
  double best = DBL_MAX;
  int best_a = INT_MAX;
  uint32_t w = cand;
  while (w) {
    const int b = __ffs(w) - 1;
    w &= w - 1;
    const int a = lane * 32 + b;
    const double key = ((prev_needed >> b) & 1u) ? prev_now : last_used[a];
    if (key < best || (key == best && a < best_a)) {
      best = key;
      best_a = a;
    }
  }
  __syncwarp();
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(kFull, best, o);
    const int oa = __shfl_xor_sync(kFull, best_a, o);
    if (ob < best || (ob == best && oa < best_a)) {
      best = ob;
      best_a = oa;
    }
  }
  return best_a == INT_MAX ? -1 : best_a;
}

__device__ __forceinline__ uint64_t fold64(uint64_t h, uint64_t w) {
  h ^= w;
  h *= 0x100000001b3ULL;
  return h;
}

#ifdef LT_SCAN_STATS
#define LT_STAT(k) (++st[k])
#else
#define LT_STAT(k) ((void)0)
#endif

// Non-lane-mode helpers of the fresh scan (rare: more than 32 adapters can
// act), kept out of line so the hot loop stays compact in the instruction cache.
// Lane-local minimum of act_key over this lane's adapters a = lane + 32 m.
static __device__ __noinline__ int2 lane_best(const int32_t* act_key, int N, int lane) {
  int best = INT_MAX, bi = -1;
#pragma unroll 1
  for (int a = lane; a < N; a += 32) {
    const int k = act_key[a];
    if (k < best) {
      best = k;
      bi = a;
    }
  }
  return make_int2(best, bi);
}

// Lane-local minimum chain head over this lane's adapters a = lane + 32 m
// (q_head -1, an empty chain, compares above every id).
static __device__ __noinline__ int2 lane_best_head(const int32_t* q_head, int N, int lane) {
  int best = INT_MAX, bi = -1;
#pragma unroll 1
  for (int a = lane; a < N; a += 32) {
    const int k = q_head[a];
    if (static_cast<unsigned>(k) < static_cast<unsigned>(best)) {
      best = k;
      bi = a;
    }
  }
  return make_int2(best, bi);
}

// act_key for every adapter (round-robin layout: lane owns a = lane + 32 m,
// whose mask bit is bit `lane` of word m).
static __device__ __noinline__ void act_keys(int32_t* act_key, const int32_t* q_head, int N, int lane, uint32_t blocked_w,
                                      uint32_t slotful_w, uint32_t claimed_w, uint32_t nonempty_w, bool mass,
                                      bool only_mass_exclusion) {
#pragma unroll 1
  for (int m = 0; m * 32 < N; ++m) {
    const uint32_t wb = __shfl_sync(kFull, blocked_w, m);
    const uint32_t ws = __shfl_sync(kFull, slotful_w, m);
    const uint32_t wc = __shfl_sync(kFull, claimed_w, m);
    const uint32_t wn = __shfl_sync(kFull, nonempty_w, m);
    const int a = lane + 32 * m;
    if (a < N) {
      const bool excl = mass && ((ws >> lane) & 1u) && !((wc >> lane) & 1u);
      if (only_mass_exclusion) {
        if (excl) act_key[a] = INT_MAX;
      } else {
        const bool acting = ((wn >> lane) & 1u) && !((wb >> lane) & 1u) && !excl;
        act_key[a] = acting ? q_head[a] : INT_MAX;
      }
    }
  }
}

// Running-set tiers of one engine (shared-memory slots < run_cap, HBM beyond).
struct RunTiers {
  int4* runs;
  int4* run;
  int2* links;
  int2* linkg;
  int32_t* cal;
  int32_t* cmin;
  int run_cap;
};

// Stable compaction of the live running entries, then the retire calendar
// rebuilt for the new slots (next links by atomic head exchange, then each
// node's successor learns its predecessor). Rare, so out of line: it keeps
// the engine loop's instruction footprint small. Returns the new length.
static __device__ __noinline__ int compact_running(RunTiers t, int R_end, int lane) {
  auto get = [&](int pos) { return pos < t.run_cap ? t.runs[pos] : t.run[pos]; };
  auto lk = [&](int pos) -> int2& { return pos < t.run_cap ? t.links[pos] : t.linkg[pos]; };
  int w = 0;
  for (int base = 0; base < R_end; base += 32) {
    const int i = base + lane;
    const int4 e = (i < R_end) ? get(i) : make_int4(-1, INT_MAX, 0, 0);
    const unsigned lm = __ballot_sync(kFull, e.x >= 0);
    __syncwarp();  // every lane's read of this chunk precedes the stores into it
    if (e.x >= 0) {
      const int d = w + __popc(lm & lanemask_lt());
      if (d < t.run_cap)
        t.runs[d] = e;
      else
        t.run[d] = e;
    }
    w += __popc(lm);
    __syncwarp();
  }
  for (int b = lane; b < kCalBuckets; b += 32) {
    t.cal[b] = -1;
    t.cmin[b] = INT_MAX;
  }
  __syncwarp();
  for (int i = lane; i < w; i += 32) {
    const int fin = get(i).y;
    lk(i) = make_int2(atomicExch(&t.cal[fin & (kCalBuckets - 1)], i), -1);
    atomicMin(&t.cmin[fin & (kCalBuckets - 1)], fin);
  }
  __syncwarp();
  for (int i = lane; i < w; i += 32) {
    const int nx = lk(i).x;
    if (nx >= 0) lk(nx).y = i;
  }
  __syncwarp();
  return w;
}

// Preempted-queue ring (shared-memory slots < kPqSmem, HBM beyond).
struct PqRing {
  int4* pqs;
  int4* pq;
  int pq_h;
  int pq_cap;
};

// A preempted request inserted into waiting_preempted ordered by (arrival,
// request_id) (kv_scheduler.cpp:206-215) at a position inside the queue: the
// backward scan for the first entry that does not sort after it, then the
// tail shifted by one (back to front). Out of line: the append / prepend
// cases cover every victim of generated workloads.
static __device__ __noinline__ void pq_insert_middle(PqRing q, int Wp, int4 ent, bool ids_sorted, const double* arr,
                                              int lane) {
  auto slot = [&](int i) {
    const int j = q.pq_h + i;
    return j >= q.pq_cap ? j - q.pq_cap : j;
  };
  auto get = [&](int i) {
    const int j = slot(i);
    return j < kPqSmem ? q.pqs[j] : q.pq[j];
  };
  auto put = [&](int i, int4 e) {
    const int j = slot(i);
    if (j < kPqSmem)
      q.pqs[j] = e;
    else
      q.pq[j] = e;
  };
  const int idx = ent.x;
  const double a_idx = arr[idx];
  int pos = 0;
  for (int hi = Wp; hi > 0; hi -= 32) {
    const int i = hi - 32 + lane;
    bool greater = false;  // entry i sorts after the victim
    if (i >= 0) {
      const int j = get(i).x;
      if (ids_sorted) {
        greater = idx < j;
      } else {
        const double aj = arr[j];
        greater = (a_idx < aj) || (a_idx == aj && idx < j);
      }
    }
    const unsigned notg = __ballot_sync(kFull, i >= 0 && !greater);
    if (notg) {
      pos = hi - 32 + (31 - __clz(notg)) + 1;
      break;
    }
  }
  for (int hi = Wp; hi > pos; hi -= 32) {
    const int lo = max(pos, hi - 32);
    const int i = lo + lane;
    int4 e;
    if (i < hi) e = get(i);
    __syncwarp();
    if (i < hi) put(i + 1, e);
    __syncwarp();
  }
  if (lane == 0) put(pos, ent);
  __syncwarp();
}

struct WarpEngine {
#ifdef LT_SCAN_STATS
  // diagnostics build: fresh scans, stop-cache hits, non-lane scans,
  // lane-set rebuilds, scan events, fresh admissions
  long long st[6] = {0, 0, 0, 0, 0, 0};
#endif
  // --- warp-uniform scalars
  double clock = 0.0, prev_now = 0.0, duration = 0.0;
  int64_t used = 0, cap = 0;
  int32_t iter = 0, iter_cap = 0;
  int32_t R = 0, Wp = 0, Wf = 0, ingest = 0, n_req = 0;
  int32_t resident_count = 0, G = 1, N = 1;
  int32_t R_end = 0;  // running array length incl. tombstones (x = -1)
  int32_t waived = -1;
  int32_t status = LT_OK, status_kind = LT_K_NONE;
  int64_t status_a = 0, status_b = 0;
  int32_t truncated = 0;
  long long finished = 0, preempts = 0, loads_n = 0, tok_win = 0, tok_tot = 0;
  long long sum_r = 0, sum_v = 0, sum_a = 0, sum_m = 0;
  uint64_t digest = 0xcbf29ce484222325ULL;
  // --- per-lane words of adapter masks
  uint32_t slotful_w = 0, resident_w = 0, claimed_w = 0, prev_needed_w = 0;
  uint32_t nonempty_w = 0;  // adapters with a non-empty fresh chain
  // --- scan-local SlotPlan state
  uint32_t evicted_w = 0, blocked_w = 0;
  int32_t free_slots = 0;
  // --- report pass: bases of this scenario's load-event and stint-log rows
  int64_t ld_base = 0, sl_base = 0;
  int32_t sl_n = 0;
  // --- pointers
  int64_t rb = 0, ab = 0;
  int lane = 0;
  double* last_used = nullptr;
  int32_t* run_cnt = nullptr;
  // fresh queue = per-adapter FIFO chains in request-id order (+ oversized
  // FIFO); q_head[a] is adapter a's first request not yet admitted, and the
  // chain is non-empty (nonempty_w) while that request has arrived (q_head in
  // [0, ingest)). Linked builds (kLinks) take the links from link_kernel and
  // may leave a head that has not arrived yet; the others append arrivals at
  // q_tail (-1: empty), so their heads have always arrived.
  int32_t* q_head = nullptr;
  int32_t* q_tail = nullptr;
  int32_t* act_key = nullptr;  // scan-local: chain head if the adapter can act, else INT_MAX
  // Lane mode of the fresh scan (<= 32 acting adapters), persistent across
  // scans: lane L owns adapter pl_a (-1: none) whose chain head is pl_k with
  // node fields pl_nd {in, out, next} (loaded without the adapter word, whose
  // dead register would otherwise be reused while the load is in flight and
  // stall the warp on it); pl_sf / pl_cl are its slot-needing /
  // claimed flags. built_w is the lane's word of the owned-adapter set.
  int32_t pl_a = -1, pl_k = INT_MAX;
  int3 pl_nd = make_int3(0, 0, -1);
  bool pl_sf = false, pl_cl = false, pl_valid = false;
  uint32_t built_w = 0;
  // Fresh admissions of the current iteration (first-token times): lane j
  // holds the j-th request id; n_fresh > 32 falls back to a running-set walk.
  int32_t fresh_id = 0, n_fresh = 0;
  // Re-admissions from the preempted queue this iteration (recording pass).
  int32_t readmit_id = 0, n_readmit = 0;
  // Retire calendar: cal[b] heads a doubly linked list ({next, prev} per
  // slot: links[] for shared slots, linkg[] for global ones; prev -1 at the
  // head) of the running slots whose retire iteration is = b mod kCalBuckets.
  // cmin[b] is a lower bound on the bucket's retire iterations (INT_MAX when
  // empty; exact after each walk), so buckets holding only later laps are
  // neither walked nor mistaken for the next retirement.
  int32_t* cal = nullptr;
  int32_t* cmin = nullptr;
  int2* links = nullptr;
  int2* linkg = nullptr;
  int32_t ov_head = 0, ov_tail = 0;
  // fresh-scan stop cache (see scan_fresh)
  int32_t last_stop = -1;
  int64_t last_stop_demand = 0;
  uint32_t act_epoch = 0, stop_epoch = 0;
  bool stop_mass = false;
  int4* run = nullptr;   // global tier of the running set (positions >= run_cap)
  int4* runs = nullptr;  // shared-memory tier (positions < run_cap)
  int32_t run_cap = 0;
  // Preempted queue: a ring of pq_cap slots holding {request, adapter|over,
  // demand, remaining tokens}; logical entry i is ring slot pq_h + i (mod
  // pq_cap). Ring slots < kPqSmem live in shared memory (pqs), the rest in HBM.
  int4* pq = nullptr;
  int4* pqs = nullptr;
  int32_t pq_h = 0, pq_cap = 1;
  bool ids_sorted = true;  // request ids follow arrival order: (arrival, id) order == id order
  int4* node = nullptr;  // per arrived fresh request: {in, out, next chained (-1: none), adapter}
  int32_t* ov = nullptr;

  __device__ __forceinline__ void fail(int32_t code, int32_t kind, int64_t a, int64_t b) {
    status = code;
    status_kind = kind;
    status_a = a;
    status_b = b;
  }

  __device__ __forceinline__ bool claimed(int a) const { return mask_bit(claimed_w, a); }

  // An adapter left the running batch: its slot is no longer claimed.
  __device__ __forceinline__ void release_adapter(int a, bool dec_to_zero) {
    if (dec_to_zero) {
      mask_clear(claimed_w, a, lane);
      ++act_epoch;
    }
  }

  __device__ __forceinline__ bool pool_any() const {
    return __any_sync(kFull, (resident_w & ~claimed_w & ~evicted_w) != 0);
  }

  __device__ __forceinline__ void block_adapter(int a) {
    mask_set(blocked_w, a, lane);
  }

  // SlotPlan::can_claim (kv_scheduler.cpp:68-72), warp-uniform a.
  __device__ __forceinline__ bool can_claim(int a) const {
    const uint32_t pool = resident_w & ~claimed_w & ~evicted_w;
    const bool in_claimed = mask_bit(claimed_w, a);
    const bool in_pool = mask_bit(pool, a);
    if (in_claimed || in_pool) return true;
    if (free_slots > 0) return true;
    return __any_sync(kFull, pool != 0);
  }

  // SlotPlan::claim (kv_scheduler.cpp:74-88).
  __device__ __forceinline__ void claim(int a) {
    if (mask_bit(claimed_w, a)) return;
    const uint32_t pool = resident_w & ~claimed_w & ~evicted_w;
    if (!mask_bit(pool, a)) {
      if (free_slots > 0) {
        --free_slots;
      } else {
        const int v = lru_victim(pool, prev_needed_w, prev_now, last_used, lane);
        if (v >= 0) mask_set(evicted_w, v, lane);
      }
    }
    mask_set(claimed_w, a, lane);
    ++act_epoch;
  }

  // Running set = run[0, R_end) in admission order with tombstones (x = -1)
  // for retired entries; cmin[c] bounds the retire iteration of chunk c from
  // below, so an iteration only touches the chunks that hold a retiree. The
  // last entry is always live (trim), so LIFO preemption pops run[R_end-1].
  // Running-set slot `pos`: the first run_cap slots live in shared memory.
  // (separate accesses per tier keep the shared one an LDS/STS, not a generic access)
  __device__ __forceinline__ int4 run_get(int pos) const {
    int4 v;
    if (pos < run_cap)
      v = runs[pos];
    else
      v = run[pos];
    return v;
  }
  __device__ __forceinline__ void run_put(int pos, int4 e) const {
    if (pos < run_cap)
      runs[pos] = e;
    else
      run[pos] = e;
  }

  __device__ __forceinline__ int pq_slot(int i) const {
    const int j = pq_h + i;
    return j >= pq_cap ? j - pq_cap : j;
  }
  __device__ __forceinline__ int4 pq_get(int i) const {
    const int j = pq_slot(i);
    int4 v;
    if (j < kPqSmem)
      v = pqs[j];
    else
      v = pq[j];
    return v;
  }
  __device__ __forceinline__ void pq_put(int i, int4 e) const {
    const int j = pq_slot(i);
    if (j < kPqSmem)
      pqs[j] = e;
    else
      pq[j] = e;
  }

  __device__ __forceinline__ int2 lk_get(int pos) const { return pos < run_cap ? links[pos] : linkg[pos]; }
  __device__ __forceinline__ void lk_put(int pos, int2 v) const {
    if (pos < run_cap)
      links[pos] = v;
    else
      linkg[pos] = v;
  }
  __device__ __forceinline__ void lk_next(int pos, int v) const {
    if (pos < run_cap)
      links[pos].x = v;
    else
      linkg[pos].x = v;
  }
  __device__ __forceinline__ void lk_prev(int pos, int v) const {
    if (pos < run_cap)
      links[pos].y = v;
    else
      linkg[pos].y = v;
  }

  // Link slot `pos` at the head of the bucket of its retire iteration (one lane).
  __device__ __forceinline__ void cal_push(int pos, int fin) const {
    const int b = fin & (kCalBuckets - 1);
    const int old = cal[b];
    lk_put(pos, make_int2(old, -1));
    if (old >= 0) lk_prev(old, pos);
    cal[b] = pos;
    cmin[b] = min(cmin[b], fin);
  }

  __device__ __forceinline__ void run_append(int4 e) {
    const int pos = R_end;
    if (lane == 0) {
      run_put(pos, e);
      cal_push(pos, e.y);
    }
    ++R_end;
    ++R;
  }

  // Unlink slot `pos` (retire iteration fin) from its bucket in O(1): a
  // popped (preempted) entry must not stay listed, its slot is reused.
  __device__ __forceinline__ void cal_unlink(int pos, int fin) {
    if (lane == 0) {
      const int2 l = lk_get(pos);
      if (l.y < 0) {
        const int b = fin & (kCalBuckets - 1);
        cal[b] = l.x;
        if (l.x < 0) cmin[b] = INT_MAX;
      } else
        lk_next(l.y, l.x);
      if (l.x >= 0) lk_prev(l.x, l.y);
    }
    __syncwarp();
  }

  // A lower bound on every live retire iteration: the first iteration
  // iter + j (j < kCalBuckets) whose bucket may retire something then, else
  // the least bucket minimum (every retirement is a lap or more away).
  __device__ __forceinline__ int next_retire_bound() const {
#pragma unroll 1
    for (int j0 = 0; j0 < kCalBuckets; j0 += 32) {
      const int it = iter + j0 + lane;
      const unsigned m = __ballot_sync(kFull, cmin[it & (kCalBuckets - 1)] <= it);
      if (m) return iter + j0 + __ffs(m) - 1;
    }
    int m = INT_MAX;
#pragma unroll 4
    for (int j = 0; j < kCalBuckets / 32; ++j) m = min(m, cmin[j * 32 + lane]);
    return __reduce_min_sync(kFull, m);
  }

  __device__ __forceinline__ void trim() {
    while (R_end > 0) {
      const int lo = max(0, R_end - 32);
      const int i = lo + lane;
      const bool live = i < R_end && run_get(i).x >= 0;
      const unsigned lm = __ballot_sync(kFull, live);
      if (lm) {
        R_end = lo + 32 - __clz(lm);
        break;
      }
      R_end = lo;
    }
    __syncwarp();  // the slots read above may be rewritten by lane 0's next append
  }

  // Stable compaction of the live entries (amortised: only when tombstones
  // outnumber live entries), out of line (compact_running).
  __device__ __forceinline__ void compact() {
    R_end = compact_running(RunTiers{runs, run, links, linkg, cal, cmin, run_cap}, R_end, lane);
  }

  // complete_finished (kv_scheduler.cpp:238-259): the retirees of this
  // iteration are exactly the current bucket's entries with y == iter (the
  // others are later laps and stay listed).
  __device__ __forceinline__ void retire(const EngineParams& P) {
    const int b = iter & (kCalBuckets - 1);
    const int m0 = cmin[b];
    int p = cal[b];
    if (m0 > iter) return;  // empty, or later laps only
    long long released = 0;
    int nf = 0, kept_head = -1, kept_tail = -1, kept_min = INT_MAX;
    while (p >= 0) {
      const int4 e = run_get(p);
      const int nxt = lk_get(p).x;
      if (e.y == iter) {
        const int idx = e.x;
        const int a = e.z & kAdapterMask;
        released += static_cast<long long>(e.w) - (idx == waived ? 1 : 0);
        const int left = run_cnt[a] - 1;
        __syncwarp();  // every lane has read run_cnt[a] and slot p before lane 0 rewrites them
        if (lane == 0) {
          P.r_phase[rb + idx] = kFinished;
          P.r_last[rb + idx] = clock;  // completion == the final emit (engine.cpp:134)
          run_cnt[a] = left;
          run_put(p, make_int4(-1, INT_MAX, 0, 0));
        }
        if (left == 0) release_adapter(a, true);
        ++nf;
      } else {
        if (lane == 0) {
          if (kept_tail < 0)
            kept_head = p;
          else
            lk_next(kept_tail, p);
          lk_prev(p, kept_tail);
        }
        kept_tail = p;
        kept_min = min(kept_min, e.y);
      }
      __syncwarp();
      p = nxt;
    }
    if (lane == 0) {
      if (kept_tail >= 0) lk_next(kept_tail, -1);
      cal[b] = kept_head;
      cmin[b] = kept_min;
    }
    __syncwarp();
    if (nf == 0) return;
    used -= released;
    finished += nf;
    sum_m += nf;
    waived = -1;
    R -= nf;
    if (R_end > 0 && run_get(R_end - 1).x < 0) trim();
    if (LT_UNLIKELY(R_end - R > max(R, 32))) compact();
  }

  // Insert a preempted request into waiting_preempted ordered by
  // (arrival, request_id) (kv_scheduler.cpp:206-215).
  // Victims are the latest admissions: fresh ones sort at the back, and
  // re-admitted preempted ones (the queue's oldest, admitted first) sort at
  // the front again -- both O(1) on the ring; other positions shift the tail.
  __device__ __forceinline__ void pq_insert(const EngineParams& P, int idx, int adapter_word, int demand,
                                            int rem) {
    const int4 ent = make_int4(idx, adapter_word, demand, rem);
    if (ids_sorted) {
      if (Wp == 0 || idx > pq_get(Wp - 1).x) {  // append
        if (lane == 0) pq_put(Wp, ent);
        __syncwarp();
        ++Wp;
        return;
      }
      if (idx < pq_get(0).x) {  // prepend
        pq_h = (pq_h == 0 ? pq_cap : pq_h) - 1;
        if (lane == 0) pq_put(0, ent);
        __syncwarp();
        ++Wp;
        return;
      }
    }
    pq_insert_middle(PqRing{pqs, pq, pq_h, pq_cap}, Wp, ent, ids_sorted, P.r_arr + rb, lane);
    ++Wp;
  }

  // decode_step_alloc (kv_scheduler.cpp:183-236).
  template <bool kRep>
  __device__ __forceinline__ bool alloc(const EngineParams& P) {
    if (R == 0) return true;
    int64_t demand = R;
    while (LT_UNLIKELY(used + demand > cap && R > 1)) {
      const int4 e = run_get(R_end - 1);
      cal_unlink(R_end - 1, e.y);
      --R;
      --R_end;
      trim();
      const int idx = e.x;
      const int a = e.z & kAdapterMask;
      const int outv = P.r_out[rb + idx];
      const int rem = e.y - iter;
      const int gen = outv - rem;
      const int in = e.w - outv;
      used -= static_cast<int64_t>(in) + gen;
      bool zero = false;
      if (lane == 0) {
        P.r_phase[rb + idx] = kPreempted;
        atomicAdd(&P.r_pre[rb + idx], 1);  // no return value: nothing waits on the load
        P.r_gen[rb + idx] = gen;
        P.r_last[rb + idx] = clock;
        zero = atomicSub(&run_cnt[a], 1) == 1;
        if (kRep && P.report) P.sl_log[sl_base + sl_n] = make_int2(idx, iter);
      }
      if constexpr (kRep) ++sl_n;
      zero = __shfl_sync(kFull, zero, 0);
      release_adapter(a, zero);
      const bool over = static_cast<int64_t>(in) + gen + 1 > cap;
      pq_insert(P, idx, a | (over ? kOverBit : 0), in + gen + 1, rem);
      ++preempts;
      ++sum_m;
      --demand;
    }
    if (used + demand > cap) {
      const int4 e = run_get(R_end - 1);  // the sole survivor
      const int rem = e.y - iter;
      if (rem > 1 || used + demand - 1 > cap) {
        fail(LT_ERR_SIMULATION, LT_K_SOLE_SURVIVOR, e.x, 0);
        return false;
      }
      waived = e.x;  // the final token needs no new reservation
      return true;
    }
    used += R;
    return true;
  }

  // scan_queue (kv_scheduler.cpp:109-166) over one waiting queue, in place.
  // Returns false if the scan stopped.
  // Entries carry their demand (in + gen + 1) and remaining tokens, so the
  // scan reads no per-request arrays.
  __device__ __forceinline__ int scan(const EngineParams& P, const int W, bool* keep_scanning) {
    int read = 0, write = 0;
    bool stopped = false;
    const unsigned lt_mask = lanemask_lt();
    while (read < W) {
      const int i = read + lane;
      const bool v = i < W;
      int4 e = make_int4(0, 0, 0, 0);
      if (v) e = pq_get(i);
      const int a = e.y & kAdapterMask;
      const bool over = v && (e.y & kOverBit);
      // every lane must execute the shuffles (no short-circuit around warp intrinsics)
      const bool sf_bit = mask_bit(slotful_w, a);
      const bool kb_bit = mask_bit(blocked_w, a);
      const bool sf = v && sf_bit;
      const bool kb = sf && kb_bit;
      const unsigned vm = __ballot_sync(kFull, v);
      const unsigned rejm = __ballot_sync(kFull, over);
      const unsigned kbm = __ballot_sync(kFull, v && !over && kb);
      unsigned cand = __ballot_sync(kFull, v && !over && !kb);
      int stop = 32;
      if (!P.priority && kbm) stop = __ffs(kbm) - 1;
      cand &= (stop >= 32) ? kFull : ((1u << stop) - 1);
      const int64_t demand = ((cand >> lane) & 1u) ? static_cast<int64_t>(e.z) : 0;
      const unsigned sfm = __ballot_sync(kFull, sf);
      unsigned admitted = 0;
      while (cand) {
        const int c = __ffs(cand) - 1;
        const int ac = __shfl_sync(kFull, a, c);
        const bool sfc = (sfm >> c) & 1u;
        if (sfc && !can_claim(ac)) {
          block_adapter(ac);
          // every later entry of this adapter is now a known-blocked keep
          cand &= ~__ballot_sync(kFull, v && a == ac);
          if (!P.priority) {
            stop = c;
            break;
          }
          continue;
        }
        const int64_t dc = __shfl_sync(kFull, demand, c);
        if (used + dc > cap) {
          stop = c;  // strict FCFS on memory
          break;
        }
        used += dc;
        if (sfc) claim(ac);
        if (lane == 0) run_cnt[ac] += 1;
        __syncwarp();
        admitted |= 1u << c;
        cand &= ~(1u << c);
      }
      const unsigned processed = (stop >= 32) ? kFull : ((1u << stop) - 1);
      const unsigned rejected = rejm & processed;
      const unsigned removed = rejected | admitted;
      {
        int fin_l = 0, s_l = 0;
        if ((admitted >> lane) & 1u) {
          fin_l = iter + e.w;    // + remaining tokens
          s_l = e.z - 1 + e.w;   // in + out
          P.r_phase[rb + e.x] = kRunning;
        }
        unsigned am = admitted;
        while (am) {
          const int src = __ffs(am) - 1;
          am &= am - 1;
          const int idx = __shfl_sync(kFull, e.x, src);
          const int ad = __shfl_sync(kFull, a, src);
          const int f = __shfl_sync(kFull, fin_l, src);
          const int sv = __shfl_sync(kFull, s_l, src);
          run_append(make_int4(idx, f, ad, sv));
          if (lane == (n_readmit & 31)) readmit_id = idx;
          ++n_readmit;
        }
      }
      if ((rejected >> lane) & 1u) P.r_phase[rb + e.x] = kRejected;
      __syncwarp();
      sum_m += __popc(admitted);
      const unsigned keep = vm & ~removed;
      __syncwarp();
      if ((keep >> lane) & 1u) pq_put(write + __popc(keep & lt_mask), e);
      write += __popc(keep);
      sum_v += (stop < 32) ? stop + 1 : __popc(vm);
      read += 32;
      __syncwarp();
      if (stop < 32) {
        stopped = true;
        break;
      }
    }
    if (stopped && read < W) {
      if (write < read) {
        for (int base = read; base < W; base += 32) {
          const int i = base + lane;
          int4 e;
          if (i < W) e = pq_get(i);
          __syncwarp();
          if (i < W) pq_put(write + (i - read), e);
          __syncwarp();
        }
      }
      write += W - read;
    }
    *keep_scanning = !stopped;
    return write;
  }

  // The preempted queue's head needs no slot decision and does not fit: the
  // scan (kv_scheduler.cpp:115-152) stops right there, admitting and
  // rejecting nothing (known-blocked adapters are reset per admit).
  __device__ __forceinline__ bool pq_stops_at_head() {
    const int4 e = pq_get(0);
    const int a = e.y & kAdapterMask;
    const bool sf = mask_bit(slotful_w, a), cl = mask_bit(claimed_w, a);
    if ((e.y & kOverBit) || (sf && !cl) || used + static_cast<int64_t>(e.z) <= cap) return false;
    ++sum_v;
    return true;
  }

  __device__ __forceinline__ void local_best(int* bkey, int* ba) const {
    const int2 r = lane_best(act_key, N, lane);
    *bkey = r.x;
    *ba = r.y;
  }

  __device__ __forceinline__ void build_act_keys(bool mass, bool only_mass_exclusion) {
    act_keys(act_key, q_head, N, lane, blocked_w, slotful_w, claimed_w, nonempty_w, mass, only_mass_exclusion);
  }

  // Lane mode (at most 32 acting adapters, act_w): reconcile the persistent
  // lane set with this acting set -- adapters whose chain filled or emptied,
  // claims and releases -- or rebuild it when many changed.
  __device__ __forceinline__ void enter_lane_mode(uint32_t act_w) {
    bool rebuild = !pl_valid;
    if (!rebuild && __any_sync(kFull, act_w != built_w)) {
      const uint32_t removed = built_w & ~act_w;
      if (__any_sync(kFull, removed != 0)) {
        const bool rm = mask_bit(removed, pl_a < 0 ? 0 : pl_a);
        if (pl_a >= 0 && rm) {
          pl_a = -1;
          pl_k = INT_MAX;
        }
        built_w &= ~removed;
      }
      uint32_t add = act_w & ~built_w;
      const int n_add = __reduce_add_sync(kFull, __popc(add));
      if (LT_UNLIKELY(n_add > 8)) {
        rebuild = true;
      } else {
#pragma unroll 1
        for (int k = 0; k < n_add; ++k) {
          const int a = mask_lowest(add);
          mask_clear(add, a, lane);
          const bool sfa = mask_bit(slotful_w, a);
          const int fl = __ffs(__ballot_sync(kFull, pl_a < 0)) - 1;  // exists: n_act <= 32
          if (lane == fl) {
            pl_a = a;
            pl_k = q_head[a];
            pl_nd = node_head(node, pl_k);
            pl_sf = sfa;
          }
          mask_set(built_w, a, lane);
        }
      }
    }
    if (LT_UNLIKELY(rebuild)) {
      LT_STAT(3);
      const int cnt_w = __popc(act_w);
      int pre = cnt_w;  // inclusive prefix over lanes
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(kFull, pre, o);
        if (lane >= o) pre += t;
      }
      const int excl = pre - cnt_w;  // exclusive prefix of this lane's word
      pl_a = -1;
      pl_k = INT_MAX;
#pragma unroll 1
      for (int m = 0; m * 32 < N; ++m) {
        const uint32_t wm = __shfl_sync(kFull, act_w, m);
        const int base = __shfl_sync(kFull, excl, m);
        const int k = lane - base;
        if (wm && k >= 0 && k < __popc(wm)) {
          pl_a = m * 32 + static_cast<int>(__fns(wm, 0, k + 1));
          pl_k = q_head[pl_a];
        }
      }
      if (pl_k != INT_MAX) pl_nd = node_head(node, pl_k);
      pl_sf = mask_bit(slotful_w, pl_a < 0 ? 0 : pl_a);
      built_w = act_w;
      pl_valid = true;
    }
    pl_cl = mask_bit(claimed_w, pl_a < 0 ? 0 : pl_a);  // claims/releases since the last scan
    __syncwarp();  // chain heads read above are rewritten by lane 0 as the scan admits
  }

  __device__ __forceinline__ void nonlane_best(bool direct, int* bkey, int* ba) const {
    const int2 r = direct ? lane_best_head(q_head, N, lane) : lane_best(act_key, N, lane);
    *bkey = r.x;
    *ba = r.y;
  }

  // scan_queue over waiting_fresh (kv_scheduler.cpp:109-166), event-driven.
  // The reference visits every waiting entry in order; here the fresh queue
  // is kept as per-adapter FIFO chains (request-id order), and the scan jumps
  // from one *acting* entry to the next in id order: an admission, the first
  // entry of an adapter that must be claimed or blocked, or the entry that
  // stops the scan. Entries of blocked adapters are kept without being
  // touched. Once no free slot and no idle resident remain (with the
  // loaded-adapter priority on), every unclaimed adapter is blocked for the
  // rest of the scan, so only claimed adapters' chains are walked. Oversized
  // entries (can never fit) sit in their own FIFO and are rejected up to the
  // stop point, as the reference rejects them when the scan passes them.
  template <bool kLinks>
  __device__ __forceinline__ void scan_fresh(const EngineParams& P) {
    LT_STAT(0);
    bool mass = P.priority && free_slots == 0 && !pool_any();
    // Steady-state shortcut: the previous fresh scan stopped on memory at
    // entry last_stop and no adapter has been claimed or released since (the
    // same adapters act, and every entry that arrived since sorts after it),
    // so this scan's first acting entry is last_stop again. If it still does
    // not fit, the scan stops right there, exactly as the full scan would.
    if (P.priority && last_stop >= 0 && stop_epoch == act_epoch && mass == stop_mass &&
        used + last_stop_demand > cap) {
      LT_STAT(1);
      ++sum_v;
      reject_oversized(P, last_stop);
      return;
    }
    last_stop = -1;
    // Acting adapters of this scan. When at most 32 can act (always for
    // N <= 32; and in the slot-starved steady state, where only the <= G
    // claimed adapters act), each lane owns one of them (lane mode) and an
    // event is one redux.sync argmin. The lane set persists across scans and
    // is reconciled with this scan's acting set (adapters whose chain filled
    // or emptied, claims and releases); otherwise act_key[] holds the heads.
    const uint32_t act_w = nonempty_w & ~blocked_w & ~(mass ? (slotful_w & ~claimed_w) : 0u);
    const int n_act = __reduce_add_sync(kFull, __popc(act_w));
    bool lane_mode = n_act <= 32;
    // Non-lane mode: lane L's best (head, adapter) over adapters a = L + 32 m,
    // from act_key[], or straight from the chain heads when every non-empty
    // chain acts ("direct": loaded-adapter priority with a free slot or an
    // idle resident left, so nothing is blocked or excluded -- the slot
    // turnover scan of a slot-starved engine).
    int lk = INT_MAX, la = -1;
    bool direct = false;
    // enter_lane_mode has one call site, at the head of the event loop (it is
    // large: a second inlined copy for the mid-scan switch doubled the scan's
    // code and its instruction-cache footprint)
    bool enter = lane_mode;
    uint32_t enter_w = act_w;
    if (LT_UNLIKELY(!lane_mode)) {
      LT_STAT(2);
      direct = P.priority && !mass && !__any_sync(kFull, blocked_w != 0);
      if (!direct) {
        build_act_keys(mass, false);
        __syncwarp();
      }
      nonlane_best(direct, &lk, &la);
    }
    int stop_id = INT_MAX;
    for (;;) {
      if (enter) {
        enter_lane_mode(enter_w);
        enter = false;
      }
      int id, a;
      bool sf, cl;
      int4 nd;  // {in, out, next, adapter}
      if (LT_LIKELY(lane_mode)) {
        const unsigned kmin = __reduce_min_sync(kFull, static_cast<unsigned>(pl_k));
        if (kmin == static_cast<unsigned>(INT_MAX)) break;
        const int src = __ffs(__ballot_sync(kFull, static_cast<unsigned>(pl_k) == kmin)) - 1;
        id = static_cast<int>(kmin);
        const int packed = pl_a | (pl_sf ? (1 << 29) : 0) | (pl_cl ? (1 << 28) : 0);
        const int pk = __shfl_sync(kFull, packed, src);
        a = pk & kAdapterMask;
        sf = (pk >> 29) & 1;
        cl = (pk >> 28) & 1;
        nd.x = __shfl_sync(kFull, pl_nd.x, src);
        nd.y = __shfl_sync(kFull, pl_nd.y, src);
        nd.z = __shfl_sync(kFull, pl_nd.z, src);
        nd.w = a;
      } else {
        const unsigned kmin = __reduce_min_sync(kFull, static_cast<unsigned>(lk));
        // (direct mode reads the raw heads, -1 sorting after every id; in the
        // linked builds one not yet arrived sorts after every arrived one)
        if (kLinks ? kmin >= static_cast<unsigned>(ingest) : kmin == static_cast<unsigned>(INT_MAX)) break;
        const int src = __ffs(__ballot_sync(kFull, static_cast<unsigned>(lk) == kmin)) - 1;
        id = static_cast<int>(kmin);
        a = __shfl_sync(kFull, la, src);
        nd = node[id];
        sf = mask_bit(slotful_w, a);
        cl = mask_bit(claimed_w, a);
      }
      const bool mine = lane_mode ? (pl_a == a) : (lane == (a & 31));  // the lane that owns a
      ++sum_v;
      LT_STAT(4);
      if (LT_UNLIKELY(sf && !cl) && !can_claim(a)) {
        block_adapter(a);
        if (!P.priority) {
          stop_id = id;
          break;
        }
        if (lane_mode) {
          if (mine) {
            pl_a = -1;
            pl_k = INT_MAX;
          }
          mask_clear(built_w, a, lane);
        } else if (direct) {  // (not reached: nothing blocks while a slot is free)
          __syncwarp();
          build_act_keys(mass, false);
          direct = false;
          __syncwarp();
          local_best(&lk, &la);
        } else if (mine) {
          act_key[a] = INT_MAX;
          local_best(&lk, &la);
        }
        continue;
      }
      const int64_t demand = static_cast<int64_t>(nd.x) + 1;
      if (used + demand > cap) {
        stop_id = id;  // strict FCFS on memory
        last_stop = id;
        last_stop_demand = demand;
        stop_epoch = act_epoch;
        stop_mass = mass;
        break;
      }
      used += demand;
      LT_STAT(5);
      const bool claiming = sf && !cl;
      if (LT_UNLIKELY(claiming)) claim(a);
      run_append(make_int4(id, iter + nd.y, a | kFreshBit, nd.x + nd.y));
      if (lane == (n_fresh & 31)) fresh_id = id;
      ++n_fresh;
      const int next = nd.z;
      if (lane == 0) {
        run_cnt[a] += 1;
        P.r_phase[rb + id] = kRunning;
        q_head[a] = next;
        if (!kLinks && next < 0) q_tail[a] = -1;
      }
      // the chain empties: no next request, or (linked builds) not arrived yet
      const bool gone = kLinks ? (next < 0 || next >= ingest) : next < 0;
      if (gone) mask_clear(nonempty_w, a, lane);
      --Wf;
      ++sum_m;
      // the lane set follows every chain it holds, in both modes
      if (pl_a == a) {
        if (lane_mode) pl_cl = pl_cl || claiming;
        if (gone) {
          pl_a = -1;
          pl_k = INT_MAX;
        } else {
          pl_k = next;
          pl_nd = node_head(node, next);  // in flight until this lane wins again
        }
      }
      if (gone) mask_clear(built_w, a, lane);
      if (!lane_mode && !direct && mine) act_key[a] = gone ? INT_MAX : next;
      if (LT_UNLIKELY(claiming)) {
        const bool mass2 = P.priority && free_slots == 0 && !pool_any();
        if (mass2 != mass) {
          mass = mass2;
          // every unclaimed adapter that needs a slot is now blocked
          if (lane_mode) {
            if (pl_a >= 0 && pl_sf && !pl_cl) {
              pl_a = -1;
              pl_k = INT_MAX;
            }
            built_w &= ~(slotful_w & ~claimed_w);
          } else {
            __syncwarp();
            const uint32_t aw = nonempty_w & ~blocked_w & ~(slotful_w & ~claimed_w);
            if (__reduce_add_sync(kFull, __popc(aw)) <= 32) {  // only claimed chains act now
              enter_w = aw;
              enter = true;
              lane_mode = true;
              continue;
            }
            if (direct) {
              build_act_keys(mass, false);
              direct = false;
            } else {
              build_act_keys(mass, true);
            }
            __syncwarp();
            local_best(&lk, &la);
            continue;
          }
        }
      }
      if (!lane_mode) {
        if (direct) {
          __syncwarp();  // lane 0's q_head store
          if (mine) nonlane_best(true, &lk, &la);
        } else if (mine) {
          local_best(&lk, &la);
        }
      }
      __syncwarp();
    }
    reject_oversized(P, stop_id);
  }

  // Oversized fresh entries in front of the stop point are rejected in place
  // (kv_scheduler.cpp:119-124): the reference rejects them when its scan
  // passes them.
  __device__ __forceinline__ void reject_oversized(const EngineParams& P, int stop_id) {
    while (ov_head < ov_tail) {
      const int i = ov_head + lane;
      const int id = i < ov_tail ? ov[i] : INT_MAX;
      const bool rej = i < ov_tail && id < stop_id;
      const unsigned m = __ballot_sync(kFull, rej);
      if (rej) P.r_phase[rb + id] = kRejected;
      const int n = __popc(m);  // ov is in id order: the rejected ones are a prefix
      ov_head += n;
      Wf -= n;
      sum_v += n;
      __syncwarp();
      if (n < 32) break;
    }
  }

  // SlotCache::ensure_loaded (adapter_cache.cpp:40-78) with needed = the
  // running batch's adapters (engine.cpp:108-114). Returns Σ load latency.
  // SimOptions.check_invariants (the debug engine build, kRep): the
  // reference's check_scheduler_invariants (kv_scheduler.cpp:261-290) on the
  // device state before the emit -- every running request Running and short
  // of its output, the ledger equal to the holds (in + generated + the
  // reserved next token, less a waived final reservation) and within
  // capacity, every preempted-queue entry Preempted. The first violation, in
  // the reference's order, fails the engine with its InternalError text.
  __device__ __forceinline__ bool check_invariants(const EngineParams& P) {
    long long held = 0;
    int bad_phase = INT_MAX, bad_gen = INT_MAX;  // lowest running-set slot of each kind
    for (int base = 0; base < R_end; base += 32) {
      const int i = base + lane;
      if (i >= R_end) continue;
      const int4 e = run_get(i);
      if (e.x < 0) continue;
      const int rem = e.y - iter;  // tokens left: the request has generated out - rem
      held += static_cast<long long>(e.w) - rem + 1 - (e.x == waived ? 1 : 0);
      if (P.r_phase[rb + e.x] != kRunning && i < bad_phase) bad_phase = i;
      if (rem < 1 && i < bad_gen) bad_gen = i;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) held += __shfl_xor_sync(kFull, held, d);
    const int first_phase = __reduce_min_sync(kFull, static_cast<unsigned>(bad_phase));
    const int first_gen = __reduce_min_sync(kFull, static_cast<unsigned>(bad_gen));
    const int first = first_phase < first_gen ? first_phase : first_gen;
    if (first != INT_MAX) {
      const int4 e = run_get(first);
      fail(LT_ERR_INTERNAL, first == first_phase ? LT_K_NOT_RUNNING : LT_K_PAST_OUTPUT, e.x, 0);
      return false;
    }
    if (held != used) {
      fail(LT_ERR_INTERNAL, LT_K_LEDGER_BALANCE, held, used);
      return false;
    }
    if (used > cap) {
      fail(LT_ERR_INTERNAL, LT_K_LEDGER_OVER, 0, 0);
      return false;
    }
    bool bad_pq = false;
    for (int i = lane; i < Wp; i += 32) bad_pq |= P.r_phase[rb + pq_get(i).x] != kPreempted;
    if (__any_sync(kFull, bad_pq)) {
      fail(LT_ERR_INTERNAL, LT_K_QUEUE_PHASE, 0, 0);
      return false;
    }
    return true;
  }

  template <bool kRep>
  __device__ __forceinline__ bool ensure_loaded(const EngineParams& P, double* loads_sum, int* loads_cnt) {
    const uint32_t needed_w = claimed_w;
    const int n_needed = __reduce_add_sync(kFull, __popc(needed_w));
    if (n_needed > G) {
      fail(LT_ERR_INTERNAL, LT_K_SLOT_OVERFLOW, n_needed, G);
      return false;
    }
    uint32_t missing_w = needed_w & ~resident_w;
    double sum = 0.0;
    int cnt = 0;
    for (;;) {
      const int a = mask_lowest(missing_w);
      if (a < 0) break;
      if (resident_count >= G) {
        const int v = lru_victim(resident_w & ~needed_w, prev_needed_w, prev_now, last_used, lane);
        if (v < 0) {
          fail(LT_ERR_INTERNAL, LT_K_NO_EVICTABLE, P.adapters[ab + a].id, 0);
          return false;
        }
        mask_clear(resident_w, v, lane);
        --resident_count;
      }
      mask_set(resident_w, a, lane);
      ++resident_count;
      const DAdapter& ad = P.adapters[ab + a];
      const double ll = ad.load_lat;
      if (ll != ll) {
        fail(LT_ERR_CONFIG, LT_K_NO_LOAD_ENTRY, ad.rank, 0);
        return false;
      }
      sum = sum + ll;
      if (kRep && P.report && lane == 0) P.ld[ld_base + loads_n + cnt] = DLoadEvent{clock, ll, ad.id, ad.rank};
      ++cnt;
      mask_clear(missing_w, a, lane);
    }
    // last_used refresh (adapter_cache.cpp:74-77), applied lazily: adapters
    // that just left the needed set keep the clock of their last use.
    uint32_t dropped = prev_needed_w & ~needed_w;
    while (dropped) {
      const int b = __ffs(dropped) - 1;
      dropped &= dropped - 1;
      last_used[lane * 32 + b] = prev_now;
    }
    __syncwarp();
    prev_needed_w = needed_w;
    prev_now = clock;
    *loads_sum = sum;
    *loads_cnt = cnt;
    return true;
  }
};

template <bool kRep, bool kRec, bool kQuietUnroll>
__device__ void engine_run(const EngineParams& P, int s, int slot, char* smem_warp) {
  // Linked ingest (link_kernel's links, no per-arrival append) in the latency,
  // report and recording builds: heavy C2 engines -7 % cycles per iteration.
  // The throughput builds keep the append (their C3 / C5 engines were 2-3 %
  // slower with the links at the 168-register cap). Their code is sensitive
  // to branch layout: `gone` below, written as !(next >= 0), flipped one
  // branch of the admission path and cost C3 / C5 3.5 % with otherwise
  // identical SASS.
  constexpr bool kLinks = !kQuietUnroll;
  const long long t_start = clock64();
#ifdef LT_PHASE_PROF
  long long ph[6] = {0, 0, 0, 0, 0, 0};
  long long tp = clock64();
#define LT_PH(k)                 \
  do {                           \
    const long long t_ = clock64(); \
    ph[k] += t_ - tp;            \
    tp = t_;                     \
  } while (0)
#else
#define LT_PH(k) \
  do {           \
  } while (0)
#endif
  WarpEngine E;
  E.lane = threadIdx.x & 31;
  const int lane = E.lane;
  const DScen sc = P.scen[s];
  lt_sim_summary o;
  memset(&o, 0, sizeof(o));
  if (sc.status != LT_OK) {  // failed before the loop (validation / Engine ctor): status only
    o.status = sc.status;
    o.status_kind = sc.status_kind;
    o.status_a = sc.status_a;
    o.status_b = sc.status_b;
    if (lane == 0) P.out[s] = o;
    return;
  }
  o.n_requests = sc.n_req;
  o.duration_s = sc.duration;
  o.slots = sc.G;
  o.served_adapters = sc.n_adapters;
  o.kv_capacity_tokens = sc.capacity;
  o.ideal_throughput_tok_s = sc.ideal;
  E.rb = sc.req_begin;
  E.ab = sc.adapter_begin;
  E.n_req = sc.n_req;
  E.N = sc.n_adapters;
  E.G = sc.G;
  E.cap = sc.capacity;
  E.duration = sc.duration;
  E.iter_cap = static_cast<int32_t>(sc.iter_cap > 0x7ff00000LL ? 0x7ff00000LL : sc.iter_cap);
  const int NA = P.max_adapters;
  E.last_used = reinterpret_cast<double*>(smem_warp);
  E.run_cnt = reinterpret_cast<int32_t*>(E.last_used + NA);
  E.q_head = E.run_cnt + NA;
  E.q_tail = E.q_head + NA;
  E.act_key = E.q_tail + NA;
  E.runs = reinterpret_cast<int4*>(E.act_key + NA);  // NA is a multiple of 32: 16-byte aligned
  E.run_cap = P.run_cap;
  E.cal = reinterpret_cast<int32_t*>(E.runs + E.run_cap);
  E.cmin = E.cal + kCalBuckets;
  E.links = reinterpret_cast<int2*>(E.cmin + kCalBuckets);
  E.pqs = reinterpret_cast<int4*>(E.links + E.run_cap);  // run_cap is a multiple of 32: 16-byte aligned
  const int64_t wsb = P.ws_per_scenario ? sc.req_begin : static_cast<int64_t>(slot) * P.ws_stride;
  E.run = P.ws_run + wsb;
  E.linkg = P.ws_link + wsb;
  E.pq = P.ws_pq + wsb;
  E.pq_cap = static_cast<int32_t>(P.ws_per_scenario ? (sc.n_req > 0 ? sc.n_req : 1) : P.ws_stride);
  E.ids_sorted = sc.ids_sorted != 0;
  E.node = P.ws_node + wsb;
  const int32_t* r_link = kLinks ? P.r_link + sc.req_begin : nullptr;
  E.ov = P.ws_ov + wsb;
  for (int a = lane; a < E.N; a += 32) {
    E.last_used[a] = 0.0;
    E.run_cnt[a] = 0;
    E.q_head[a] = -1;
    E.q_tail[a] = -1;
    E.act_key[a] = INT_MAX;
  }
  for (int b = lane; b < kCalBuckets; b += 32) {
    E.cal[b] = -1;
    E.cmin[b] = INT_MAX;
  }
  __syncwarp();
#pragma unroll 1
  for (int b = 0; b < 32; ++b) {
    const int a = lane * 32 + b;
    if (a < E.N && P.adapters[E.ab + a].rank > 0) E.slotful_w |= 1u << b;
  }
  __syncwarp();
  const bool capped_by_range = sc.iter_cap > 0x7ff00000LL;
  double pf_t = INFINITY;
  int pf_a = 0, pf_in = 0, pf_out = 0, pf_lk = 0;
  if (E.n_req > 0) {
    const int jc = lane < E.n_req ? lane : E.n_req - 1;
    pf_t = lane < E.n_req ? P.r_arr[E.rb + jc] : INFINITY;
    pf_a = P.r_adp[E.rb + jc];
    pf_in = P.r_in[E.rb + jc];
    pf_out = P.r_out[E.rb + jc];
    if constexpr (kLinks) pf_lk = r_link[jc];
  }
  double next_arr = __shfl_sync(kFull, pf_t, 0);  // arrival time of request `ingest`
  const int64_t rec_base = P.record ? P.rec_off[s] : 0;
  int64_t rec_n = 0;
  // single-pass recording (kRec): lane 0 appends to its chunk list
  int rc_cur = s, rc_pos = 0;
  int64_t rc_total = 0;
  bool rc_dead = false;
  auto rec_put = [&](double d, int c) {
    if (rc_dead) return;
    if (rc_pos == kRecChunk) {
      const int nxt = atomicAdd(P.rec_pool_next, 1);
      if (nxt >= P.rec_pool_chunks) {
        rc_dead = true;
        atomicExch(P.rec_overflow, 1);
        return;
      }
      P.rec_chunk_next[rc_cur] = nxt;
      rc_cur = nxt;
      rc_pos = 0;
    }
    const int64_t o = static_cast<int64_t>(rc_cur) * kRecChunk + rc_pos;
    P.rec_d[o] = d;
    P.rec_c[o] = c;
    ++rc_pos;
    ++rc_total;
  };
  // Consecutive records of one value are kept as one record of their summed
  // weight (the percentiles are a weighted rank select over the multiset, so
  // this is exact): a quiet stretch's equal emit gaps cost one record. Lane 0.
  double rl_d = 0.0;
  int rl_w = 0;
  auto rec_add = [&](double d, int c) {
    if (c <= 0) return;  // (weightless records never select a percentile)
    if (rl_w > 0 && d == rl_d && rl_w <= (1 << 30) - c) {
      rl_w += c;
      return;
    }
    if (rl_w > 0) rec_put(rl_d, rl_w);
    rl_d = d;
    rl_w = c;
  };
  int64_t tr_base = 0;
  if (kRep && P.report) {
    tr_base = P.tr_off[s];
    E.ld_base = P.ld_off[s];
    E.sl_base = P.sl_off[s];
  }

  while (true) {
    __syncwarp();
    if (E.R == 0 && E.Wp + E.Wf == 0) {
      if (E.ingest >= E.n_req) break;  // fully drained
      E.clock = E.clock < next_arr ? next_arr : E.clock;  // std::max(clock_, arrival)
    }
    // ingest arrivals <= clock (engine.cpp:88-92): append to the adapter's
    // FIFO chain, or to the oversized FIFO when in + 1 > capacity. The next
    // 32 arrivals are kept prefetched in registers (pf_*), so an iteration
    // with no arrival costs one comparison and one with arrivals no waiting.
    while (E.ingest < E.n_req && next_arr <= E.clock) {
      const int i = E.ingest + lane;
      const bool ok = (i < E.n_req) & (pf_t <= E.clock);
      const unsigned b = __ballot_sync(kFull, ok);
      const int n = (b == kFull) ? 32 : __ffs(~b) - 1;
      const int a_l = pf_a;
      const bool over_l = static_cast<int64_t>(pf_in) + 1 > E.cap;
      const unsigned live = (n >= 32) ? kFull : ((1u << n) - 1);
      const unsigned overm = __ballot_sync(kFull, over_l) & live;
      if ((overm >> lane) & 1u) E.ov[E.ov_tail + __popc(overm & lanemask_lt())] = i;
      E.ov_tail += __popc(overm);
      if constexpr (kLinks) {
        const bool chained = ((live & ~overm) >> lane) & 1u;
        const int nx = pf_lk & kLinkNone;
        if (chained) E.node[i] = make_int4(pf_in, pf_out, nx == kLinkNone ? -1 : nx, a_l);
        // A chain turns non-empty when its head arrives: the adapter's first
        // chained request, or the one an admission left in q_head before it
        // had arrived. (Two arrivals of one adapter never both qualify.)
        const bool first = (pf_lk & kLinkFirst) != 0;
        const bool head = chained && (first || E.q_head[a_l] == i);
        unsigned m = __ballot_sync(kFull, head);
        if (head && first) E.q_head[a_l] = i;
        while (m) {
          const int src = __ffs(m) - 1;
          m &= m - 1;
          mask_set(E.nonempty_w, __shfl_sync(kFull, a_l, src), lane);
        }
      } else {
        unsigned m = live & ~overm;
        if ((m >> lane) & 1u) E.node[i] = make_int4(pf_in, pf_out, -1, a_l);
        __syncwarp();
        while (m) {  // append to the adapter's chain, one arrival at a time
          const int src = __ffs(m) - 1;
          m &= m - 1;
          const int a = __shfl_sync(kFull, a_l, src);
          const int id = E.ingest + src;
          const int t = E.q_tail[a];
          __syncwarp();  // every lane has read q_tail[a] before lane 0 rewrites it
          if (lane == 0) {
            if (t < 0)
              E.q_head[a] = id;
            else
              reinterpret_cast<int*>(&E.node[t])[2] = id;
            E.q_tail[a] = id;
          }
          // the lane holding this chain's head node in registers sees its link
          if (E.pl_a == a && E.pl_k == t) E.pl_nd.z = id;
          mask_set(E.nonempty_w, a, lane);
          __syncwarp();
        }
      }
      E.Wf += n;
      E.ingest += n;
      E.sum_a += n;
      {  // slide the prefetch window by n
        const int srcl = lane + n;
        const double t2 = __shfl_sync(kFull, pf_t, srcl & 31);
        const int a2 = __shfl_sync(kFull, pf_a, srcl & 31);
        const int in2 = __shfl_sync(kFull, pf_in, srcl & 31);
        const int out2 = __shfl_sync(kFull, pf_out, srcl & 31);
        const int lk2 = kLinks ? __shfl_sync(kFull, pf_lk, srcl & 31) : 0;
        const double nxt = __shfl_sync(kFull, t2, 0);  // lane 0's new head when n < 32
        if (srcl < 32) {
          pf_t = t2;
          pf_a = a2;
          pf_in = in2;
          pf_out = out2;
          pf_lk = lk2;
        } else {
          const int j = E.ingest + lane;
          const int jc = j < E.n_req ? j : E.n_req - 1;
          pf_t = j < E.n_req ? P.r_arr[E.rb + jc] : INFINITY;
          pf_a = P.r_adp[E.rb + jc];
          pf_in = P.r_in[E.rb + jc];
          pf_out = P.r_out[E.rb + jc];
          if constexpr (kLinks) pf_lk = r_link[jc];
        }
        // (n == 32: lane 0 refilled from memory, wait for it)
        next_arr = (n < 32) ? nxt : __shfl_sync(kFull, pf_t, 0);
      }
      __syncwarp();
      if (n < 32) break;
    }
    __syncwarp();
    LT_PH(0);
    if (E.R > 0) E.retire(P);
    LT_PH(1);
    if (!E.template alloc<kRep>(P)) break;
    LT_PH(2);
    const int r_before = E.R_end;
    const int w_before = E.Wp + E.Wf, rcount_before = E.R;
    // admit (kv_scheduler.cpp:170-181): preempted queue first, then fresh
    E.free_slots = E.G - E.resident_count;
    E.evicted_w = 0;
    E.blocked_w = 0;
    E.n_fresh = 0;
    E.n_readmit = 0;
    {
      bool go = true;
      if (E.Wp > 0 && E.pq_stops_at_head()) {
        go = false;  // the scan would stop at its first entry (memory)
      } else {
        E.Wp = E.scan(P, E.Wp, &go);
      }
      LT_PH(3);
      if (go) E.template scan_fresh<kLinks>(P);
    }
    __syncwarp();
    LT_PH(4);
    if (kRep && P.report) {  // stint log: this iteration's admissions, in running-set order
      for (int base = r_before; base < E.R_end; base += 32) {
        const int i = base + lane;
        const int4 e = i < E.R_end ? E.run_get(i) : make_int4(-1, 0, 0, 0);
        const unsigned m = __ballot_sync(kFull, e.x >= 0);
        if (e.x >= 0) P.sl_log[E.sl_base + E.sl_n + __popc(m & lanemask_lt())] = make_int2(e.x, E.iter);
        E.sl_n += __popc(m);
      }
    }
    if (E.R == 0) {
      if (E.Wp + E.Wf != 0) {
        E.fail(LT_ERR_INTERNAL, LT_K_ADMISSION_STUCK, 0, 0);
        break;
      }
      continue;
    }
    if (kRep && P.check_invariants) {  // check_invariants_pre_emit (engine.cpp:105, :168-183)
      if (LT_UNLIKELY(P.inject_iteration == E.iter)) E.used += 1;  // test hook: a ledger fault
      if (!E.check_invariants(P)) break;
    }
    double loads = 0.0;
    int nl = 0;
    if (!E.template ensure_loaded<kRep>(P, &loads, &nl)) break;
    E.loads_n += nl;
    // lat_step (estimators.cpp:110-139), no contraction (--fmad=false).
    const int W = E.Wp + E.Wf;
    const int A = __reduce_add_sync(kFull, __popc(E.claimed_w));
    const double rr = static_cast<double>(E.R), ww = static_cast<double>(W);
    const double ratio_raw = static_cast<double>(E.G) / static_cast<double>(E.N);
    const double ratio = (1.0 < ratio_raw) ? 1.0 : ratio_raw;
    const double v = P.k1 * rr + P.k2 * ww + P.k3 * ww * ratio;
    const double sched = (v < 0.0) ? 0.0 : v;
    const double model = P.k4 * rr + P.k5;
    const double adapters = (A == 0) ? 1.0 : P.k6 * static_cast<double>(A) + P.k7;
    const double lat = sched + loads + model * adapters;
    const double emit = E.clock + lat;
    if (kRep && P.report) {  // IterationTraceRow (engine.cpp:137-140)
      if (lane == 0) {
        P.tr_time[tr_base + E.iter] = E.clock;
        P.tr_lat[tr_base + E.iter] = lat;
        P.tr_rwal[tr_base + E.iter] = make_int4(E.R, W, A, nl);
      }
    }
    if (kRec && P.rec_chunked) {  // the same ITL records, appended by lane 0
      if (lane == 0) rec_add(emit - E.clock, E.R - E.n_fresh - E.n_readmit);
      if (E.n_readmit <= 32) {
        const double dv = lane < E.n_readmit ? emit - P.r_last[E.rb + E.readmit_id] : 0.0;
        for (int j = 0; j < E.n_readmit; ++j) {
          const double x = __shfl_sync(kFull, dv, j);
          if (lane == 0) rec_add(x, 1);
        }
      } else {
        for (int base = r_before; base < E.R_end; base += 32) {
          const int i = base + lane;
          bool re = false;
          double dv = 0.0;
          if (i < E.R_end) {
            const int4 e = E.run_get(i);
            re = e.x >= 0 && !(e.z & kFreshBit);
            if (re) dv = emit - P.r_last[E.rb + e.x];
          }
          unsigned m = __ballot_sync(kFull, re);
          while (m) {
            const int j = __ffs(m) - 1;
            m &= m - 1;
            const double x = __shfl_sync(kFull, dv, j);
            if (lane == 0) rec_add(x, 1);
          }
        }
      }
    }
    if (LT_UNLIKELY(P.record)) {  // ITL multiset of compute_metrics (metrics.cpp:92-105)
      const int64_t r0 = rec_base + rec_n;
      if (lane == 0) {
        P.rec_d[r0] = emit - E.clock;
        P.rec_c[r0] = E.R - E.n_fresh - E.n_readmit;
      }
      int wrote = 1;
      if (E.n_readmit <= 32) {
        if (lane < E.n_readmit) {
          P.rec_d[r0 + 1 + lane] = emit - P.r_last[E.rb + E.readmit_id];
          P.rec_c[r0 + 1 + lane] = 1;
        }
        wrote += E.n_readmit;
      } else {  // this iteration's admissions without the fresh bit
        for (int base = r_before; base < E.R_end; base += 32) {
          const int i = base + lane;
          bool re = false;
          int idx = 0;
          if (i < E.R_end) {
            const int4 e = E.run_get(i);
            re = e.x >= 0 && !(e.z & kFreshBit);
            idx = e.x;
          }
          const unsigned m = __ballot_sync(kFull, re);
          if (re) {
            const int64_t o = r0 + wrote + __popc(m & lanemask_lt());
            P.rec_d[o] = emit - P.r_last[E.rb + idx];
            P.rec_c[o] = 1;
          }
          wrote += __popc(m);
        }
      }
      rec_n += wrote;
    }
    // first tokens of this iteration's fresh admissions (engine.cpp:131)
    if (LT_LIKELY(E.n_fresh <= 32)) {
      if (lane < E.n_fresh) P.r_first[E.rb + E.fresh_id] = emit;
    } else {
      for (int i = r_before + lane; i < E.R_end; i += 32) {
        const int4 e = E.run_get(i);
        if (e.z & kFreshBit) P.r_first[E.rb + e.x] = emit;
      }
    }
    __syncwarp();
    E.tok_tot += E.R;
    if (emit <= E.duration) E.tok_win += E.R;
    E.sum_r += E.R;
    if (LT_UNLIKELY(P.want_digest)) {
      E.digest = fold64(E.digest, static_cast<uint32_t>(E.R) | (static_cast<uint64_t>(static_cast<uint32_t>(W)) << 32));
      E.digest = fold64(E.digest, static_cast<uint32_t>(A) | (static_cast<uint64_t>(static_cast<uint32_t>(nl)) << 32));
      E.digest = fold64(E.digest, static_cast<uint64_t>(__double_as_longlong(lat)));
    }
    E.clock = emit;
    ++E.iter;
    LT_PH(5);
    if (LT_UNLIKELY(E.iter >= E.iter_cap)) {
      if (capped_by_range) {
        E.fail(LT_ERR_UNSUPPORTED, LT_K_ITERATION_RANGE, E.iter, 0);
      } else {
        E.truncated = 1;
      }
      break;
    }
    // Quiet stretch. This iteration's admission scan admitted and rejected
    // nothing, so until the next arrival (engine.cpp:88-92), the next
    // retirement (kv_scheduler.cpp:245), the next preemption
    // (kv_scheduler.cpp:190: used + R > cap) or the iteration cap, every
    // iteration of the reference repeats the same decisions: the same
    // SlotPlan (resident/claimed sets unchanged), a scan that stops at the
    // same entry (memory only tightens) or keeps the same slot-blocked
    // entries, no loads, and the same (R, W, A) -> the same lat_step. Such
    // iterations only advance the clock by `lat` (one rounded add each, as
    // the reference does), grow the ledger by R and count R tokens.
    if (E.Wp + E.Wf == w_before && E.R == rcount_before && E.waived < 0 &&
        (E.ingest >= E.n_req || next_arr > E.clock) && E.used + E.R <= E.cap &&
        E.cmin[E.iter & (kCalBuckets - 1)] > E.iter) {
      const long long n_fin = static_cast<long long>(E.next_retire_bound()) - E.iter;
      const long long n_mem = (E.cap - E.used) / E.R;
      const long long n_cap = static_cast<long long>(E.iter_cap) - 1 - E.iter;
      long long n_max = n_fin < n_mem ? n_fin : n_mem;
      n_max = n_max < n_cap ? n_max : n_cap;
      const double t_next = E.ingest < E.n_req ? next_arr : INFINITY;
      if (n_max > 0 && t_next > E.clock) {
        const double lat_q = sched + model * adapters;  // loads == 0
        double clk = E.clock, start = E.clock;
        int n = 0, win = 0;
        if (kQuietUnroll && !kRep && !kRec && !P.record && !P.want_digest && lat_q >= 0.0) {
          // Four iterations per loop test: the adds are the reference's, one
          // after the other; the clock only grows, so t_next above the clock
          // before the block's last add covers the block's other tests.
          // (Throughput variants only: C3 / C5 engines -3 %, the latency
          // variant's C2 critical path +0.6 %.)
          while (n + 4 <= n_max) {
            const double c1 = clk + lat_q;
            const double c2 = c1 + lat_q;
            const double c3 = c2 + lat_q;
            if (!(t_next > c3)) break;
            const double c4 = c3 + lat_q;
            win += (c1 <= E.duration) + (c2 <= E.duration) + (c3 <= E.duration) + (c4 <= E.duration);
            start = c3;
            clk = c4;
            n += 4;
          }
        }
        while (n < n_max && t_next > clk) {
          start = clk;
          clk = clk + lat_q;
          if (P.record && lane == 0) {
            P.rec_d[rec_base + rec_n + n] = clk - start;
            P.rec_c[rec_base + rec_n + n] = E.R;
          }
          if (kRec && P.rec_chunked && lane == 0) rec_add(clk - start, E.R);
          if (kRep && P.report) {
            if (lane == 0) {
              P.tr_time[tr_base + E.iter + n] = start;
              P.tr_lat[tr_base + E.iter + n] = lat_q;
              P.tr_rwal[tr_base + E.iter + n] = make_int4(E.R, W, A, 0);
            }
          }
          win += (clk <= E.duration);
          ++n;
          if (LT_UNLIKELY(P.want_digest)) {
            E.digest = fold64(E.digest, static_cast<uint32_t>(E.R) | (static_cast<uint64_t>(static_cast<uint32_t>(W)) << 32));
            E.digest = fold64(E.digest, static_cast<uint32_t>(A));
            E.digest = fold64(E.digest, static_cast<uint64_t>(__double_as_longlong(lat_q)));
          }
        }
        const long long rn = static_cast<long long>(E.R) * n;
        rec_n += n;
        E.clock = clk;
        E.prev_now = start;  // ensure_loaded's last_used refresh of the last skipped iteration
        E.used += rn;
        E.iter += n;
        E.tok_tot += rn;
        E.tok_win += static_cast<long long>(E.R) * win;
        E.sum_r += rn;
      }
    }
  }
  __syncwarp();
  // Requests still running keep their emitted tokens (truncation / error).
  for (int i = lane; i < E.R_end; i += 32) {
    const int4 e = E.run_get(i);
    if (e.x < 0) continue;
    const int outv = P.r_out[E.rb + e.x];
    P.r_gen[E.rb + e.x] = outv - (e.y - E.iter);
    P.r_last[E.rb + e.x] = E.clock;
  }
  __syncwarp();

  o.status = E.status;
  o.status_kind = E.status_kind;
  o.status_a = E.status_a;
  o.status_b = E.status_b;
  o.iterations = E.iter;
  o.final_clock_s = E.clock;
  o.truncated = E.truncated;
  o.preemptions = E.preempts;
  o.load_events = E.loads_n;
  o.tokens_in_window = E.tok_win;
  o.tokens_total = E.tok_tot;
  o.digest = P.want_digest ? E.digest : 0;
  o.sum_running = E.sum_r;
  o.sum_visited = E.sum_v;
  o.sum_arrivals = E.sum_a;
  o.sum_moves = E.sum_m;

  // Throughput (metrics.cpp:96); the rest of compute_metrics -- counts, the
  // ordered TTFT / ITL / rejected-demand sums and the starved verdict -- is
  // metrics_kernel (K2), launched after this kernel.
  if (E.status == LT_OK && E.n_req > 0) o.throughput_tok_s = static_cast<double>(E.tok_win) / E.duration;
  LT_PH(5);
#ifdef LT_PHASE_PROF
  for (int k = 0; k < 6; ++k) o.phase_cycles[k] = ph[k];
#endif
#ifdef LT_SCAN_STATS
  for (int k = 0; k < 6; ++k) o.phase_cycles[k] = E.st[k];
#endif
  o.device_cycles = clock64() - t_start;
  if (lane == 0) P.out[s] = o;
  if (kRep && P.report && lane == 0) P.sl_cnt[s] = E.sl_n;
  if (kRec && P.rec_chunked && lane == 0) {
    if (rl_w > 0) rec_put(rl_d, rl_w);
    P.rec_total[s] = rc_total;
    P.rec_chunk_next[rc_cur] = -1;
  }
}

// Persistent kernel: each warp pulls scenarios (cost-descending order) from a
// global counter until the batch is drained. kMinBlocks = 1: ~200 registers,
// one 8-warp block per SM, the shortest per-engine latency (the batch's
// longest engines set its time). kMinBlocks = 2: <= 128 registers, 16 warps
// per SM, for batches with many rounds of engines per warp (throughput).
template <int kThreads, int kMinBlocks, bool kRep = false, bool kRec = kRep>
__global__ void __launch_bounds__(kThreads, kMinBlocks) engine_kernel(EngineParams P) {
  extern __shared__ __align__(16) char smem[];
  const int warp = threadIdx.x >> 5;
  const int slot = blockIdx.x * (blockDim.x >> 5) + warp;
  char* mine = smem + static_cast<size_t>(warp) * P.smem_per_warp;
  // First round: scenario warp * gridDim + block, so the most expensive
  // scenarios (the head of the cost order) land on different SMs instead of
  // sharing one SM's schedulers; then a global counter hands out the rest.
  // Warps w and w + 4 share a scheduler (SMSP w % 4): the other SMSP-0
  // warps (4, 8) are filled last, so when a batch leaves spare slots the
  // heaviest engines (warp 0 of each block) keep their scheduler to themselves.
  const int warps = blockDim.x >> 5;
  const int rank = (warp & 3) ? warp - (warp >> 2) : (warp == 0 ? 0 : warps - (warps >> 2) + (warp >> 2));
  const int first = rank * gridDim.x + blockIdx.x;
  // (one call site: engine_run is inlined once)
  for (int k = first; k < P.n_scen;) {
    engine_run<kRep, kRec, (kThreads > 256 || kMinBlocks > 1)>(P, P.order[k], slot, mine);
    int nk = 0;
    if ((threadIdx.x & 31) == 0) nk = atomicAdd(P.counter, 1) + gridDim.x * warps;
    k = __shfl_sync(kFull, nk, 0);
  }
}

}  // namespace lt
