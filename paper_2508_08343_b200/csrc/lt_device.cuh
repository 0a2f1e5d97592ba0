// Device-side data layout of the DT sweep (shared by all kernels).
//
// HBM layout (SoA, one segment per scenario, all sized by the host):
//   scenarios  DScen[n]                     per-engine scalars
//   adapters   DAdapter[sum N]              per scenario, sorted by adapter_id
//   requests   arrival f64 / in / out / adapter i32   [sum n_req]   (inputs)
//              phase u8 / gen i32 / first f64 / last f64 / preempt i32  (state + outputs)
//   workspace  per persistent warp slot: running int4[cap], preempted int2[cap],
//              chain node int4[cap] {in, out, next, adapter}, oversized FIFO i32[cap]
//              (cap = max n_req of the batch)
//   smem       per warp: last_used f64[NA], run_count, chain head/tail/count,
//              block epoch, flags i32[NA] (NA = max adapters)
#pragma once
#include <stdint.h>

#include "loratwin_gpu.h"

namespace lt {

constexpr int kMaxAdapters = 1024;  // 32 lanes x 32-bit adapter bitmask words

enum Phase : int8_t { kWaiting = 0, kRunning = 1, kPreempted = 2, kFinished = 3, kRejected = 4 };

// Queue entry (int2): x = request index within the scenario,
// y = dense adapter index | kOverBit (demand can never fit: reject on visit).
constexpr int kOverBit = 1 << 30;
constexpr int kAdapterMask = (1 << 20) - 1;
// Running entry (int4): x = request index, y = retire iteration (iteration at
// whose start gen >= out), z = dense adapter | kFreshBit (first admission this
// iteration), w = input + output tokens.
constexpr int kFreshBit = 1 << 30;
// Chain link of a request (int32, link_kernel): the low 30 bits are the
// adapter's next chained request (kLinkNone: none); kLinkFirst marks the
// adapter's first chained request. Oversized requests are never chained.
constexpr int kLinkFirst = 1 << 30;
constexpr int kLinkNone = (1 << 30) - 1;
constexpr int kMaxScenarioRequests = kLinkNone;  // requests per scenario (link index range)

// Engine shared-memory layout (k_engine.cuh; sized on the host in size_engine).
// per-warp shared memory per adapter: last_used f64 + run_cnt, q_head, q_tail,
// act_key (i32)
constexpr int kSmemPerAdapter = 8 + 4 * 4;
// Retire calendar: running entries are linked into bucket (retire iteration
// mod kCalBuckets); the bucket of the current iteration holds every retiree.
constexpr int kCalBuckets = 512;
// Preempted-queue slots kept in shared memory (the rest in HBM).
constexpr int kPqSmem = 64;

// Records per chunk of the single-pass percentile recording pool.
constexpr int kRecChunk = 512;

struct DScen {
  int64_t req_begin;
  int32_t n_req;
  int32_t n_adapters;
  int64_t adapter_begin;
  int32_t G;
  int32_t generated;
  int64_t capacity;
  double duration;
  double ideal;
  int64_t iter_cap;
  int32_t status;
  int32_t status_kind;
  int64_t status_a;
  int64_t status_b;
  int32_t length_param;  // scenario-level Mean parameters (index into DLen)
  int32_t ids_sorted;    // arrivals non-decreasing in request id (generated: always)
};

struct DAdapter {
  int32_t id;
  int32_t rank;
  double rate;
  double load_lat;  // NaN: rank missing from cpu_load_seconds (lazy ConfigError)
  int32_t key;      // RNG table key (generated scenarios)
  int32_t length_param;
  int32_t deck;     // >= 0: Full-mode lengths from DDeck[deck] (sample_lengths, workload.cpp:149-161)
  int32_t _pad;
  int64_t list_off; // Full mode: first (in, out) pair of the adapter's length list
};

// LoadEvent (adapter_cache.hpp:28-34) as the report pass writes it; the
// source is the config's default_source for every event (engine.cpp:113-114).
struct DLoadEvent {
  double time;
  double latency;
  int32_t adapter_id;
  int32_t rank;
};

// Full-mode length deck of one (RNG key, list size D): the lengths stream
// {2, id} shuffles the deck once, then again every D requests
// (workload.cpp:149-161). tab[table_off + j] is the list index of arrival j.
struct DDeck {
  int64_t table_off;
  int32_t key;
  int32_t D;
};

struct DLen {
  double mean_in, std_in, mean_out, std_out;
};

// One (seed, adapter_id) RNG key: E table (arrivals stream {1, id}) and Z
// table (lengths stream {2, id}), shared by every scenario using the key.
struct DKey {
  uint64_t seed;
  int64_t id;
  double rate_max;
  double dur_max;
  int64_t e_off;
  int64_t z_off;
  int32_t cap;    // entries reserved in E (and Z)
  int32_t e_len;  // E entries written (arrivals + the terminating draw)
  int32_t z_len;  // Z pairs written
  int32_t overflow;
};

struct EngineParams {
  const DScen* scen;
  const int32_t* order;
  int32_t n_scen;
  int32_t max_adapters;  // adapters per warp in shared memory
  int32_t run_cap;       // running-set slots per warp in shared memory
  int32_t smem_per_warp; // bytes
  int32_t* counter;
  const DAdapter* adapters;
  const double* r_arr;
  const int32_t* r_in;
  const int32_t* r_out;
  const int32_t* r_adp;
  int8_t* r_phase;
  int32_t* r_gen;
  double* r_first;
  double* r_last;
  int32_t* r_pre;
  int4* ws_run;
  int4* ws_pq;
  int4* ws_node;
  int2* ws_link;  // retire-calendar {next, prev} links of the global running-set tier
  int32_t* ws_ov;
  int64_t ws_stride;  // entries per warp slot
  int32_t ws_per_scenario;  // 1: workspace indexed by the scenario's request offset
  double k1, k2, k3, k4, k5, k6, k7;
  int32_t priority;
  int32_t want_digest;
  lt_sim_summary* out;
  // recording pass (want_percentiles): per iteration one ITL record
  // (emit_k - emit_{k-1}, requests emitting in both iterations) and one
  // (gap, 1) record per re-admitted preempted request, at rec_off[s]
  int32_t record;
  const int64_t* rec_off;
  double* rec_d;
  int32_t* rec_c;
  // report pass (lt_simulate_report, engine_kernel<.., true>): trace row k of
  // scenario s at tr_off[s] + k (engine.cpp:137-140), its load events at
  // ld_off[s] in emission order (:141), and a stint log at sl_off[s]: one
  // {request, iteration} per admission and per preemption, in the order they
  // happen (a request's entries alternate admit / preempt); sl_cnt[s] = entries
  const int64_t* tr_off;
  double* tr_time;
  double* tr_lat;
  int4* tr_rwal;  // {R, W, A, loads}
  const int64_t* ld_off;
  DLoadEvent* ld;
  const int64_t* sl_off;
  int2* sl_log;
  int32_t* sl_cnt;
  // single-pass percentile recording (engine_kernel<256,1,true>): the ITL
  // records go to chunks of kRecChunk in a pool -- scenario s starts in chunk
  // s, further chunks come from rec_pool_next and are linked by
  // rec_chunk_next; rec_total[s] counts them; rec_overflow is set (and the
  // scenario stops recording) when the pool runs out
  int32_t rec_chunked;
  int32_t rec_pool_chunks;
  int32_t* rec_pool_next;
  int32_t* rec_chunk_next;
  int64_t* rec_total;
  int32_t* rec_overflow;
  int32_t report;            // the report pass writes the rows above
  int32_t check_invariants;  // SimOptions.check_invariants: checked engine pass
  int64_t inject_iteration;  // test hook (LT_INVARIANT_INJECT): ledger fault at this iteration, -1 none
  // chain links per request (link_kernel), linked builds only. (Last, so the
  // fields above keep their parameter-bank offsets: the k1..k7 pairs stay
  // 16-byte aligned for the uniform constant loads of lat_step.)
  const int32_t* r_link;
};

}  // namespace lt
