// loratwin_gpu.h implementation: host orchestration of the B200 DT sweep.
//
// Host work is limited to what the reference does before its hot loop and
// that cannot differ per device: input validation with the reference's exact
// messages (workload.cpp:97-141, server_config.cpp:21-27,
// estimators.cpp:38-98, engine.cpp:32-71), ideal throughput
// (metrics.cpp:36-45), and packing POD inputs into the device SoA layout
// (lt_device.cuh). Arrival generation, merging, every engine iteration, the
// metrics epilogue and the placement reduction run on the GPU.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "engine_launch.h"
#include "k_metrics.cuh"
#include "k_predict.cuh"
#include "k_report.cuh"
#include "k_sweep.cuh"
#include "k_workload.cuh"
#include "loratwin_gpu.h"
#include "lt_device.cuh"

using namespace lt;

namespace {

// Persistent host workers for the plan-building passes (thread start-up
// would otherwise cost more than the small batches' work): run(nt, fn)
// calls fn(t) for t in [0, nt) on up to nt threads, the caller running t = 0.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool* p = new HostPool();  // never destroyed (outlives static plans)
    return *p;
  }
  static int width(int64_t work, int64_t min_per_thread) {
    const int64_t hw = std::max(1u, std::thread::hardware_concurrency());
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(hw, 16), work / min_per_thread)));
  }
  template <typename F>
  void run(int nt, F&& fn) {
    if (nt <= 1) {
      fn(0);
      return;
    }
    std::unique_lock<std::mutex> call(call_mu_);  // one parallel pass at a time
    ensure(nt - 1);
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = [&fn](int t) { fn(t); };
      n_ = nt;
      next_ = 1;
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    std::exception_ptr err;
    try {
      fn(0);
    } catch (...) {
      err = std::current_exception();
    }
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return done_ == nt - 1; });  // the workers still use fn
    job_ = nullptr;
    if (!err) err = worker_err_;
    worker_err_ = nullptr;
    if (err) std::rethrow_exception(err);
  }

 private:
  void ensure(int k) {
    while (static_cast<int>(threads_.size()) < k) threads_.emplace_back([this] { loop(); });
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return gen_ != seen && next_ < n_; });
      seen = gen_;
      while (next_ < n_) {
        const int t = next_++;
        auto job = job_;
        lk.unlock();
        std::exception_ptr err;
        try {
          job(t);
        } catch (...) {
          err = std::current_exception();
        }
        lk.lock();
        if (err && !worker_err_) worker_err_ = err;
        if (++done_ == n_ - 1) done_cv_.notify_one();
      }
    }
  }
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  std::vector<std::thread> threads_;
  std::function<void(int)> job_;
  std::exception_ptr worker_err_;
  int n_ = 0, next_ = 0, done_ = 0;
  uint64_t gen_ = 0;
};

struct CudaError {
  std::string what;
};

#define LT_CUDA(call)                                                                      \
  do {                                                                                     \
    cudaError_t err_ = (call);                                                             \
    if (err_ != cudaSuccess)                                                               \
      throw CudaError{std::string(#call) + ": " + cudaGetErrorString(err_)};               \
  } while (0)

// LT_SYNC_DEBUG=1: synchronise after every launch and name the failing kernel.
bool sync_debug() {
  static const bool on = [] {
    const char* v = std::getenv("LT_SYNC_DEBUG");
    return v && v[0] == '1';
  }();
  return on;
}

void after_launch(const char* name, cudaStream_t st) {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && sync_debug()) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) throw CudaError{std::string(name) + ": " + cudaGetErrorString(e)};
}

void set_status(lt_status* st, int32_t code, int32_t kind, int64_t index, int64_t a, int64_t b,
                const std::string& msg) {
  if (!st) return;
  st->code = code;
  st->kind = kind;
  st->index = index;
  st->detail_a = a;
  st->detail_b = b;
  std::snprintf(st->message, sizeof(st->message), "%s", msg.c_str());
}

void ok_status(lt_status* st) {
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->index = -1;
  }
}

// Host-side error of one scenario: code + reference message.
struct HostErr {
  int32_t code = LT_OK;
  int32_t kind = LT_K_NONE;
  int64_t a = 0, b = 0;
  std::string msg;
  bool set(int32_t c, const std::string& m, int32_t k = LT_K_VALIDATION_MSG, int64_t aa = 0,
           int64_t bb = 0) {
    code = c;
    kind = k;
    msg = m;
    a = aa;
    b = bb;
    return false;
  }
};

std::string render(int32_t code, int32_t kind, int64_t a, int64_t b) {
  char buf[320];
  lt_format_status(code, kind, a, b, buf, sizeof(buf));
  return buf;
}

// ----------------------------------------------------------------------------
// Reference validation (exact messages).

bool validate_lengths(const lt_length_spec& l, const int32_t* full, const std::string& path,
                      HostErr* e) {
  if (l.mode == LT_MODE_FULL) {
    if (l.full_count <= 0)
      return e->set(LT_ERR_VALIDATION, path + ".full_lengths: Full mode requires a non-empty length list");
    for (int64_t i = 0; i < l.full_count; ++i) {
      if (full[2 * (l.full_offset + i)] < 1 || full[2 * (l.full_offset + i) + 1] < 1)
        return e->set(LT_ERR_VALIDATION, path + ".full_lengths[" + std::to_string(i) +
                                              "]: token counts must be >= 1");
    }
    return true;
  }
  if (l.mean_input <= 0.0)
    return e->set(LT_ERR_VALIDATION, path + ".mean_input: must be > 0, got " + std::to_string(l.mean_input));
  if (l.mean_output <= 0.0)
    return e->set(LT_ERR_VALIDATION, path + ".mean_output: must be > 0, got " + std::to_string(l.mean_output));
  if (l.std_input < 0.0)
    return e->set(LT_ERR_VALIDATION, path + ".std_input: must be >= 0, got " + std::to_string(l.std_input));
  if (l.std_output < 0.0)
    return e->set(LT_ERR_VALIDATION, path + ".std_output: must be >= 0, got " + std::to_string(l.std_output));
  return true;
}

// ServerConfig::validate (server_config.cpp:21-27) without the slots check.
bool validate_config_body(const lt_server_config& c, HostErr* e) {
  if (c.iteration_cap < 1) return e->set(LT_ERR_VALIDATION, "config.iteration_cap: must be >= 1");
  if (c.k4 < 0.0) return e->set(LT_ERR_VALIDATION, "estimators.latency.k4: must be >= 0");
  if (c.k5 <= 0.0)
    return e->set(LT_ERR_VALIDATION, "estimators.latency.k5: must be > 0 (a forward pass takes time)");
  if (c.k6 < 0.0) return e->set(LT_ERR_VALIDATION, "estimators.latency.k6: must be >= 0");
  if (c.k7 < 1.0)
    return e->set(LT_ERR_VALIDATION, "estimators.latency.k7: must be >= 1 (adapters never speed up the model)");
  if (c.total_kv_budget <= 0)
    return e->set(LT_ERR_VALIDATION, "estimators.memory.total_kv_budget: must be > 0");
  if (c.n_slot_cost == 0 && !c.has_slot_cost_base_rank8)
    return e->set(LT_ERR_VALIDATION,
                  "estimators.memory: one of slot_cost_tokens or slot_cost_base_rank8 is required");
  if (c.has_slot_cost_base_rank8 && c.slot_cost_base_rank8 <= 0.0)
    return e->set(LT_ERR_VALIDATION, "estimators.memory.slot_cost_base_rank8: must be > 0");
  {
    std::map<int, int64_t> t;
    for (int i = 0; i < c.n_slot_cost; ++i) t[c.slot_cost_rank[i]] = c.slot_cost_tokens[i];
    int64_t prev = 0;
    int prev_rank = 0;
    for (const auto& [rank, cost] : t) {
      if (rank <= 0) return e->set(LT_ERR_VALIDATION, "estimators.memory.slot_cost_tokens: ranks must be > 0");
      if (cost <= prev)
        return e->set(LT_ERR_VALIDATION,
                      "estimators.memory.slot_cost_tokens: cost must increase with rank (rank " +
                          std::to_string(rank) + " vs rank " + std::to_string(prev_rank) + ")");
      prev = cost;
      prev_rank = rank;
    }
  }
  if (c.disk_multiplier < 1.0) return e->set(LT_ERR_VALIDATION, "estimators.load.disk_multiplier: must be >= 1");
  {
    std::map<int, double> t;
    for (int i = 0; i < c.n_load; ++i) t[c.load_rank[i]] = c.load_seconds[i];
    double prev = 0.0;
    int prev_rank = 0;
    for (const auto& [rank, seconds] : t) {
      if (rank <= 0) return e->set(LT_ERR_VALIDATION, "estimators.load.cpu_load_seconds: ranks must be > 0");
      if (seconds < prev)
        return e->set(LT_ERR_VALIDATION,
                      "estimators.load.cpu_load_seconds: latency must not decrease with rank (rank " +
                          std::to_string(rank) + " vs rank " + std::to_string(prev_rank) + ")");
      prev = seconds;
      prev_rank = rank;
    }
  }
  return true;
}

// Parsed config tables.
struct Config {
  lt_server_config raw;
  std::map<int, int64_t> slot_cost;
  std::map<int, double> load;
  HostErr body_err;  // config.validate() failure other than slots
  bool body_ok = true;
  std::vector<double> lat_cache;
  int variant = 1;
};

// MemoryModel::slot_cost_tokens (estimators.cpp:46-55).
bool slot_cost(const Config& c, int rank, int64_t* out, HostErr* e) {
  if (rank == 0) {
    *out = 0;
    return true;
  }
  if (rank < 0) return e->set(LT_ERR_VALIDATION, "slot rank must be >= 0, got " + std::to_string(rank));
  auto it = c.slot_cost.find(rank);
  if (it != c.slot_cost.end()) {
    *out = it->second;
    return true;
  }
  if (c.raw.has_slot_cost_base_rank8) {
    *out = static_cast<int64_t>(std::llround(c.raw.slot_cost_base_rank8 * rank / 8.0));
    return true;
  }
  return e->set(LT_ERR_CONFIG, render(LT_ERR_CONFIG, LT_K_NO_SLOT_COST, rank, 0), LT_K_NO_SLOT_COST, rank);
}

// LoadLatencyTable::load_latency (estimators.cpp:78-83); NaN when missing
// (the reference raises lazily, at the first load of that rank).
double load_latency(const Config& c, int rank) {
  auto it = c.load.find(rank);
  if (it == c.load.end()) return NAN;
  return c.raw.load_source == LT_SOURCE_CPU ? it->second : it->second * c.raw.disk_multiplier;
}

double load_latency_cached(Config& c, int rank) {
  if (rank >= 0 && rank < 1024) {
    if (c.lat_cache.empty()) c.lat_cache.assign(1024, -2.0);
    double& v = c.lat_cache[rank];
    if (v == -2.0) v = load_latency(c, rank);
    return v;
  }
  return load_latency(c, rank);
}

struct Stats {
  double max, min, mean, std;
};

// list_stats (workload.cpp:31-50).
Stats list_stats(const int32_t* full, int64_t off, int64_t n, bool input) {
  Stats s{0.0, 0.0, 0.0, 0.0};
  if (n == 0) return s;
  s.max = -1.79769313486231570815e+308;
  s.min = 1.79769313486231570815e+308;
  double sum = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double v = full[2 * (off + i) + (input ? 0 : 1)];
    s.max = std::max(s.max, v);
    s.min = std::min(s.min, v);
    sum += v;
  }
  s.mean = sum / static_cast<double>(n);
  double sq = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double v = full[2 * (off + i) + (input ? 0 : 1)];
    sq += (v - s.mean) * (v - s.mean);
  }
  s.std = std::sqrt(sq / static_cast<double>(n));
  return s;
}

double output_mean(const lt_length_spec& l, const int32_t* full) {
  if (l.mode == LT_MODE_FULL) return list_stats(full, l.full_offset, l.full_count, false).mean;
  return l.mean_output;
}
double input_mean(const lt_length_spec& l, const int32_t* full) {
  if (l.mode == LT_MODE_FULL) return list_stats(full, l.full_offset, l.full_count, true).mean;
  return l.mean_input;
}

// LengthSpec::as_mean (workload.cpp:91-95) for Mean-mode sampling.
DLen as_dlen(const lt_length_spec& l, const int32_t* full) {
  if (l.mode == LT_MODE_FULL) {
    const Stats in = list_stats(full, l.full_offset, l.full_count, true);
    const Stats out = list_stats(full, l.full_offset, l.full_count, false);
    return DLen{in.mean, in.std, out.mean, out.std};
  }
  return DLen{l.mean_input, l.std_input, l.mean_output, l.std_output};
}

// ----------------------------------------------------------------------------
// Device buffers

// Grow-only caching allocator: device buffers are recycled across plans and
// calls (cudaMalloc/cudaFree of GB-sized workspaces would otherwise dominate
// small end-to-end calls). Blocks are keyed by device and size class.
struct BlockCache {
  std::mutex mu;
  std::multimap<std::pair<int, size_t>, void*> free_blocks;
  static BlockCache& get() {
    static BlockCache* c = new BlockCache();  // never destroyed: outlives static DBufs
    return *c;
  }
  static size_t size_class(size_t bytes) {
    size_t c = 256;
    while (c < bytes) c <<= 1;  // power-of-two classes bound waste at 2x
    return c;
  }
  void* take(size_t bytes, size_t* got, int* device) {
    int dev = 0;
    cudaGetDevice(&dev);
    *device = dev;
    const size_t cls = size_class(bytes);
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = free_blocks.find({dev, cls});
      if (it != free_blocks.end()) {
        void* p = it->second;
        free_blocks.erase(it);
        *got = cls;
        return p;
      }
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, cls);
    if (e != cudaSuccess) {
      // release cached blocks of this device and retry once
      trim(dev);
      cudaGetLastError();
      e = cudaMalloc(&p, cls);
    }
    if (e != cudaSuccess) throw CudaError{std::string("cudaMalloc: ") + cudaGetErrorString(e)};
    *got = cls;
    return p;
  }
  void give(void* p, size_t cls, int dev) {
    std::lock_guard<std::mutex> lk(mu);
    free_blocks.emplace(std::make_pair(dev, cls), p);
  }
  void trim(int dev) {
    std::lock_guard<std::mutex> lk(mu);
    for (auto it = free_blocks.begin(); it != free_blocks.end();) {
      if (it->first.first == dev) {
        cudaFree(it->second);
        it = free_blocks.erase(it);
      } else {
        ++it;
      }
    }
  }
};

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  size_t cls = 0;
  int dev = 0;  // the block goes back to its own device's free list, whichever thread releases it
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) BlockCache::get().give(p, cls, dev);
    p = nullptr;
    n = 0;
    cls = 0;
  }
  void alloc(size_t count) {
    if (p && count * sizeof(T) <= cls) {  // reuse the current block
      n = count;
      return;
    }
    release();
    n = count;
    if (count) p = static_cast<T*>(BlockCache::get().take(count * sizeof(T), &cls, &dev));
  }
  void upload(const std::vector<T>& v, cudaStream_t s) { upload(v.data(), v.size(), s); }
  void upload(const T* src, size_t count, cudaStream_t s) {
    alloc(count);
    if (count) LT_CUDA(cudaMemcpyAsync(p, src, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
};

}  // namespace

struct lt_ctx {
  std::vector<std::string> messages;  // per scenario / condition of the last call
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t stream2 = nullptr;  // every other chunk of a chunked lt_simulate_batch
  cudaStream_t stream_up = nullptr;  // packed-scenario uploads, beside K0
  int smem_optin = 0;              // max dynamic shared memory per block (opt-in)
  int sm_count = 0;
  lt_timing timing{};
  cudaEvent_t ev[8]{};
  // multi-device context (lt_create_devices): one single-device member per
  // entry; the group's own streams are the first member's
  std::vector<lt_ctx*> members;
  std::vector<void*> comms;  // ncclComm_t per member (LT_GATHER_NCCL)
  int32_t transport = LT_GATHER_NONE;
};

// A prepared batch: everything the kernels need, resident in HBM.
struct lt_plan {
  lt_ctx* ctx = nullptr;
  cudaStream_t st = nullptr;  // the stream this plan's work runs on
  cudaEvent_t ev[8]{};        // this plan's timing events
  cudaEvent_t ev_up = nullptr;  // packed-scenario uploads done (ctx->stream_up)
  int warps_per_block = 8;
  ~lt_plan() {
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
    if (ev_up) cudaEventDestroy(ev_up);
  }
  Config cfg;
  int64_t n_scen = 0;
  int max_adapters = 32;
  int64_t max_req = 0;
  int64_t total_req = 0;
  std::vector<DScen> h_scen;
  std::vector<HostErr> errs;
  std::vector<int32_t> h_order;
  std::vector<int32_t> adapter_ids;  // dense -> adapter_id, per scenario segment
  DBuf<DScen> scen;
  DBuf<DAdapter> adapters;
  DBuf<DLen> lens;
  DBuf<DKey> keys;
  DBuf<uint64_t> seed_state;   // K0a -> K0b: seeded MT19937-64 states of one key chunk
  // Full-mode length decks
  std::vector<DDeck> h_decks;
  DBuf<DDeck> decks;
  DBuf<int32_t> deck_tab, big_deck, full;
  DBuf<int64_t> big_off;
  size_t deck_smem = 0;
  DBuf<int32_t> tab_overflow;  // set when some key's table was too short
  DBuf<double> E;
  DBuf<double2> Z;
  DBuf<int32_t> order;
  DBuf<int32_t> counter;
  DBuf<double> r_arr, r_first, r_last;
  DBuf<int32_t> r_in, r_out, r_adp, r_gen, r_pre;
  DBuf<int8_t> r_phase;
  DBuf<int4> ws_run;
  DBuf<int4> ws_pq;
  DBuf<int4> ws_node;
  DBuf<int32_t> ws_ov;
  DBuf<int2> ws_link;
  DBuf<lt_sim_summary> out;
  // percentiles (want_percentiles): recording pass + segmented sorts
  int want_pct = 0;
  int want_check = 0;  // SimOptions.check_invariants: the checked engine build (engine_kernel<256,1,true>)
  DBuf<int64_t> rec_off, rec_len;
  DBuf<double> rec_d, rec_d_sorted, ttft_keys, ttft_sorted;
  DBuf<int32_t> rec_c, rec_c_sorted, pct_seg_b, pct_seg_e, pct_rseg_b, pct_rseg_e;
  DBuf<char> pct_tmp;
  // re-run state (lt_plan_run recomputes K0 tables, counts, offsets, merge)
  DBuf<int32_t> pair_scen, pair_adp, adp_count, overflow;
  DBuf<int64_t> pair_begin;
  DBuf<unsigned long long> scen_count, base_count, scen_off;
  DBuf<char> scan_tmp;
  size_t scan_tmp_bytes = 0;
  // sort-based merge of adapter streams
  DBuf<unsigned long long> pair_excl, sv_in, sv_out;
  DBuf<double> st_in, st_out;
  DBuf<int32_t> pos_a, pos_b;      // radix merge: positions, sorted by time, then by scenario
  DBuf<uint32_t> skey_a, skey_b;   // radix merge: scenario of each time-sorted position
  size_t radix_tmp_bytes = 0;
  int scen_bits = 1;
  DBuf<int> seg_begin, seg_end;
  DBuf<char> sort_tmp, pscan_tmp;
  size_t sort_tmp_bytes = 0, pscan_tmp_bytes = 0;
  int64_t n_pairs = 0;
  int n_keys = 0;
  bool fresh = true;
  int64_t ws_stride = 0;
  int ws_per_scenario = 0;
  int grid = 0;
  int block = 256;
  size_t smem = 0;
  int32_t run_cap = 0, smem_per_warp = 0;
  int engine_variant = 1;  // engine_kernel<1> (latency) or <2> (occupancy)
  int pair_g = 32;         // lanes per (scenario, adapter) pair in count / expand (pair_group)
  int want_digest = 0;
  double tables_ms = 0, h2d_ms = 0;
  int64_t h2d_bytes = 0;
  int64_t launches_prep = 0;
  int64_t launches_run = 0;
  // lt_plan_trim: the per-request arrays, RNG tables, merge buffers and
  // engine workspace go back to the block cache between runs (sizes kept)
  bool has_scripted = false;  // scripted requests live in r_*: never trimmed
  bool trimmed = false;
  std::vector<size_t> trimmed_sizes;
};

namespace {

// ----------------------------------------------------------------------------
// Batch preparation

// Page-locked host memory for the packed arrays uploaded every plan: the
// copies run as DMA straight from them (no driver staging copy). Prep keeps
// them per host thread across plans, so the allocation is paid once.
template <class T>
struct PinnedAlloc {
  using value_type = T;
  PinnedAlloc() = default;
  template <class U>
  PinnedAlloc(const PinnedAlloc<U>&) {}
  T* allocate(size_t n) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, n * sizeof(T), cudaHostAllocDefault) != cudaSuccess) throw std::bad_alloc();
    return static_cast<T*>(p);
  }
  void deallocate(T* p, size_t) { cudaFreeHost(p); }
  template <class U>
  bool operator==(const PinnedAlloc<U>&) const { return true; }
  template <class U>
  bool operator!=(const PinnedAlloc<U>&) const { return false; }
};
template <class T>
using PinnedVec = std::vector<T, PinnedAlloc<T>>;

// DAdapter without value-initialisation: the packed array is sized up front
// for scenarios packed later by several host threads (Prep::deferred).
struct DAdapterNI : DAdapter {
  DAdapterNI() {}
  DAdapterNI(const DAdapter& d) : DAdapter(d) {}
};
static_assert(sizeof(DAdapterNI) == sizeof(DAdapter), "layout");
struct DKeyNI : DKey {
  DKeyNI() {}
  DKeyNI(const DKey& d) : DKey(d) {}
};
static_assert(sizeof(DKeyNI) == sizeof(DKey), "layout");

struct Prep {
  PinnedVec<DAdapterNI> adapters;
  // Generated Mean-mode scenarios with ascending adapter ids that passed
  // validation: their adapter records are packed after the serial pass, in
  // parallel, into slots reserved in order (scenario, adapter offset, pair offset).
  struct Deferred {
    int64_t i, a_off, p_off;
  };
  std::vector<Deferred> deferred;
  bool allow_defer = false;
  std::vector<DLen> lens;
  PinnedVec<DKeyNI> keys;
  // Scenarios whose seed no other scenario uses, with strictly ascending ids:
  // their keys are their adapters, at keys[key_base[i] + k] (else -1).
  std::vector<int64_t> key_base;
  PinnedVec<int32_t> pair_scen, pair_adp;
  PinnedVec<int64_t> pair_begin;
  std::unordered_map<std::string, int> len_index;
  // (seed, adapter_id) -> key index. Keys are looked up per seed: a batch has
  // few distinct seeds with many adapters each (sweeps share one seed across
  // every grid point), and ids are small (instantiate_condition: 1..N), so
  // each seed keeps a dense id table (hash map for ids outside [0, 65536)).
  struct SeedKeys {
    std::vector<int32_t> dense;
    std::unordered_map<int64_t, int32_t> sparse;
  };
  std::unordered_map<uint64_t, int32_t> seed_index;
  std::vector<SeedKeys> seeds;
  std::vector<DDeck> decks;                        // Full-mode decks, table_off set after sizing
  std::map<std::pair<int32_t, int32_t>, int32_t> deck_index;  // (key, D) -> deck
  std::vector<double> cost;
  // a key appeared (or grew) after the early K0 launch (collect_keys)
  bool late_keys = false;

  // Empties every table but keeps the vectors' memory (already paged in) for
  // the next plan on this host thread; very large buffers are released.
  void reset() {
    const bool big = keys.capacity() * sizeof(DKey) + adapters.capacity() * sizeof(DAdapter) > (size_t(1536) << 20);
    if (big) {
      *this = Prep();
      return;
    }
    adapters.clear();
    deferred.clear();
    allow_defer = false;
    lens.clear();
    keys.clear();
    key_base.clear();
    pair_scen.clear();
    pair_adp.clear();
    pair_begin.clear();
    len_index.clear();
    seed_index.clear();
    seeds.clear();
    decks.clear();
    deck_index.clear();
    cost.clear();
    late_keys = false;
  }

  SeedKeys& seed_keys(uint64_t seed) {
    auto it = seed_index.find(seed);
    if (it != seed_index.end()) return seeds[it->second];
    seed_index.emplace(seed, static_cast<int32_t>(seeds.size()));
    seeds.emplace_back();
    return seeds.back();
  }
  // Key index of (seed, id) or -1, without inserting (safe from several threads).
  int32_t find_key(uint64_t seed, int64_t id) const {
    auto it = seed_index.find(seed);
    if (it == seed_index.end()) return -1;
    const SeedKeys& sk = seeds[it->second];
    if (id >= 0 && id < 65536) return id < static_cast<int64_t>(sk.dense.size()) ? sk.dense[id] : -1;
    auto j = sk.sparse.find(id);
    return j == sk.sparse.end() ? -1 : j->second;
  }
  // Returns the key index of (seed, id) in `sk`, inserting `fresh` when absent.
  static int32_t find_or_insert(SeedKeys& sk, int64_t id, int32_t fresh, bool* inserted) {
    int32_t* slot;
    if (id >= 0 && id < 65536) {
      if (static_cast<int64_t>(sk.dense.size()) <= id) sk.dense.resize(static_cast<size_t>(id) + 1, -1);
      slot = &sk.dense[static_cast<size_t>(id)];
    } else {
      slot = &sk.sparse.emplace(id, -1).first->second;
    }
    *inserted = *slot < 0;
    if (*inserted) *slot = fresh;
    return *slot;
  }
};

int intern_len(Prep& p, const DLen& d) {
  std::string k(reinterpret_cast<const char*>(&d), sizeof(d));
  auto it = p.len_index.find(k);
  if (it != p.len_index.end()) return it->second;
  const int idx = static_cast<int>(p.lens.size());
  p.lens.push_back(d);
  p.len_index.emplace(k, idx);
  return idx;
}

int libm_variant_for(const lt_sim_options* o) {
  if (o && o->libm_variant >= 0) return o->libm_variant ? 1 : 0;
  return lt_host_libm_variant();
}

// Validates scenario `i` in reference order and fills its device record.
// Screen of prepare_scenario's checks for plain generated scenarios (Mean
// mode, workload-level lengths, ascending ids, valid ranks and rates, a
// feasible slot cost), run on host threads before the serial pass: a
// scenario that passes takes the serial pass's deferred branch in O(1)
// (plain_scenario); anything else -- every error included, so the messages
// stay the reference's -- takes prepare_scenario.
struct PlainPre {
  int32_t plain = 0;
  int32_t G = 0;
  int64_t capacity = 0;
  double ideal = 0.0;
};

void prescreen_plain(const lt_plan& P, const lt_workload_batch& b, std::vector<PlainPre>& pre) {
  const int64_t n = b.n_scenarios;
  pre.assign(n, PlainPre{});
  std::vector<char> len_ok(std::max<int64_t>(b.n_lengths, 1), 0);
  for (int64_t l = 0; l < b.n_lengths; ++l) {
    HostErr e;
    len_ok[l] = b.lengths[l].mode == LT_MODE_MEAN && validate_lengths(b.lengths[l], b.full_lengths, "workload.lengths", &e);
  }
  if (!P.cfg.body_ok) return;
  auto work = [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) {
      const lt_scenario& s = b.scenarios[i];
      const int G = s.slots > 0 ? s.slots : P.cfg.raw.slots;
      if (s.n_requests >= 0 || s.n_adapters <= 0 || s.n_adapters > kMaxAdapters || !(s.duration_s > 0.0) ||
          s.mode == LT_MODE_FULL || G < 1 || s.length_index < 0 || s.length_index >= b.n_lengths || !len_ok[s.length_index])
        continue;
      const lt_adapter* ad = b.adapters + s.adapter_offset;
      bool ok = true;
      int max_rank = 0;
      for (int k = 0; k < s.n_adapters && ok; ++k) {
        ok = ad[k].rank >= 0 && ad[k].rate > 0.0 && ad[k].length_index < 0 && (k == 0 || ad[k - 1].adapter_id < ad[k].adapter_id);
        max_rank = std::max(max_rank, ad[k].rank);
      }
      if (!ok) continue;
      int64_t c_slot;
      HostErr e;
      if (!slot_cost(P.cfg, max_rank, &c_slot, &e)) continue;
      const int64_t capacity = P.cfg.raw.total_kv_budget - static_cast<int64_t>(G) * c_slot;
      if (capacity <= 0) continue;
      // ideal_throughput (metrics.cpp:36-45) in spec order, as prepare_scenario
      const lt_length_spec& l = b.lengths[s.length_index];
      double tokens = output_mean(l, b.full_lengths);
      if (P.cfg.raw.ideal_includes_input) tokens += input_mean(l, b.full_lengths);
      double ideal = 0.0;
      for (int k = 0; k < s.n_adapters; ++k) ideal += ad[k].rate * tokens;
      pre[i] = PlainPre{1, G, capacity, ideal};
    }
  };
  const int nt = HostPool::width(n, 512);
  HostPool::get().run(nt, [&](int t) { work(n * t / nt, n * (t + 1) / nt); });
}

// prepare_scenario's deferred branch for a screened plain scenario.
void plain_scenario(lt_plan& P, Prep& pr, const lt_workload_batch& b, int64_t i, const PlainPre& q,
                    int32_t& last_len_index, int32_t& last_len_param) {
  const lt_scenario& s = b.scenarios[i];
  DScen& d = P.h_scen[i];
  std::memset(&d, 0, sizeof(d));
  d.G = q.G;
  d.duration = s.duration_s;
  d.n_adapters = s.n_adapters;
  d.adapter_begin = static_cast<int64_t>(pr.adapters.size());
  d.generated = 1;
  d.ids_sorted = 1;
  d.iter_cap = P.cfg.raw.iteration_cap;
  d.capacity = q.capacity;
  d.ideal = q.ideal;
  if (s.length_index != last_len_index) {
    last_len_index = s.length_index;
    last_len_param = intern_len(pr, as_dlen(b.lengths[s.length_index], b.full_lengths));
  }
  d.length_param = last_len_param;
  pr.deferred.push_back(Prep::Deferred{i, static_cast<int64_t>(pr.adapters.size()),
                                       static_cast<int64_t>(pr.pair_scen.size())});
  pr.adapters.resize(pr.adapters.size() + s.n_adapters);
  P.adapter_ids.resize(P.adapter_ids.size() + s.n_adapters);
  pr.pair_scen.resize(pr.pair_scen.size() + s.n_adapters);
  pr.pair_adp.resize(pr.pair_adp.size() + s.n_adapters);
  P.max_adapters = std::max(P.max_adapters, s.n_adapters);
}

void prepare_scenario(lt_plan& P, Prep& pr, const lt_workload_batch& b, int64_t i) {
  const lt_scenario& s = b.scenarios[i];
  DScen& d = P.h_scen[i];
  std::memset(&d, 0, sizeof(d));
  HostErr& e = P.errs[i];
  const int G = s.slots > 0 ? s.slots : P.cfg.raw.slots;
  d.G = G;
  d.duration = s.duration_s;
  d.n_adapters = s.n_adapters;
  d.adapter_begin = static_cast<int64_t>(pr.adapters.size());
  d.generated = s.n_requests < 0;
  d.ids_sorted = 1;  // generated: request ids are the (arrival, adapter) order
  d.iter_cap = P.cfg.raw.iteration_cap;
  const bool scripted = s.n_requests >= 0;
  const lt_adapter* ad = b.adapters + s.adapter_offset;
  const int32_t* full = b.full_lengths;
  auto fail = [&]() {
    d.status = e.code;
    d.status_kind = e.kind;
    d.status_a = e.a;
    d.status_b = e.b;
    d.n_adapters = 0;
  };
  auto lengths_of = [&](const lt_adapter& a) -> const lt_length_spec& {
    return a.length_index >= 0 ? b.lengths[a.length_index] : b.lengths[s.length_index];
  };
  if (!scripted) {
    // WorkloadSpec::validate(for_simulation=true) (workload.cpp:118-141)
    if (s.n_adapters <= 0) return e.set(LT_ERR_VALIDATION, "workload.adapters: must be non-empty"), fail();
    if (s.duration_s <= 0.0)
      return e.set(LT_ERR_VALIDATION, "workload.duration_s: must be > 0, got " + std::to_string(s.duration_s)), fail();
    // fast screen; the exact first error (in spec order) is rebuilt only on failure
    bool suspect = false;
    for (int k = 0; k < s.n_adapters && !suspect; ++k)
      suspect = ad[k].rank < 0 || !(ad[k].rate > 0.0) || ad[k].length_index >= 0;
    if (!suspect) {
      // ids are usually ascending already (instantiate_condition: 1..N)
      bool asc = true;
      for (int k = 1; k < s.n_adapters && asc; ++k) asc = ad[k - 1].adapter_id < ad[k].adapter_id;
      if (!asc) {
        std::vector<int> ids(s.n_adapters);
        for (int k = 0; k < s.n_adapters; ++k) ids[k] = ad[k].adapter_id;
        std::sort(ids.begin(), ids.end());
        suspect = std::adjacent_find(ids.begin(), ids.end()) != ids.end();
      }
    }
    if (suspect) {
      std::set<int> seen;
      for (int k = 0; k < s.n_adapters; ++k) {
        const std::string path = "workload.adapters[" + std::to_string(k) + "]";
        if (ad[k].rank < 0)
          return e.set(LT_ERR_VALIDATION, path + ".rank: must be >= 0, got " + std::to_string(ad[k].rank)), fail();
        if (ad[k].rate <= 0.0)
          return e.set(LT_ERR_VALIDATION, path + ".rate: must be > 0, got " + std::to_string(ad[k].rate)), fail();
        if (!seen.insert(ad[k].adapter_id).second)
          return e.set(LT_ERR_VALIDATION, path + ".adapter_id: duplicate id " + std::to_string(ad[k].adapter_id)), fail();
        if (ad[k].length_index >= 0 &&
            !validate_lengths(b.lengths[ad[k].length_index], full, path + ".lengths", &e))
          return fail();
      }
    }
    if (!validate_lengths(b.lengths[s.length_index], full, "workload.lengths", &e)) return fail();
    // generate_arrivals mode handling (workload.cpp:185-192)
    for (int k = 0; k < s.n_adapters; ++k) {
      const lt_length_spec& l = lengths_of(ad[k]);
      if (s.mode != l.mode && s.mode == LT_MODE_FULL)
        return e.set(LT_ERR_VALIDATION, "workload.lengths: cannot force Full mode without a length list"), fail();
    }
  }
  // Engine::Engine (engine.cpp:32-71)
  if (G < 1) return e.set(LT_ERR_VALIDATION, "config.slots: must be >= 1, got " + std::to_string(G)), fail();
  if (!P.cfg.body_ok) return (e = P.cfg.body_err), fail();
  if (s.n_adapters <= 0) return e.set(LT_ERR_VALIDATION, "workload.adapters: must be non-empty"), fail();
  if (s.duration_s <= 0.0) return e.set(LT_ERR_VALIDATION, "workload.duration_s: must be > 0"), fail();
  if (s.n_adapters > kMaxAdapters)
    return e.set(LT_ERR_UNSUPPORTED, render(LT_ERR_UNSUPPORTED, LT_K_TOO_MANY_ADAPTERS, s.n_adapters, kMaxAdapters),
                 LT_K_TOO_MANY_ADAPTERS, s.n_adapters, kMaxAdapters),
           fail();
  int max_rank = 0;
  std::vector<int> perm(s.n_adapters);
  for (int k = 0; k < s.n_adapters; ++k) {
    perm[k] = k;
    max_rank = std::max(max_rank, ad[k].rank);
  }
  bool ascending = true;
  for (int k = 1; k < s.n_adapters && ascending; ++k) ascending = ad[k - 1].adapter_id < ad[k].adapter_id;
  if (!ascending)
    std::sort(perm.begin(), perm.end(), [&](int x, int y) { return ad[x].adapter_id < ad[y].adapter_id; });
  for (int k = 1; k < s.n_adapters; ++k)
    if (ad[perm[k]].adapter_id == ad[perm[k - 1]].adapter_id)
      return e.set(LT_ERR_VALIDATION, "workload.adapters: duplicate adapter_id"), fail();
  // mem_max (estimators.cpp:100-108): budget - G * slot_cost(max_rank), floored at 0
  int64_t c_slot;
  if (!slot_cost(P.cfg, max_rank, &c_slot, &e)) return fail();
  int64_t capacity = P.cfg.raw.total_kv_budget - static_cast<int64_t>(G) * c_slot;
  capacity = std::max<int64_t>(capacity, 0);
  if (capacity <= 0)
    return e.set(LT_ERR_CONFIG, render(LT_ERR_CONFIG, LT_K_INFEASIBLE_SLOTS, G, 0), LT_K_INFEASIBLE_SLOTS, G), fail();
  d.capacity = capacity;
  // ideal_throughput (metrics.cpp:36-45), spec order
  double ideal = 0.0;
  for (int k = 0; k < s.n_adapters; ++k) {
    const lt_length_spec& l = lengths_of(ad[k]);
    double tokens = output_mean(l, full);
    if (P.cfg.raw.ideal_includes_input) tokens += input_mean(l, full);
    ideal += ad[k].rate * tokens;
  }
  d.ideal = ideal;
  d.length_param = intern_len(pr, as_dlen(b.lengths[s.length_index], full));
  if (pr.allow_defer && !scripted && ascending && s.mode != LT_MODE_FULL) {
    bool simple = true;  // no per-adapter length specs (interning stays serial)
    for (int k = 0; k < s.n_adapters && simple; ++k) simple = ad[k].length_index < 0;
    if (simple) {
      pr.deferred.push_back(Prep::Deferred{i, static_cast<int64_t>(pr.adapters.size()),
                                           static_cast<int64_t>(pr.pair_scen.size())});
      pr.adapters.resize(pr.adapters.size() + s.n_adapters);
      P.adapter_ids.resize(P.adapter_ids.size() + s.n_adapters);
      pr.pair_scen.resize(pr.pair_scen.size() + s.n_adapters);
      pr.pair_adp.resize(pr.pair_adp.size() + s.n_adapters);
      P.max_adapters = std::max(P.max_adapters, s.n_adapters);
      return;
    }
  }
  double cost = 0.0;
  Prep::SeedKeys* sk = (scripted || (!pr.key_base.empty() && pr.key_base[i] >= 0)) ? nullptr : &pr.seed_keys(s.seed);
  for (int k = 0; k < s.n_adapters; ++k) {
    const lt_adapter& a = ad[perm[k]];
    DAdapter x{};
    x.id = a.adapter_id;
    x.rank = a.rank;
    x.rate = a.rate;
    x.load_lat = load_latency_cached(P.cfg, a.rank);
    x.length_param = a.length_index >= 0 ? intern_len(pr, as_dlen(b.lengths[a.length_index], full)) : -1;
    x.key = -1;
    x.deck = -1;
    if (!scripted) {
      bool inserted = false;
      const bool own = !pr.key_base.empty() && pr.key_base[i] >= 0;  // (perm is the identity then)
      const int kidx = own ? static_cast<int>(pr.key_base[i] + k)
                           : Prep::find_or_insert(*sk, a.adapter_id, static_cast<int32_t>(pr.keys.size()), &inserted);
      if (own) {
      } else if (inserted) {
        DKey k{};
        k.seed = s.seed;
        k.id = a.adapter_id;
        k.rate_max = a.rate;
        k.dur_max = s.duration_s;
        pr.keys.push_back(k);
        pr.late_keys = true;
      } else {
        DKey& k = pr.keys[kidx];
        if (a.rate > k.rate_max || s.duration_s > k.dur_max) pr.late_keys = true;
        k.rate_max = std::max(k.rate_max, a.rate);
        k.dur_max = std::max(k.dur_max, s.duration_s);
      }
      x.key = kidx;
      const lt_length_spec& la = lengths_of(a);
      if (s.mode == LT_MODE_FULL && la.mode == LT_MODE_FULL) {  // deck sampling (workload.cpp:149-161)
        const auto dkey = std::make_pair(static_cast<int32_t>(kidx), static_cast<int32_t>(la.full_count));
        auto it = pr.deck_index.find(dkey);
        if (it == pr.deck_index.end()) {
          it = pr.deck_index.emplace(dkey, static_cast<int32_t>(pr.decks.size())).first;
          pr.decks.push_back(DDeck{0, dkey.first, dkey.second});
        }
        x.deck = it->second;
        x.list_off = la.full_offset;
      }
      pr.pair_scen.push_back(static_cast<int32_t>(i));
      pr.pair_adp.push_back(k);
      const lt_length_spec& l = lengths_of(a);
      cost += a.rate * s.duration_s * (output_mean(l, full) + 1.0);
    }
    pr.adapters.push_back(x);
    P.adapter_ids.push_back(a.adapter_id);
  }
  if (scripted) {
    const lt_request* rq = b.requests + s.request_offset;
    std::unordered_map<int, int> dense;
    for (int k = 0; k < s.n_adapters; ++k) dense[ad[perm[k]].adapter_id] = k;
    for (int64_t r = 0; r < s.n_requests; ++r) {
      if (rq[r].request_id != r)
        return e.set(LT_ERR_VALIDATION, "requests must be sorted with request_id = position, got id " +
                                            std::to_string(rq[r].request_id) + " at position " + std::to_string(r)),
               fail();
      if (!dense.count(rq[r].adapter_id))
        return e.set(LT_ERR_VALIDATION, "request " + std::to_string(rq[r].request_id) +
                                            " references unknown adapter " + std::to_string(rq[r].adapter_id)),
               fail();
      cost += rq[r].output_tokens + 1.0;
      if (r > 0 && rq[r].arrival_time_s < rq[r - 1].arrival_time_s) d.ids_sorted = 0;
    }
    d.n_req = static_cast<int32_t>(s.n_requests);
  }
  pr.cost[i] = cost;
  P.max_adapters = std::max(P.max_adapters, s.n_adapters);
}

void load_config(Config& c, const lt_server_config* cfg, const lt_sim_options* opts) {
  c.raw = *cfg;
  for (int i = 0; i < cfg->n_slot_cost; ++i) c.slot_cost[cfg->slot_cost_rank[i]] = cfg->slot_cost_tokens[i];
  for (int i = 0; i < cfg->n_load; ++i) c.load[cfg->load_rank[i]] = cfg->load_seconds[i];
  c.body_ok = validate_config_body(*cfg, &c.body_err);
  if (opts && opts->iteration_cap_override > 0) c.raw.iteration_cap = opts->iteration_cap_override;
  c.variant = libm_variant_for(opts);
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

void launch_count(const lt_plan& P, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>((P.n_pairs * P.pair_g + 255) / 256);
  if (P.pair_g == 4)
    count_kernel<4><<<grid, 256, 0, st>>>(P.scen.p, P.pair_scen.p, P.pair_adp.p, P.n_pairs, P.adapters.p, P.keys.p,
                                          P.E.p, P.adp_count.p, P.scen_count.p, P.overflow.p);
  else
    count_kernel<32><<<grid, 256, 0, st>>>(P.scen.p, P.pair_scen.p, P.pair_adp.p, P.n_pairs, P.adapters.p, P.keys.p,
                                           P.E.p, P.adp_count.p, P.scen_count.p, P.overflow.p);
  after_launch("count_kernel", st);
}

void launch_expand(const lt_plan& P, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>((P.n_pairs * P.pair_g + 255) / 256);
  if (P.pair_g == 4)
    expand_kernel<4><<<grid, 256, 0, st>>>(P.scen.p, P.pair_scen.p, P.pair_adp.p, P.n_pairs, P.pair_begin.p,
                                           P.adapters.p, P.keys.p, P.E.p, P.adp_count.p, P.pair_excl.p, P.st_in.p,
                                           P.sv_in.p);
  else
    expand_kernel<32><<<grid, 256, 0, st>>>(P.scen.p, P.pair_scen.p, P.pair_adp.p, P.n_pairs, P.pair_begin.p,
                                            P.adapters.p, P.keys.p, P.E.p, P.adp_count.p, P.pair_excl.p, P.st_in.p,
                                            P.sv_in.p);
  after_launch("expand_kernel", st);
}

// Mean expected arrivals per (scenario, adapter) pair of a batch, from up to
// 4,096 evenly spaced scenarios (it only picks count / expand's lanes per pair).
double mean_pair_draws(const lt_workload_batch* b) {
  const int64_t n = b->n_scenarios;
  const int64_t step = std::max<int64_t>(1, n / 4096);
  double draws = 0.0;
  int64_t pairs = 0;
  for (int64_t i = 0; i < n; i += step) {
    const lt_scenario& s = b->scenarios[i];
    if (s.n_requests >= 0) continue;
    for (int32_t k = 0; k < s.n_adapters; ++k)
      draws += std::max(b->adapters[s.adapter_offset + k].rate, 0.0) * std::max(s.duration_s, 0.0);
    pairs += s.n_adapters;
  }
  return pairs ? draws / static_cast<double>(pairs) : 1e9;
}

// Arrival merge: the merge tree of each scenario's per-adapter lists
// (merge_kernel, default); LT_MERGE=segmented selects CUB's per-scenario
// stable segmented sort, LT_MERGE=radix two global stable radix sorts. All
// three order the arrivals identically (tested).
int merge_mode() {
  const char* e = std::getenv("LT_MERGE");
  return (e && std::strcmp(e, "segmented") == 0) ? 2 : 1;
}

bool radix_merge(int64_t n_requests) {
  // the merge tree is faster at every measured size (C2, C3 plans, C5 plans:
  // 2.26 / 9.19 / 72.0 ms pre-engine with the segmented sort, 7.23 / 73.6
  // with the radix sorts, 2.13 / 5.54 / 68.7 with the tree); the radix form
  // stays selectable (LT_MERGE=radix)
  (void)n_requests;
  const char* e = std::getenv("LT_MERGE");
  return e && std::strcmp(e, "radix") == 0;
}

// Keys seeded and drawn per chunk (the seeded states take 5 KB per key).
constexpr int64_t kSeedChunk = 1 << 18;  // keys per seed_kernel + tables_draw_kernel pair (upper bound)
// Keys per launch pair: the 2.5 KB MT states a seed_kernel launch writes are
// read back by the draw kernel right after, so a launch's states should fit
// in L2 instead of going to HBM and back. LT_SEED_CHUNK overrides.
int64_t seed_chunk() {
  static const int64_t v = [] {
    const char* e = std::getenv("LT_SEED_CHUNK");
    return e ? std::max<int64_t>(1, std::min<int64_t>(std::atoll(e), kSeedChunk)) : kSeedChunk;
  }();
  return v;
}

int launch_decks(lt_plan& P, cudaStream_t st);

// K0: seed_kernel (seed_seq, one thread per stream) then tables_draw_kernel
// (one warp per key), chunk by chunk, then the decks. Returns the launches.
int launch_tables(lt_plan& P, int nk, cudaStream_t st) {
  LT_CUDA(cudaFuncSetAttribute(seed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(kSeedSmem)));
  LT_CUDA(cudaFuncSetAttribute(seed_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared));
  int launches = 0;
  const int64_t chunk = seed_chunk();
  for (int64_t k0 = 0; k0 < nk; k0 += chunk) {
    const int n = static_cast<int>(std::min<int64_t>(chunk, nk - k0));
    seed_kernel<<<(2 * n + kSeedThreads - 1) / kSeedThreads, kSeedThreads, kSeedSmem, st>>>(
        P.keys.p, static_cast<int>(k0), n, P.seed_state.p);
    after_launch("seed_kernel", st);
    const unsigned g = static_cast<unsigned>((n + 3) / 4);
    if (P.cfg.variant)
      tables_draw_kernel<true><<<g, 128, 0, st>>>(P.keys.p, static_cast<int>(k0), n, P.seed_state.p, P.E.p, P.Z.p,
                                                  P.tab_overflow.p);
    else
      tables_draw_kernel<false><<<g, 128, 0, st>>>(P.keys.p, static_cast<int>(k0), n, P.seed_state.p, P.E.p, P.Z.p,
                                                   P.tab_overflow.p);
    after_launch("tables_draw_kernel", st);
    launches += 2;
  }
  return launches + launch_decks(P, st);
}

// Full-mode decks (deck_kernel) of the plan's keys, once their tables are sized.
int launch_decks(lt_plan& P, cudaStream_t st) {
  if (P.h_decks.empty()) return 0;
  LT_CUDA(cudaFuncSetAttribute(deck_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, P.ctx->smem_optin));
  deck_kernel<<<static_cast<unsigned>(P.h_decks.size()), 32, P.deck_smem, st>>>(P.keys.p, P.decks.p, P.deck_tab.p,
                                                                                P.big_deck.p, P.big_off.p);
  after_launch("deck_kernel", st);
  return 1;
}

// Full-mode deck tables: one slot per possible arrival of the deck's key.
void size_decks(lt_plan& P, const PinnedVec<DKeyNI>& keys, cudaStream_t st) {
  if (P.h_decks.empty()) return;
  int64_t off = 0, big = 0;
  int max_small = 0;
  std::vector<int64_t> boff(P.h_decks.size(), 0);
  for (size_t d = 0; d < P.h_decks.size(); ++d) {
    DDeck& dk = P.h_decks[d];
    dk.table_off = off;
    off += keys[dk.key].cap;
    if (dk.D > kDeckSmemMax) {
      boff[d] = big;
      big += dk.D;
    } else {
      max_small = std::max(max_small, dk.D);
    }
  }
  P.decks.upload(P.h_decks, st);
  P.deck_tab.alloc(std::max<int64_t>(off, 1));
  P.big_off.upload(boff, st);
  P.big_deck.alloc(std::max<int64_t>(big, 1));
  P.deck_smem = 624 * sizeof(uint32_t) + kMtN * sizeof(uint64_t) + static_cast<size_t>(max_small) * sizeof(int32_t);
}

// Packs the deferred scenarios' adapter records (the adapter loop of
// prepare_scenario for generated Mean-mode scenarios with ascending ids) on
// several host threads. Returns false if a key was missing (never expected:
// collect_keys saw every such adapter); the caller then repacks serially.
bool pack_deferred(lt_plan& P, Prep& pr, const lt_workload_batch& b) {
  const int64_t nd = static_cast<int64_t>(pr.deferred.size());
  if (nd == 0) return true;
  std::atomic<bool> ok{true};
  auto work = [&](int64_t d0, int64_t d1) {
    for (int64_t d = d0; d < d1; ++d) {
      const Prep::Deferred& df = pr.deferred[d];
      const lt_scenario& s = b.scenarios[df.i];
      const lt_adapter* ad = b.adapters + s.adapter_offset;
      const lt_length_spec& l = b.lengths[s.length_index];
      const double out_mean = output_mean(l, b.full_lengths) + 1.0;
      double cost = 0.0;
      for (int k = 0; k < s.n_adapters; ++k) {
        const lt_adapter& a = ad[k];
        DAdapter x{};
        x.id = a.adapter_id;
        x.rank = a.rank;
        x.rate = a.rate;
        x.load_lat = (a.rank >= 0 && a.rank < 1024) ? P.cfg.lat_cache[a.rank] : load_latency(P.cfg, a.rank);
        x.length_param = -1;
        x.deck = -1;
        x.key = pr.key_base[df.i] >= 0 ? static_cast<int32_t>(pr.key_base[df.i] + k) : pr.find_key(s.seed, a.adapter_id);
        if (x.key < 0) ok = false;
        pr.adapters[df.a_off + k] = x;
        P.adapter_ids[df.a_off + k] = a.adapter_id;
        pr.pair_scen[df.p_off + k] = static_cast<int32_t>(df.i);
        pr.pair_adp[df.p_off + k] = k;
        cost += a.rate * s.duration_s * out_mean;
      }
      pr.cost[df.i] = cost;
    }
  };
  // the load-latency cache is filled serially first (read-only in the workers)
  for (const Prep::Deferred& df : pr.deferred) {
    const lt_scenario& s = b.scenarios[df.i];
    for (int k = 0; k < s.n_adapters; ++k) load_latency_cached(P.cfg, b.adapters[s.adapter_offset + k].rank);
  }
  const int64_t total = pr.deferred.back().a_off + b.scenarios[pr.deferred.back().i].n_adapters -
                        pr.deferred.front().a_off;
  const int nt = std::min<int64_t>(HostPool::width(total, 8192), std::max<int64_t>(nd, 1));
  HostPool::get().run(nt, [&](int t) { work(nd * t / nt, nd * (t + 1) / nt); });
  return ok;
}

// First pass of build_plan: the RNG keys (seed, adapter id) with their
// largest rate and duration over every generated scenario that can pass the
// workload screen, so K0 runs on the device while the second pass validates
// and packs the scenarios. Keys of scenarios that fail later only lengthen
// tables (each table is a prefix-stable draw sequence), never change them.
void collect_keys(Prep& pr, const lt_workload_batch& b) {
  const int64_t n = b.n_scenarios;
  auto screened = [&](const lt_scenario& s) {
    return s.n_requests < 0 && s.n_adapters > 0 && s.n_adapters <= kMaxAdapters && s.duration_s > 0.0;
  };
  // seeds used by exactly one screened scenario with strictly ascending ids
  // and positive rates: one key per adapter, written in parallel below
  std::unordered_map<uint64_t, int32_t> uses;
  uses.reserve(static_cast<size_t>(n) * 2);
  for (int64_t i = 0; i < n; ++i)
    if (screened(b.scenarios[i])) ++uses[b.scenarios[i].seed];
  pr.key_base.assign(n, -1);
  int64_t base = 0;
  for (int64_t i = 0; i < n; ++i) {
    const lt_scenario& s = b.scenarios[i];
    if (!screened(s) || uses[s.seed] != 1) continue;
    const lt_adapter* ad = b.adapters + s.adapter_offset;
    bool ok = ad[0].rate > 0.0;
    for (int k = 1; k < s.n_adapters && ok; ++k) ok = ad[k - 1].adapter_id < ad[k].adapter_id && ad[k].rate > 0.0;
    if (!ok) continue;
    pr.key_base[i] = base;
    base += s.n_adapters;
  }
  pr.keys.resize(static_cast<size_t>(base));
  auto fill = [&](int64_t i0, int64_t i1) {
    for (int64_t i = i0; i < i1; ++i) {
      if (pr.key_base[i] < 0) continue;
      const lt_scenario& s = b.scenarios[i];
      const lt_adapter* ad = b.adapters + s.adapter_offset;
      DKey* out = pr.keys.data() + pr.key_base[i];
      for (int k = 0; k < s.n_adapters; ++k) {
        DKey key{};
        key.seed = s.seed;
        key.id = ad[k].adapter_id;
        key.rate_max = ad[k].rate;
        key.dur_max = s.duration_s;
        out[k] = key;
      }
    }
  };
  const int nt = std::min<int64_t>(HostPool::width(base, 8192), std::max<int64_t>(n, 1));
  HostPool::get().run(nt, [&](int t) { fill(n * t / nt, n * (t + 1) / nt); });
  // the rest (shared seeds) deduplicated per (seed, id)
  for (int64_t i = 0; i < n; ++i) {
    const lt_scenario& s = b.scenarios[i];
    if (!screened(s) || pr.key_base[i] >= 0) continue;
    const lt_adapter* ad = b.adapters + s.adapter_offset;
    Prep::SeedKeys& sk = pr.seed_keys(s.seed);
    for (int k = 0; k < s.n_adapters; ++k) {
      const lt_adapter& a = ad[k];
      if (!(a.rate > 0.0)) continue;
      bool inserted = false;
      const int kidx = Prep::find_or_insert(sk, a.adapter_id, static_cast<int32_t>(pr.keys.size()), &inserted);
      if (inserted) {
        DKey key{};
        key.seed = s.seed;
        key.id = a.adapter_id;
        key.rate_max = a.rate;
        key.dur_max = s.duration_s;
        pr.keys.push_back(key);
      } else {
        DKey& key = pr.keys[kidx];
        key.rate_max = std::max(key.rate_max, a.rate);
        key.dur_max = std::max(key.dur_max, s.duration_s);
      }
    }
  }
}

// Table capacity per key: rate_max * dur_max + 8 sigma + slack draws.
// (On host threads for large key sets: the capacities and partial sums per
// range, then the offsets; the K0 launch waits on this.)
int64_t size_keys(PinnedVec<DKeyNI>& keys) {
  const int64_t n = static_cast<int64_t>(keys.size());
  auto cap_of = [](const DKey& k) {
    const double lam = k.rate_max * k.dur_max;
    const double capd = lam + 8.0 * std::sqrt(lam) + 32.0;
    return static_cast<int32_t>(std::min(capd, 2.0e9));
  };
  const int nt = HostPool::width(n, 8192);
  std::vector<int64_t> part(nt + 1, 0);
  auto caps = [&](int t) {
    int64_t sum = 0;
    for (int64_t i = n * t / nt; i < n * (t + 1) / nt; ++i) {
      keys[i].cap = cap_of(keys[i]);
      sum += keys[i].cap;
    }
    part[t + 1] = sum;
  };
  auto offsets = [&](int t) {
    int64_t off = part[t];
    for (int64_t i = n * t / nt; i < n * (t + 1) / nt; ++i) {
      keys[i].e_off = off;
      keys[i].z_off = off;
      off += keys[i].cap;
    }
  };
  HostPool::get().run(nt, caps);
  for (int t = 0; t < nt; ++t) part[t + 1] += part[t];
  HostPool::get().run(nt, offsets);
  return part[nt];
}

// Request arrays and merge scratch for P.total_req requests of P.n_pairs
// (scenario, adapter) streams over P.n_scen scenarios.
void alloc_requests(lt_plan& P) {
  cudaStream_t st = P.st;
  const int64_t nr = std::max<int64_t>(P.total_req, 1);
  P.r_arr.alloc(nr);
  P.r_in.alloc(nr);
  P.r_out.alloc(nr);
  P.r_adp.alloc(nr);
  P.r_phase.alloc(nr);
  P.r_gen.alloc(nr);
  P.r_first.alloc(nr);
  P.r_last.alloc(nr);
  P.r_pre.alloc(nr);
  if (P.total_req >= (int64_t(1) << 31)) throw CudaError{"batch too large: more than 2^31 requests in one plan"};
  if (P.n_pairs > 0) {
    P.pair_excl.alloc(P.n_pairs);
    P.st_in.alloc(nr);
    P.st_out.alloc(nr);
    P.sv_in.alloc(nr);
    P.sv_out.alloc(nr);
    P.seg_begin.alloc(P.n_scen);
    P.seg_end.alloc(P.n_scen);
    LT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, P.pscan_tmp_bytes, P.adp_count.p, P.pair_excl.p,
                                          static_cast<int>(P.n_pairs), st));
    P.pscan_tmp.alloc(std::max<size_t>(P.pscan_tmp_bytes, 1));
    if (radix_merge(nr)) {
      P.pos_a.alloc(nr);
      P.pos_b.alloc(nr);
      P.skey_a.alloc(nr);
      P.skey_b.alloc(nr);
      P.scen_bits = 1;
      while ((int64_t(1) << P.scen_bits) < P.n_scen) ++P.scen_bits;
      size_t b1 = 0, b2 = 0;
      LT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b1, P.st_in.p, P.st_out.p, P.pos_a.p, P.pos_b.p,
                                              static_cast<int>(nr), 0, 64, st));
      LT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b2, P.skey_a.p, P.skey_b.p, P.pos_b.p, P.pos_a.p,
                                              static_cast<int>(nr), 0, P.scen_bits, st));
      P.sort_tmp_bytes = std::max(b1, b2);
    } else {
      LT_CUDA(cub::DeviceSegmentedSort::StableSortPairs(nullptr, P.sort_tmp_bytes, P.st_in.p, P.st_out.p, P.sv_in.p,
                                                        P.sv_out.p, static_cast<int>(nr), static_cast<int>(P.n_scen),
                                                        P.seg_begin.p, P.seg_end.p, st));
    }
    P.sort_tmp.alloc(std::max<size_t>(P.sort_tmp_bytes, 1));
  }
}

// Engine launch shape of a plan (order, variant, warps, shared memory,
// persistent grid, workspace) from the per-scenario cost estimates and the
// plan's request counts (max_req, total_req) and max_adapters.
void size_engine(lt_plan& P, const std::vector<double>& cost, int max_run_cap) {
  lt_ctx* ctx = P.ctx;
  cudaStream_t st = P.st;
  // engine order: most expensive first
  P.h_order.resize(P.n_scen);
  for (int64_t i = 0; i < P.n_scen; ++i) P.h_order[i] = static_cast<int32_t>(i);
  std::stable_sort(P.h_order.begin(), P.h_order.end(),
                   [&](int32_t x, int32_t y) { return cost[x] > cost[y]; });
  P.order.upload(P.h_order, st);
  P.counter.alloc(1);
  P.out.alloc(std::max<int64_t>(P.n_scen, 1));
  // occupancy-sized persistent grid: 8 warps per block, one block per SM
  // (the engine kernel runs at ~200 registers). Per warp: the adapter tables
  // plus as much of the running set as fits in shared memory.
  {
    // engine_kernel<1> (~200 registers, 8 warps per SM) is the default: the
    // longest engines set every batch's time, even C3's 65,536 (3.25 s vs
    // 3.93 s with engine_kernel<2>: <=128 registers with spills, 16 warps per
    // SM, half the shared memory per warp). LT_ENGINE_VARIANT=2 selects it.
    // Variant 3: 12 warps per block (<= 170 registers), one block per SM.
    // Batches whose mean work per warp slot exceeds their longest engine are
    // throughput-bound (C3 / C5 chunks: 12% / 17% faster with 12 warps);
    // one-round batches are set by their longest engines, which run ~7%
    // faster at the latency variant's register budget (C2).
    // LT_ENGINE_VARIANT overrides.
    P.engine_variant = 1;
    if (P.warps_per_block == 8 && P.n_scen > 0) {
      double total = 0.0, longest = 0.0;
      for (int64_t i = 0; i < P.n_scen; ++i) {
        total += cost[i];
        longest = std::max(longest, cost[i]);
      }
      if (total / (static_cast<double>(ctx->sm_count) * 8.0) > longest) P.engine_variant = 3;
    }
    if (const char* env = std::getenv("LT_ENGINE_VARIANT")) {
      const int v = std::atoi(env);
      P.engine_variant = (v == 2 || v == 3) ? v : 1;
    }
    if (P.engine_variant == 3 && P.warps_per_block == 8) P.warps_per_block = 12;
    // per SM, below the 227 KB opt-in limit (variant 2: two blocks per SM)
    size_t budget = (static_cast<size_t>(ctx->smem_optin) - 1024) / (P.engine_variant == 2 ? 2 : 1);
    // per warp: adapter tables, retire calendar, then the running-set slots
    // (int4 entry + int32 calendar link each) that fit
    const size_t adapters = static_cast<size_t>(P.max_adapters) * kSmemPerAdapter + 2 * kCalBuckets * sizeof(int32_t) +
                            kPqSmem * sizeof(int4);
    // Every warp's adapter tables must fit in the block: many-adapter batches
    // (24 B per adapter per warp) leave the occupancy variants and then drop
    // warps per block until they do (1,024 adapters: 7 warps of 29.7 KB).
    if (static_cast<size_t>(P.warps_per_block) * adapters > budget && P.engine_variant != 1) {
      P.engine_variant = 1;
      P.warps_per_block = std::min(P.warps_per_block, 8);
      budget = static_cast<size_t>(ctx->smem_optin) - 1024;
    }
    while (P.warps_per_block > 1 && static_cast<size_t>(P.warps_per_block) * adapters > budget) --P.warps_per_block;
    const int warps = P.warps_per_block;
    const size_t per_slot = sizeof(int4) + sizeof(int2);
    const size_t per_warp_max = budget / warps;
    int64_t cap = per_warp_max > adapters ? static_cast<int64_t>((per_warp_max - adapters) / per_slot) : 0;
    cap = std::min<int64_t>(cap, max_run_cap) / 32 * 32;
    P.run_cap = static_cast<int32_t>(cap);
    P.smem_per_warp = static_cast<int32_t>(adapters + static_cast<size_t>(cap) * per_slot);
    P.block = warps * 32;
    P.smem = static_cast<size_t>(P.smem_per_warp) * warps;
  }
  // The device's opt-in maximum (a constant, so plans built concurrently on
  // other host threads never lower it under each other) and the max-shared
  // carveout, so an engine block and the K0 seed kernel of the next chunk can
  // share an SM.
  const void* ek = engine_kernel_fn(P.engine_variant);
  LT_CUDA(cudaFuncSetAttribute(ek, cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->smem_optin));
  LT_CUDA(cudaFuncSetAttribute(ek, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
  int per_sm = 0;
  LT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ek, P.block, P.smem));
  per_sm = std::max(per_sm, 1);
  // at least one block per SM while there are scenarios for them (the first
  // round spreads the heaviest engines one per SM)
  const int64_t want = std::max<int64_t>((P.n_scen + P.block / 32 - 1) / (P.block / 32),
                                         std::min<int64_t>(P.n_scen, ctx->sm_count));
  P.grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(ctx->sm_count) * per_sm)));
}

// The engine workspace, once the request counts are known (size_engine ran
// before them: it needs only the cost estimates).
void size_workspace(lt_plan& P) {
  P.ws_stride = std::max<int64_t>(P.max_req, 1);
  {
    // Workspace per persistent warp slot (slots x longest scenario) or per
    // scenario (at its request offset), whichever is smaller.
    const int64_t slots = int64_t(P.grid) * (P.block / 32);
    const int64_t per_slot = slots * P.ws_stride;
    const int64_t per_scen = std::max<int64_t>(P.total_req, 1);
    P.ws_per_scenario = per_scen < per_slot;
    const int64_t entries = P.ws_per_scenario ? per_scen : per_slot;
    P.ws_run.alloc(entries);
    P.ws_pq.alloc(entries);
    P.ws_node.alloc(entries);
    P.ws_link.alloc(entries);
    P.ws_ov.alloc(entries);
  }
}

// Adapter records the batch's scenarios reference (a chunk of a larger batch
// shares the caller's adapter array, so b->n_adapters would over-reserve).
int64_t batch_adapters(const lt_workload_batch* b) {
  int64_t n = 0;
  for (int64_t i = 0; i < b->n_scenarios; ++i) n += std::max<int32_t>(b->scenarios[i].n_adapters, 0);
  return std::min<int64_t>(n, b->n_adapters);
}

// Builds a plan: validation, RNG tables, counting, merge, request arrays,
// workspace. Leaves everything resident; returns nullptr + status on error.
lt_plan* build_plan(lt_ctx* ctx, const lt_workload_batch* b, const lt_server_config* cfg,
                    const lt_sim_options* opts, int warps_per_block = 8, int max_run_cap = 1024,
                    cudaStream_t stream = nullptr) {
  auto plan = std::make_unique<lt_plan>();
  lt_plan& P = *plan;
  P.ctx = ctx;
  P.st = stream ? stream : ctx->stream;
  for (cudaEvent_t& e : P.ev) LT_CUDA(cudaEventCreate(&e));
  P.warps_per_block = warps_per_block;
  cudaStream_t st = P.st;
  load_config(P.cfg, cfg, opts);
  P.want_digest = opts ? opts->want_digest : 0;
  P.want_pct = opts ? opts->want_percentiles : 0;
  P.want_check = opts ? opts->check_invariants : 0;
  P.n_scen = b->n_scenarios;
  P.h_scen.resize(P.n_scen);
  P.errs.resize(P.n_scen);
  using hclk = std::chrono::steady_clock;
  const auto h0 = hclk::now();
  auto hms = [&](hclk::time_point t) { return std::chrono::duration<double, std::milli>(t - h0).count(); };
  // (the pinned Prep buffers are rewritten below: no upload of an earlier
  // plan may still read them)
  LT_CUDA(cudaStreamSynchronize(ctx->stream_up));
  static thread_local Prep t_prep;
  Prep& pr = t_prep;
  pr.reset();
  pr.cost.assign(P.n_scen, 0.0);
  const int64_t n_ad = batch_adapters(b);
  pr.keys.reserve(n_ad);
  P.adapter_ids.reserve(n_ad);
  pr.adapters.reserve(n_ad);
  pr.pair_scen.reserve(n_ad);
  pr.pair_adp.reserve(n_ad);
  pr.pair_begin.resize(P.n_scen);
  // pass 1 + early K0 (seed_seq and table draws; Full-mode decks follow pass 2)
  const auto h_setup = hclk::now();
  collect_keys(pr, *b);
  const auto h_keys = hclk::now();
  int64_t e_total = size_keys(pr.keys);
  const auto h_size = hclk::now();
  cudaEventRecord(P.ev[0], st);
  if (!pr.keys.empty())
    P.seed_state.alloc(std::min<int64_t>(static_cast<int64_t>(pr.keys.size()), kSeedChunk) * 2 * kMtN);
  P.tab_overflow.alloc(1);
  LT_CUDA(cudaMemsetAsync(P.tab_overflow.p, 0, sizeof(int32_t), st));
  const size_t early_keys = pr.keys.size();
  auto h_up = h_size;
  if (early_keys > 0) {
    P.keys.upload(pr.keys.data(), pr.keys.size(), st);
    P.E.alloc(std::max<int64_t>(e_total, 1));
    P.Z.alloc(std::max<int64_t>(e_total, 1));
    P.h2d_bytes += pr.keys.size() * sizeof(DKey);
    h_up = hclk::now();
    P.launches_prep += launch_tables(P, static_cast<int>(early_keys), st);
  }
  if (std::getenv("LT_HOST_TIMING"))
    std::fprintf(stderr, "[lt]   K0 launch: size_keys %.2f, allocs+upload %.2f, launches %.2f ms\n", hms(h_size),
                 hms(h_up), hms(hclk::now()));
  // pass 2: validation and packing in reference order; the adapter records
  // of plain generated scenarios are packed afterwards on several threads
  const auto h_k0 = hclk::now();
  std::vector<PlainPre> pre;
  auto h_screen = h_k0, h_serial = h_k0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    pr.allow_defer = attempt == 0 && !std::getenv("LT_SERIAL_PREP");
    const bool screen = pr.allow_defer && !std::getenv("LT_NO_PRESCREEN");
    if (screen) prescreen_plain(P, *b, pre);
    h_screen = hclk::now();
    int32_t last_len_index = -1, last_len_param = -1;
    for (int64_t i = 0; i < P.n_scen; ++i) {
      pr.pair_begin[i] = static_cast<int64_t>(pr.pair_scen.size());
      if (screen && pre[i].plain) {
        plain_scenario(P, pr, *b, i, pre[i], last_len_index, last_len_param);
        continue;
      }
      prepare_scenario(P, pr, *b, i);
      if (P.errs[i].code != LT_OK) {
        // drop partially appended pairs of a failed scenario
        pr.pair_scen.resize(pr.pair_begin[i]);
        pr.pair_adp.resize(pr.pair_begin[i]);
      }
    }
    h_serial = hclk::now();
    if (pack_deferred(P, pr, *b)) break;
    // a key was missing: repack everything serially
    pr.deferred.clear();
    pr.adapters.clear();
    P.adapter_ids.clear();
    pr.pair_scen.clear();
    pr.pair_adp.clear();
    pr.lens.clear();
    pr.len_index.clear();
    pr.decks.clear();
    pr.deck_index.clear();
    P.max_adapters = 0;
  }
  P.max_adapters = (P.max_adapters + 31) / 32 * 32;
  if (pr.lens.empty()) pr.lens.push_back(DLen{1, 0, 1, 0});
  // The packed scenarios go up on their own stream while K0 runs.
  {
    cudaStream_t su = ctx->stream_up;
    LT_CUDA(cudaEventCreateWithFlags(&P.ev_up, cudaEventDisableTiming));
    P.scen.upload(P.h_scen, su);
    P.adapters.upload(pr.adapters.data(), pr.adapters.size(), su);  // (DAdapterNI: DAdapter layout)
    P.lens.upload(pr.lens, su);
    P.h2d_bytes += P.h_scen.size() * sizeof(DScen) + pr.adapters.size() * sizeof(DAdapter);
    std::vector<unsigned long long> base(std::max<int64_t>(P.n_scen, 1), 0ULL);
    for (int64_t i = 0; i < P.n_scen; ++i)
      if (!P.h_scen[i].generated && P.h_scen[i].status == LT_OK) base[i] = P.h_scen[i].n_req;
    P.base_count.upload(base, su);
    if (!pr.pair_scen.empty()) {
      P.pair_scen.upload(pr.pair_scen.data(), pr.pair_scen.size(), su);
      P.pair_adp.upload(pr.pair_adp.data(), pr.pair_adp.size(), su);
      P.pair_begin.upload(pr.pair_begin.data(), pr.pair_begin.size(), su);
    }
    LT_CUDA(cudaEventRecord(P.ev_up, su));
  }
  const auto h_prep = hclk::now();
  P.h_decks = pr.decks;
  if (!P.h_decks.empty() && b->n_full_pairs > 0) {
    std::vector<int32_t> fl(b->full_lengths, b->full_lengths + 2 * b->n_full_pairs);
    P.full.upload(fl, st);
  }
  // (pass 2 found every key pass 1 did, unchanged, unless late_keys)
  bool relaunch = (pr.late_keys || std::getenv("LT_K0_RELAUNCH")) && !pr.keys.empty();  // (env: test hook)
  if (relaunch) e_total = size_keys(pr.keys);
  if (!relaunch && !P.h_decks.empty()) {  // decks of the early tables
    size_decks(P, pr.keys, st);
    P.launches_prep += launch_decks(P, st);
  }
  for (int attempt = 0;; ++attempt) {
    if (relaunch) {
      P.seed_state.alloc(std::min<int64_t>(static_cast<int64_t>(pr.keys.size()), kSeedChunk) * 2 * kMtN);
      size_decks(P, pr.keys, st);
      P.keys.upload(pr.keys.data(), pr.keys.size(), st);
      LT_CUDA(cudaMemsetAsync(P.tab_overflow.p, 0, sizeof(int32_t), st));
      P.E.alloc(std::max<int64_t>(e_total, 1));
      P.Z.alloc(std::max<int64_t>(e_total, 1));
      P.h2d_bytes += pr.keys.size() * sizeof(DKey);
      P.launches_prep += launch_tables(P, static_cast<int>(pr.keys.size()), st);
    }
    relaunch = true;
    int32_t any = 0;
    LT_CUDA(cudaMemcpyAsync(&any, P.tab_overflow.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaStreamSynchronize(st));
    if (!any) break;
    std::vector<DKey> back(pr.keys.size());
    LT_CUDA(cudaMemcpyAsync(back.data(), P.keys.p, back.size() * sizeof(DKey), cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaStreamSynchronize(st));
    if (attempt > 4) throw CudaError{"RNG table sizing failed"};
    e_total = 0;
    for (size_t k = 0; k < pr.keys.size(); ++k) {
      DKey& key = pr.keys[k];
      if (back[k].overflow) key.cap = static_cast<int32_t>(std::min<int64_t>(int64_t(key.cap) * 4, 2000000000));
      key.e_off = key.z_off = e_total;
      e_total += key.cap;
    }
  }
  cudaEventRecord(P.ev[1], st);
  const auto h_tables = hclk::now();
  // count arrivals per (scenario, adapter): sizes the request arrays
  const int64_t n_pairs = static_cast<int64_t>(pr.pair_scen.size());
  P.n_pairs = n_pairs;
  P.n_keys = static_cast<int>(pr.keys.size());
  P.scen_count.alloc(std::max<int64_t>(P.n_scen, 1));
  P.scen_off.alloc(std::max<int64_t>(P.n_scen, 1));
  P.overflow.alloc(1);
  LT_CUDA(cudaStreamWaitEvent(st, P.ev_up, 0));  // the packed-scenario uploads
  if (n_pairs > 0) {
    P.adp_count.alloc(n_pairs);
    LT_CUDA(cudaMemsetAsync(P.scen_count.p, 0, P.n_scen * sizeof(unsigned long long), st));
    LT_CUDA(cudaMemsetAsync(P.overflow.p, 0, sizeof(int32_t), st));
    P.pair_g = pair_group(mean_pair_draws(b));
    launch_count(P, st);
    ++P.launches_prep;
  }
  // the engine's order, variant and grid need only the cost estimates: sized
  // while K0 and the counts run
  size_engine(P, pr.cost, max_run_cap);
  if (n_pairs > 0) {
    std::vector<unsigned long long> counts(P.n_scen);
    int32_t ovf = 0;
    LT_CUDA(cudaMemcpyAsync(counts.data(), P.scen_count.p, P.n_scen * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaMemcpyAsync(&ovf, P.overflow.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaStreamSynchronize(st));
    if (ovf) throw CudaError{"internal: RNG table shorter than an arrival stream"};
    for (int64_t i = 0; i < P.n_scen; ++i)
      if (P.h_scen[i].generated && P.h_scen[i].status == LT_OK) P.h_scen[i].n_req = static_cast<int32_t>(counts[i]);
  }
  LT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, P.scan_tmp_bytes, P.scen_count.p, P.scen_off.p,
                                        static_cast<int>(std::max<int64_t>(P.n_scen, 1)), st));
  P.scan_tmp.alloc(std::max<size_t>(P.scan_tmp_bytes, 1));
  int64_t off = 0;
  for (int64_t i = 0; i < P.n_scen; ++i) {
    P.h_scen[i].req_begin = off;
    off += P.h_scen[i].n_req;
    P.max_req = std::max<int64_t>(P.max_req, P.h_scen[i].n_req);
  }
  P.total_req = off;
  P.scen.upload(P.h_scen, st);
  alloc_requests(P);
  // scripted requests
  {
    std::vector<double> arr;
    std::vector<int32_t> in, outv, adp;
    std::vector<int64_t> where;
    for (int64_t i = 0; i < P.n_scen; ++i) {
      const lt_scenario& s = b->scenarios[i];
      if (s.n_requests < 0 || P.h_scen[i].status != LT_OK) continue;
      std::unordered_map<int, int> dense;
      const int64_t ab = P.h_scen[i].adapter_begin;
      for (int k = 0; k < s.n_adapters; ++k) dense[P.adapter_ids[ab + k]] = k;
      for (int64_t r = 0; r < s.n_requests; ++r) {
        const lt_request& q = b->requests[s.request_offset + r];
        arr.push_back(q.arrival_time_s);
        in.push_back(q.input_tokens);
        outv.push_back(q.output_tokens);
        adp.push_back(dense[q.adapter_id]);
      }
      where.push_back(i);
    }
    P.has_scripted = !where.empty();
    int64_t cursor = 0;
    for (int64_t i : where) {
      const int64_t n = P.h_scen[i].n_req;
      const int64_t at = P.h_scen[i].req_begin;
      LT_CUDA(cudaMemcpyAsync(P.r_arr.p + at, arr.data() + cursor, n * sizeof(double), cudaMemcpyHostToDevice, st));
      LT_CUDA(cudaMemcpyAsync(P.r_in.p + at, in.data() + cursor, n * sizeof(int32_t), cudaMemcpyHostToDevice, st));
      LT_CUDA(cudaMemcpyAsync(P.r_out.p + at, outv.data() + cursor, n * sizeof(int32_t), cudaMemcpyHostToDevice, st));
      LT_CUDA(cudaMemcpyAsync(P.r_adp.p + at, adp.data() + cursor, n * sizeof(int32_t), cudaMemcpyHostToDevice, st));
      cursor += n;
    }
    P.h2d_bytes += cursor * 20;  // (pageable sources: the copies are staged before the calls return)
  }
  size_workspace(P);
  P.tables_ms = elapsed(P.ev[0], P.ev[1]);
  P.fresh = true;
  if (std::getenv("LT_HOST_TIMING"))
    std::fprintf(stderr,
                 "[lt] build_plan host: setup %.2f, keys %.2f, K0 launch %.2f, screen %.2f, serial pass %.2f, "
                 "packing+uploads %.2f -> prep %.2f ms, +tables sync %.2f ms, total %.2f ms (%lld scenarios)\n",
                 hms(h_setup), hms(h_keys), hms(h_k0), hms(h_screen), hms(h_serial), hms(h_prep), hms(h_prep),
                 hms(h_tables), hms(hclk::now()), static_cast<long long>(P.n_scen));
  return plan.release();
}

// Buffers a run regenerates from the plan's inputs (K0 tables, request
// arrays, merge scratch, engine workspace): what lt_plan_trim releases.
template <typename F>
void for_transient(lt_plan& P, F&& f) {
  f(P.seed_state);
  f(P.E);
  f(P.Z);
  f(P.r_arr);
  f(P.r_first);
  f(P.r_last);
  f(P.r_in);
  f(P.r_out);
  f(P.r_adp);
  f(P.r_gen);
  f(P.r_pre);
  f(P.r_phase);
  f(P.ws_run);
  f(P.ws_pq);
  f(P.ws_node);
  f(P.ws_ov);
  f(P.ws_link);
  f(P.pair_excl);
  f(P.st_in);
  f(P.st_out);
  f(P.sv_in);
  f(P.sv_out);
  f(P.pos_a);
  f(P.pos_b);
  f(P.skey_a);
  f(P.skey_b);
  f(P.sort_tmp);
}

void trim_plan(lt_plan& P) {
  if (P.trimmed || P.has_scripted) return;
  P.trimmed_sizes.clear();
  for_transient(P, [&](auto& b) {
    P.trimmed_sizes.push_back(b.n);
    b.release();
  });
  P.trimmed = true;
  P.fresh = false;  // the next run regenerates the tables
}

void untrim_plan(lt_plan& P) {
  if (!P.trimmed) return;
  size_t k = 0;
  for_transient(P, [&](auto& b) { b.alloc(P.trimmed_sizes[k++]); });
  P.trimmed = false;
}

int64_t merge_requests(lt_plan& P);

// K0 + merge: (re)generates every request of every generated scenario.
void prepare_requests(lt_plan& P) {
  cudaStream_t st = P.st;
  cudaEventRecord(P.ev[0], st);
  // K0: RNG tables, arrival counts and request offsets are recomputed on
  // device every run (the first run after lt_plan_simulate reuses the ones
  // computed while sizing the buffers).
  int64_t launches = 0;
  if (!P.fresh && P.n_keys > 0) launches += launch_tables(P, P.n_keys, st);
  cudaEventRecord(P.ev[1], st);
  if (!P.fresh && P.n_scen > 0) {
    LT_CUDA(cudaMemcpyAsync(P.scen_count.p, P.base_count.p, P.n_scen * sizeof(unsigned long long),
                            cudaMemcpyDeviceToDevice, st));
    if (P.n_pairs > 0) {
      launch_count(P, st);
      ++launches;
    }
    size_t tb = P.scan_tmp_bytes;
    LT_CUDA(cub::DeviceScan::ExclusiveSum(P.scan_tmp.p, tb, P.scen_count.p, P.scen_off.p,
                                          static_cast<int>(P.n_scen), st));
    set_offsets_kernel<<<static_cast<unsigned>((P.n_scen + 255) / 256), 256, 0, st>>>(
        P.scen.p, static_cast<int>(P.n_scen), P.scen_count.p, P.scen_off.p);
    after_launch("set_offsets_kernel", st);
    launches += 2;
  }
  cudaEventRecord(P.ev[2], st);
  launches += merge_requests(P);
  cudaEventRecord(P.ev[3], st);
  P.fresh = false;
  P.launches_run = launches + 2;  // + engine, metrics (launch_engine)
}

// Arrival merge of the counted streams: per-pair times (expand), stable sort
// by time per scenario, gather into the request arrays. Returns own launches.
int64_t merge_requests(lt_plan& P) {
  cudaStream_t st = P.st;
  int64_t launches = 0;
  if (P.n_pairs > 0) {
    // sort-based merge: unsorted times per (scenario, adapter), stable
    // segmented sort by time, gather into request arrays
    size_t tb = P.pscan_tmp_bytes;
    LT_CUDA(cub::DeviceScan::ExclusiveSum(P.pscan_tmp.p, tb, P.adp_count.p, P.pair_excl.p,
                                          static_cast<int>(P.n_pairs), st));
    launch_expand(P, st);
    size_t sb = P.sort_tmp_bytes;
    const int nr = static_cast<int>(std::max<int64_t>(P.total_req, 1));
    const unsigned gr = static_cast<unsigned>((nr + 255) / 256);
    const int32_t* perm = nullptr;
    if (P.pos_a.p) {  // two global stable radix sorts (see scen_key_kernel)
      iota_kernel<<<gr, 256, 0, st>>>(P.pos_a.p, nr);
      after_launch("iota_kernel", st);
      LT_CUDA(cub::DeviceRadixSort::SortPairs(P.sort_tmp.p, sb, P.st_in.p, P.st_out.p, P.pos_a.p, P.pos_b.p, nr, 0,
                                              64, st));
      scen_key_kernel<<<gr, 256, 0, st>>>(P.scen.p, static_cast<int>(P.n_scen), nr, P.pos_b.p, P.skey_a.p);
      after_launch("scen_key_kernel", st);
      sb = P.sort_tmp_bytes;
      LT_CUDA(cub::DeviceRadixSort::SortPairs(P.sort_tmp.p, sb, P.skey_a.p, P.skey_b.p, P.pos_b.p, P.pos_a.p, nr, 0,
                                              P.scen_bits, st));
      perm = P.pos_a.p;
      launches += 2;  // iota, scen_key
    } else if (merge_mode() == 2) {  // the per-scenario stable segmented sort (CUB)
      segments_kernel<<<static_cast<unsigned>((P.n_scen + 255) / 256), 256, 0, st>>>(
          P.scen.p, static_cast<int>(P.n_scen), P.seg_begin.p, P.seg_end.p);
      after_launch("segments_kernel", st);
      LT_CUDA(cub::DeviceSegmentedSort::StableSortPairs(P.sort_tmp.p, sb, P.st_in.p, P.st_out.p, P.sv_in.p,
                                                        P.sv_out.p, nr, static_cast<int>(P.n_scen), P.seg_begin.p,
                                                        P.seg_end.p, st));
      launches += 1;  // segments
    } else {  // merge tree of the per-adapter lists, one block per scenario
      merge_kernel<<<static_cast<unsigned>(P.n_scen), 512, 0, st>>>(P.scen.p, P.pair_begin.p, P.pair_excl.p,
                                                                    P.st_in.p, P.sv_in.p, P.st_out.p, P.sv_out.p);
      after_launch("merge_kernel", st);
      launches += 1;
    }
    gather_kernel<<<gr, 256, 0, st>>>(P.scen.p, static_cast<int>(P.n_scen), P.total_req, P.adapters.p, P.keys.p,
                                      P.lens.p, P.Z.p, perm ? P.st_in.p : P.st_out.p, perm ? P.sv_in.p : P.sv_out.p,
                                      P.r_arr.p, P.r_in.p, P.r_out.p, P.r_adp.p, P.decks.p, P.deck_tab.p, P.full.p,
                                      perm);
    after_launch("gather_kernel", st);
    launches += 2;  // expand, gather (own kernels; CUB's scan and sorts not counted)
  }
  return launches;
}

// The report / checked engine build (engine_kernel<256,1,true>) on the plan's
// warp layout, at most 8 warps per block.
void launch_engine_checked(lt_plan& P, const EngineParams& E, cudaStream_t st) {
  const int warps = std::min(P.block / 32, 8);
  LT_CUDA(cudaFuncSetAttribute(engine_kernel_fn(kEngineChecked), cudaFuncAttributeMaxDynamicSharedMemorySize,
                               P.ctx->smem_optin));
  launch_engine_build(kEngineChecked, static_cast<unsigned>(P.grid), static_cast<unsigned>(warps * 32),
                      static_cast<size_t>(P.smem_per_warp) * warps, st, E);
}

// K1 (the engine kernel) then K2 (metrics_kernel) over the plan's scenarios.
void launch_engine(lt_plan& P, const EngineParams& E, cudaStream_t st) {
  if (E.check_invariants)
    launch_engine_checked(P, E, st);
  else
    launch_engine_build(P.engine_variant, static_cast<unsigned>(P.grid), static_cast<unsigned>(P.block), P.smem, st,
                        E);
  after_launch("engine_kernel", st);
  metrics_kernel<<<static_cast<unsigned>((P.n_scen + 7) / 8), 256, 0, st>>>(
      E.scen, E.n_scen, E.r_phase, E.r_first, E.r_arr, E.r_last, E.r_out, E.r_gen, E.out);
}

// Per-request engine state before an engine pass.
void reset_state(lt_plan& P) {
  cudaStream_t st = P.st;
  const int64_t nr = std::max<int64_t>(P.total_req, 1);
  LT_CUDA(cudaMemsetAsync(P.r_phase.p, 0, nr, st));
  LT_CUDA(cudaMemsetAsync(P.r_gen.p, 0, nr * sizeof(int32_t), st));
  LT_CUDA(cudaMemsetAsync(P.r_pre.p, 0, nr * sizeof(int32_t), st));
  LT_CUDA(cudaMemsetAsync(P.r_first.p, 0xff, nr * sizeof(double), st));  // NaN: no first token
  LT_CUDA(cudaMemsetAsync(P.r_last.p, 0, nr * sizeof(double), st));
  LT_CUDA(cudaMemsetAsync(P.counter.p, 0, sizeof(int32_t), st));
}

// Kernel parameters of a plan's engine pass.
EngineParams engine_params(const lt_plan& P) {
  EngineParams E{};
  E.scen = P.scen.p;
  E.order = P.order.p;
  E.n_scen = static_cast<int32_t>(P.n_scen);
  E.max_adapters = P.max_adapters;
  E.run_cap = P.run_cap;
  E.smem_per_warp = P.smem_per_warp;
  E.counter = P.counter.p;
  E.adapters = P.adapters.p;
  E.r_arr = P.r_arr.p;
  E.r_in = P.r_in.p;
  E.r_out = P.r_out.p;
  E.r_adp = P.r_adp.p;
  E.r_phase = P.r_phase.p;
  E.r_gen = P.r_gen.p;
  E.r_first = P.r_first.p;
  E.r_last = P.r_last.p;
  E.r_pre = P.r_pre.p;
  E.ws_run = P.ws_run.p;
  E.ws_pq = P.ws_pq.p;
  E.ws_node = P.ws_node.p;
  E.ws_link = P.ws_link.p;
  E.ws_ov = P.ws_ov.p;
  E.ws_stride = P.ws_stride;
  E.ws_per_scenario = P.ws_per_scenario;
  E.k1 = P.cfg.raw.k1;
  E.k2 = P.cfg.raw.k2;
  E.k3 = P.cfg.raw.k3;
  E.k4 = P.cfg.raw.k4;
  E.k5 = P.cfg.raw.k5;
  E.k6 = P.cfg.raw.k6;
  E.k7 = P.cfg.raw.k7;
  E.priority = P.cfg.raw.loaded_adapter_priority;
  E.want_digest = P.want_digest;
  E.out = P.out.p;
  E.check_invariants = P.want_check;
  const char* inject = std::getenv("LT_INVARIANT_INJECT");  // test hook: a ledger fault at this iteration
  E.inject_iteration = inject ? std::atoll(inject) : -1;
  return E;
}

void run_percentiles(lt_plan& P, EngineParams E);

void run_plan(lt_plan& P) {
  cudaStream_t st = P.st;
  untrim_plan(P);
  prepare_requests(P);
  reset_state(P);
  const EngineParams E = engine_params(P);
  cudaEventRecord(P.ev[4], st);
  if (P.n_scen > 0) {
    launch_engine(P, E, st);
    after_launch("metrics_kernel", st);
  }
  cudaEventRecord(P.ev[5], st);
  if (P.want_pct && P.n_scen > 0) run_percentiles(P, E);
}

// TTFT/ITL p50/p99 (metrics.cpp:47-54): a second, recording engine pass sized
// by the first pass's iteration and preemption counts, then segmented sorts
// and a weighted rank select (k_metrics.cuh).
void run_percentiles(lt_plan& P, EngineParams E) {
  cudaStream_t st = P.st;
  const int64_t n = P.n_scen;
  std::vector<lt_sim_summary> h(n);
  LT_CUDA(cudaMemcpyAsync(h.data(), P.out.p, n * sizeof(lt_sim_summary), cudaMemcpyDeviceToHost, st));
  LT_CUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> off(n), len(n);
  std::vector<int32_t> rb(n), re(n), tb(n), te(n);
  int64_t tot = 0;
  for (int64_t i = 0; i < n; ++i) {
    len[i] = (h[i].status == LT_OK) ? h[i].iterations + h[i].preemptions : 0;
    off[i] = tot;
    tot += len[i];
    tb[i] = static_cast<int32_t>(P.h_scen[i].req_begin);
    te[i] = static_cast<int32_t>(P.h_scen[i].req_begin + P.h_scen[i].n_req);
  }
  if (tot >= (int64_t(1) << 31)) throw CudaError{"percentiles: more than 2^31 ITL records in one plan"};
  for (int64_t i = 0; i < n; ++i) {
    rb[i] = static_cast<int32_t>(off[i]);
    re[i] = static_cast<int32_t>(off[i] + len[i]);
  }
  const int64_t nt = std::max<int64_t>(tot, 1), nr = std::max<int64_t>(P.total_req, 1);
  P.rec_off.upload(off, st);
  P.rec_len.upload(len, st);
  P.pct_rseg_b.upload(rb, st);
  P.pct_rseg_e.upload(re, st);
  P.pct_seg_b.upload(tb, st);
  P.pct_seg_e.upload(te, st);
  P.rec_d.alloc(nt);
  P.rec_c.alloc(nt);
  P.rec_d_sorted.alloc(nt);
  P.rec_c_sorted.alloc(nt);
  P.ttft_keys.alloc(nr);
  P.ttft_sorted.alloc(nr);
  LT_CUDA(cudaMemsetAsync(P.rec_c.p, 0, nt * sizeof(int32_t), st));
  reset_state(P);
  E.record = 1;
  E.rec_off = P.rec_off.p;
  E.rec_d = P.rec_d.p;
  E.rec_c = P.rec_c.p;
  launch_engine(P, E, st);
  after_launch("metrics_kernel(record)", st);
  ttft_keys_kernel<<<static_cast<unsigned>((nr + 255) / 256), 256, 0, st>>>(P.r_arr.p, P.r_first.p, nr,
                                                                            P.ttft_keys.p);
  after_launch("ttft_keys_kernel", st);
  size_t b1 = 0, b2 = 0;
  LT_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, b1, P.ttft_keys.p, P.ttft_sorted.p, static_cast<int>(nr),
                                             static_cast<int>(n), P.pct_seg_b.p, P.pct_seg_e.p, st));
  LT_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, b2, P.rec_d.p, P.rec_d_sorted.p, P.rec_c.p,
                                              P.rec_c_sorted.p, static_cast<int>(nt), static_cast<int>(n),
                                              P.pct_rseg_b.p, P.pct_rseg_e.p, st));
  P.pct_tmp.alloc(static_cast<int64_t>(std::max<size_t>(std::max(b1, b2), 1)));
  LT_CUDA(cub::DeviceSegmentedSort::SortKeys(P.pct_tmp.p, b1, P.ttft_keys.p, P.ttft_sorted.p, static_cast<int>(nr),
                                             static_cast<int>(n), P.pct_seg_b.p, P.pct_seg_e.p, st));
  LT_CUDA(cub::DeviceSegmentedSort::SortPairs(P.pct_tmp.p, b2, P.rec_d.p, P.rec_d_sorted.p, P.rec_c.p,
                                              P.rec_c_sorted.p, static_cast<int>(nt), static_cast<int>(n),
                                              P.pct_rseg_b.p, P.pct_rseg_e.p, st));
  percentile_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, 0, st>>>(
      P.scen.p, static_cast<int>(n), P.ttft_sorted.p, P.rec_off.p, P.rec_len.p, P.rec_d_sorted.p,
      P.rec_c_sorted.p, P.out.p);
  after_launch("percentile_kernel", st);
  P.launches_run += 5;  // engine + metrics (recording pass), ttft keys, percentiles
}

// lt_simulate_report's second engine pass (engine_kernel<256, 1, true>),
// sized by the first pass's counts, and the emit-time expansion
// (k_report.cuh). The rows stay on the device in R until copied out.
struct ReportRun {
  std::vector<int64_t> tr_off, ld_off, ld_len;
  int64_t n_tr = 0, n_ld = 0, n_log = 0, n_emit = 0;
  DBuf<int64_t> d_tr_off, d_ld_off, d_sl_off, tokens, emit_off;
  DBuf<double> tr_time, tr_lat, emit;
  DBuf<int4> tr_rwal;
  DBuf<lt_trace_row> trace;
  DBuf<DLoadEvent> ld;
  DBuf<int2> sl_log;
  DBuf<int32_t> sl_cnt, iters, iters_sorted;
  DBuf<uint32_t> keys, keys_sorted;
  DBuf<char> tmp;
};

void run_report(lt_plan& P, ReportRun& R) {
  cudaStream_t st = P.st;
  const int64_t n = P.n_scen;
  const int64_t nr = std::max<int64_t>(P.total_req, 1);
  std::vector<lt_sim_summary> h(n);
  LT_CUDA(cudaMemcpyAsync(h.data(), P.out.p, n * sizeof(lt_sim_summary), cudaMemcpyDeviceToHost, st));
  LT_CUDA(cudaStreamSynchronize(st));
  // rows per scenario: a trace row per iteration, the load events, and at
  // most one stint-log entry per first admission, re-admission and
  // preemption. A scenario that fails in the engine still writes the rows of
  // its completed iterations, plus the loads of the failing call (<= N).
  R.tr_off.resize(n);
  R.ld_off.resize(n);
  R.ld_len.resize(n);
  std::vector<int64_t> sl_off(n);
  int64_t n_sl = 0;
  for (int64_t i = 0; i < n; ++i) {
    R.tr_off[i] = R.n_tr;
    R.ld_off[i] = R.n_ld;
    sl_off[i] = n_sl;
    R.ld_len[i] = h[i].load_events;
    R.n_tr += h[i].iterations;
    R.n_ld += h[i].load_events + (h[i].status != LT_OK ? h[i].served_adapters : 0);
    n_sl += P.h_scen[i].n_req + 2 * h[i].preemptions;
  }
  if (n_sl >= (int64_t(1) << 31) || P.total_req >= (int64_t(1) << 32) - 1)
    throw CudaError{"lt_simulate_report: batch too large for one report (2^31 stint entries)"};
  R.n_log = n_sl;
  R.d_tr_off.upload(R.tr_off, st);
  R.d_ld_off.upload(R.ld_off, st);
  R.d_sl_off.upload(sl_off, st);
  R.tr_time.alloc(std::max<int64_t>(R.n_tr, 1));
  R.tr_lat.alloc(std::max<int64_t>(R.n_tr, 1));
  R.tr_rwal.alloc(std::max<int64_t>(R.n_tr, 1));
  R.ld.alloc(std::max<int64_t>(R.n_ld, 1));
  R.sl_log.alloc(std::max<int64_t>(n_sl, 1));
  R.sl_cnt.alloc(std::max<int64_t>(n, 1));
  LT_CUDA(cudaMemsetAsync(R.sl_cnt.p, 0, R.sl_cnt.n * sizeof(int32_t), st));
  reset_state(P);
  EngineParams E = engine_params(P);
  E.tr_off = R.d_tr_off.p;
  E.tr_time = R.tr_time.p;
  E.tr_lat = R.tr_lat.p;
  E.tr_rwal = R.tr_rwal.p;
  E.ld_off = R.d_ld_off.p;
  E.ld = R.ld.p;
  E.sl_off = R.d_sl_off.p;
  E.sl_log = R.sl_log.p;
  E.sl_cnt = R.sl_cnt.p;
  E.report = 1;
  launch_engine_checked(P, E, st);
  after_launch("engine_kernel(report)", st);
  metrics_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, 0, st>>>(E.scen, E.n_scen, E.r_phase, E.r_first, E.r_arr,
                                                                     E.r_last, E.r_out, E.r_gen, E.out);
  after_launch("metrics_kernel(report)", st);
  // trace rows as lt_trace_row
  R.trace.alloc(std::max<int64_t>(R.n_tr, 1));
  if (R.n_tr > 0) {
    trace_pack_kernel<<<static_cast<unsigned>((R.n_tr + 255) / 256), 256, 0, st>>>(
        R.d_tr_off.p, static_cast<int>(n), R.n_tr, R.tr_time.p, R.tr_lat.p, R.tr_rwal.p, R.trace.p);
    after_launch("trace_pack_kernel", st);
  }
  // emit times: stint log grouped by request (stable), then expanded
  R.keys.alloc(std::max<int64_t>(n_sl, 1));
  R.keys_sorted.alloc(std::max<int64_t>(n_sl, 1));
  R.iters.alloc(std::max<int64_t>(n_sl, 1));
  R.iters_sorted.alloc(std::max<int64_t>(n_sl, 1));
  LT_CUDA(cudaMemsetAsync(R.keys.p, 0xff, R.keys.n * sizeof(uint32_t), st));
  stint_keys_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, 0, st>>>(P.scen.p, static_cast<int>(n), R.d_sl_off.p,
                                                                        R.sl_cnt.p, R.sl_log.p, R.keys.p, R.iters.p);
  after_launch("stint_keys_kernel", st);
  R.tokens.alloc(nr);
  R.emit_off.alloc(nr);
  request_tokens_kernel<<<static_cast<unsigned>((nr + 255) / 256), 256, 0, st>>>(
      P.scen.p, static_cast<int>(n), P.out.p, P.r_phase.p, P.r_gen.p, P.r_out.p, P.total_req, R.tokens.p);
  after_launch("request_tokens_kernel", st);
  size_t b1 = 0, b2 = 0;
  LT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b1, R.keys.p, R.keys_sorted.p, R.iters.p, R.iters_sorted.p,
                                          static_cast<int>(std::max<int64_t>(n_sl, 1)), 0, 32, st));
  LT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b2, R.tokens.p, R.emit_off.p, static_cast<int>(nr), st));
  R.tmp.alloc(std::max<size_t>(std::max(b1, b2), 1));
  LT_CUDA(cub::DeviceRadixSort::SortPairs(R.tmp.p, b1, R.keys.p, R.keys_sorted.p, R.iters.p, R.iters_sorted.p,
                                          static_cast<int>(std::max<int64_t>(n_sl, 1)), 0, 32, st));
  LT_CUDA(cub::DeviceScan::ExclusiveSum(R.tmp.p, b2, R.tokens.p, R.emit_off.p, static_cast<int>(nr), st));
  int64_t last_off = 0, last_tok = 0;
  if (P.total_req > 0) {
    LT_CUDA(cudaMemcpyAsync(&last_off, R.emit_off.p + P.total_req - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaMemcpyAsync(&last_tok, R.tokens.p + P.total_req - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  }
  LT_CUDA(cudaStreamSynchronize(st));
  R.n_emit = last_off + last_tok;
  R.emit.alloc(std::max<int64_t>(R.n_emit, 1));
  if (P.total_req > 0) {
    emit_times_kernel<<<static_cast<unsigned>((P.total_req + 255) / 256), 256, 0, st>>>(
        P.scen.p, static_cast<int>(n), P.total_req, R.keys_sorted.p, R.iters_sorted.p, n_sl, R.tokens.p,
        R.emit_off.p, R.d_tr_off.p, R.tr_time.p, R.tr_lat.p, R.emit.p);
    after_launch("emit_times_kernel", st);
  }
  P.launches_run += 7;
}

void fetch_results(lt_plan& P, lt_sim_summary* out, lt_request_states* states) {
  lt_ctx* ctx = P.ctx;
  cudaStream_t st = P.st;
  if (P.n_scen > 0)
    LT_CUDA(cudaMemcpyAsync(out, P.out.p, P.n_scen * sizeof(lt_sim_summary), cudaMemcpyDeviceToHost, st));
  int64_t d2h = P.n_scen * sizeof(lt_sim_summary);
  std::vector<int8_t> phase;
  std::vector<int32_t> gen, pre, in, outv, adp;
  std::vector<double> first, last, arr;
  if (states && P.trimmed) throw CudaError{"lt_plan_results: per-request states were released by lt_plan_trim"};
  if (states) {
    const int64_t n = P.total_req;
    phase.resize(n);
    gen.resize(n);
    pre.resize(n);
    in.resize(n);
    outv.resize(n);
    adp.resize(n);
    first.resize(n);
    last.resize(n);
    arr.resize(n);
    if (n) {
      LT_CUDA(cudaMemcpyAsync(phase.data(), P.r_phase.p, n, cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(gen.data(), P.r_gen.p, n * 4, cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(pre.data(), P.r_pre.p, n * 4, cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(in.data(), P.r_in.p, n * 4, cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(outv.data(), P.r_out.p, n * 4, cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(adp.data(), P.r_adp.p, n * 4, cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(first.data(), P.r_first.p, n * 8, cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(last.data(), P.r_last.p, n * 8, cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(arr.data(), P.r_arr.p, n * 8, cudaMemcpyDeviceToHost, st));
    }
    d2h += n * 45;
  }
  cudaEventRecord(P.ev[6], st);
  LT_CUDA(cudaStreamSynchronize(st));
  ctx->messages.assign(P.n_scen, std::string());
  for (int64_t i = 0; i < P.n_scen; ++i) {
    const HostErr& e = P.errs[i];
    if (e.code != LT_OK) {
      out[i].status = e.code;
      out[i].status_kind = e.kind;
      out[i].status_a = e.a;
      out[i].status_b = e.b;
      ctx->messages[i] = e.msg;
    } else if (out[i].status != LT_OK) {
      ctx->messages[i] = render(out[i].status, out[i].status_kind, out[i].status_a, out[i].status_b);
    }
  }
  if (states) {
    int64_t off = 0;
    for (int64_t i = 0; i < P.n_scen; ++i) {
      if (states->req_offset) states->req_offset[i] = off;
      const DScen& d = P.h_scen[i];
      for (int64_t r = 0; r < d.n_req; ++r, ++off) {
        if (off >= states->capacity) continue;
        const int64_t g = d.req_begin + r;
        const int8_t ph = phase[g];
        int32_t tg = gen[g];
        if (ph == kFinished) tg = outv[g];
        if (states->phase) states->phase[off] = ph;
        if (states->tokens_generated) states->tokens_generated[off] = tg;
        if (states->first_token_time_s) states->first_token_time_s[off] = first[g];
        if (states->completion_time_s)
          states->completion_time_s[off] =
              (ph == kFinished || (ph == kRunning && tg == outv[g])) ? last[g] : 0.0;
        if (states->preemption_count) states->preemption_count[off] = pre[g];
        if (states->adapter_id) states->adapter_id[off] = P.adapter_ids[d.adapter_begin + adp[g]];
        if (states->input_tokens) states->input_tokens[off] = in[g];
        if (states->output_tokens) states->output_tokens[off] = outv[g];
        if (states->arrival_time_s) states->arrival_time_s[off] = arr[g];
      }
    }
  }
  lt_timing& t = ctx->timing;
  t.tables_ms = elapsed(P.ev[0], P.ev[1]);
  t.merge_ms = elapsed(P.ev[1], P.ev[3]);
  t.engine_ms = elapsed(P.ev[4], P.ev[5]);
  t.d2h_ms = elapsed(P.ev[5], P.ev[6]);
  t.run_ms = elapsed(P.ev[0], P.ev[5]);
  t.d2h_bytes = d2h;
  t.h2d_bytes = P.h2d_bytes;
  t.engine_launches = P.launches_run;
  int64_t bytes = 0;
  for (int64_t i = 0; i < P.n_scen; ++i) {
    const lt_sim_summary& o = out[i];
    bytes += 20 * o.sum_running + 16 * o.sum_visited + 24 * o.sum_arrivals + 16 * o.sum_moves + 64 * o.iterations;
  }
  t.algorithmic_bytes = bytes;
}

int32_t first_error(lt_ctx* ctx, const lt_sim_summary* out, int64_t n, lt_status* st) {
  for (int64_t i = 0; i < n; ++i) {
    if (out[i].status != LT_OK) {
      set_status(st, out[i].status, out[i].status_kind, i, out[i].status_a, out[i].status_b,
                 ctx->messages[i]);
      return out[i].status;
    }
  }
  return LT_OK;
}

// Requests a scenario can generate: the Poisson mean of every adapter plus
// 8 sigma and slack (the same bound that sizes the RNG tables), or the
// scripted list.
double est_requests(const lt_workload_batch* b, int64_t i) {
  const lt_scenario& s = b->scenarios[i];
  if (s.n_requests >= 0) return static_cast<double>(s.n_requests);
  double e = 0.0;
  for (int32_t k = 0; k < s.n_adapters; ++k) {
    const double lam = std::max(b->adapters[s.adapter_offset + k].rate, 0.0) * std::max(s.duration_s, 0.0);
    e += lam + 8.0 * std::sqrt(lam) + 32.0;
  }
  return e;
}

}  // namespace

#include "host_sweep.h"
#include "host_group.h"

// ============================================================================
// C-ABI

extern "C" {

int32_t lt_abi_version(void) { return LT_ABI_VERSION; }

// Diagnostics (not in the public header): host wall time of the plan's
// validation + packing pass alone, no device calls.
double lt__host_prep_ms(const lt_workload_batch* b, const lt_server_config* cfg) {
  const auto t0 = std::chrono::steady_clock::now();
  lt_plan P;
  load_config(P.cfg, cfg, nullptr);
  P.n_scen = b->n_scenarios;
  P.h_scen.resize(P.n_scen);
  P.errs.resize(P.n_scen);
  static thread_local Prep t_prep;
  Prep& pr = t_prep;
  pr.reset();
  pr.cost.assign(P.n_scen, 0.0);
  const int64_t n_ad = batch_adapters(b);
  pr.keys.reserve(n_ad);
  P.adapter_ids.reserve(n_ad);
  pr.adapters.reserve(n_ad);
  pr.pair_scen.reserve(n_ad);
  pr.pair_adp.reserve(n_ad);
  const auto t05 = std::chrono::steady_clock::now();
  collect_keys(pr, *b);
  const auto t1 = std::chrono::steady_clock::now();
  pr.allow_defer = !std::getenv("LT_SERIAL_PREP");
  for (int64_t i = 0; i < P.n_scen; ++i) prepare_scenario(P, pr, *b, i);
  const auto t2 = std::chrono::steady_clock::now();
  pack_deferred(P, pr, *b);
  if (std::getenv("LT_HOST_TIMING")) {
    auto ms = [](auto x, auto y) { return std::chrono::duration<double, std::milli>(y - x).count(); };
    std::fprintf(stderr, "[lt] host prep: setup %.2f ms, keys %.2f ms, serial pass %.2f ms, parallel packing %.2f ms\n", ms(t0, t05), ms(t05, t1),
                 ms(t1, t2), ms(t2, std::chrono::steady_clock::now()));
  }
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

int32_t lt_host_libm_variant(void) {
  static int cached = -1;
  if (cached >= 0) return cached;
  std::mt19937_64 g(12345);
  for (int i = 0; i < 1000000; ++i) {
    const double x = -static_cast<double>(g() >> 11) * 0x1.0p-53;
    const double a = glibc_log1p<true>(x), b = glibc_log1p<false>(x);
    if (as_u64(a) != as_u64(b)) {
      volatile double xv = x;
      const double w = std::log1p(xv);
      cached = as_u64(w) == as_u64(a) ? 1 : 0;
      return cached;
    }
  }
  cached = 1;
  return cached;
}

void lt_format_status(int32_t code, int32_t kind, int64_t a, int64_t b, char* buf, size_t len) {
  if (!buf || !len) return;
  switch (kind) {
    case LT_K_INFEASIBLE_SLOTS:
      std::snprintf(buf, len, "infeasible configuration: %lld slots consume the entire KV budget (mem_max = 0)",
                    static_cast<long long>(a));
      return;
    case LT_K_NO_LOAD_ENTRY:
      std::snprintf(buf, len, "estimators.load.cpu_load_seconds: no entry for rank %lld", static_cast<long long>(a));
      return;
    case LT_K_SOLE_SURVIVOR:
      std::snprintf(buf, len, "single request exceeds KV capacity: request %lld", static_cast<long long>(a));
      return;
    case LT_K_NO_SLOT_COST:
      std::snprintf(buf, len,
                    "estimators.memory: no slot cost for rank %lld (add a slot_cost_tokens entry or "
                    "slot_cost_base_rank8)",
                    static_cast<long long>(a));
      return;
    case LT_K_ADMISSION_STUCK:
      std::snprintf(buf, len, "empty batch with a non-empty waiting queue: admission stuck");
      return;
    case LT_K_TOO_MANY_ADAPTERS:
      std::snprintf(buf, len, "device path supports at most %lld adapters per scenario, got %lld",
                    static_cast<long long>(b), static_cast<long long>(a));
      return;
    case LT_K_ITERATION_RANGE:
      std::snprintf(buf, len, "device path iteration index limit reached at %lld", static_cast<long long>(a));
      return;
    case LT_K_TABLE_EXHAUSTED:
      std::snprintf(buf, len, "internal: RNG table exhausted");
      return;
    case LT_K_SLOT_OVERFLOW:
      std::snprintf(buf, len, "SlotCache: running batch needs %lld adapters but only %lld slots exist (admission bug)",
                    static_cast<long long>(a), static_cast<long long>(b));
      return;
    case LT_K_NOT_RUNNING:
      std::snprintf(buf, len, "request %lld in the batch but not Running", static_cast<long long>(a));
      return;
    case LT_K_PAST_OUTPUT:
      std::snprintf(buf, len, "request %lld generated past its output length", static_cast<long long>(a));
      return;
    case LT_K_LEDGER_BALANCE:
      std::snprintf(buf, len, "KV ledger out of balance: holds sum to %lld, ledger says %lld",
                    static_cast<long long>(a), static_cast<long long>(b));
      return;
    case LT_K_LEDGER_OVER:
      std::snprintf(buf, len, "KV ledger over capacity");
      return;
    case LT_K_QUEUE_PHASE:
      std::snprintf(buf, len, "non-preempted request in the preempted queue");
      return;
    case LT_K_NO_EVICTABLE:
      std::snprintf(buf, len, "SlotCache: no evictable slot for adapter %lld (admission bug)",
                    static_cast<long long>(a));
      return;
    default:
      buf[0] = 0;
      if (code == LT_OK) std::snprintf(buf, len, "ok");
      return;
  }
}

lt_ctx* lt_create(int32_t device, lt_status* status) {
  ok_status(status);
  try {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count <= device || device < 0) {
      set_status(status, LT_ERR_DEVICE, LT_K_MESSAGE, -1, 0, 0, "no CUDA device available for the B200 path");
      return nullptr;
    }
    auto ctx = std::make_unique<lt_ctx>();
    ctx->device = device;
    LT_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    LT_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
      set_status(status, LT_ERR_DEVICE, LT_K_MESSAGE, -1, prop.major, prop.minor,
                 std::string("device is not sm_100 (B200): ") + prop.name);
      return nullptr;
    }
    ctx->sm_count = prop.multiProcessorCount;
    ctx->smem_optin = static_cast<int>(prop.sharedMemPerBlockOptin);
    LT_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    LT_CUDA(cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking));
    LT_CUDA(cudaStreamCreateWithFlags(&ctx->stream_up, cudaStreamNonBlocking));
    for (auto& e : ctx->ev) LT_CUDA(cudaEventCreate(&e));
    return ctx.release();
  } catch (const CudaError& e) {
    set_status(status, LT_ERR_DEVICE, LT_K_MESSAGE, -1, 0, 0, e.what);
    return nullptr;
  }
}

lt_ctx* lt_create_devices(const int32_t* devices, int32_t n_devices, lt_status* status) {
  ok_status(status);
  if (!devices || n_devices <= 0) {
    set_status(status, LT_ERR_VALIDATION, LT_K_MESSAGE, -1, n_devices, 0, "lt_create_devices: no devices given");
    return nullptr;
  }
  if (n_devices == 1) return lt_create(devices[0], status);
  auto g = std::make_unique<lt_ctx>();
  auto fail = [&](lt_ctx* grp) {
    for (lt_ctx* m : grp->members) lt_destroy(m);
    grp->members.clear();
    return nullptr;
  };
  for (int32_t i = 0; i < n_devices; ++i) {
    lt_ctx* m = lt_create(devices[i], status);
    if (!m) return fail(g.get());
    g->members.push_back(m);
  }
  lt_ctx* m0 = g->members[0];
  g->device = m0->device;
  g->stream = m0->stream;
  g->sm_count = m0->sm_count;
  g->smem_optin = m0->smem_optin;
  // NCCL needs distinct devices (one communicator rank per GPU); repeated
  // entries (one GPU split into several members) gather with peer copies.
  std::set<int32_t> distinct(devices, devices + n_devices);
  const char* env = std::getenv("LT_GATHER");
  const bool want_peer = env && std::string(env) == "peer";
  g->transport = LT_GATHER_PEER;
  if (!want_peer && static_cast<int32_t>(distinct.size()) == n_devices && NcclApi::get().ok) {
    std::vector<ncclComm_t> comms(n_devices);
    const ncclResult_t r = NcclApi::get().CommInitAll(comms.data(), n_devices, devices);
    if (r == ncclSuccess) {
      g->comms.assign(comms.begin(), comms.end());
      g->transport = LT_GATHER_NCCL;
    }
  }
  if (g->transport == LT_GATHER_PEER) {
    for (size_t i = 1; i < g->members.size(); ++i) {
      int can = 0;
      const int d = g->members[i]->device;
      if (d != m0->device && cudaDeviceCanAccessPeer(&can, m0->device, d) == cudaSuccess && can) {
        cudaSetDevice(m0->device);
        cudaDeviceEnablePeerAccess(d, 0);  // already enabled is fine
        cudaGetLastError();
      }
    }
  }
  return g.release();
}

lt_ctx* lt_create_mask(uint64_t device_mask, lt_status* status) {
  std::vector<int32_t> devs;
  for (int d = 0; d < 64; ++d)
    if (device_mask >> d & 1) devs.push_back(d);
  if (devs.empty()) {
    ok_status(status);
    set_status(status, LT_ERR_VALIDATION, LT_K_MESSAGE, -1, 0, 0, "lt_create_mask: empty device mask");
    return nullptr;
  }
  return lt_create_devices(devs.data(), static_cast<int32_t>(devs.size()), status);
}

int32_t lt_device_count(lt_ctx* ctx) {
  if (!ctx) return 0;
  return ctx->members.empty() ? 1 : static_cast<int32_t>(ctx->members.size());
}

int32_t lt_gather_transport(lt_ctx* ctx) { return ctx ? ctx->transport : LT_GATHER_NONE; }

void lt_destroy(lt_ctx* ctx) {
  if (!ctx) return;
  if (!ctx->members.empty()) {  // a group: its streams belong to the members
    for (void* c : ctx->comms)
      if (c) NcclApi::get().CommDestroy(static_cast<ncclComm_t>(c));
    for (lt_ctx* m : ctx->members) lt_destroy(m);
    delete ctx;
    return;
  }
  cudaSetDevice(ctx->device);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->stream2) cudaStreamDestroy(ctx->stream2);
  if (ctx->stream_up) cudaStreamDestroy(ctx->stream_up);
  delete ctx;
}

void* lt_stream(lt_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int32_t lt_last_message(lt_ctx* ctx, int64_t index, char* buf, size_t len) {
  if (!ctx || !buf || !len) return LT_ERR_VALIDATION;
  if (index < 0 || static_cast<size_t>(index) >= ctx->messages.size()) {
    buf[0] = 0;
    return LT_ERR_VALIDATION;
  }
  std::snprintf(buf, len, "%s", ctx->messages[static_cast<size_t>(index)].c_str());
  return LT_OK;
}

int32_t lt_last_timing(lt_ctx* ctx, lt_timing* out) {
  if (!ctx || !out) return LT_ERR_VALIDATION;
  *out = ctx->timing;
  return LT_OK;
}

lt_plan* lt_plan_simulate(lt_ctx* ctx, const lt_workload_batch* batch, const lt_server_config* config,
                          const lt_sim_options* options, lt_status* status) {
  ok_status(status);
  if (!ctx->members.empty()) ctx = ctx->members[0];  // a plan lives on one device
  try {
    cudaSetDevice(ctx->device);
    return build_plan(ctx, batch, config, options);
  } catch (const CudaError& e) {
    set_status(status, LT_ERR_DEVICE, LT_K_MESSAGE, -1, 0, 0, e.what);
    return nullptr;
  }
}

int32_t lt_plan_run(lt_plan* plan, lt_status* status) {
  ok_status(status);
  try {
    cudaSetDevice(plan->ctx->device);
    run_plan(*plan);
    return LT_OK;
  } catch (const CudaError& e) {
    set_status(status, LT_ERR_DEVICE, LT_K_MESSAGE, -1, 0, 0, e.what);
    return LT_ERR_DEVICE;
  }
}

int32_t lt_plan_results(lt_plan* plan, lt_sim_summary* out, lt_request_states* states, lt_status* status) {
  ok_status(status);
  try {
    cudaSetDevice(plan->ctx->device);
    fetch_results(*plan, out, states);
    return first_error(plan->ctx, out, plan->n_scen, status);
  } catch (const CudaError& e) {
    set_status(status, LT_ERR_DEVICE, LT_K_MESSAGE, -1, 0, 0, e.what);
    return LT_ERR_DEVICE;
  }
}

int32_t lt_plan_trim(lt_plan* plan) {
  if (!plan) return LT_ERR_VALIDATION;
  cudaSetDevice(plan->ctx->device);
  trim_plan(*plan);
  return LT_OK;
}

int32_t lt_plan_summaries_device(lt_plan* plan, void** ptr, int64_t* bytes) {
  if (!plan || !ptr || !bytes) return LT_ERR_VALIDATION;
  *ptr = plan->out.p;
  *bytes = plan->n_scen * static_cast<int64_t>(sizeof(lt_sim_summary));
  return LT_OK;
}

void lt_plan_destroy(lt_plan* plan) {
  if (!plan) return;
  cudaSetDevice(plan->ctx->device);
  delete plan;
}

// One plan over the whole batch (the caller bounds its size).
static int32_t simulate_one(lt_ctx* ctx, const lt_workload_batch* batch, const lt_server_config* config,
                            const lt_sim_options* options, lt_sim_summary* out, lt_request_states* states,
                            lt_status* status, double* plan_ms) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  lt_plan* plan = lt_plan_simulate(ctx, batch, config, options, status);
  if (!plan) return status ? status->code : LT_ERR_DEVICE;
  *plan_ms += std::chrono::duration<double, std::milli>(clk::now() - t0).count();
  int32_t rc = lt_plan_run(plan, status);
  if (rc == LT_OK) rc = lt_plan_results(plan, out, states, status);
  lt_plan_destroy(plan);
  return rc;
}

int32_t lt_simulate_batch(lt_ctx* ctx, const lt_workload_batch* batch, const lt_server_config* config,
                          const lt_sim_options* options, lt_sim_summary* out, lt_request_states* states,
                          lt_status* status) {
  ok_status(status);
  if (!ctx->members.empty()) return group_simulate(ctx, batch, config, options, out, states, status);
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  // Device memory is bounded by splitting the batch into consecutive chunks of
  // at most kChunkScenarios scenarios and kChunkRequests estimated requests
  // (~100 B of device state each). Chunks are pipelined on two streams: the
  // host validates and packs chunk c+1 (and launches its tables) while the
  // device runs chunk c, then collects chunk c.
  double kChunkRequests = 2.5e8;
  int64_t kChunkScenarios = 65536;
  if (const char* env = std::getenv("LT_CHUNK_REQUESTS")) kChunkRequests = std::max(1.0, std::atof(env));
  if (const char* env = std::getenv("LT_CHUNK_SCENARIOS")) kChunkScenarios = std::max(1, std::atoi(env));
  const int64_t n = batch->n_scenarios;
  std::vector<int64_t> cuts{0};
  double acc = 0.0;
  int64_t cnt = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double e = est_requests(batch, i);
    if (cnt > 0 && (acc + e > kChunkRequests || cnt >= kChunkScenarios)) {
      cuts.push_back(i);
      acc = 0.0;
      cnt = 0;
    }
    acc += e;
    ++cnt;
  }
  cuts.push_back(n);
  double plan_ms = 0.0;
  int32_t rc = LT_OK;
  if (cuts.size() <= 2) {
    rc = simulate_one(ctx, batch, config, options, out, states, status, &plan_ms);
  } else {
    try {
      cudaSetDevice(ctx->device);
      std::vector<std::string> msgs(n);
      lt_timing tsum{};
      int64_t req_off = 0;
      lt_status first{};
      first.code = LT_OK;
      // collects chunk [c0, c0 + nc) of plan P into the caller's arrays
      auto finish = [&](lt_plan& P, int64_t c0, int64_t nc) {
        lt_request_states sst;
        lt_request_states* sp = nullptr;
        if (states) {
          sst = *states;
          sst.capacity = std::max<int64_t>(states->capacity - req_off, 0);
          sst.req_offset = states->req_offset ? states->req_offset + c0 : nullptr;
          auto shift = [&](auto*& q) {
            if (q) q += req_off;
          };
          shift(sst.phase);
          shift(sst.tokens_generated);
          shift(sst.first_token_time_s);
          shift(sst.completion_time_s);
          shift(sst.preemption_count);
          shift(sst.adapter_id);
          shift(sst.input_tokens);
          shift(sst.output_tokens);
          shift(sst.arrival_time_s);
          sp = &sst;
        }
        fetch_results(P, out + c0, sp);
        lt_status st{};
        const int32_t r = first_error(ctx, out + c0, nc, &st);
        const int64_t base = req_off;
        for (int64_t i = 0; i < nc; ++i) {
          msgs[c0 + i] = ctx->messages[i];
          if (states && states->req_offset) states->req_offset[c0 + i] += base;
          req_off += out[c0 + i].n_requests;
        }
        if (r != LT_OK && first.code == LT_OK) {
          first = st;
          first.index += c0;
          rc = r;
        }
        const lt_timing& t = ctx->timing;
        tsum.tables_ms += t.tables_ms;
        tsum.merge_ms += t.merge_ms;
        tsum.engine_ms += t.engine_ms;
        tsum.d2h_ms += t.d2h_ms;
        tsum.run_ms += t.run_ms;
        tsum.h2d_bytes += t.h2d_bytes;
        tsum.d2h_bytes += t.d2h_bytes;
        tsum.engine_launches += t.engine_launches;
        tsum.algorithmic_bytes += t.algorithmic_bytes;
      };
      std::unique_ptr<lt_plan> prev;
      int64_t prev_c0 = 0, prev_nc = 0;
      for (size_t c = 0; c + 1 < cuts.size(); ++c) {
        const int64_t c0 = cuts[c], nc = cuts[c + 1] - c0;
        lt_workload_batch sub = *batch;
        sub.scenarios = batch->scenarios + c0;
        sub.n_scenarios = nc;
        const auto tb = clk::now();
        std::unique_ptr<lt_plan> plan(
            build_plan(ctx, &sub, config, options, 8, 1024, (c & 1) ? ctx->stream2 : ctx->stream));
        plan_ms += std::chrono::duration<double, std::milli>(clk::now() - tb).count();
        run_plan(*plan);
        if (prev) finish(*prev, prev_c0, prev_nc);
        prev = std::move(plan);
        prev_c0 = c0;
        prev_nc = nc;
      }
      finish(*prev, prev_c0, prev_nc);
      prev.reset();
      ctx->messages = std::move(msgs);
      ctx->timing = tsum;
      if (status && rc != LT_OK) *status = first;
    } catch (const CudaError& e) {
      set_status(status, LT_ERR_DEVICE, LT_K_MESSAGE, -1, 0, 0, e.what);
      return LT_ERR_DEVICE;
    }
  }
  ctx->timing.total_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
  ctx->timing.plan_ms = plan_ms;
  ctx->timing.run_wait_ms = ctx->timing.total_ms - plan_ms;
  return rc;
}

int32_t lt_simulate_report(lt_ctx* ctx, const lt_workload_batch* batch, const lt_server_config* config,
                           const lt_sim_options* options, lt_sim_summary* out, lt_request_states* states,
                           lt_report* report, lt_status* status) {
  ok_status(status);
  if (!states || !report) {
    set_status(status, LT_ERR_VALIDATION, LT_K_MESSAGE, -1, 0, 0, "lt_simulate_report: states and report are required");
    return LT_ERR_VALIDATION;
  }
  if (!ctx->members.empty()) {  // one plan: the first device
    const int32_t rc = lt_simulate_report(ctx->members[0], batch, config, options, out, states, report, status);
    ctx->messages = ctx->members[0]->messages;
    ctx->timing = ctx->members[0]->timing;
    return rc;
  }
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  try {
    cudaSetDevice(ctx->device);
    std::unique_ptr<lt_plan> plan(build_plan(ctx, batch, config, options));
    lt_plan& P = *plan;
    const double plan_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
    const int want_pct = P.want_pct;
    P.want_pct = 0;  // the report pass rewrites the summaries: percentiles last
    run_plan(P);
    ReportRun R;
    if (P.n_scen > 0) {
      run_report(P, R);
      if (want_pct) run_percentiles(P, engine_params(P));
      // the exact ITL mean from the emit times, after every pass that rewrites the summaries
      itl_exact_kernel<<<static_cast<unsigned>((P.n_scen + 127) / 128), 128, 0, P.st>>>(
          P.scen.p, static_cast<int>(P.n_scen), P.out.p, R.tokens.p, R.emit_off.p, R.emit.p);
      after_launch("itl_exact_kernel", P.st);
    }
    fetch_results(P, out, states);
    cudaStream_t st = P.st;
    const int64_t n = P.n_scen;
    // trace rows (dense: iterations per scenario)
    for (int64_t i = 0; i < n; ++i) {
      if (report->trace_offset) report->trace_offset[i] = R.tr_off[i];
    }
    const int64_t nt = std::min<int64_t>(R.n_tr, std::max<int64_t>(report->trace_capacity, 0));
    if (nt > 0 && report->trace)
      LT_CUDA(cudaMemcpyAsync(report->trace, R.trace.p, nt * sizeof(lt_trace_row), cudaMemcpyDeviceToHost, st));
    // emit times, one offset per request row (device request order = row order)
    const int64_t nr = std::min<int64_t>(P.total_req, std::max<int64_t>(states->capacity, 0));
    if (nr > 0 && report->emit_offset)
      LT_CUDA(cudaMemcpyAsync(report->emit_offset, R.emit_off.p, nr * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    const int64_t ne = std::min<int64_t>(R.n_emit, std::max<int64_t>(report->emit_capacity, 0));
    if (ne > 0 && report->emit_times)
      LT_CUDA(cudaMemcpyAsync(report->emit_times, R.emit.p, ne * sizeof(double), cudaMemcpyDeviceToHost, st));
    std::vector<DLoadEvent> ld(R.n_ld);
    if (R.n_ld > 0) LT_CUDA(cudaMemcpyAsync(ld.data(), R.ld.p, R.n_ld * sizeof(DLoadEvent), cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaStreamSynchronize(st));
    // load events, dense in scenario order (the device rows of a failed
    // scenario carry slack for its failing call)
    int64_t lo = 0;
    for (int64_t i = 0; i < n; ++i) {
      if (report->load_offset) report->load_offset[i] = lo;
      for (int64_t k = 0; k < R.ld_len[i]; ++k, ++lo) {
        if (lo >= report->load_capacity || !report->loads) continue;
        const DLoadEvent& e = ld[R.ld_off[i] + k];
        lt_load_event& o = report->loads[lo];
        o.time_s = e.time;
        o.adapter_id = e.adapter_id;
        o.rank = e.rank;
        o.source = P.cfg.raw.load_source;
        o._pad = 0;
        o.latency_s = e.latency;
      }
    }
    ctx->timing.d2h_bytes += nt * static_cast<int64_t>(sizeof(lt_trace_row)) + ne * 8 + nr * 8 +
                             R.n_ld * static_cast<int64_t>(sizeof(DLoadEvent));
    ctx->timing.total_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
    ctx->timing.plan_ms = plan_ms;
    return first_error(ctx, out, n, status);
  } catch (const CudaError& e) {
    set_status(status, LT_ERR_DEVICE, LT_K_MESSAGE, -1, 0, 0, e.what);
    return LT_ERR_DEVICE;
  }
}

int32_t lt_generate_arrivals_batch(lt_ctx* ctx, const lt_workload_batch* batch, const lt_sim_options* options,
                                   lt_request* out, int64_t capacity, int64_t* offsets, int64_t* counts,
                                   lt_status* status) {
  ok_status(status);
  if (!ctx->members.empty()) {  // a data-format call: the first device does it
    const int32_t rc = lt_generate_arrivals_batch(ctx->members[0], batch, options, out, capacity, offsets, counts, status);
    ctx->messages = ctx->members[0]->messages;
    ctx->timing = ctx->members[0]->timing;
    return rc;
  }
  lt_server_config cfg{};
  // generate_arrivals needs no server config; a permissive one keeps the
  // engine-level checks out of the way.
  cfg.slots = 1;
  cfg.iteration_cap = 1;
  cfg.k5 = 1.0;
  cfg.k7 = 1.0;
  cfg.total_kv_budget = INT64_MAX / 4;
  cfg.has_slot_cost_base_rank8 = 1;
  cfg.slot_cost_base_rank8 = 1.0;
  cfg.disk_multiplier = 1.0;
  std::unique_ptr<lt_plan> plan;
  try {
    cudaSetDevice(ctx->device);
    plan.reset(build_plan(ctx, batch, &cfg, options));
    prepare_requests(*plan);
    cudaStream_t st = ctx->stream;
    const int64_t n = plan->total_req;
    std::vector<double> arr(n);
    std::vector<int32_t> in(n), outv(n), adp(n);
    if (n) {
      LT_CUDA(cudaMemcpyAsync(arr.data(), plan->r_arr.p, n * 8, cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(in.data(), plan->r_in.p, n * 4, cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(outv.data(), plan->r_out.p, n * 4, cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(adp.data(), plan->r_adp.p, n * 4, cudaMemcpyDeviceToHost, st));
    }
    LT_CUDA(cudaStreamSynchronize(st));
    int64_t off = 0;
    int32_t rc = LT_OK;
    for (int64_t i = 0; i < plan->n_scen; ++i) {
      const DScen& d = plan->h_scen[i];
      const HostErr& e = plan->errs[i];
      offsets[i] = off;
      counts[i] = d.n_req;
      if (e.code != LT_OK && rc == LT_OK) {
        rc = e.code;
        set_status(status, e.code, e.kind, i, e.a, e.b, e.msg);
      }
      for (int64_t r = 0; r < d.n_req; ++r, ++off) {
        if (off >= capacity) continue;
        const int64_t g = d.req_begin + r;
        lt_request& q = out[off];
        q.request_id = r;
        q.adapter_id = plan->adapter_ids[d.adapter_begin + adp[g]];
        q.input_tokens = in[g];
        q.output_tokens = outv[g];
        q._pad = 0;
        q.arrival_time_s = arr[g];
      }
    }
    return rc;
  } catch (const CudaError& e) {
    set_status(status, LT_ERR_DEVICE, LT_K_MESSAGE, -1, 0, 0, e.what);
    return LT_ERR_DEVICE;
  }
}


int32_t lt_sweep_frontier_capacity(const lt_sweep_grid* grid) {
  if (!grid) return 0;
  int32_t cap = 0;
  for (int i = 0; i < grid->n_count; ++i) cap += std::max<int32_t>(4, grid->g_count);
  return std::max<int32_t>(cap, 1);
}

int32_t lt_sweep_batch(lt_ctx* ctx, const lt_condition_batch* batch, const lt_server_config* config,
                       const lt_sweep_grid* grid, double duration_s, uint64_t seed,
                       const lt_sweep_options* options, const lt_sim_options* sim_options,
                       lt_placement* out, lt_frontier_point* frontier, int32_t max_frontier,
                       lt_status* status) {
  ok_status(status);
  if (!ctx->members.empty())
    return group_sweep(ctx, batch, config, grid, duration_s, seed, options, sim_options, out, frontier, max_frontier,
                       status);
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t n_cond = batch->n_conditions;
  ctx->messages.assign(n_cond, std::string());
  try {
    SweepRun R;
    sweep_run(ctx, batch, config, grid, duration_s, seed, options, sim_options, max_frontier, R);
    cudaStream_t st = ctx->stream;
    cudaEventRecord(ctx->ev[6], st);
    if (n_cond > 0) {
      LT_CUDA(cudaMemcpyAsync(out, R.d_out.p, n_cond * sizeof(lt_placement), cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(frontier, R.d_front.p, n_cond * max_frontier * sizeof(lt_frontier_point),
                              cudaMemcpyDeviceToHost, st));
    }
    cudaEventRecord(ctx->ev[7], st);
    LT_CUDA(cudaStreamSynchronize(st));
    std::vector<lt_placement*> rows(n_cond);
    for (int64_t c = 0; c < n_cond; ++c) rows[c] = out + c;
    sweep_statuses(R, rows.data(), ctx->messages.data());
    sweep_timing(ctx, R, elapsed(ctx->ev[6], ctx->ev[7]));
    ctx->timing.total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return first_condition_error(ctx, out, n_cond, status);
  } catch (const CudaError& e) {
    set_status(status, LT_ERR_DEVICE, LT_K_MESSAGE, -1, 0, 0, e.what);
    return LT_ERR_DEVICE;
  }
}

}  // extern "C"
#include "host_dataset.h"
#include "host_predict.h"
