// Host-side utilities of the C-ABI library (one translation unit: capi.cu
// includes this first): CUDA error handling, reference-text statuses,
// configuration validation and lookups, length statistics, the device block
// cache and buffers, the persistent host worker pool.
#pragma once

namespace {

// Writes back a host range that a worker thread just wrote (CLWB per 64-byte
// line, then a store fence) so the DMA of the following upload reads memory,
// not dirty lines in other cores' private caches: measured on the GPU box's
// VM, 8.6 MB of keys written by 16 threads uploaded at ~7 GB/s without it
// (0.8-1.4 ms) against ~50 GB/s from memory. The caches keep the lines.
inline void write_back(const void* p, size_t bytes) {
#if defined(__x86_64__)
  if (bytes == 0) return;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(63);
  const uintptr_t a1 = reinterpret_cast<uintptr_t>(p) + bytes;
  if (std::getenv("LT_NO_WRITE_BACK")) return;
  for (uintptr_t a = a0; a < a1; a += 64) asm volatile("clwb (%0)" ::"r"(a) : "memory");
  asm volatile("sfence" ::: "memory");
#else
  (void)p;
  (void)bytes;
#endif
}

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
