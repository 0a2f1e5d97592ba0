// The library's context and plan types and everything that builds and runs
// a plan (capi.cu includes this after host_common.h): validation and packing
// of a batch into the device layout on host threads, K0 / merge / engine
// launches, percentiles, the report pass, result collection.
#pragma once


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
  double rec_per_req = 0.0;  // ITL records per request seen by single-pass percentile runs (pool sizing)
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
  DBuf<int32_t> r_link;  // chain links per request (link_kernel)
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
  // single-pass recording pool (run_percentiles_single)
  DBuf<double> pool_d;
  DBuf<int32_t> pool_c, chunk_next, pool_next;
  DBuf<int64_t> rec_total;
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
  bool run_fresh = false;  // the last run used the tables built with the plan
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
    if (d1 > d0) {  // this thread's contiguous share of the uploaded arrays
      const int64_t a0 = pr.deferred[d0].a_off, p0 = pr.deferred[d0].p_off;
      const int64_t na = pr.deferred[d1 - 1].a_off + b.scenarios[pr.deferred[d1 - 1].i].n_adapters - a0;
      const int64_t np = pr.deferred[d1 - 1].p_off + b.scenarios[pr.deferred[d1 - 1].i].n_adapters - p0;
      write_back(pr.adapters.data() + a0, na * sizeof(pr.adapters[0]));
      write_back(pr.pair_scen.data() + p0, np * sizeof(int32_t));
      write_back(pr.pair_adp.data() + p0, np * sizeof(int32_t));
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
    const int64_t i0 = n * t / nt, i1 = n * (t + 1) / nt;
    for (int64_t i = i0; i < i1; ++i) {
      keys[i].e_off = off;
      keys[i].z_off = off;
      off += keys[i].cap;
    }
    write_back(keys.data() + i0, (i1 - i0) * sizeof(DKeyNI));  // uploaded next
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
  if (P.max_req > kMaxScenarioRequests) throw CudaError{"scenario too large: more than 2^30 - 1 requests"};
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
void size_engine(lt_plan& P, const std::vector<double>& cost, int max_run_cap, bool narrow_blocks = true) {
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
    // Latency-bound batches whose work per warp slot stays under half the
    // longest engine with half the warps per block take the smaller blocks:
    // each warp gets a larger running-set tier in shared memory (1,024 slots
    // at 4 warps vs 704 at 8 for 256-adapter batches) and the heaviest
    // engines (warp 0 of each block, one per SM) share their SM with fewer
    // others. C2 (1,024 scenarios: 0.21 of the longest engine per slot at 8
    // warps) takes 4: engine 27.2 -> 26.9 ms (same-box A/B). Not for the
    // sweep waves (narrow_blocks false), which are measured without it.
    if (narrow_blocks && P.engine_variant == 1 && P.warps_per_block == 8 && P.n_scen > 0 &&
        !std::getenv("LT_WIDE_BLOCKS")) {
      double total = 0.0, longest = 0.0;
      for (int64_t i = 0; i < P.n_scen; ++i) {
        total += cost[i];
        longest = std::max(longest, cost[i]);
      }
      while (P.warps_per_block > 2 &&
             total / (static_cast<double>(ctx->sm_count) * (P.warps_per_block / 2)) <= 0.5 * longest)
        P.warps_per_block /= 2;
      if (std::getenv("LT_HOST_TIMING"))
        std::fprintf(stderr, "[lt] size_engine: %lld scenarios, work per slot / longest at 8 warps %.3f -> %d warps per block\n",
                     static_cast<long long>(P.n_scen), total / (static_cast<double>(ctx->sm_count) * 8.0) / longest,
                     P.warps_per_block);
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
  cudaEvent_t dbg_k0 = nullptr;
  if (std::getenv("LT_HOST_TIMING")) cudaEventCreate(&dbg_k0);
  // tables_ms: ev[0] just before the first K0 launch, ev[1] after the last
  // (in a chunk pipeline it includes waiting for the previous chunk's SMs)
  cudaEventRecord(P.ev[0], st);
  cudaEventRecord(P.ev[1], st);
  if (!pr.keys.empty())
    P.seed_state.alloc(std::min<int64_t>(static_cast<int64_t>(pr.keys.size()), kSeedChunk) * 2 * kMtN);
  P.tab_overflow.alloc(1);
  LT_CUDA(cudaMemsetAsync(P.tab_overflow.p, 0, sizeof(int32_t), st));
  const size_t early_keys = pr.keys.size();
  auto h_up = h_size;
  cudaEvent_t dbg_a = nullptr, dbg_b = nullptr;
  if (dbg_k0) {
    cudaEventCreate(&dbg_a);
    cudaEventCreate(&dbg_b);
    cudaEventRecord(dbg_a, st);
  }
  if (early_keys > 0) {
    P.keys.upload(pr.keys.data(), pr.keys.size(), st);
    if (dbg_b) cudaEventRecord(dbg_b, st);
    P.E.alloc(std::max<int64_t>(e_total, 1));
    P.Z.alloc(std::max<int64_t>(e_total, 1));
    P.h2d_bytes += pr.keys.size() * sizeof(DKey);
    h_up = hclk::now();
    if (dbg_k0) cudaEventRecord(dbg_k0, st);
    cudaEventRecord(P.ev[0], st);
    P.launches_prep += launch_tables(P, static_cast<int>(early_keys), st);
    cudaEventRecord(P.ev[1], st);
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
  // The arrival counts are queued right behind K0 and read back with its
  // overflow flag in one synchronisation; the engine is sized on the host
  // meanwhile. An overflowing table (never expected: the tables hold the
  // Poisson bound + 8 sigma) relaunches K0 with larger tables and recounts.
  const int64_t n_pairs = static_cast<int64_t>(pr.pair_scen.size());
  P.n_pairs = n_pairs;
  P.n_keys = static_cast<int>(pr.keys.size());
  P.scen_count.alloc(std::max<int64_t>(P.n_scen, 1));
  P.scen_off.alloc(std::max<int64_t>(P.n_scen, 1));
  P.overflow.alloc(1);
  if (n_pairs > 0) {
    P.adp_count.alloc(n_pairs);
    P.pair_g = pair_group(mean_pair_draws(b));
  }
  LT_CUDA(cudaStreamWaitEvent(st, P.ev_up, 0));  // the packed-scenario uploads
  std::vector<unsigned long long> counts(std::max<int64_t>(P.n_scen, 1));
  int32_t ovf = 0;
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
      cudaEventRecord(P.ev[1], st);
    }
    relaunch = true;
    if (n_pairs > 0) {  // count arrivals per (scenario, adapter): sizes the request arrays
      LT_CUDA(cudaMemsetAsync(P.scen_count.p, 0, P.n_scen * sizeof(unsigned long long), st));
      LT_CUDA(cudaMemsetAsync(P.overflow.p, 0, sizeof(int32_t), st));
      launch_count(P, st);
      ++P.launches_prep;
    }
    // the engine's order, variant and grid need only the cost estimates:
    // sized while K0 and the counts run (the pageable read-backs below block)
    if (attempt == 0) size_engine(P, pr.cost, max_run_cap);
    int32_t any = 0;
    LT_CUDA(cudaMemcpyAsync(&any, P.tab_overflow.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    if (n_pairs > 0) {
      LT_CUDA(cudaMemcpyAsync(counts.data(), P.scen_count.p, P.n_scen * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaMemcpyAsync(&ovf, P.overflow.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    }
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
  const auto h_tables = hclk::now();
  if (dbg_k0) {
    std::fprintf(stderr, "[lt]   device: keys upload %.3f ms (%zu B), K0 %.3f ms\n", elapsed(dbg_a, dbg_b),
                 pr.keys.size() * sizeof(DKey), elapsed(dbg_k0, P.ev[1]));
    cudaEventDestroy(dbg_a);
    cudaEventDestroy(dbg_b);
    cudaEventDestroy(dbg_k0);
  }
  if (n_pairs > 0) {
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

}  // namespace
