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

#include "host_common.h"
#include "host_plan.h"
#include "host_run.h"

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
  // per-scenario request estimates on the host pool (a pass over every
  // adapter record: ~0.2 s single-threaded for a 524k-scenario C5 part)
  std::vector<double> est(n);
  {
    const int nt = HostPool::width(n, 4096);
    HostPool::get().run(nt, [&](int t) {
      for (int64_t i = n * t / nt; i < n * (t + 1) / nt; ++i) est[i] = est_requests(batch, i);
    });
  }
  // (A first chunk a quarter of the rest, so the device starts sooner, gained
  // 0.4 % on C5 and lost 6.5 % on C3: one more engine tail. Not kept.)
  std::vector<int64_t> cuts{0};
  double acc = 0.0;
  int64_t cnt = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double e = est[i];
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
        const auto tf = clk::now();
        if (prev) finish(*prev, prev_c0, prev_nc);
        if (std::getenv("LT_HOST_TIMING")) {
          auto ms = [&](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
          std::fprintf(stderr, "[lt] chunk %zu (%lld scenarios): build from %.1f ms for %.1f ms, run launched %.1f, "
                       "previous chunk collected %.1f ms later\n", c, static_cast<long long>(nc), ms(t0, tb),
                       ms(tb, tf), ms(t0, tf), ms(tf, clk::now()));
        }
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
