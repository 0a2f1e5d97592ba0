/* loratwin_gpu.h — C-ABI of the B200 Digital-Twin sweep (drop-in for the
 * reference's batched simulator / placement-search hot path).
 *
 * The reference (C++20, /root/reference/proj) has no FFI; its hot-path API is
 * the core C++ functions below. Each entry point here replaces one of them
 * for a whole batch at once, with plain-old-data inputs and caller-owned
 * outputs, so the existing C++ host (CLI, generate_dataset) can call it
 * through the shim in INTEGRATION.md:
 *
 *   lt_simulate_batch  <- run_simulation     (engine.hpp:70-71, engine.cpp:198-204)
 *                      <- run_scripted       (engine.hpp:76-78, engine.cpp:206-211)
 *                      +  compute_metrics    (metrics.hpp:49-50, metrics.cpp:70-113)
 *   lt_generate_arrivals_batch <- generate_arrivals (workload.hpp:111-113, workload.cpp:170-211)
 *   lt_sweep_batch     <- sweep_optimal      (placement.hpp:100-102, placement.cpp:185-264)
 *                         (one call = many conditions; generate_dataset's loop,
 *                          placement.cpp:492-522, becomes one batch)
 *
 * Errors: the reference throws ValidationError / ConfigError /
 * SimulationError / InternalError (errors.hpp:25-54). Every failure here is
 * reported as an lt_status whose `code` names that class and whose `message`
 * is the reference's exact what() text, so a shim can rethrow the identical
 * exception. Per-scenario failures are reported per scenario (the batch keeps
 * going, like generate_dataset); the call-level status reports the
 * lowest-index failure first (run_parallel, placement.cpp:93-95).
 *
 * Threading: one lt_ctx per host thread; calls are synchronous. The context
 * owns its device memory and stream; the caller owns every host buffer.
 * Device: NVIDIA B200 (sm_100a). There is no CPU fallback: without a usable
 * device lt_create fails with LT_ERR_DEVICE.
 */
#ifndef LORATWIN_GPU_H_
#define LORATWIN_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LT_ABI_VERSION 4

/* Exception classes of errors.hpp, plus two conditions of this library. */
enum lt_code {
  LT_OK = 0,
  LT_ERR_VALIDATION = 1, /* ValidationError (errors.hpp:25-29) */
  LT_ERR_CONFIG = 2,     /* ConfigError     (errors.hpp:31-36) */
  LT_ERR_SIMULATION = 3, /* SimulationError (errors.hpp:44-49) */
  LT_ERR_INTERNAL = 4,   /* InternalError   (errors.hpp:51-54) */
  LT_ERR_UNSUPPORTED = 5, /* input outside what the device path implements */
  LT_ERR_DEVICE = 6       /* CUDA failure / no device */
};

/* Which reference message template a per-scenario status carries. */
enum lt_status_kind {
  LT_K_NONE = 0,
  LT_K_INFEASIBLE_SLOTS = 1,   /* engine.cpp:51-53          a = slots */
  LT_K_NO_LOAD_ENTRY = 2,      /* estimators.cpp:79-81      a = rank */
  LT_K_SOLE_SURVIVOR = 3,      /* kv_scheduler.cpp:226-227  a = request_id */
  LT_K_NO_SLOT_COST = 4,       /* estimators.cpp:52-54      a = rank */
  LT_K_ADMISSION_STUCK = 5,    /* engine.cpp:100-101 */
  LT_K_TOO_MANY_ADAPTERS = 6,  /* device limit: a = adapters, b = limit */
  LT_K_ITERATION_RANGE = 7,    /* device limit: iteration index beyond int32 */
  LT_K_TABLE_EXHAUSTED = 8,    /* internal: RNG table shorter than needed */
  LT_K_MESSAGE = 9,            /* free-form, message holds the text */
  LT_K_SLOT_OVERFLOW = 10,     /* adapter_cache.cpp:45-48   a = needed, b = slots */
  LT_K_NO_EVICTABLE = 11,      /* adapter_cache.cpp:64-66   a = adapter_id */
  LT_K_VALIDATION_MSG = 12,    /* host validation; message holds the text */
  /* check_invariants (kv_scheduler.cpp:261-290): InternalError texts */
  LT_K_NOT_RUNNING = 13,       /* a = request_id: "request a in the batch but not Running" */
  LT_K_PAST_OUTPUT = 14,       /* a = request_id: "request a generated past its output length" */
  LT_K_LEDGER_BALANCE = 15,    /* a = holds, b = ledger: "KV ledger out of balance: ..." */
  LT_K_LEDGER_OVER = 16,       /* "KV ledger over capacity" */
  LT_K_QUEUE_PHASE = 17        /* "non-preempted request in the preempted queue" */
};

typedef struct lt_status {
  int32_t code;   /* enum lt_code */
  int32_t kind;   /* enum lt_status_kind */
  int64_t index;  /* failing scenario / condition index, -1 when n/a */
  int64_t detail_a;
  int64_t detail_b;
  char message[320]; /* reference what() text */
} lt_status;

/* LengthMode (workload.hpp:26): enum class LengthMode { Full, Mean }. */
enum lt_length_mode { LT_MODE_FULL = 0, LT_MODE_MEAN = 1 };
/* LoadSource (estimators.hpp:29). */
enum lt_load_source { LT_SOURCE_CPU = 0, LT_SOURCE_DISK = 1 };

/* ServerConfig (server_config.hpp:26-43) with its LatencyCoefficients,
 * MemoryModel and LoadLatencyTable (estimators.hpp:33-71) flattened. */
typedef struct lt_server_config {
  int32_t slots; /* G; a scenario's `slots` overrides it (placement.cpp:210-211) */
  int32_t loaded_adapter_priority;
  int64_t iteration_cap;
  int32_t ideal_includes_input;
  int32_t load_source; /* enum lt_load_source (default_source) */
  double k1, k2, k3, k4, k5, k6, k7;
  int64_t total_kv_budget;
  double kv_bytes_per_token; /* informational (estimators.hpp:54) */
  int32_t has_slot_cost_base_rank8;
  double slot_cost_base_rank8;
  int32_t n_slot_cost; /* slot_cost_tokens table: rank -> tokens */
  const int32_t* slot_cost_rank;
  const int64_t* slot_cost_tokens;
  int32_t n_load; /* cpu_load_seconds table: rank -> seconds */
  const int32_t* load_rank;
  const double* load_seconds;
  double disk_multiplier;
} lt_server_config;

/* LengthSpec (workload.hpp:31-65). Full-mode pairs live in a shared array. */
typedef struct lt_length_spec {
  int32_t mode; /* enum lt_length_mode */
  int32_t _pad;
  double mean_input, std_input, mean_output, std_output;
  int64_t full_offset; /* first (in, out) pair in lt_workload_batch.full_lengths */
  int64_t full_count;
} lt_length_spec;

/* AdapterSpec (workload.hpp:71-76). */
typedef struct lt_adapter {
  int32_t adapter_id;
  int32_t rank;
  double rate;
  int32_t length_index; /* -1: the scenario's workload-level spec */
  int32_t _pad;
} lt_adapter;

/* Request (workload.hpp:91-99); 32 bytes. */
typedef struct lt_request {
  int64_t request_id;
  int32_t adapter_id;
  int32_t input_tokens;
  int32_t output_tokens;
  int32_t _pad;
  double arrival_time_s;
} lt_request;

/* One simulation: a WorkloadSpec (workload.hpp:78-89) run under the batch's
 * ServerConfig with `slots` overriding G, or (n_requests >= 0) a
 * run_scripted over an explicit request list. */
typedef struct lt_scenario {
  int64_t adapter_offset;
  int32_t n_adapters;
  int32_t length_index; /* WorkloadSpec.lengths */
  double duration_s;
  uint64_t seed;
  int32_t slots; /* > 0 overrides lt_server_config.slots */
  int32_t mode;  /* run_simulation's LengthMode argument */
  int64_t request_offset;
  int64_t n_requests; /* -1: generate arrivals (run_simulation); >= 0: scripted */
} lt_scenario;

typedef struct lt_workload_batch {
  const lt_scenario* scenarios;
  int64_t n_scenarios;
  const lt_adapter* adapters;
  int64_t n_adapters;
  const lt_length_spec* lengths;
  int64_t n_lengths;
  const int32_t* full_lengths; /* 2 * n_full_pairs ints: in, out, in, out, ... */
  int64_t n_full_pairs;
  const lt_request* requests; /* scripted requests */
  int64_t n_requests;
} lt_workload_batch;

/* SimOptions (engine.hpp:29-35) plus device knobs. */
typedef struct lt_sim_options {
  int32_t check_invariants;      /* the reference's scheduler invariants, checked every simulated iteration
                                    (a checked engine build; InternalError on a violation) */
  int32_t want_digest;           /* fold each iteration's decisions into summary.digest */
  int64_t iteration_cap_override; /* <= 0: none */
  int32_t libm_variant;          /* -1: match the host glibc; 0: generic build; 1: FMA build */
  int32_t want_percentiles;      /* fill the TTFT/ITL p50/p99 of compute_metrics (a second, recording
                                    engine pass + segmented sorts); sweeps never need them */
} lt_sim_options;

/* SimulationResult (engine.hpp:47-64) scalars + MetricsSummary
 * (metrics.hpp:27-40) of compute_metrics, per scenario. */
typedef struct lt_sim_summary {
  int32_t status;      /* enum lt_code */
  int32_t status_kind; /* enum lt_status_kind */
  int64_t status_a, status_b;
  int64_t n_requests;
  int64_t iterations;
  double final_clock_s;
  double duration_s;
  int32_t truncated;
  int32_t slots;
  int32_t served_adapters;
  int32_t starved;
  int64_t kv_capacity_tokens;
  int64_t finished_count;
  int64_t rejected_count;
  int64_t preemptions;
  int64_t load_events;
  int64_t tokens_in_window;
  int64_t tokens_total;
  double throughput_tok_s;
  double ideal_throughput_tok_s;
  double ttft_mean_s;
  double itl_mean_s;
  double ttft_p50_s, ttft_p99_s; /* nearest rank (metrics.cpp:47-54); 0 unless want_percentiles */
  double itl_p50_s, itl_p99_s;
  int32_t degenerate;
  int32_t _pad;
  uint64_t digest; /* FNV-1a over per-iteration (R, W, A, loads, lat bits) */
  /* roofline counters: sums over iterations */
  int64_t sum_running;  /* R */
  int64_t sum_visited;  /* waiting entries the admission scans touched (device: events) */
  int64_t sum_arrivals; /* A */
  int64_t sum_moves;    /* admissions + finishes + preemptions */
  int64_t device_cycles; /* SM clock cycles the engine warp spent on this scenario (0 on CPU) */
  int64_t phase_cycles[6]; /* profiling builds only (-DLT_PHASE_PROF): ingest, retire, alloc,
                              preempted-queue scan, fresh scan, load+price+emit; 0 otherwise */
} lt_sim_summary;

/* Optional per-request final states (RequestState, kv_scheduler.hpp:30-41),
 * indexed by lt_sim_summary offsets: scenario s owns rows
 * [req_offset[s], req_offset[s] + n_requests). Any pointer may be NULL. */
typedef struct lt_request_states {
  int64_t capacity;  /* rows available */
  int64_t* req_offset; /* n_scenarios entries, filled by the library */
  int8_t* phase;     /* Phase: 0 Waiting 1 Running 2 Preempted 3 Finished 4 Rejected */
  int32_t* tokens_generated;
  double* first_token_time_s; /* NaN when never emitted */
  double* completion_time_s;  /* 0 unless the final token was emitted */
  int32_t* preemption_count;
  int32_t* adapter_id;
  int32_t* input_tokens;
  int32_t* output_tokens;
  double* arrival_time_s;
} lt_request_states;

/* Condition (placement.hpp:37-40), its AdapterTemplate legs (:32-35). */
typedef struct lt_template {
  int32_t rank;
  int32_t _pad;
  double rate;
} lt_template;

typedef struct lt_condition {
  int64_t mix_offset;
  int32_t mix_count;
  int32_t length_index;
} lt_condition;

typedef struct lt_condition_batch {
  const lt_condition* conditions;
  int64_t n_conditions;
  const lt_template* templates;
  int64_t n_templates;
  const lt_length_spec* lengths;
  int64_t n_lengths;
  const int32_t* full_lengths;
  int64_t n_full_pairs;
} lt_condition_batch;

/* SweepGrid (placement.hpp:77-88). */
enum lt_g_mode { LT_G_GEOMETRIC = 0, LT_G_EXPLICIT = 1 };
typedef struct lt_sweep_grid {
  const int32_t* n_values;
  int32_t n_count;
  int32_t g_mode;
  const int32_t* g_values;
  int32_t g_count;
  int32_t _pad;
} lt_sweep_grid;

/* SweepOptions (placement.hpp:90-95). `jobs` is accepted and ignored. */
typedef struct lt_sweep_options {
  int32_t early_exit;
  int32_t early_exit_k;
  int32_t jobs;
  int32_t mode;
} lt_sweep_options;

/* FrontierPoint (placement.hpp:60-66). */
typedef struct lt_frontier_point {
  int32_t n;
  int32_t g;
  double throughput_tok_s;
  int32_t starved;
  int32_t skipped;
} lt_frontier_point;

/* PlacementResult (placement.hpp:68-75) + the sweep-level status. */
typedef struct lt_placement {
  int32_t status; /* the exception sweep_optimal would throw (lowest G index of the first failing evaluated row) */
  int32_t status_kind;
  int64_t status_a, status_b;
  double max_throughput_tok_s;
  int32_t n_star;
  int32_t g_star; /* max_loras */
  int32_t all_starved;
  int32_t frontier_open;
  int32_t frontier_count; /* points written to this condition's frontier rows */
  int32_t _pad;
  int64_t points_simulated; /* grid points consumed by the reduction (as the reference simulates them) */
  int64_t iterations;       /* engine-iterations summed over those points */
  int64_t status_point;     /* internal: failing grid point, -1 when none */
} lt_placement;

typedef struct lt_ctx lt_ctx;

/* Timing of the last call, from CUDA events on the context's stream. */
typedef struct lt_timing {
  double h2d_ms, tables_ms, merge_ms, engine_ms, reduce_ms, d2h_ms, total_ms;
  double run_ms; /* whole device pipeline of the last run (K0 tables .. engine) */
  int64_t h2d_bytes, d2h_bytes;
  int64_t engine_launches; /* kernels this library launched in the call */
  int64_t algorithmic_bytes; /* B_iter summed over the engine launches */
  double plan_ms;    /* host wall time of building the plan (validation, packing, sizing passes) */
  double run_wait_ms; /* host wall time from lt_plan_run to results copied back */
  /* multi-device contexts: device phases above are the slowest member's */
  double gather_ms;     /* wall time of the cross-device gather + the one copy back (sweeps) */
  int64_t gather_bytes; /* bytes moved between devices by that gather */
  int32_t devices;      /* members that ran the call (0 for a single-device context) */
  int32_t _pad;
} lt_timing;

int32_t lt_abi_version(void);
/* 1 when the host glibc runs its FMA libm build, 0 for the generic build. */
int32_t lt_host_libm_variant(void);
/* Renders the reference message for (code, kind, a, b) into buf. */
void lt_format_status(int32_t code, int32_t kind, int64_t a, int64_t b, char* buf, size_t len);

lt_ctx* lt_create(int32_t device, lt_status* status);

/* Multi-device context (SURVEY 8b `lt_create(device_mask)`, 8e). Replaces the
 * reference's thread pool over conditions (run_parallel, placement.cpp:65-96,
 * as generate_dataset uses it at :492-522) with the GPUs of one box:
 * lt_simulate_batch / lt_sweep_batch / lt_generate_dataset on it shard the
 * scenarios / conditions by estimated cost (LPT) over one member context per
 * entry, run the members on their own host threads, and gather the sweeps'
 * per-condition placements + frontiers to the first device (NCCL send/recv
 * when the devices are distinct, peer copies otherwise) before one copy back.
 * Results, statuses and messages are those of the single-device call.
 * lt_create_devices may repeat a device (members then share that GPU);
 * plans and lt_generate_arrivals_batch run on the first member. */
lt_ctx* lt_create_devices(const int32_t* devices, int32_t n_devices, lt_status* status);
lt_ctx* lt_create_mask(uint64_t device_mask, lt_status* status); /* bit d = CUDA device d */
int32_t lt_device_count(lt_ctx* ctx);
enum lt_gather_transport { LT_GATHER_NONE = 0, LT_GATHER_NCCL = 1, LT_GATHER_PEER = 2 };
int32_t lt_gather_transport(lt_ctx* ctx);
void lt_destroy(lt_ctx* ctx);
/* The cudaStream_t (as void*) all work of this context runs on. */
void* lt_stream(lt_ctx* ctx);
int32_t lt_last_timing(lt_ctx* ctx, lt_timing* out);
/* The reference what() text of scenario / condition `index` of the last
 * batch call ("" when it succeeded). */
int32_t lt_last_message(lt_ctx* ctx, int64_t index, char* buf, size_t len);

/* generate_arrivals for every non-scripted scenario: writes the merged,
 * request_id-ordered list of scenario s at out[offsets[s] .. offsets[s] + counts[s]).
 * `capacity` rows are available; counts are always filled. */
int32_t lt_generate_arrivals_batch(lt_ctx* ctx, const lt_workload_batch* batch,
                                   const lt_sim_options* options, lt_request* out,
                                   int64_t capacity, int64_t* offsets, int64_t* counts,
                                   lt_status* status);

/* run_simulation / run_scripted + compute_metrics for every scenario. */
int32_t lt_simulate_batch(lt_ctx* ctx, const lt_workload_batch* batch,
                          const lt_server_config* config, const lt_sim_options* options,
                          lt_sim_summary* out, lt_request_states* states, lt_status* status);

/* ---- Full simulation report ----------------------------
 * What run_simulation / run_scripted return beyond the summary: the
 * IterationTraceRow trace (engine.hpp:39-47, engine.cpp:137-140), the
 * LoadEvent list (adapter_cache.hpp:28-34, engine.cpp:141) and every
 * request's token_emit_times_s (kv_scheduler.hpp:30-41, engine.cpp:132),
 * i.e. the inputs of simulation_report_json (json_io.cpp:608-687). */
typedef struct lt_trace_row {
  double time_s;   /* clock at the start of the iteration */
  int64_t iteration;
  int32_t r_running, r_waiting, a_running, loads;
  double lat_step_s;
} lt_trace_row;

typedef struct lt_load_event {
  double time_s;
  int32_t adapter_id;
  int32_t rank;
  int32_t source; /* enum lt_load_source */
  int32_t _pad;
  double latency_s;
} lt_load_event;

/* Caller-owned output rows. Scenario s's trace is trace[trace_offset[s] ..
 * + summary.iterations), its loads loads[load_offset[s] .. + load_events);
 * request row j (lt_request_states order) emitted at emit_times[emit_offset[j]
 * .. + tokens_generated). Rows past a capacity are not written (the counts
 * still are), so a first lt_simulate_batch call can size the buffers. */
typedef struct lt_report {
  lt_trace_row* trace;
  int64_t trace_capacity;
  int64_t* trace_offset; /* n_scenarios entries */
  lt_load_event* loads;
  int64_t load_capacity;
  int64_t* load_offset;  /* n_scenarios entries */
  double* emit_times;
  int64_t emit_capacity;
  int64_t* emit_offset;  /* one per request row (states->capacity entries) */
} lt_report;

/* lt_simulate_batch plus the full report: a second engine pass over the same
 * batch records the trace rows, load events and every admission / preemption
 * (the request's running stints); the emit times are expanded on the device
 * from the stints and the per-iteration emit times. One device plan (no
 * chunking): meant for report-sized batches. `states` is required. */
int32_t lt_simulate_report(lt_ctx* ctx, const lt_workload_batch* batch,
                           const lt_server_config* config, const lt_sim_options* options,
                           lt_sim_summary* out, lt_request_states* states, lt_report* report,
                           lt_status* status);

/* sweep_optimal for every condition: frontier rows of condition c are
 * frontier[c * max_frontier ...]. lt_sweep_frontier_capacity gives the
 * maximum frontier length of a grid. */
int32_t lt_sweep_frontier_capacity(const lt_sweep_grid* grid);
int32_t lt_sweep_batch(lt_ctx* ctx, const lt_condition_batch* batch,
                       const lt_server_config* config, const lt_sweep_grid* grid,
                       double duration_s, uint64_t seed, const lt_sweep_options* options,
                       const lt_sim_options* sim_options, lt_placement* out,
                       lt_frontier_point* frontier, int32_t max_frontier, lt_status* status);

/* ---- Dataset generation (placement.hpp:104-158) -------------------------- */

/* DatasetSpec (placement.hpp:126-137). lengths.full_offset / full_count index
 * full_lengths (in, out pairs). */
typedef struct lt_dataset_spec {
  const double* rates;
  int32_t n_rates;
  int32_t triple_size;
  const int32_t* ranks;
  int32_t n_ranks;
  int32_t condition_stride;
  lt_length_spec lengths;
  const int32_t* full_lengths;
  int64_t n_full_pairs;
  double duration_s;
  uint64_t seed;
  lt_sweep_grid grid;
  lt_sweep_options sweep; /* jobs is accepted and ignored: conditions run as one device batch */
} lt_dataset_spec;

/* DatasetProgress (placement.hpp:143-147). */
typedef struct lt_dataset_progress {
  int64_t total_conditions;
  int64_t completed; /* includes rows found on resume */
  int64_t failed;
} lt_dataset_progress;

/* on_error of generate_dataset: called in canonical condition order. */
typedef void (*lt_error_fn)(const char* message, void* user);

/* generate_dataset (placement.cpp:415-527): enumerates the conditions, resumes
 * from the hashes already in out_csv (truncating a torn tail), sweeps every
 * pending condition on the device in one batched lt_sweep_batch per chunk and
 * appends the rows in canonical order. Same file bytes as the reference. */
int32_t lt_generate_dataset(lt_ctx* ctx, const lt_dataset_spec* spec, const lt_server_config* config,
                            const char* out_csv, lt_error_fn on_error, void* user,
                            lt_dataset_progress* progress, lt_status* status);

/* condition_hash (placement.cpp:266-296): FNV-1a over the canonical text. */
uint64_t lt_condition_hash(const lt_template* mix, int32_t n_mix, const lt_length_spec* lengths,
                           const int32_t* full_lengths, double duration_s, uint64_t seed,
                           const lt_sweep_grid* grid);

/* encode_workload (placement.cpp:117-137): the 16 features. */
int32_t lt_encode_workload(const lt_template* mix, int32_t n_mix, const lt_length_spec* lengths,
                           const int32_t* full_lengths, double* features16, lt_status* status);

/* ---- Placement-model training on the device -------------
 * train_tree / train_forest / train_placement_model and ForestModel::predict
 * (predictor.hpp:41-118, predictor.cpp:202-269). Features are the 16
 * WorkloadFeatures values per row (row-major, n_rows x 16); trees come back
 * as the reference's node vectors (preorder, nodes[0] the root). */
typedef struct lt_tree_params { /* TreeParams */
  int32_t max_depth;
  int32_t min_leaf;
  int32_t feature_subset; /* features considered per node, 1..16 */
  int32_t _pad;
} lt_tree_params;

typedef struct lt_forest_params { /* ForestParams */
  int32_t n_trees;
  int32_t bootstrap;
  lt_tree_params tree;
} lt_forest_params;

typedef struct lt_tree_node { /* TreeNode */
  int32_t feature_index; /* -1: leaf */
  int32_t left, right;
  int32_t _pad;
  double threshold;
  double value;
  int64_t coverage;
} lt_tree_node;

/* train_tree(x, y, params, seed, tree_tag): node_count[0] nodes at nodes[0..]. */
int32_t lt_train_tree(lt_ctx* ctx, const double* x, int64_t n_rows, const double* y,
                      const lt_tree_params* params, uint64_t seed, uint64_t tree_tag,
                      lt_tree_node* nodes, int64_t node_capacity, int32_t* node_count,
                      lt_status* status);

/* train_forest for each of n_targets targets (y: n_targets rows of n_rows;
 * target_tags: PredictTarget 0 throughput, 1 n_star, 2 g_star) over the same
 * features -- train_placement_model is the three targets at once. Tree t of
 * target g is tree g * n_trees + t, its nodes at nodes[node_offset[..]] with
 * node_count[..] entries. All trees grow on the device in one call. */
int32_t lt_train_forests(lt_ctx* ctx, const double* x, int64_t n_rows, const double* y,
                         const int32_t* target_tags, int32_t n_targets, const lt_forest_params* params,
                         uint64_t seed, lt_tree_node* nodes, int64_t node_capacity,
                         int64_t* node_offset, int32_t* node_count, lt_status* status);

/* ForestModel::predict of n_targets forests of n_trees trees each (the
 * lt_train_forests layout) for n_rows feature rows: out[g * n_rows + i]; a
 * negative target tag gives predict_raw (the plain mean of the trees). */
int32_t lt_predict_forests(lt_ctx* ctx, const lt_tree_node* nodes, int64_t n_nodes,
                           const int64_t* node_offset, int32_t n_trees, const int32_t* target_tags,
                           int32_t n_targets, const double* x, int64_t n_rows, double* out,
                           lt_status* status);

/* Resident-input form for timing the device path alone: upload once, run
 * many times with inputs already in HBM, read results back once. */
typedef struct lt_plan lt_plan;
lt_plan* lt_plan_simulate(lt_ctx* ctx, const lt_workload_batch* batch,
                          const lt_server_config* config, const lt_sim_options* options,
                          lt_status* status);
int32_t lt_plan_run(lt_plan* plan, lt_status* status); /* asynchronous on lt_stream */
int32_t lt_plan_results(lt_plan* plan, lt_sim_summary* out, lt_request_states* states,
                        lt_status* status);
void lt_plan_destroy(lt_plan* plan);
/* Device address of the plan's lt_sim_summary array (for device-side
 * collectives, e.g. an NCCL all-gather of per-scenario records). */
int32_t lt_plan_summaries_device(lt_plan* plan, void** ptr, int64_t* bytes);
/* Returns the plan's regenerated buffers (RNG tables, per-request arrays,
 * merge scratch, engine workspace) to the context's block cache; the
 * summaries stay. The next lt_plan_run re-acquires and regenerates them, so
 * a chain of trimmed plans run on one context needs the device memory of the
 * largest, not of all (stream order makes the reuse safe). Per-request states
 * are unavailable from lt_plan_results until the next run. Plans holding
 * scripted requests are not trimmed. */
int32_t lt_plan_trim(lt_plan* plan);

#ifdef __cplusplus
}
#endif

#endif /* LORATWIN_GPU_H_ */
