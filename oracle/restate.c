/* ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/README.md).
 *
 * A plain-C restatement of the reference's hot path (arXiv 2508.08343
 * `loratwin`, proj/core/src), exported with the loratwin_gpu.h C-ABI under
 * the `ltor_` prefix. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / reference legs may load it, as the checker or the timed CPU
 * baseline. It follows the reference line by line (citations below), keeps
 * its data structures (linear scans, explicit per-token emit records) and
 * calls the HOST libm exactly where the reference does, so on the same host
 * it reproduces the reference bit for bit -- including the ITL mean, which
 * the device path only matches to 1e-9. Parity of this file against the
 * compiled reference (oracle/_ref/libloratwin_ref.so) and the golden vectors
 * in tests/golden is pinned by tests/test_oracle.py.
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "loratwin_gpu.h"

/* ------------------------------------------------------------------ RNG */
/* rng.hpp:33-73: std::seed_seq -> std::mt19937_64 per (seed, stream ids). */
typedef struct {
  uint64_t x[312];
  int i;
  int has_spare;
  double spare;
} Rng;

static uint32_t ss_T(uint32_t v) { return v ^ (v >> 27); }

/* [rand.util.seedseq] generate(624 words) + [rand.eng.mers] seed(seq) */
static void rng_init(Rng* r, uint64_t seed, uint64_t a, uint64_t b) {
  uint32_t v[6] = {(uint32_t)seed, (uint32_t)(seed >> 32), (uint32_t)a, (uint32_t)(a >> 32),
                   (uint32_t)b, (uint32_t)(b >> 32)};
  const int s = 6, n = 624, t = 11, p = (n - t) / 2, q = p + t, m = n;
  uint32_t bw[624];
  for (int k = 0; k < n; ++k) bw[k] = 0x8b8b8b8bu;
  for (int k = 0; k < m; ++k) {
    const int kn = k % n, kp = (k + p) % n, kq = (k + q) % n, km = (k + n - 1) % n;
    const uint32_t r1 = 1664525u * ss_T(bw[kn] ^ bw[kp] ^ bw[km]);
    uint32_t r2 = r1 + (k == 0 ? (uint32_t)s : (k <= s ? (uint32_t)kn + v[k - 1] : (uint32_t)kn));
    bw[kp] += r1;
    bw[kq] += r2;
    bw[kn] = r2;
  }
  for (int k = m; k < m + n; ++k) {
    const int kn = k % n, kp = (k + p) % n, kq = (k + q) % n, km = (k + n - 1) % n;
    const uint32_t r3 = 1566083941u * ss_T(bw[kn] + bw[kp] + bw[km]);
    const uint32_t r4 = r3 - (uint32_t)kn;
    bw[kp] ^= r3;
    bw[kq] ^= r4;
    bw[kn] = r4;
  }
  int zero = 1;
  for (int k = 0; k < 312; ++k) {
    r->x[k] = (uint64_t)bw[2 * k] | ((uint64_t)bw[2 * k + 1] << 32);
    if (k == 0 ? (r->x[0] & ~((1ULL << 31) - 1)) != 0 : r->x[k] != 0) zero = 0;
  }
  if (zero) r->x[0] = 1ULL << 63;
  r->i = 312;
  r->has_spare = 0;
  r->spare = 0.0;
}

static uint64_t rng_next(Rng* r) {
  if (r->i >= 312) { /* whole-array twist, as libstdc++ does */
    for (int k = 0; k < 312; ++k) {
      const uint64_t y = (r->x[k] & 0xffffffff80000000ULL) | (r->x[(k + 1) % 312] & 0x7fffffffULL);
      r->x[k] = r->x[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1ULL) ? 0xb5026f5aa96619e9ULL : 0ULL);
    }
    r->i = 0;
  }
  uint64_t z = r->x[r->i++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71d67fffeda60000ULL;
  z ^= (z << 37) & 0xfff7eee000000000ULL;
  z ^= z >> 43;
  return z;
}

static double uniform01(Rng* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }             /* rng.hpp:51 */
static double exponential(Rng* r, double rate) { return -log1p(-uniform01(r)) / rate; }          /* rng.hpp:54 */
static double normal01(Rng* r) {                                                                 /* rng.hpp:57-71 */
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double u1 = uniform01(r);
  double u2 = uniform01(r);
  while (u1 <= 0.0) u1 = uniform01(r);
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = 2.0 * M_PI * u2;
  r->spare = radius * sin(angle);
  r->has_spare = 1;
  return radius * cos(angle);
}
static double normal(Rng* r, double mean, double sd) {                                           /* rng.hpp:73 */
  const double z = normal01(r);
  const double p = sd * z;
  return mean + p;
}
static uint64_t uniform_below(Rng* r, uint64_t bound) {                                          /* rng.hpp:76-82 */
  if (bound <= 1) return 0;
  const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
  uint64_t d = rng_next(r);
  while (d >= limit) d = rng_next(r);
  return d % bound;
}
static int round_clamp_token(double v) {                                                         /* workload.cpp:52-55 */
  const double r = round(v);
  return r < 1.0 ? 1 : (int)r;
}

/* ------------------------------------------------------------------ inputs */
typedef struct {
  int mode; /* LT_MODE_* */
  double mi, si, mo, so;
  const int32_t* full; /* pairs */
  int64_t n_full;
} Len;

static Len len_of(const lt_length_spec* l, const int32_t* full) {
  Len x;
  x.mode = l->mode;
  x.mi = l->mean_input;
  x.si = l->std_input;
  x.mo = l->mean_output;
  x.so = l->std_output;
  x.full = full + 2 * l->full_offset;
  x.n_full = l->full_count;
  return x;
}

/* list_stats (workload.cpp:31-50) */
static void list_stats(const Len* l, int input, double* mean, double* sd) {
  if (l->n_full == 0) {
    *mean = *sd = 0.0;
    return;
  }
  double sum = 0.0;
  for (int64_t i = 0; i < l->n_full; ++i) sum += (double)l->full[2 * i + (input ? 0 : 1)];
  const double m = sum / (double)l->n_full;
  double sq = 0.0;
  for (int64_t i = 0; i < l->n_full; ++i) {
    const double v = (double)l->full[2 * i + (input ? 0 : 1)];
    sq += (v - m) * (v - m);
  }
  *mean = m;
  *sd = sqrt(sq / (double)l->n_full);
}
static double len_out_mean(const Len* l) {
  if (l->mode == LT_MODE_FULL) {
    double m, s;
    list_stats(l, 0, &m, &s);
    return m;
  }
  return l->mo;
}
static double len_in_mean(const Len* l) {
  if (l->mode == LT_MODE_FULL) {
    double m, s;
    list_stats(l, 1, &m, &s);
    return m;
  }
  return l->mi;
}

typedef struct {
  int id, rank;
  double rate;
  Len len;
} Adp;

typedef struct {
  int64_t id;
  int adapter;
  double t;
  int in, out;
} Req;

typedef struct {
  int code, kind;
  int64_t a, b;
  char msg[320];
} Err;

static int err_set(Err* e, int code, const char* fmt, ...) __attribute__((format(printf, 3, 4)));
#include <stdarg.h>
static int err_set(Err* e, int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(e->msg, sizeof(e->msg), fmt, ap);
  va_end(ap);
  e->code = code;
  e->kind = LT_K_MESSAGE;
  return 0;
}

/* std::to_string(double) == "%f" */
static const char* f6(double v, char* buf) {
  snprintf(buf, 64, "%f", v);
  return buf;
}

static int validate_len(const Len* l, const char* path, Err* e) { /* workload.cpp:97-116 */
  char b[64];
  if (l->mode == LT_MODE_FULL) {
    if (l->n_full <= 0) return err_set(e, LT_ERR_VALIDATION, "%s.full_lengths: Full mode requires a non-empty length list", path);
    for (int64_t i = 0; i < l->n_full; ++i)
      if (l->full[2 * i] < 1 || l->full[2 * i + 1] < 1)
        return err_set(e, LT_ERR_VALIDATION, "%s.full_lengths[%lld]: token counts must be >= 1", path, (long long)i);
    return 1;
  }
  if (l->mi <= 0.0) return err_set(e, LT_ERR_VALIDATION, "%s.mean_input: must be > 0, got %s", path, f6(l->mi, b));
  if (l->mo <= 0.0) return err_set(e, LT_ERR_VALIDATION, "%s.mean_output: must be > 0, got %s", path, f6(l->mo, b));
  if (l->si < 0.0) return err_set(e, LT_ERR_VALIDATION, "%s.std_input: must be >= 0, got %s", path, f6(l->si, b));
  if (l->so < 0.0) return err_set(e, LT_ERR_VALIDATION, "%s.std_output: must be >= 0, got %s", path, f6(l->so, b));
  return 1;
}

/* ------------------------------------------------------------------ arrivals */
/* sample_lengths (workload.cpp:143-168) for adapter stream id `stream`. */
static void sample_lengths(const Len* l, size_t n, uint64_t seed, uint64_t stream, int* in, int* out) {
  Rng* r = (Rng*)malloc(sizeof(Rng));
  rng_init(r, seed, 2, stream);
  if (l->mode == LT_MODE_FULL) {
    const int64_t d = l->n_full;
    int* deck = (int*)malloc(sizeof(int) * 2 * (size_t)d);
    memcpy(deck, l->full, sizeof(int) * 2 * (size_t)d);
    for (int64_t i = d; i > 1; --i) { /* rng.hpp:86-91 Fisher-Yates */
      const int64_t j = (int64_t)uniform_below(r, (uint64_t)i);
      int t0 = deck[2 * (i - 1)], t1 = deck[2 * (i - 1) + 1];
      deck[2 * (i - 1)] = deck[2 * j];
      deck[2 * (i - 1) + 1] = deck[2 * j + 1];
      deck[2 * j] = t0;
      deck[2 * j + 1] = t1;
    }
    int64_t cur = 0;
    for (size_t i = 0; i < n; ++i) {
      if (cur == d) {
        for (int64_t k = d; k > 1; --k) {
          const int64_t j = (int64_t)uniform_below(r, (uint64_t)k);
          int t0 = deck[2 * (k - 1)], t1 = deck[2 * (k - 1) + 1];
          deck[2 * (k - 1)] = deck[2 * j];
          deck[2 * (k - 1) + 1] = deck[2 * j + 1];
          deck[2 * j] = t0;
          deck[2 * j + 1] = t1;
        }
        cur = 0;
      }
      in[i] = deck[2 * cur];
      out[i] = deck[2 * cur + 1];
      ++cur;
    }
    free(deck);
  } else {
    for (size_t i = 0; i < n; ++i) {
      in[i] = round_clamp_token(normal(r, l->mi, l->si));
      out[i] = round_clamp_token(normal(r, l->mo, l->so));
    }
  }
  free(r);
}

static int req_cmp(const void* a, const void* b) { /* (time, adapter_id, seq) -- stable via seq */
  const Req* x = (const Req*)a;
  const Req* y = (const Req*)b;
  if (x->t != y->t) return x->t < y->t ? -1 : 1;
  if (x->adapter != y->adapter) return x->adapter < y->adapter ? -1 : 1;
  return x->id < y->id ? -1 : (x->id > y->id);
}

/* generate_arrivals (workload.cpp:170-211). Returns count, *out malloc'd. */
static int64_t generate_arrivals(const Adp* ads, int n_ad, const Len* wl, double duration, uint64_t seed, int mode,
                                 Req** out, Err* e) {
  size_t cap = 64, n = 0;
  Req* v = (Req*)malloc(sizeof(Req) * cap);
  int64_t seq = 0;
  for (int a = 0; a < n_ad; ++a) {
    Rng* r = (Rng*)malloc(sizeof(Rng));
    rng_init(r, seed, 1, (uint64_t)(int64_t)ads[a].id);
    size_t nt = 0, ct = 64;
    double* times = (double*)malloc(sizeof(double) * ct);
    double t = 0.0;
    for (;;) {
      t += exponential(r, ads[a].rate);
      if (t >= duration) break;
      if (nt == ct) times = (double*)realloc(times, sizeof(double) * (ct *= 2));
      times[nt++] = t;
    }
    free(r);
    Len l = ads[a].len;
    if (mode != l.mode) {
      if (mode == LT_MODE_FULL) {
        free(times);
        free(v);
        err_set(e, LT_ERR_VALIDATION, "workload.lengths: cannot force Full mode without a length list");
        return -1;
      }
      double m1, s1, m2, s2; /* LengthSpec::as_mean (workload.cpp:91-95) */
      list_stats(&l, 1, &m1, &s1);
      list_stats(&l, 0, &m2, &s2);
      l.mode = LT_MODE_MEAN;
      l.mi = m1;
      l.si = s1;
      l.mo = m2;
      l.so = s2;
    }
    int* in = (int*)malloc(sizeof(int) * (nt + 1));
    int* ou = (int*)malloc(sizeof(int) * (nt + 1));
    sample_lengths(&l, nt, seed, (uint64_t)(int64_t)ads[a].id, in, ou);
    for (size_t i = 0; i < nt; ++i) {
      if (n == cap) v = (Req*)realloc(v, sizeof(Req) * (cap *= 2));
      v[n].id = seq++;
      v[n].adapter = ads[a].id;
      v[n].t = times[i];
      v[n].in = in[i];
      v[n].out = ou[i];
      ++n;
    }
    free(in);
    free(ou);
    free(times);
  }
  (void)wl;
  qsort(v, n, sizeof(Req), req_cmp);
  for (size_t i = 0; i < n; ++i) v[i].id = (int64_t)i;
  *out = v;
  return (int64_t)n;
}

/* ------------------------------------------------------------------ config */
typedef struct {
  lt_server_config c;
  int slots;
} Cfg;

static int slot_cost(const lt_server_config* c, int rank, int64_t* out, Err* e) { /* estimators.cpp:46-55 */
  if (rank == 0) {
    *out = 0;
    return 1;
  }
  if (rank < 0) return err_set(e, LT_ERR_VALIDATION, "slot rank must be >= 0, got %d", rank);
  for (int i = 0; i < c->n_slot_cost; ++i)
    if (c->slot_cost_rank[i] == rank) {
      *out = c->slot_cost_tokens[i];
      return 1;
    }
  if (c->has_slot_cost_base_rank8) {
    *out = (int64_t)llround(c->slot_cost_base_rank8 * rank / 8.0);
    return 1;
  }
  err_set(e, LT_ERR_CONFIG,
          "estimators.memory: no slot cost for rank %d (add a slot_cost_tokens entry or slot_cost_base_rank8)", rank);
  return 0;
}

static int load_latency(const lt_server_config* c, int rank, double* out, Err* e) { /* estimators.cpp:78-83 */
  for (int i = 0; i < c->n_load; ++i)
    if (c->load_rank[i] == rank) {
      *out = c->load_source == LT_SOURCE_CPU ? c->load_seconds[i] : c->load_seconds[i] * c->disk_multiplier;
      return 1;
    }
  err_set(e, LT_ERR_CONFIG, "estimators.load.cpu_load_seconds: no entry for rank %d", rank);
  return 0;
}

static int cmp_int(const void* a, const void* b) {
  const int x = *(const int*)a, y = *(const int*)b;
  return (x > y) - (x < y);
}

static int validate_config(const lt_server_config* c, int slots, Err* e) { /* server_config.cpp:21-27 */
  if (slots < 1) return err_set(e, LT_ERR_VALIDATION, "config.slots: must be >= 1, got %d", slots);
  if (c->iteration_cap < 1) return err_set(e, LT_ERR_VALIDATION, "config.iteration_cap: must be >= 1");
  if (c->k4 < 0.0) return err_set(e, LT_ERR_VALIDATION, "estimators.latency.k4: must be >= 0");
  if (c->k5 <= 0.0) return err_set(e, LT_ERR_VALIDATION, "estimators.latency.k5: must be > 0 (a forward pass takes time)");
  if (c->k6 < 0.0) return err_set(e, LT_ERR_VALIDATION, "estimators.latency.k6: must be >= 0");
  if (c->k7 < 1.0) return err_set(e, LT_ERR_VALIDATION, "estimators.latency.k7: must be >= 1 (adapters never speed up the model)");
  if (c->total_kv_budget <= 0) return err_set(e, LT_ERR_VALIDATION, "estimators.memory.total_kv_budget: must be > 0");
  if (c->n_slot_cost == 0 && !c->has_slot_cost_base_rank8)
    return err_set(e, LT_ERR_VALIDATION, "estimators.memory: one of slot_cost_tokens or slot_cost_base_rank8 is required");
  if (c->has_slot_cost_base_rank8 && c->slot_cost_base_rank8 <= 0.0)
    return err_set(e, LT_ERR_VALIDATION, "estimators.memory.slot_cost_base_rank8: must be > 0");
  /* ascending-rank checks (estimators.cpp:64-75, :86-97) */
  {
    int n = c->n_slot_cost;
    int* idx = (int*)malloc(sizeof(int) * (size_t)(n + 1));
    for (int i = 0; i < n; ++i) idx[i] = i;
    for (int i = 1; i < n; ++i)
      for (int j = i; j > 0 && c->slot_cost_rank[idx[j]] < c->slot_cost_rank[idx[j - 1]]; --j) {
        int t = idx[j];
        idx[j] = idx[j - 1];
        idx[j - 1] = t;
      }
    int64_t prev = 0;
    int prev_rank = 0;
    for (int i = 0; i < n; ++i) {
      const int r = c->slot_cost_rank[idx[i]];
      const int64_t cost = c->slot_cost_tokens[idx[i]];
      if (r <= 0) {
        free(idx);
        return err_set(e, LT_ERR_VALIDATION, "estimators.memory.slot_cost_tokens: ranks must be > 0");
      }
      if (cost <= prev) {
        free(idx);
        return err_set(e, LT_ERR_VALIDATION,
                       "estimators.memory.slot_cost_tokens: cost must increase with rank (rank %d vs rank %d)", r, prev_rank);
      }
      prev = cost;
      prev_rank = r;
    }
    free(idx);
  }
  if (c->disk_multiplier < 1.0) return err_set(e, LT_ERR_VALIDATION, "estimators.load.disk_multiplier: must be >= 1");
  {
    int n = c->n_load;
    int* idx = (int*)malloc(sizeof(int) * (size_t)(n + 1));
    for (int i = 0; i < n; ++i) idx[i] = i;
    for (int i = 1; i < n; ++i)
      for (int j = i; j > 0 && c->load_rank[idx[j]] < c->load_rank[idx[j - 1]]; --j) {
        int t = idx[j];
        idx[j] = idx[j - 1];
        idx[j - 1] = t;
      }
    double prev = 0.0;
    int prev_rank = 0;
    for (int i = 0; i < n; ++i) {
      const int r = c->load_rank[idx[i]];
      const double sec = c->load_seconds[idx[i]];
      if (r <= 0) {
        free(idx);
        return err_set(e, LT_ERR_VALIDATION, "estimators.load.cpu_load_seconds: ranks must be > 0");
      }
      if (sec < prev) {
        free(idx);
        return err_set(e, LT_ERR_VALIDATION,
                       "estimators.load.cpu_load_seconds: latency must not decrease with rank (rank %d vs rank %d)", r,
                       prev_rank);
      }
      prev = sec;
      prev_rank = r;
    }
    free(idx);
  }
  return 1;
}

/* ------------------------------------------------------------------ engine */
enum { P_WAITING = 0, P_RUNNING = 1, P_PREEMPTED = 2, P_FINISHED = 3, P_REJECTED = 4 };

typedef struct {
  int phase, gen, pre, dense, rank;
  int64_t kv, seq;
  int has_first;
  double first, completion;
  /* emitted-token record: runs of consecutive iterations (start, count) */
  int* runs;
  int n_runs, cap_runs;
} St;

typedef struct {
  int* v;
  int n, cap;
} Vec;

static void vpush(Vec* q, int x) {
  if (q->n == q->cap) q->v = (int*)realloc(q->v, sizeof(int) * (size_t)(q->cap = q->cap ? 2 * q->cap : 16));
  q->v[q->n++] = x;
}

typedef struct {
  /* output */
  lt_sim_summary* o;
  Err* e;
} Out;

typedef struct {
  const Req* req;
  int64_t n;
  St* st;
  const Adp* ads; /* spec order */
  int n_ad;
  int* ids_sorted;     /* dense index -> adapter id (ascending) */
  int* rank_of_dense;
  /* slot cache (adapter_cache.cpp) */
  int* resident;       /* dense -> 1 */
  double* last_used;
  int n_resident;
  int G;
} Sim;

static int dense_of(const Sim* s, int id) {
  int lo = 0, hi = s->n_ad - 1;
  while (lo <= hi) {
    const int m = (lo + hi) / 2;
    if (s->ids_sorted[m] == id) return m;
    if (s->ids_sorted[m] < id) lo = m + 1;
    else hi = m - 1;
  }
  return -1;
}

static void run_push(St* r, int it) {
  if (r->n_runs > 0) {
    int* last = &r->runs[2 * (r->n_runs - 1)];
    if (last[0] + last[1] == it) {
      last[1]++;
      return;
    }
  }
  if (r->n_runs == r->cap_runs) r->runs = (int*)realloc(r->runs, sizeof(int) * 2 * (size_t)(r->cap_runs = r->cap_runs ? 2 * r->cap_runs : 2));
  r->runs[2 * r->n_runs] = it;
  r->runs[2 * r->n_runs + 1] = 1;
  r->n_runs++;
}

/* Engine::run + metrics (engine.cpp:73-161, kv_scheduler.cpp:49-259,
 * adapter_cache.cpp:40-78, estimators.cpp:110-139, metrics.cpp:70-113). */
/* percentile_nearest_rank (metrics.cpp:47-54): sort, 1-based rank ceil(p/100 n) clamped to [1, n] */
static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}
static double nearest_rank_sorted(const double* v, int64_t n, double pct) {
  if (n == 0) return 0.0;
  int64_t rank = (int64_t)ceil(pct / 100.0 * (double)n);
  if (rank < 1) rank = 1;
  if (rank > n) rank = n;
  return v[rank - 1];
}

static void simulate(const lt_server_config* c, int G, const Adp* ads, int n_ad, double duration, const Req* req,
                     int64_t n, double ideal, lt_sim_summary* o, Err* e, int want_digest, int64_t cap_override,
                     lt_request_states* states, int64_t st_off) {
  memset(o, 0, sizeof(*o));
  Sim S;
  memset(&S, 0, sizeof(S));
  S.req = req;
  S.n = n;
  S.ads = ads;
  S.n_ad = n_ad;
  S.G = G;
  S.ids_sorted = (int*)malloc(sizeof(int) * (size_t)n_ad);
  S.rank_of_dense = (int*)malloc(sizeof(int) * (size_t)n_ad);
  int max_rank = 0;
  for (int a = 0; a < n_ad; ++a) {
    S.ids_sorted[a] = ads[a].id;
    if (ads[a].rank > max_rank) max_rank = ads[a].rank;
  }
  qsort(S.ids_sorted, (size_t)n_ad, sizeof(int), cmp_int);
  for (int a = 0; a < n_ad; ++a) S.rank_of_dense[dense_of(&S, ads[a].id)] = ads[a].rank;
  S.resident = (int*)calloc((size_t)n_ad, sizeof(int));
  S.last_used = (double*)calloc((size_t)n_ad, sizeof(double));
  S.st = (St*)calloc((size_t)(n > 0 ? n : 1), sizeof(St));
  for (int64_t i = 0; i < n; ++i) {
    S.st[i].dense = dense_of(&S, req[i].adapter);
    S.st[i].rank = S.rank_of_dense[S.st[i].dense];
    S.st[i].seq = -1;
  }
  /* mem_max (estimators.cpp:100-108; engine.cpp:46-54) */
  int64_t capacity = c->total_kv_budget;
  for (int g = 0; g < G; ++g) {
    int64_t sc;
    if (!slot_cost(c, max_rank, &sc, e)) goto done_err;
    capacity -= sc;
  }
  if (capacity < 0) capacity = 0;
  if (capacity <= 0) {
    err_set(e, LT_ERR_CONFIG, "infeasible configuration: %d slots consume the entire KV budget (mem_max = 0)", G);
    goto done_err;
  }
  o->kv_capacity_tokens = capacity;
  {
    const int64_t cap_it = cap_override > 0 ? cap_override : c->iteration_cap;
    Vec running = {0}, wp = {0}, wf = {0};
    int64_t used = 0, next_seq = 0, ingest = 0, iterations = 0;
    double clock = 0.0;
    size_t n_emit_cap = 1024, n_emit = 0;
    double* emit_at = (double*)malloc(sizeof(double) * n_emit_cap); /* emit time of each iteration */
    int* r_at = (int*)malloc(sizeof(int) * n_emit_cap);
    uint64_t digest = 0xcbf29ce484222325ULL;
    int64_t loads_total = 0;
    unsigned char* claimed = (unsigned char*)malloc((size_t)n_ad);
    unsigned char* evicted = (unsigned char*)malloc((size_t)n_ad);
    unsigned char* blocked = (unsigned char*)malloc((size_t)n_ad);
    unsigned char* needed = (unsigned char*)malloc((size_t)n_ad);
    int* pool = (int*)malloc(sizeof(int) * (size_t)(n_ad + 1));
    for (;;) {
      if (running.n == 0 && wp.n + wf.n == 0) { /* engine.cpp:82-85 */
        if (ingest >= n) break;
        if (req[ingest].t > clock) clock = req[ingest].t;
      }
      while (ingest < n && req[ingest].t <= clock) vpush(&wf, (int)ingest++); /* :88-92 */
      /* complete_finished (kv_scheduler.cpp:238-259) */
      {
        int w = 0;
        for (int k = 0; k < running.n; ++k) {
          St* r = &S.st[running.v[k]];
          if (r->gen >= req[running.v[k]].out) {
            used -= r->kv;
            r->kv = 0;
            r->phase = P_FINISHED;
          } else {
            running.v[w++] = running.v[k];
          }
        }
        running.n = w;
      }
      /* decode_step_alloc (kv_scheduler.cpp:183-236) */
      if (running.n > 0) {
        int64_t demand = running.n;
        while (used + demand > capacity && running.n > 1) {
          int vp = 0;
          for (int k = 1; k < running.n; ++k)
            if (S.st[running.v[k]].seq > S.st[running.v[vp]].seq) vp = k;
          const int victim = running.v[vp];
          St* r = &S.st[victim];
          used -= r->kv;
          r->kv = 0;
          r->phase = P_PREEMPTED;
          r->pre++;
          memmove(&running.v[vp], &running.v[vp + 1], sizeof(int) * (size_t)(running.n - vp - 1));
          running.n--;
          /* lower_bound by (arrival, request_id) */
          int lo = 0, hi = wp.n;
          while (lo < hi) {
            const int mid = (lo + hi) / 2;
            const Req* a = &req[wp.v[mid]];
            const Req* b = &req[victim];
            const int less = a->t != b->t ? a->t < b->t : a->id < b->id;
            if (less) lo = mid + 1;
            else hi = mid;
          }
          vpush(&wp, 0);
          memmove(&wp.v[lo + 1], &wp.v[lo], sizeof(int) * (size_t)(wp.n - 1 - lo));
          wp.v[lo] = victim;
          --demand;
        }
        if (used + demand > capacity) {
          St* r = &S.st[running.v[0]];
          if (r->gen + 1 < req[running.v[0]].out || used + demand - 1 > capacity) {
            err_set(e, LT_ERR_SIMULATION, "single request exceeds KV capacity: request %lld",
                    (long long)req[running.v[0]].id);
            free(emit_at);
            free(r_at);
            free(running.v);
            free(wp.v);
            free(wf.v);
            free(claimed);
            free(evicted);
            free(blocked);
            free(needed);
            free(pool);
            goto done_err;
          }
        } else {
          for (int k = 0; k < running.n; ++k) {
            used += 1;
            S.st[running.v[k]].kv += 1;
          }
        }
      }
      /* admit: SlotPlan (kv_scheduler.cpp:49-98) + scan_queue (:109-181) */
      {
        int free_slots = G - S.n_resident;
        memset(claimed, 0, (size_t)n_ad);
        memset(evicted, 0, (size_t)n_ad);
        memset(blocked, 0, (size_t)n_ad);
        for (int k = 0; k < running.n; ++k)
          if (S.st[running.v[k]].rank > 0) claimed[S.st[running.v[k]].dense] = 1;
        int np = 0; /* idle pool sorted by (last_used, id) */
        for (int a = 0; a < n_ad; ++a)
          if (S.resident[a] && !claimed[a]) pool[np++] = a;
        for (int i = 1; i < np; ++i)
          for (int j = i; j > 0; --j) {
            const int x = pool[j], y = pool[j - 1];
            if (S.last_used[x] < S.last_used[y] || (S.last_used[x] == S.last_used[y] && x < y)) {
              pool[j] = y;
              pool[j - 1] = x;
            } else {
              break;
            }
          }
        Vec* queues[2] = {&wp, &wf};
        for (int qi = 0; qi < 2; ++qi) {
          Vec* q = queues[qi];
          int read = 0, write = 0, keep = 1;
          for (; read < q->n; ++read) {
            const int idx = q->v[read];
            St* r = &S.st[idx];
            const int64_t demand = (int64_t)req[idx].in + r->gen + 1;
            if (demand > capacity) {
              r->phase = P_REJECTED;
              continue;
            }
            const int needs = r->rank > 0;
            const int a = r->dense;
            if (needs && blocked[a]) {
              q->v[write++] = idx;
              if (!c->loaded_adapter_priority) {
                keep = 0;
                ++read;
                break;
              }
              continue;
            }
            int claimable = 1;
            if (needs) {
              int vres = 0; /* is_virtually_resident */
              if (!evicted[a])
                for (int k = 0; k < np; ++k)
                  if (pool[k] == a) vres = 1;
              claimable = claimed[a] || vres || free_slots > 0 || np > 0;
            }
            if (needs && !claimable) {
              blocked[a] = 1;
              q->v[write++] = idx;
              if (!c->loaded_adapter_priority) {
                keep = 0;
                ++read;
                break;
              }
              continue;
            }
            if (used + demand > capacity) {
              q->v[write++] = idx;
              keep = 0;
              ++read;
              break;
            }
            used += demand;
            r->kv = demand;
            r->phase = P_RUNNING;
            r->seq = next_seq++;
            if (needs && !claimed[a]) { /* SlotPlan::claim */
              int pos = -1;
              for (int k = 0; k < np; ++k)
                if (pool[k] == a) pos = k;
              if (pos >= 0 && !evicted[a]) {
                memmove(&pool[pos], &pool[pos + 1], sizeof(int) * (size_t)(np - pos - 1));
                np--;
              } else if (free_slots > 0) {
                free_slots--;
              } else {
                evicted[pool[0]] = 1;
                memmove(&pool[0], &pool[1], sizeof(int) * (size_t)(np - 1));
                np--;
              }
              claimed[a] = 1;
            }
            vpush(&running, idx);
          }
          for (; read < q->n; ++read) q->v[write++] = q->v[read];
          q->n = write;
          if (!keep) break;
        }
      }
      if (running.n == 0) {
        if (wp.n + wf.n != 0) {
          err_set(e, LT_ERR_INTERNAL, "empty batch with a non-empty waiting queue: admission stuck");
          goto loop_err;
        }
        continue;
      }
      /* ensure_loaded (adapter_cache.cpp:40-78), needed in ascending id */
      double loads = 0.0;
      int nl = 0, A = 0;
      memset(needed, 0, (size_t)n_ad);
      for (int k = 0; k < running.n; ++k)
        if (S.st[running.v[k]].rank > 0) needed[S.st[running.v[k]].dense] = 1;
      for (int a = 0; a < n_ad; ++a) {
        if (!needed[a]) continue;
        A++;
      }
      if (A > G) {
        err_set(e, LT_ERR_INTERNAL, "SlotCache: running batch needs %d adapters but only %d slots exist (admission bug)", A, G);
        goto loop_err;
      }
      for (int a = 0; a < n_ad; ++a) {
        if (!needed[a] || S.resident[a]) continue;
        if (S.n_resident >= G) {
          int victim = -1;
          for (int b = 0; b < n_ad; ++b) {
            if (!S.resident[b] || needed[b]) continue;
            if (victim < 0 || S.last_used[b] < S.last_used[victim]) victim = b; /* ties: smaller id first */
          }
          if (victim < 0) {
            err_set(e, LT_ERR_INTERNAL, "SlotCache: no evictable slot for adapter %d (admission bug)", S.ids_sorted[a]);
            goto loop_err;
          }
          S.resident[victim] = 0;
          S.n_resident--;
        }
        S.resident[a] = 1;
        S.n_resident++;
        S.last_used[a] = clock;
        double ll;
        if (!load_latency(c, S.rank_of_dense[a], &ll, e)) goto loop_err;
        loads += ll;
        nl++;
      }
      for (int a = 0; a < n_ad; ++a)
        if (needed[a]) S.last_used[a] = clock;
      loads_total += nl;
      /* lat_step (estimators.cpp:110-139) */
      const int R = running.n, W = wp.n + wf.n;
      double ratio = (double)G / (double)n_ad;
      if (1.0 < ratio) ratio = 1.0;
      double v = c->k1 * R + c->k2 * W + c->k3 * W * ratio;
      const double sched = v < 0.0 ? 0.0 : v;
      const double model = c->k4 * R + c->k5;
      const double adapters = A == 0 ? 1.0 : c->k6 * A + c->k7;
      const double lat = sched + loads + model * adapters;
      const double emit = clock + lat;
      if (n_emit == n_emit_cap) {
        emit_at = (double*)realloc(emit_at, sizeof(double) * (n_emit_cap *= 2));
        r_at = (int*)realloc(r_at, sizeof(int) * n_emit_cap);
      }
      emit_at[n_emit] = emit;
      r_at[n_emit] = R;
      for (int k = 0; k < R; ++k) { /* engine.cpp:128-135 */
        St* r = &S.st[running.v[k]];
        r->gen++;
        if (!r->has_first) {
          r->has_first = 1;
          r->first = emit;
        }
        run_push(r, (int)n_emit);
        if (r->gen == req[running.v[k]].out) r->completion = emit;
      }
      n_emit++;
      if (want_digest) {
        uint64_t lb;
        memcpy(&lb, &lat, 8);
        digest ^= (uint64_t)(uint32_t)R | ((uint64_t)(uint32_t)W << 32);
        digest *= 0x100000001b3ULL;
        digest ^= (uint64_t)(uint32_t)A | ((uint64_t)(uint32_t)nl << 32);
        digest *= 0x100000001b3ULL;
        digest ^= lb;
        digest *= 0x100000001b3ULL;
      }
      clock = emit;
      ++iterations;
      if (iterations >= cap_it) {
        o->truncated = 1;
        break;
      }
    }
    /* compute_metrics (metrics.cpp:70-113): sums in request_id order, ITL gap by gap */
    o->iterations = iterations;
    o->final_clock_s = clock;
    o->load_events = loads_total;
    o->digest = want_digest ? digest : 0;
    o->n_requests = n;
    if (n == 0) {
      o->degenerate = 1;
    } else {
      const double window = duration;
      double rej = 0.0, ttft = 0.0, itl = 0.0;
      int64_t nttft = 0, nitl = 0, win = 0, tot = 0, pre = 0;
      double* ttft_v = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
      size_t itl_cap = 1024, itl_n = 0;
      double* itl_v = (double*)malloc(sizeof(double) * itl_cap);
      for (int64_t i = 0; i < n; ++i) {
        St* r = &S.st[i];
        if (r->phase == P_REJECTED) {
          o->rejected_count++;
          rej += (double)req[i].out / window;
        }
        if (r->phase == P_FINISHED) o->finished_count++;
        if (r->has_first) {
          ttft += r->first - req[i].t;
          ttft_v[nttft] = r->first - req[i].t;
          nttft++;
        }
        double prev = 0.0;
        int have = 0;
        for (int k = 0; k < r->n_runs; ++k)
          for (int j = 0; j < r->runs[2 * k + 1]; ++j) {
            const double t = emit_at[r->runs[2 * k] + j];
            if (t <= window) win++;
            if (have) {
              itl += t - prev;
              nitl++;
              if (itl_n == itl_cap) {
                itl_cap *= 2;
                itl_v = (double*)realloc(itl_v, sizeof(double) * itl_cap);
              }
              itl_v[itl_n++] = t - prev;
            }
            prev = t;
            have = 1;
            tot++;
          }
        pre += r->pre;
      }
      o->tokens_in_window = win;
      o->tokens_total = tot;
      o->preemptions = pre;
      o->throughput_tok_s = (double)win / window;
      o->ttft_mean_s = nttft ? ttft / (double)nttft : 0.0;
      o->itl_mean_s = nitl ? itl / (double)nitl : 0.0;
      qsort(ttft_v, (size_t)nttft, sizeof(double), cmp_double);
      qsort(itl_v, itl_n, sizeof(double), cmp_double);
      o->ttft_p50_s = nearest_rank_sorted(ttft_v, nttft, 50.0);
      o->ttft_p99_s = nearest_rank_sorted(ttft_v, nttft, 99.0);
      o->itl_p50_s = nearest_rank_sorted(itl_v, (int64_t)itl_n, 50.0);
      o->itl_p99_s = nearest_rank_sorted(itl_v, (int64_t)itl_n, 99.0);
      free(ttft_v);
      free(itl_v);
      const double eff_raw = ideal - rej;
      const double eff = eff_raw < 0.0 ? 0.0 : eff_raw;
      o->starved = o->throughput_tok_s < 0.9 * eff;
    }
    for (size_t k = 0; k < n_emit; ++k) o->sum_running += r_at[k];
    if (states) {
      for (int64_t i = 0; i < n; ++i) {
        const int64_t off = st_off + i;
        if (off >= states->capacity) continue;
        St* r = &S.st[i];
        if (states->phase) states->phase[off] = (int8_t)r->phase;
        if (states->tokens_generated) states->tokens_generated[off] = r->gen;
        if (states->first_token_time_s) states->first_token_time_s[off] = r->has_first ? r->first : NAN;
        if (states->completion_time_s) states->completion_time_s[off] = r->completion;
        if (states->preemption_count) states->preemption_count[off] = r->pre;
        if (states->adapter_id) states->adapter_id[off] = req[i].adapter;
        if (states->input_tokens) states->input_tokens[off] = req[i].in;
        if (states->output_tokens) states->output_tokens[off] = req[i].out;
        if (states->arrival_time_s) states->arrival_time_s[off] = req[i].t;
      }
    }
    free(emit_at);
    free(r_at);
    free(running.v);
    free(wp.v);
    free(wf.v);
    free(claimed);
    free(evicted);
    free(blocked);
    free(needed);
    free(pool);
    goto done;
  loop_err:
    free(emit_at);
    free(r_at);
    free(running.v);
    free(wp.v);
    free(wf.v);
    free(claimed);
    free(evicted);
    free(blocked);
    free(needed);
    free(pool);
    goto done_err;
  }
done_err:
  o->status = e->code;
  o->status_kind = LT_K_MESSAGE;
done:
  o->duration_s = duration;
  o->slots = G;
  o->served_adapters = n_ad;
  o->ideal_throughput_tok_s = ideal;
  for (int64_t i = 0; i < n; ++i) free(S.st[i].runs);
  free(S.st);
  free(S.ids_sorted);
  free(S.rank_of_dense);
  free(S.resident);
  free(S.last_used);
}

/* ------------------------------------------------------------------ batch */
static int g_threads = 1;
static char (*g_msgs)[320] = NULL;
static int64_t g_nmsgs = 0;

typedef struct {
  void (*fn)(void*, int64_t);
  void* ctx;
  int64_t n;
  int64_t next;
  pthread_mutex_t mu;
} Pool;

static void* pool_worker(void* arg) {
  Pool* p = (Pool*)arg;
  for (;;) {
    pthread_mutex_lock(&p->mu);
    const int64_t i = p->next++;
    pthread_mutex_unlock(&p->mu);
    if (i >= p->n) break;
    p->fn(p->ctx, i);
  }
  return NULL;
}

/* run_parallel pattern (placement.cpp:65-96): a shared counter over tasks */
static void run_pool(int64_t n, void (*fn)(void*, int64_t), void* ctx) {
  Pool p;
  p.fn = fn;
  p.ctx = ctx;
  p.n = n;
  p.next = 0;
  pthread_mutex_init(&p.mu, NULL);
  int w = g_threads < 1 ? 1 : g_threads;
  if (w > n) w = (int)(n > 0 ? n : 1);
  pthread_t th[256];
  if (w > 256) w = 256;
  for (int k = 1; k < w; ++k) pthread_create(&th[k], NULL, pool_worker, &p);
  pool_worker(&p);
  for (int k = 1; k < w; ++k) pthread_join(th[k], NULL);
  pthread_mutex_destroy(&p.mu);
}

static void msgs_reset(int64_t n) {
  free(g_msgs);
  g_msgs = (char(*)[320])calloc((size_t)(n > 0 ? n : 1), 320);
  g_nmsgs = n;
}

typedef struct {
  const lt_workload_batch* b;
  const lt_server_config* c;
  const lt_sim_options* o;
  lt_sim_summary* out;
  Req** gen;
  int64_t* gen_n;
  int arrivals_only;
} SimJob;

static void sim_task(void* vctx, int64_t i) {
  SimJob* J = (SimJob*)vctx;
  const lt_workload_batch* b = J->b;
  const lt_scenario* s = &b->scenarios[i];
  Err e;
  memset(&e, 0, sizeof(e));
  lt_sim_summary tmp;
  lt_sim_summary* o = J->out ? &J->out[i] : &tmp;
  memset(o, 0, sizeof(*o));
  const int G = s->slots > 0 ? s->slots : (J->c ? J->c->slots : 1);
  Adp* ads = (Adp*)malloc(sizeof(Adp) * (size_t)(s->n_adapters > 0 ? s->n_adapters : 1));
  const Len wl = len_of(&b->lengths[s->length_index], b->full_lengths);
  for (int k = 0; k < s->n_adapters; ++k) {
    const lt_adapter* a = &b->adapters[s->adapter_offset + k];
    ads[k].id = a->adapter_id;
    ads[k].rank = a->rank;
    ads[k].rate = a->rate;
    ads[k].len = a->length_index >= 0 ? len_of(&b->lengths[a->length_index], b->full_lengths) : wl;
  }
  Req* req = NULL;
  int64_t n = 0;
  int ok = 1;
  char db[64];
  if (s->n_requests < 0) {
    /* WorkloadSpec::validate(for_simulation) (workload.cpp:118-141) */
    if (s->n_adapters <= 0) ok = err_set(&e, LT_ERR_VALIDATION, "workload.adapters: must be non-empty");
    else if (s->duration_s <= 0.0)
      ok = err_set(&e, LT_ERR_VALIDATION, "workload.duration_s: must be > 0, got %s", f6(s->duration_s, db));
    for (int k = 0; ok && k < s->n_adapters; ++k) {
      char path[64];
      snprintf(path, sizeof(path), "workload.adapters[%d]", k);
      if (ads[k].rank < 0) ok = err_set(&e, LT_ERR_VALIDATION, "%s.rank: must be >= 0, got %d", path, ads[k].rank);
      else if (ads[k].rate <= 0.0)
        ok = err_set(&e, LT_ERR_VALIDATION, "%s.rate: must be > 0, got %s", path, f6(ads[k].rate, db));
      else {
        for (int j = 0; j < k && ok; ++j)
          if (ads[j].id == ads[k].id)
            ok = err_set(&e, LT_ERR_VALIDATION, "%s.adapter_id: duplicate id %d", path, ads[k].id);
        const lt_adapter* a = &b->adapters[s->adapter_offset + k];
        if (ok && a->length_index >= 0) {
          char p2[80];
          snprintf(p2, sizeof(p2), "%s.lengths", path);
          ok = validate_len(&ads[k].len, p2, &e);
        }
      }
    }
    if (ok) ok = validate_len(&wl, "workload.lengths", &e);
    if (ok) {
      n = generate_arrivals(ads, s->n_adapters, &wl, s->duration_s, s->seed, s->mode, &req, &e);
      if (n < 0) ok = 0;
    }
  } else {
    n = s->n_requests;
    req = (Req*)malloc(sizeof(Req) * (size_t)(n > 0 ? n : 1));
    for (int64_t k = 0; k < n; ++k) {
      const lt_request* q = &b->requests[s->request_offset + k];
      req[k].id = q->request_id;
      req[k].adapter = q->adapter_id;
      req[k].t = q->arrival_time_s;
      req[k].in = q->input_tokens;
      req[k].out = q->output_tokens;
    }
  }
  if (J->arrivals_only) {
    J->gen[i] = ok ? req : NULL;
    J->gen_n[i] = ok ? n : 0;
    if (!ok) {
      free(req);
      o->status = e.code;
      snprintf(g_msgs[i], 320, "%s", e.msg);
    }
    free(ads);
    return;
  }
  /* Engine::Engine (engine.cpp:32-71) */
  if (ok) ok = validate_config(J->c, G, &e);
  if (ok && s->n_adapters <= 0) ok = err_set(&e, LT_ERR_VALIDATION, "workload.adapters: must be non-empty");
  if (ok && s->duration_s <= 0.0) ok = err_set(&e, LT_ERR_VALIDATION, "workload.duration_s: must be > 0");
  if (ok) {
    for (int k = 0; k < s->n_adapters && ok; ++k)
      for (int j = 0; j < k && ok; ++j)
        if (ads[j].id == ads[k].id) ok = err_set(&e, LT_ERR_VALIDATION, "workload.adapters: duplicate adapter_id");
  }
  if (ok && s->n_requests >= 0) {
    /* rank check via mem_max happens in simulate(); request checks after it (engine.cpp:56-69) */
  }
  if (ok) {
    double ideal = 0.0; /* ideal_throughput (metrics.cpp:36-45) */
    for (int k = 0; k < s->n_adapters; ++k) {
      double tok = len_out_mean(&ads[k].len);
      if (J->c->ideal_includes_input) tok += len_in_mean(&ads[k].len);
      ideal += ads[k].rate * tok;
    }
    if (s->n_requests >= 0) {
      /* Engine ctor order: mem_max first, then per-request checks */
      int max_rank = 0;
      for (int k = 0; k < s->n_adapters; ++k)
        if (ads[k].rank > max_rank) max_rank = ads[k].rank;
      int64_t cap = J->c->total_kv_budget, sc;
      for (int g = 0; g < G && ok; ++g) {
        ok = slot_cost(J->c, max_rank, &sc, &e);
        cap -= sc;
      }
      if (ok && cap <= 0)
        ok = err_set(&e, LT_ERR_CONFIG, "infeasible configuration: %d slots consume the entire KV budget (mem_max = 0)", G);
      for (int64_t k = 0; ok && k < n; ++k) {
        if (req[k].id != k)
          ok = err_set(&e, LT_ERR_VALIDATION, "requests must be sorted with request_id = position, got id %lld at position %lld",
                       (long long)req[k].id, (long long)k);
        else {
          int found = 0;
          for (int a = 0; a < s->n_adapters; ++a) found |= ads[a].id == req[k].adapter;
          if (!found)
            ok = err_set(&e, LT_ERR_VALIDATION, "request %lld references unknown adapter %d", (long long)req[k].id,
                         req[k].adapter);
        }
      }
    }
    if (ok) {
      simulate(J->c, G, ads, s->n_adapters, s->duration_s, req, n, ideal, o, &e, J->o ? J->o->want_digest : 0,
               J->o ? J->o->iteration_cap_override : 0, NULL, 0);
      if (o->status != LT_OK) ok = 0;
    }
  }
  if (!ok) {
    o->status = e.code;
    o->status_kind = LT_K_MESSAGE;
    snprintf(g_msgs[i], 320, "%s", e.msg);
  }
  free(req);
  free(ads);
}

void ltor_set_threads(int32_t n) { g_threads = n < 1 ? 1 : n; }

int32_t ltor_message(int64_t index, char* buf, size_t len) {
  if (index < 0 || index >= g_nmsgs) return -1;
  snprintf(buf, len, "%s", g_msgs[index]);
  return 0;
}

int32_t ltor_simulate_batch(void* ctx, const lt_workload_batch* b, const lt_server_config* c, const lt_sim_options* o,
                            lt_sim_summary* out, lt_request_states* states, lt_status* st) {
  (void)ctx;
  msgs_reset(b->n_scenarios);
  SimJob J;
  memset(&J, 0, sizeof(J));
  J.b = b;
  J.c = c;
  J.o = o;
  J.out = out;
  if (states) {
    /* sequential, with per-request states (oracle path for small cases) */
    int64_t off = 0;
    for (int64_t i = 0; i < b->n_scenarios; ++i) {
      sim_task(&J, i);
      if (states->req_offset) states->req_offset[i] = off;
      off += out[i].n_requests;
    }
    /* re-run with state capture (simulate() fills states directly) */
    off = 0;
    for (int64_t i = 0; i < b->n_scenarios; ++i) {
      const lt_scenario* s = &b->scenarios[i];
      if (out[i].status != LT_OK) continue;
      const int G = s->slots > 0 ? s->slots : c->slots;
      Adp* ads = (Adp*)malloc(sizeof(Adp) * (size_t)s->n_adapters);
      const Len wl = len_of(&b->lengths[s->length_index], b->full_lengths);
      for (int k = 0; k < s->n_adapters; ++k) {
        const lt_adapter* a = &b->adapters[s->adapter_offset + k];
        ads[k].id = a->adapter_id;
        ads[k].rank = a->rank;
        ads[k].rate = a->rate;
        ads[k].len = a->length_index >= 0 ? len_of(&b->lengths[a->length_index], b->full_lengths) : wl;
      }
      Req* req = NULL;
      int64_t n;
      Err e;
      memset(&e, 0, sizeof(e));
      if (s->n_requests < 0) {
        n = generate_arrivals(ads, s->n_adapters, &wl, s->duration_s, s->seed, s->mode, &req, &e);
      } else {
        n = s->n_requests;
        req = (Req*)malloc(sizeof(Req) * (size_t)(n > 0 ? n : 1));
        for (int64_t k = 0; k < n; ++k) {
          const lt_request* q = &b->requests[s->request_offset + k];
          req[k].id = q->request_id;
          req[k].adapter = q->adapter_id;
          req[k].t = q->arrival_time_s;
          req[k].in = q->input_tokens;
          req[k].out = q->output_tokens;
        }
      }
      lt_sim_summary tmp;
      simulate(c, G, ads, s->n_adapters, s->duration_s, req, n, out[i].ideal_throughput_tok_s, &tmp, &e,
               o ? o->want_digest : 0, o ? o->iteration_cap_override : 0, states, states->req_offset ? states->req_offset[i] : off);
      off += n;
      free(req);
      free(ads);
    }
  } else {
    run_pool(b->n_scenarios, sim_task, &J);
  }
  if (st) {
    memset(st, 0, sizeof(*st));
    st->index = -1;
    for (int64_t i = 0; i < b->n_scenarios; ++i)
      if (out[i].status != LT_OK) {
        st->code = out[i].status;
        st->kind = LT_K_MESSAGE;
        st->index = i;
        snprintf(st->message, sizeof(st->message), "%s", g_msgs[i]);
        break;
      }
  }
  return st ? st->code : 0;
}

int32_t ltor_generate_arrivals_batch(void* ctx, const lt_workload_batch* b, const lt_sim_options* o, lt_request* out,
                                     int64_t capacity, int64_t* offsets, int64_t* counts, lt_status* st) {
  (void)ctx;
  (void)o;
  msgs_reset(b->n_scenarios);
  SimJob J;
  memset(&J, 0, sizeof(J));
  J.b = b;
  J.arrivals_only = 1;
  J.gen = (Req**)calloc((size_t)(b->n_scenarios > 0 ? b->n_scenarios : 1), sizeof(Req*));
  J.gen_n = (int64_t*)calloc((size_t)(b->n_scenarios > 0 ? b->n_scenarios : 1), sizeof(int64_t));
  lt_sim_summary* tmp = (lt_sim_summary*)calloc((size_t)(b->n_scenarios > 0 ? b->n_scenarios : 1), sizeof(lt_sim_summary));
  J.out = tmp;
  run_pool(b->n_scenarios, sim_task, &J);
  int64_t off = 0;
  if (st) {
    memset(st, 0, sizeof(*st));
    st->index = -1;
  }
  for (int64_t i = 0; i < b->n_scenarios; ++i) {
    offsets[i] = off;
    counts[i] = J.gen_n[i];
    if (tmp[i].status != LT_OK && st && st->code == LT_OK) {
      st->code = tmp[i].status;
      st->index = i;
      snprintf(st->message, sizeof(st->message), "%s", g_msgs[i]);
    }
    for (int64_t k = 0; k < J.gen_n[i]; ++k, ++off) {
      if (off >= capacity) continue;
      out[off].request_id = J.gen[i][k].id;
      out[off].adapter_id = J.gen[i][k].adapter;
      out[off].input_tokens = J.gen[i][k].in;
      out[off].output_tokens = J.gen[i][k].out;
      out[off]._pad = 0;
      out[off].arrival_time_s = J.gen[i][k].t;
    }
    free(J.gen[i]);
  }
  free(J.gen);
  free(J.gen_n);
  free(tmp);
  return st ? st->code : 0;
}

/* ------------------------------------------------------------------ sweep */
typedef struct {
  const lt_condition_batch* b;
  const lt_server_config* c;
  const lt_sweep_grid* g;
  double dur;
  uint64_t seed;
  const lt_sweep_options* so;
  lt_placement* out;
  lt_frontier_point* fr;
  int32_t maxf;
} SweepJob;

static int g_cands(const lt_sweep_grid* g, int n, int* gs) { /* placement.cpp:159-167 */
  int cand[64], nc = 0, m = 0;
  if (g->g_mode == LT_G_GEOMETRIC) {
    cand[0] = 8;
    cand[1] = n / 4;
    cand[2] = n / 2;
    cand[3] = n;
    nc = 4;
  } else {
    for (int i = 0; i < g->g_count && i < 64; ++i) cand[nc++] = g->g_values[i];
  }
  for (int i = 0; i < nc; ++i) {
    int v = cand[i] < 1 ? 1 : (cand[i] > n ? n : cand[i]);
    int dup = 0;
    for (int j = 0; j < m; ++j) dup |= gs[j] == v;
    if (!dup) gs[m++] = v;
  }
  qsort(gs, (size_t)m, sizeof(int), cmp_int);
  return m;
}

static void sweep_task(void* vctx, int64_t ci) {
  SweepJob* J = (SweepJob*)vctx;
  const lt_condition* cd = &J->b->conditions[ci];
  lt_placement* P = &J->out[ci];
  memset(P, 0, sizeof(*P));
  P->status_point = -1;
  lt_frontier_point* fr = J->fr + ci * J->maxf;
  Err e;
  memset(&e, 0, sizeof(e));
  const lt_sweep_grid* g = J->g;
  int ok = 1;
  /* SweepGrid::validate (placement.cpp:169-183) */
  if (g->n_count <= 0) ok = err_set(&e, LT_ERR_VALIDATION, "grid.n_values: must be non-empty");
  for (int i = 0; ok && i < g->n_count; ++i) {
    if (g->n_values[i] < 1) ok = err_set(&e, LT_ERR_VALIDATION, "grid.n_values: entries must be >= 1");
    else if (i > 0 && g->n_values[i] <= g->n_values[i - 1])
      ok = err_set(&e, LT_ERR_VALIDATION, "grid.n_values: must be strictly ascending");
  }
  if (ok && g->g_mode == LT_G_EXPLICIT) {
    if (g->g_count <= 0) ok = err_set(&e, LT_ERR_VALIDATION, "grid.g_values: must be non-empty in explicit mode");
    for (int i = 0; ok && i < g->g_count; ++i)
      if (g->g_values[i] < 1) ok = err_set(&e, LT_ERR_VALIDATION, "grid.g_values: entries must be >= 1");
  }
  const Len L = len_of(&J->b->lengths[cd->length_index], J->b->full_lengths);
  if (ok) ok = validate_len(&L, "condition.lengths", &e);
  if (ok && cd->mix_count <= 0) ok = err_set(&e, LT_ERR_VALIDATION, "condition.mix: must be non-empty");
  if (!ok) {
    P->status = e.code;
    snprintf(g_msgs[ci], 320, "%s", e.msg);
    return;
  }
  /* sweep_optimal (placement.cpp:185-264) */
  double best = -1.0, first_best = -1.0;
  int best_n = 0, best_g = 0, first_g = 0, any_non = 0, any_st = 0, stall = 0, nf = 0;
  int stop = g->n_count;
  for (int ni = 0; ni < g->n_count; ++ni) {
    const int n = g->n_values[ni];
    int gs[64];
    const int m = g_cands(g, n, gs);
    lt_sim_summary res[64];
    /* instantiate_condition (placement.cpp:139-157) */
    Adp* ads = (Adp*)malloc(sizeof(Adp) * (size_t)n);
    for (int k = 0; k < n; ++k) {
      const lt_template* t = &J->b->templates[cd->mix_offset + (k % cd->mix_count)];
      ads[k].id = k + 1;
      ads[k].rank = t->rank;
      ads[k].rate = t->rate;
      ads[k].len = L;
    }
    int row_err = -1;
    for (int gi = 0; gi < m; ++gi) {
      Err pe;
      memset(&pe, 0, sizeof(pe));
      memset(&res[gi], 0, sizeof(res[gi]));
      int pok = 1;
      char db[64];
      for (int k = 0; pok && k < n; ++k) {
        char path[64];
        snprintf(path, sizeof(path), "workload.adapters[%d]", k);
        if (ads[k].rank < 0) pok = err_set(&pe, LT_ERR_VALIDATION, "%s.rank: must be >= 0, got %d", path, ads[k].rank);
        else if (ads[k].rate <= 0.0)
          pok = err_set(&pe, LT_ERR_VALIDATION, "%s.rate: must be > 0, got %s", path, f6(ads[k].rate, db));
      }
      Req* req = NULL;
      int64_t nr = 0;
      if (pok) {
        nr = generate_arrivals(ads, n, &L, J->dur, J->seed, J->so->mode, &req, &pe);
        if (nr < 0) pok = 0;
      }
      if (pok) pok = validate_config(J->c, gs[gi], &pe);
      if (pok) {
        double ideal = 0.0;
        for (int k = 0; k < n; ++k) {
          double tok = len_out_mean(&ads[k].len);
          if (J->c->ideal_includes_input) tok += len_in_mean(&ads[k].len);
          ideal += ads[k].rate * tok;
        }
        simulate(J->c, gs[gi], ads, n, J->dur, req, nr, ideal, &res[gi], &pe, 0, 0, NULL, 0);
        if (res[gi].status != LT_OK) pok = 0;
      }
      free(req);
      if (!pok) {
        res[gi].status = pe.code;
        if (row_err < 0) {
          row_err = gi;
          snprintf(g_msgs[ci], 320, "%s", pe.msg);
        }
      }
    }
    free(ads);
    if (row_err >= 0) { /* run_parallel rethrows the lowest index */
      P->status = res[row_err].status;
      P->frontier_count = 0;
      return;
    }
    int improved = 0;
    for (int gi = 0; gi < m; ++gi) {
      const double t = res[gi].throughput_tok_s;
      const int starved = res[gi].starved;
      if (nf < J->maxf) {
        fr[nf].n = n;
        fr[nf].g = gs[gi];
        fr[nf].throughput_tok_s = t;
        fr[nf].starved = starved;
        fr[nf].skipped = 0;
      }
      nf++;
      P->points_simulated++;
      P->iterations += res[gi].iterations;
      if (starved) any_st = 1;
      if (!starved) {
        any_non = 1;
        if (t > best) {
          best = t;
          best_n = n;
          best_g = gs[gi];
          improved = 1;
        }
      }
      if (ni == 0 && t > first_best) {
        first_best = t;
        first_g = gs[gi];
      }
    }
    if (J->so->early_exit) {
      stall = improved ? 0 : stall + 1;
      if (stall >= J->so->early_exit_k && ni + 1 < g->n_count) {
        stop = ni + 1;
        break;
      }
    }
  }
  for (int ni = stop; ni < g->n_count; ++ni) {
    if (nf < J->maxf) {
      fr[nf].n = g->n_values[ni];
      fr[nf].g = 0;
      fr[nf].throughput_tok_s = 0.0;
      fr[nf].starved = 0;
      fr[nf].skipped = 1;
    }
    nf++;
  }
  P->frontier_count = nf;
  if (!any_non) {
    P->all_starved = 1;
    P->n_star = g->n_values[0];
    P->g_star = first_g;
    P->max_throughput_tok_s = first_best < 0.0 ? 0.0 : first_best;
    return;
  }
  P->max_throughput_tok_s = best;
  P->n_star = best_n;
  P->g_star = best_g;
  P->frontier_open = !any_st && best_n == g->n_values[stop - 1];
}

int32_t ltor_sweep_batch(void* ctx, const lt_condition_batch* b, const lt_server_config* c, const lt_sweep_grid* g,
                         double duration_s, uint64_t seed, const lt_sweep_options* so, const lt_sim_options* sim,
                         lt_placement* out, lt_frontier_point* fr, int32_t maxf, lt_status* st) {
  (void)ctx;
  (void)sim;
  msgs_reset(b->n_conditions);
  SweepJob J = {b, c, g, duration_s, seed, so, out, fr, maxf};
  run_pool(b->n_conditions, sweep_task, &J);
  if (st) {
    memset(st, 0, sizeof(*st));
    st->index = -1;
    for (int64_t i = 0; i < b->n_conditions; ++i)
      if (out[i].status != LT_OK) {
        st->code = out[i].status;
        st->index = i;
        snprintf(st->message, sizeof(st->message), "%s", g_msgs[i]);
        break;
      }
  }
  return st ? st->code : 0;
}
