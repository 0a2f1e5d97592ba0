// Host side of the batched generate_dataset: the
// reference's condition enumeration, feature encoding, condition hash, CSV
// format and resume logic (placement.cpp:100-137, :266-527), with the
// per-condition sweeps replaced by batched lt_sweep_batch calls. Included at
// the end of capi.cu (it calls the C-ABI entry points).
#pragma once
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace lt_dataset {

// format_double (placement.cpp:54-58).
inline std::string format_double(double v) {
  char buf[32];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

struct Stats4 {
  double max, min, mean, std;
};

// stats_of (placement.cpp:39-52).
inline Stats4 stats_of(const std::vector<double>& v) {
  Stats4 s{0.0, 0.0, 0.0, 0.0};
  if (v.empty()) return s;
  s.max = v[0];
  s.min = v[0];
  for (double x : v) {
    s.max = std::max(s.max, x);
    s.min = std::min(s.min, x);
  }
  double sum = 0.0;
  for (double x : v) sum += x;
  s.mean = sum / static_cast<double>(v.size());
  double sq = 0.0;
  for (double x : v) {
    const double d = x - s.mean;
    sq += d * d;
  }
  s.std = std::sqrt(sq / static_cast<double>(v.size()));
  return s;
}

// LengthSpec::input_stats / output_stats (workload.cpp:81-89): Full mode uses
// list_stats (workload.cpp:31-50), Mean mode {mean, mean, mean, std}.
inline Stats4 length_stats(const lt_length_spec& l, const int32_t* full, bool input) {
  if (l.mode == LT_MODE_FULL) {
    Stats4 s{0.0, 0.0, 0.0, 0.0};
    if (l.full_count <= 0) return s;
    s.max = std::numeric_limits<double>::lowest();
    s.min = std::numeric_limits<double>::max();
    double sum = 0.0;
    for (int64_t i = 0; i < l.full_count; ++i) {
      const double v = full[2 * (l.full_offset + i) + (input ? 0 : 1)];
      s.max = std::max(s.max, v);
      s.min = std::min(s.min, v);
      sum += v;
    }
    s.mean = sum / static_cast<double>(l.full_count);
    double sq = 0.0;
    for (int64_t i = 0; i < l.full_count; ++i) {
      const double v = full[2 * (l.full_offset + i) + (input ? 0 : 1)];
      sq += (v - s.mean) * (v - s.mean);
    }
    s.std = std::sqrt(sq / static_cast<double>(l.full_count));
    return s;
  }
  const double m = input ? l.mean_input : l.mean_output;
  return Stats4{m, m, m, input ? l.std_input : l.std_output};
}

// encode_workload (placement.cpp:117-137).
inline bool encode(const lt_template* mix, int n_mix, const lt_length_spec& l, const int32_t* full, double* f,
                   std::string* err) {
  if (n_mix <= 0) {
    *err = "condition.mix: must be non-empty";
    return false;
  }
  std::vector<double> rates, ranks;
  for (int i = 0; i < n_mix; ++i) {
    rates.push_back(mix[i].rate);
    ranks.push_back(static_cast<double>(mix[i].rank));
  }
  const Stats4 a = stats_of(rates), b = stats_of(ranks);
  const Stats4 in = length_stats(l, full, true), out = length_stats(l, full, false);
  const double v[16] = {a.max,  a.min,  a.mean,  a.std,  b.max,   b.min,   b.mean,   b.std,
                        in.max, in.min, in.mean, in.std, out.max, out.min, out.mean, out.std};
  for (int i = 0; i < 16; ++i) f[i] = v[i];
  return true;
}

// condition_hash (placement.cpp:266-296).
inline uint64_t condition_hash(const lt_template* mix, int n_mix, const lt_length_spec& l, const int32_t* full,
                               double duration_s, uint64_t seed, const lt_sweep_grid& grid) {
  std::ostringstream canon;
  canon << "v1|mix=";
  for (int i = 0; i < n_mix; ++i) canon << mix[i].rank << ':' << format_double(mix[i].rate) << ',';
  canon << "|lengths=";
  if (l.mode == LT_MODE_FULL) {
    canon << "full:";
    for (int64_t i = 0; i < l.full_count; ++i)
      canon << full[2 * (l.full_offset + i)] << '/' << full[2 * (l.full_offset + i) + 1] << ',';
  } else {
    canon << "mean:" << format_double(l.mean_input) << ',' << format_double(l.std_input) << ','
          << format_double(l.mean_output) << ',' << format_double(l.std_output);
  }
  canon << "|dur=" << format_double(duration_s) << "|seed=" << seed << "|n=";
  for (int i = 0; i < grid.n_count; ++i) canon << grid.n_values[i] << ',';
  canon << "|g=" << (grid.g_mode == LT_G_GEOMETRIC ? "geo" : "exp") << ':';
  if (grid.g_mode == LT_G_EXPLICIT)
    for (int i = 0; i < grid.g_count; ++i) canon << grid.g_values[i] << ',';
  uint64_t h = 0xcbf29ce484222325ull;
  for (unsigned char c : canon.str()) {
    h ^= c;
    h *= 0x100000001b3ull;
  }
  return h;
}

constexpr const char* kFeatureNames[16] = {
    "rate_max",      "rate_min",      "rate_mean",      "rate_std",      "rank_max",       "rank_min",
    "rank_mean",     "rank_std",      "input_len_max",  "input_len_min", "input_len_mean", "input_len_std",
    "output_len_max", "output_len_min", "output_len_mean", "output_len_std"};

// write_dataset_header (placement.cpp:342-345).
inline std::string header_line() {
  std::string h;
  for (const char* n : kFeatureNames) h += std::string(n) + ',';
  return h + "max_throughput,n_star,g_star,all_starved,condition_hash,duration_s,seed\n";
}

struct Row {
  double f[16];
  double max_tput;
  int n_star, g_star;
  bool all_starved;
  uint64_t hash;
  double duration_s;
  uint64_t seed;
};

// write_dataset_row (placement.cpp:347-352).
inline std::string row_line(const Row& r) {
  std::string s;
  for (double v : r.f) s += format_double(v) + ',';
  s += format_double(r.max_tput) + ',' + std::to_string(r.n_star) + ',' + std::to_string(r.g_star) + ',' +
       (r.all_starved ? "1" : "0") + ',' + std::to_string(r.hash) + ',' + format_double(r.duration_s) + ',' +
       std::to_string(r.seed) + '\n';
  return s;
}

struct Fail {
  std::string msg;
};

// std::stod / stoi / stoull as read_dataset_csv uses them: leading
// whitespace and a valid prefix parse; no digits or out of range throws.
inline double parse_d(const std::string& f) {
  errno = 0;
  char* end = nullptr;
  const double v = std::strtod(f.c_str(), &end);
  if (end == f.c_str() || errno == ERANGE) throw Fail{};
  return v;
}
inline int parse_i(const std::string& f) {
  errno = 0;
  char* end = nullptr;
  const long v = std::strtol(f.c_str(), &end, 10);
  if (end == f.c_str() || errno == ERANGE || v < INT32_MIN || v > INT32_MAX) throw Fail{};
  return static_cast<int>(v);
}
inline unsigned long long parse_u(const std::string& f) {
  errno = 0;
  char* end = nullptr;
  const unsigned long long v = std::strtoull(f.c_str(), &end, 10);
  if (end == f.c_str() || errno == ERANGE) throw Fail{};
  return v;
}

// read_dataset_csv (placement.cpp:367-413): the hashes of the rows on disk.
// Returns false with the reference's ValidationError text on failure.
inline bool read_hashes(const std::string& path, std::set<uint64_t>* done, std::string* err) {
  std::ifstream in(path);
  if (!in) {
    *err = "cannot open dataset CSV: " + path;
    return false;
  }
  std::string line;
  if (!std::getline(in, line)) {
    *err = "empty dataset CSV: " + path;
    return false;
  }
  std::string want = header_line();
  want.pop_back();
  if (line != want) {
    *err = "dataset CSV header mismatch in " + path + " (got \"" + line + "\")";
    return false;
  }
  size_t line_no = 1;
  while (std::getline(in, line)) {
    ++line_no;
    if (line.empty()) continue;
    std::vector<std::string> fields;
    {
      std::string field;
      std::istringstream ls(line);
      while (std::getline(ls, field, ',')) fields.push_back(field);
      if (!line.empty() && line.back() == ',') fields.push_back("");
    }
    if (fields.size() != 23) {
      if (in.eof()) break;  // torn final line of an interrupted run
      *err = path + ":" + std::to_string(line_no) + ": expected 23 columns, got " + std::to_string(fields.size());
      return false;
    }
    try {
      for (int i = 0; i < 16; ++i) parse_d(fields[i]);
      parse_d(fields[16]);
      parse_i(fields[17]);
      parse_i(fields[18]);
      parse_i(fields[19]);
      const uint64_t h = parse_u(fields[20]);
      parse_d(fields[21]);
      parse_u(fields[22]);
      done->insert(h);
    } catch (const Fail&) {
      *err = path + ":" + std::to_string(line_no) + ": unparsable numeric field";
      return false;
    }
  }
  return true;
}

// enumerate_conditions (placement.cpp:298-340): size-k non-decreasing index
// tuples of rates x ranks in lexicographic order, every stride-th kept.
inline std::vector<std::vector<size_t>> combos(size_t n_values, int k) {
  std::vector<std::vector<size_t>> out;
  std::vector<size_t> idx(static_cast<size_t>(k), 0);
  for (;;) {
    out.push_back(idx);
    int pos = k - 1;
    while (pos >= 0 && idx[static_cast<size_t>(pos)] == n_values - 1) --pos;
    if (pos < 0) break;
    const size_t bumped = ++idx[static_cast<size_t>(pos)];
    for (size_t j = static_cast<size_t>(pos) + 1; j < idx.size(); ++j) idx[j] = bumped;
  }
  return out;
}

}  // namespace lt_dataset

extern "C" {

uint64_t lt_condition_hash(const lt_template* mix, int32_t n_mix, const lt_length_spec* lengths,
                           const int32_t* full_lengths, double duration_s, uint64_t seed,
                           const lt_sweep_grid* grid) {
  return lt_dataset::condition_hash(mix, n_mix, *lengths, full_lengths, duration_s, seed, *grid);
}

int32_t lt_encode_workload(const lt_template* mix, int32_t n_mix, const lt_length_spec* lengths,
                           const int32_t* full_lengths, double* features16, lt_status* status) {
  ok_status(status);
  std::string err;
  if (!lt_dataset::encode(mix, n_mix, *lengths, full_lengths, features16, &err)) {
    set_status(status, LT_ERR_VALIDATION, LT_K_VALIDATION_MSG, -1, 0, 0, err);
    return LT_ERR_VALIDATION;
  }
  return LT_OK;
}

int32_t lt_generate_dataset(lt_ctx* ctx, const lt_dataset_spec* spec, const lt_server_config* config,
                            const char* out_csv, lt_error_fn on_error, void* user,
                            lt_dataset_progress* progress, lt_status* status) {
  namespace D = lt_dataset;
  ok_status(status);
  lt_dataset_progress prog{0, 0, 0};
  auto fail = [&](int32_t code, const std::string& msg) {
    set_status(status, code, LT_K_VALIDATION_MSG, -1, 0, 0, msg);
    if (progress) *progress = prog;
    return code;
  };
  // spec.grid.validate() (placement.cpp:169-183), then enumerate_conditions'
  // own checks (placement.cpp:298-302)
  const lt_sweep_grid& grid = spec->grid;
  if (grid.n_count <= 0) return fail(LT_ERR_VALIDATION, "grid.n_values: must be non-empty");
  for (int i = 0; i < grid.n_count; ++i) {
    if (grid.n_values[i] < 1) return fail(LT_ERR_VALIDATION, "grid.n_values: entries must be >= 1");
    if (i > 0 && grid.n_values[i] <= grid.n_values[i - 1])
      return fail(LT_ERR_VALIDATION, "grid.n_values: must be strictly ascending");
  }
  if (grid.g_mode == LT_G_EXPLICIT) {
    if (grid.g_count <= 0) return fail(LT_ERR_VALIDATION, "grid.g_values: must be non-empty in explicit mode");
    for (int i = 0; i < grid.g_count; ++i)
      if (grid.g_values[i] < 1) return fail(LT_ERR_VALIDATION, "grid.g_values: entries must be >= 1");
  }
  if (spec->triple_size < 1) return fail(LT_ERR_VALIDATION, "dataset.triple_size: must be >= 1");
  if (spec->n_rates <= 0) return fail(LT_ERR_VALIDATION, "dataset.rates: must be non-empty");
  if (spec->n_ranks <= 0) return fail(LT_ERR_VALIDATION, "dataset.ranks: must be non-empty");
  if (spec->condition_stride < 1) return fail(LT_ERR_VALIDATION, "dataset.condition_stride: must be >= 1");
  const int k = spec->triple_size;
  const auto rt = D::combos(static_cast<size_t>(spec->n_rates), k);
  const auto kt = D::combos(static_cast<size_t>(spec->n_ranks), k);
  std::vector<lt_template> tmpl;
  std::vector<lt_condition> conds;
  size_t counter = 0;
  for (const auto& r : rt)
    for (const auto& q : kt) {
      if (counter++ % static_cast<size_t>(spec->condition_stride) != 0) continue;
      conds.push_back(lt_condition{static_cast<int64_t>(tmpl.size()), k, 0});
      for (int leg = 0; leg < k; ++leg)
        tmpl.push_back(lt_template{spec->ranks[q[static_cast<size_t>(leg)]], 0, spec->rates[r[static_cast<size_t>(leg)]]});
    }
  prog.total_conditions = static_cast<int64_t>(conds.size());
  if (conds.empty()) {
    if (on_error) on_error("empty condition grid; nothing to do", user);
    if (progress) *progress = prog;
    return LT_OK;
  }
  // resume: hashes on disk, torn tail truncated (placement.cpp:428-451)
  const std::string path(out_csv);
  std::set<uint64_t> done;
  bool file_exists = false;
  {
    std::ifstream in(path, std::ios::binary);
    if (in) {
      file_exists = true;
      std::string err;
      if (!D::read_hashes(path, &done, &err)) return fail(LT_ERR_VALIDATION, "resume failed: " + err);
      const std::string content((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
      const size_t nl = content.rfind('\n');
      const size_t keep = nl == std::string::npos ? 0 : nl + 1;
      if (keep < content.size()) {
        in.close();
        std::filesystem::resize_file(path, keep);
      }
    }
  }
  std::ofstream out(path, std::ios::app);
  if (!out) return fail(LT_ERR_VALIDATION, "cannot open dataset CSV for writing: " + path);
  if (!file_exists) out << D::header_line();
  // pending conditions -> batched sweeps (chunks bound host + device memory)
  std::vector<uint64_t> hash(conds.size());
  std::vector<int64_t> pending;
  for (size_t i = 0; i < conds.size(); ++i) {
    hash[i] = D::condition_hash(tmpl.data() + conds[i].mix_offset, k, spec->lengths, spec->full_lengths,
                                spec->duration_s, spec->seed, grid);
    if (!done.count(hash[i])) pending.push_back(static_cast<int64_t>(i));
  }
  std::vector<lt_placement> place(conds.size());
  std::vector<std::string> errs(conds.size());
  const int32_t F = lt_sweep_frontier_capacity(&grid);
  lt_sweep_options so = spec->sweep;
  so.jobs = 1;
  constexpr size_t kChunk = 8192;
  for (size_t c0 = 0; c0 < pending.size(); c0 += kChunk) {
    const size_t nc = std::min(kChunk, pending.size() - c0);
    std::vector<lt_condition> sub(nc);
    for (size_t j = 0; j < nc; ++j) sub[j] = conds[static_cast<size_t>(pending[c0 + j])];
    lt_length_spec ls = spec->lengths;
    lt_condition_batch cb{sub.data(), static_cast<int64_t>(nc), tmpl.data(), static_cast<int64_t>(tmpl.size()),
                          &ls, 1, spec->full_lengths, spec->n_full_pairs};
    std::vector<lt_placement> po(nc);
    std::vector<lt_frontier_point> fr(nc * static_cast<size_t>(std::max(F, 1)));
    lt_status st{};
    const int32_t rc = lt_sweep_batch(ctx, &cb, config, &grid, spec->duration_s, spec->seed, &so, nullptr,
                                      po.data(), fr.data(), F, &st);
    if (rc == LT_ERR_DEVICE) {
      if (status) *status = st;
      if (progress) *progress = prog;
      return rc;
    }
    for (size_t j = 0; j < nc; ++j) {
      const size_t i = static_cast<size_t>(pending[c0 + j]);
      place[i] = po[j];
      if (po[j].status != LT_OK) errs[i] = ctx->messages[j];
    }
  }
  // rows in canonical order (placement.cpp:468-485)
  for (size_t i = 0; i < conds.size(); ++i) {
    if (done.count(hash[i])) {
      ++prog.completed;
      continue;
    }
    const lt_placement& p = place[i];
    D::Row row{};
    std::string err;
    if (p.status == LT_OK &&
        D::encode(tmpl.data() + conds[i].mix_offset, k, spec->lengths, spec->full_lengths, row.f, &err)) {
      row.max_tput = p.max_throughput_tok_s;
      row.n_star = p.n_star;
      row.g_star = p.g_star;
      row.all_starved = p.all_starved != 0;
      row.hash = hash[i];
      row.duration_s = spec->duration_s;
      row.seed = spec->seed;
      out << D::row_line(row);
      out.flush();
      ++prog.completed;
    } else {
      ++prog.failed;
      const std::string what = p.status != LT_OK ? errs[i] : err;
      if (on_error)
        on_error(("condition " + std::to_string(i) + " (hash " + std::to_string(hash[i]) + "): " + what).c_str(),
                 user);
    }
  }
  if (progress) *progress = prog;
  return LT_OK;
}

}  // extern "C"
