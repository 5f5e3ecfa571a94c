// TEST INFRASTRUCTURE ONLY (oracle). Exposes the UNMODIFIED reference planner
// (/root/reference/proj/include/mimose, compiled from where it lies by
// oracle/Makefile into oracle/_ref/libmimose_ref.so) over the same C ABI as
// the product's include/mimose_planner.h, with the prefix `ref_planner_`, so
// tests can diff product plans / fits / simulations against the reference.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
// load it.
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "mimose/mimose.hpp"  // resolved to the REFERENCE include dir by oracle/Makefile

extern "C" {
typedef struct {
  int64_t budget_bytes;
  int64_t reserve_bytes;
  double bucket_tolerance;
  double cache_tolerance;
  int excess_includes_constant;
} ref_sched_cfg;
}

namespace {

thread_local std::string err;

char* to_c(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

template <typename Fn>
int run(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::exception& e) {
    err = e.what();
    return 1;
  }
}

std::vector<mimose::CollectedSample> read_csv(const char* text) {
  std::vector<mimose::CollectedSample> v;
  std::istringstream in(text ? text : "");
  std::string row;
  while (std::getline(in, row)) {
    if (!row.empty() && row.back() == '\r') row.pop_back();
    if (row.empty() || row.rfind("layer_id", 0) == 0) continue;
    std::stringstream rs(row);
    std::string a, b, c, d, e;
    std::getline(rs, a, ',');
    std::getline(rs, b, ',');
    std::getline(rs, c, ',');
    std::getline(rs, d, ',');
    std::getline(rs, e, ',');
    mimose::CollectedSample s;
    s.layer_id = static_cast<int>(mimose::detail::parse_int(a, "layer_id"));
    s.input_size = mimose::detail::parse_int(b, "input_size");
    s.measured_activation_bytes = mimose::detail::parse_int(c, "bytes");
    s.measured_forward_ms = mimose::detail::parse_double(d, "ms");
    s.valid = mimose::detail::parse_int(e, "valid") != 0;
    v.push_back(s);
  }
  return v;
}

mimose::SchedulerConfig sched_of(const ref_sched_cfg* c) {
  mimose::SchedulerConfig s;
  s.budget_bytes = c->budget_bytes;
  s.reserve_bytes = c->reserve_bytes;
  s.bucket_tolerance = c->bucket_tolerance;
  s.cache_tolerance = c->cache_tolerance;
  s.excess_includes_constant = c->excess_includes_constant != 0;
  return s;
}

}  // namespace

extern "C" {

const char* ref_planner_last_error(void) { return err.c_str(); }
void ref_planner_free(char* s) { std::free(s); }

int ref_planner_fit(const char* csv, int order, char** out) {
  return run([&] { *out = to_c(mimose::estimator_to_string(mimose::fit(read_csv(csv), order))); });
}

int ref_planner_plan_sequence(const char* est_text, const char* model_text,
                              const ref_sched_cfg* cfg, const int64_t* xs, int n,
                              uint64_t* masks, int words, int* insufficient, int* hits) {
  return run([&] {
    const auto est = mimose::estimator_from_string(est_text);
    const auto model = mimose::load_model_from_string(model_text);
    const auto sc = sched_of(cfg);
    mimose::PlanCache cache;
    for (int i = 0; i < n; ++i) {
      const auto res = mimose::lookup_or_plan(cache, est, model, xs[i], sc);
      for (int w = 0; w < words; ++w) masks[i * words + w] = 0;
      for (int id : res.first.dropped_layers) masks[i * words + id / 64] |= 1ULL << (id % 64);
      insufficient[i] = res.first.insufficient_budget;
      hits[i] = res.second;
    }
  });
}

int ref_planner_simulate(const char* model_text, const int* dropped, int nd, int64_t x,
                         int64_t* peak, double* it_ms, double* rc_ms) {
  return run([&] {
    mimose::CheckpointPlan p;
    for (int i = 0; i < nd; ++i) p.dropped_layers.push_back(dropped[i]);
    p.normalize();
    const auto tl = mimose::simulate_iteration(mimose::load_model_from_string(model_text), p, x);
    *peak = tl.peak_bytes;
    *it_ms = tl.iteration_time_ms;
    *rc_ms = tl.recompute_time_ms;
  });
}

int ref_planner_sample_workload(const char* dist, int64_t mult, int64_t iters, uint64_t seed,
                                int64_t* out) {
  return run([&] {
    auto w = mimose::parse_distribution(dist);
    w.batch_multiplier = mult;
    w.iterations = iters;
    w.seed = seed;
    const auto xs = mimose::sample_workload(w);
    for (size_t i = 0; i < xs.size(); ++i) out[i] = xs[i];
  });
}

int ref_planner_run_experiment(const char* model_text, const char* dist, int64_t mult,
                               int64_t iters, uint64_t seed, const ref_sched_cfg* cfg,
                               const char* planner, char** summary, char** csv) {
  return run([&] {
    auto w = mimose::parse_distribution(dist);
    w.batch_multiplier = mult;
    w.iterations = iters;
    w.seed = seed;
    mimose::ExperimentConfig ec;
    ec.planner = mimose::planner_from_string(planner);
    ec.sched = sched_of(cfg);
    const auto rep = mimose::run_experiment(mimose::load_model_from_string(model_text), w, ec);
    std::ostringstream s, c;
    mimose::write_report_summary(rep, s);
    mimose::write_report_csv(rep, c);
    std::istringstream lines(s.str());
    std::string kept;
    for (std::string line; std::getline(lines, line);) {
      if (line.rfind("planner_wall_ms", 0) == 0 || line.rfind("fit_wall_ms", 0) == 0 ||
          line.rfind("overhead_iterations", 0) == 0)
        continue;
      kept += line + "\n";
    }
    *summary = to_c(kept);
    *csv = to_c(c.str());
  });
}

}  // extern "C"
