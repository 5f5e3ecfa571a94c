// libmimose_host.so: C ABI over the host planner headers (include/mimose).
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "mimose/mimose.hpp"
#include "mimose_planner.h"

namespace {

thread_local std::string g_err;

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

template <typename Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// "layer_id,input_size,bytes,ms,valid" (collector.hpp:198-204)
std::vector<mimose::CollectedSample> parse_samples(const char* csv) {
  std::vector<mimose::CollectedSample> out;
  std::istringstream in(csv ? csv : "");
  std::string line;
  bool header = true;
  while (std::getline(in, line)) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    if (header) {
      header = false;
      if (line.rfind("layer_id", 0) == 0) continue;
    }
    std::vector<std::string> f;
    std::stringstream ls(line);
    std::string cell;
    while (std::getline(ls, cell, ',')) f.push_back(cell);
    if (f.size() != 5) throw mimose::ParseError("bad sample row: '" + line + "'");
    mimose::CollectedSample s;
    s.layer_id = static_cast<int>(mimose::detail::parse_int(f[0], "layer_id"));
    s.input_size = mimose::detail::parse_int(f[1], "input_size");
    s.measured_activation_bytes = mimose::detail::parse_int(f[2], "bytes");
    s.measured_forward_ms = mimose::detail::parse_double(f[3], "ms");
    s.valid = mimose::detail::parse_int(f[4], "valid") != 0;
    out.push_back(s);
  }
  return out;
}

mimose::SchedulerConfig to_sched(const mimose_sched_cfg* c) {
  mimose::SchedulerConfig s;
  s.budget_bytes = c->budget_bytes;
  s.reserve_bytes = c->reserve_bytes;
  s.bucket_tolerance = c->bucket_tolerance;
  s.cache_tolerance = c->cache_tolerance;
  s.excess_includes_constant = c->excess_includes_constant != 0;
  return s;
}

}  // namespace

struct mimose_plan_session {
  mimose::EstimatorModel est;
  mimose::ModelSpec model;
  mimose::SchedulerConfig sched;
  mimose::PlanCache cache;
};

extern "C" {

int mimose_planner_session_create(const char* estimator_text, const char* model_text,
                                  const mimose_sched_cfg* cfg, mimose_plan_session** out) {
  return guard([&] {
    auto* s = new mimose_plan_session();
    try {
      s->est = mimose::estimator_from_string(estimator_text);
      s->model = mimose::load_model_from_string(model_text);
      s->sched = to_sched(cfg);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

int mimose_planner_session_set_estimator(mimose_plan_session* s, const char* estimator_text) {
  return guard([&] { s->est = mimose::estimator_from_string(estimator_text); });
}

int mimose_planner_session_plan(mimose_plan_session* s, int64_t x, int64_t reserve_bytes,
                                uint64_t* dropped_mask, int mask_words, int* insufficient,
                                int* cache_hit) {
  return guard([&] {
    mimose::SchedulerConfig sc = s->sched;
    if (reserve_bytes >= 0) sc.reserve_bytes = reserve_bytes;
    auto [plan, hit] = mimose::lookup_or_plan(s->cache, s->est, s->model, x, sc);
    for (int w = 0; w < mask_words; ++w) dropped_mask[w] = 0;
    for (int id : plan.dropped_layers) {
      if (id < 0 || id >= 64 * mask_words) throw mimose::Error("layer id beyond mask width");
      dropped_mask[id / 64] |= uint64_t{1} << (id % 64);
    }
    *insufficient = plan.insufficient_budget ? 1 : 0;
    *cache_hit = hit ? 1 : 0;
  });
}

int mimose_planner_session_destroy(mimose_plan_session* s) {
  delete s;
  return 0;
}

const char* mimose_planner_last_error(void) { return g_err.c_str(); }
void mimose_planner_free(char* s) { std::free(s); }

int mimose_planner_fit(const char* samples_csv, int order, char** estimator_text) {
  return guard([&] {
    const auto est = mimose::fit(parse_samples(samples_csv), order);
    *estimator_text = dup(mimose::estimator_to_string(est));
  });
}

int mimose_planner_plan_sequence(const char* estimator_text, const char* model_text,
                                 const mimose_sched_cfg* cfg, const int64_t* xs, int n,
                                 uint64_t* dropped_masks, int mask_words, int* insufficient,
                                 int* cache_hit) {
  return guard([&] {
    const auto est = mimose::estimator_from_string(estimator_text);
    const auto model = mimose::load_model_from_string(model_text);
    const auto sched = to_sched(cfg);
    mimose::PlanCache cache;
    for (int i = 0; i < n; ++i) {
      auto [plan, hit] = mimose::lookup_or_plan(cache, est, model, xs[i], sched);
      for (int w = 0; w < mask_words; ++w) dropped_masks[(size_t)i * mask_words + w] = 0;
      for (int id : plan.dropped_layers) {
        if (id < 0 || id >= 64 * mask_words) throw mimose::Error("layer id beyond mask width");
        dropped_masks[(size_t)i * mask_words + id / 64] |= uint64_t{1} << (id % 64);
      }
      insufficient[i] = plan.insufficient_budget ? 1 : 0;
      cache_hit[i] = hit ? 1 : 0;
    }
  });
}

int mimose_planner_simulate(const char* model_text, const int* dropped, int n_dropped,
                            int64_t x, int64_t* peak_bytes, double* iteration_ms,
                            double* recompute_ms) {
  return guard([&] {
    const auto model = mimose::load_model_from_string(model_text);
    mimose::CheckpointPlan plan;
    plan.dropped_layers.assign(dropped, dropped + n_dropped);
    plan.normalize();
    const auto tl = mimose::simulate_iteration(model, plan, x);
    *peak_bytes = tl.peak_bytes;
    *iteration_ms = tl.iteration_time_ms;
    *recompute_ms = tl.recompute_time_ms;
  });
}

int mimose_planner_sample_workload(const char* distribution, int64_t batch_multiplier,
                                   int64_t iterations, uint64_t seed, int64_t* out) {
  return guard([&] {
    auto w = mimose::parse_distribution(distribution);
    w.batch_multiplier = batch_multiplier;
    w.iterations = iterations;
    w.seed = seed;
    const auto xs = mimose::sample_workload(w);
    std::memcpy(out, xs.data(), xs.size() * sizeof(int64_t));
  });
}

int mimose_planner_run_experiment(const char* model_text, const char* distribution,
                                  int64_t batch_multiplier, int64_t iterations, uint64_t seed,
                                  const mimose_sched_cfg* cfg, const char* planner,
                                  char** summary, char** csv) {
  return guard([&] {
    const auto model = mimose::load_model_from_string(model_text);
    auto w = mimose::parse_distribution(distribution);
    w.batch_multiplier = batch_multiplier;
    w.iterations = iterations;
    w.seed = seed;
    mimose::ExperimentConfig ec;
    ec.planner = mimose::planner_from_string(planner);
    ec.sched = to_sched(cfg);
    const auto rep = mimose::run_experiment(model, w, ec);
    std::ostringstream s, c;
    mimose::write_report_summary(rep, s);
    mimose::write_report_csv(rep, c);
    std::string sum;
    std::istringstream lines(s.str());
    for (std::string line; std::getline(lines, line);) {
      if (line.rfind("planner_wall_ms", 0) == 0 || line.rfind("fit_wall_ms", 0) == 0 ||
          line.rfind("overhead_iterations", 0) == 0)
        continue;  // wall-clock dependent
      sum += line + "\n";
    }
    *summary = dup(sum);
    *csv = dup(c.str());
  });
}

}  // extern "C"
