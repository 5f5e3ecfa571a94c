/* C ABI of the host planner (libmimose_host.so), built from include/mimose.
 *
 * The reference planner is header-only C++ with no FFI
 * (reference proj/include/mimose/ headers); these entry points expose exactly
 * its planner-side calls over plain C types so non-C++ callers (and the
 * Python tests) reach the same code the B200 trainer links:
 *
 *   mimose_planner_fit            <- estimator.hpp:79   fit()
 *   mimose_planner_plan_sequence  <- scheduler.hpp:195  lookup_or_plan() (fresh PlanCache)
 *                                    scheduler.hpp:81   generate_plan()
 *   mimose_planner_simulate       <- simulator.hpp:104  simulate_iteration()
 *   mimose_planner_sample_workload<- workload.hpp:63    sample_workload() + parse_distribution()
 *   mimose_planner_run_experiment <- harness.hpp:139    run_experiment() + write_report_*()
 *
 * Text arguments use the reference's own formats: model documents
 * (model_spec.hpp:268-385), estimator dumps (estimator.hpp:182-259),
 * sample CSV (collector.hpp:198-204). Returned strings are freed with
 * mimose_planner_free. Status: 0 ok, 1 error (mimose_planner_last_error),
 * exceptions never cross the boundary.
 */
#ifndef MIMOSE_PLANNER_H_
#define MIMOSE_PLANNER_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int64_t budget_bytes;         /* scheduler.hpp:23 */
  int64_t reserve_bytes;        /* scheduler.hpp:24 (-1 = 8% default) */
  double bucket_tolerance;      /* scheduler.hpp:25 */
  double cache_tolerance;       /* scheduler.hpp:26 */
  int excess_includes_constant; /* scheduler.hpp:27 */
} mimose_sched_cfg;

const char* mimose_planner_last_error(void);
void mimose_planner_free(char* s);

int mimose_planner_fit(const char* samples_csv, int order, char** estimator_text);

/* For each x (in order) runs lookup_or_plan against one fresh cache.
 * dropped_masks: n * mask_words uint64 (bit i of word w = layer id 64*w + i). */
int mimose_planner_plan_sequence(const char* estimator_text, const char* model_text,
                                 const mimose_sched_cfg* cfg, const int64_t* xs, int n,
                                 uint64_t* dropped_masks, int mask_words, int* insufficient,
                                 int* cache_hit);

/* A planning session: the estimator, the model document, the scheduler
 * config and ONE persistent PlanCache (scheduler.hpp:169-227), as the
 * reference harness keeps them across iterations (harness.hpp:277-293).
 * set_estimator swaps in a refit estimator and keeps the cache, as
 * harness.hpp:264-276 does. reserve_bytes >= 0 overrides the session's
 * reserve for this call (per-input-size reserves). */
typedef struct mimose_plan_session mimose_plan_session;
int mimose_planner_session_create(const char* estimator_text, const char* model_text,
                                  const mimose_sched_cfg* cfg, mimose_plan_session** out);
int mimose_planner_session_set_estimator(mimose_plan_session* s, const char* estimator_text);
int mimose_planner_session_plan(mimose_plan_session* s, int64_t x, int64_t reserve_bytes,
                                uint64_t* dropped_mask, int mask_words, int* insufficient,
                                int* cache_hit);
int mimose_planner_session_destroy(mimose_plan_session* s);

int mimose_planner_simulate(const char* model_text, const int* dropped, int n_dropped,
                            int64_t x, int64_t* peak_bytes, double* iteration_ms,
                            double* recompute_ms);

int mimose_planner_sample_workload(const char* distribution, int64_t batch_multiplier,
                                   int64_t iterations, uint64_t seed, int64_t* out);

/* planner: "mimose" | "static-max" | "dtr" | "none". Summary omits the two
 * wall-clock fields (they are not seed-deterministic). */
int mimose_planner_run_experiment(const char* model_text, const char* distribution,
                                  int64_t batch_multiplier, int64_t iterations, uint64_t seed,
                                  const mimose_sched_cfg* cfg, const char* planner,
                                  char** summary, char** csv);

#ifdef __cplusplus
}
#endif

#endif /* MIMOSE_PLANNER_H_ */
