// Layer executor + Mimose training loop on one B200 (SURVEY §2.4 P1, C1, and
// §8(a) a14/a16-a18).
//
// The trainer runs the reference's two-phase machine
// (reference harness.hpp:215-296) for real: sheltered iterations measure
// every encoder block's activation bytes as the budget arena's
// requested-bytes delta around the block's forward (and its time with
// cudaEvents); the host fits the reference estimator (include/mimose/
// estimator.hpp `fit`), and responsive iterations apply
// `lookup_or_plan` plans: a dropped block forwards in no-save mode keeping
// only its output, and is re-forwarded (same kernels, same Philox streams)
// right before its backward.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <deque>
#include <map>
#include <string>
#include <unordered_set>
#include <vector>

#include "capi_common.hpp"
#include "mimose/mimose.hpp"
#include "mimose_cuda.h"
#include "dp.hpp"

namespace mimose_rt {

struct ParamRef {
  int64_t off = 0;  // element offset into the flat parameter buffers
  int64_t n = 0;
};

struct LayerParams {
  ParamRef wqkv, bqkv, wo, bo, ln1_g, ln1_b, w1, b1, w2, b2, ln2_g, ln2_b;
};

// Saved tensors of the attention half of a block. z1: pre-LN = LN1 output x1
// (post-LN halves keep no LN input: their LN backward reads the LN output,
// see Trainer::bnd_st_); st1 = LN1 {mean, rstd} (pre-LN; post-LN whole-block
// units: the block-internal h1's).
struct AttnSave {
  void *qkv = nullptr, *P = nullptr, *Pd = nullptr, *ctx = nullptr, *z1 = nullptr,
       *st1 = nullptr;
  void *lse = nullptr, *mask = nullptr;  // flash attention (attn_fused = 3) instead of P / Pd
};
// Saved tensors of the FFN half. z2: pre-LN = LN2 output x2 (the FFN input);
// u = FFN1 pre-activation, g = GELU(u).
struct FfnSave {
  void *z2 = nullptr, *st2 = nullptr, *u = nullptr, *g = nullptr;
};
// Saved set of one checkpoint unit (a whole block, or one half of it). For
// whole-block units h1 - the block-internal attention-half output - is saved
// too; for half units it is the attention unit's output (a boundary).
struct UnitSave {
  AttnSave a;
  FfnSave f;
  void* h1 = nullptr;
  bool live = false;
};

struct EmbedSave {
  void *z0 = nullptr, *st0 = nullptr;  // BERT: LN input and {mean, rstd}
};

struct StepGeo {
  int B = 0, S = 0, ld = 0;
  int64_t T = 0;
  uint64_t step = 0;
};

struct StepInputs {  // device pointers
  const int32_t* tokens = nullptr;
  const int32_t* types = nullptr;
  const int32_t* labels = nullptr;
  const int32_t* perm = nullptr;
  const int32_t* seg = nullptr;
  const int32_t* uid = nullptr;
  int n_unique = 0;
  int n_valid = 0;                     // LM: labelled (>= 0) positions
  const int32_t* mask_pos = nullptr;   // MLM: masked row indices [n_mask]
  const int32_t* mask_lab = nullptr;   // MLM: their labels [n_mask]
  int n_mask = 0;
};

class Trainer {
 public:
  Trainer(mimose_ctx* ctx, const mimose_model_cfg& m, const mimose_train_cfg& t);
  ~Trainer();

  // One forward + backward (no optimizer). Host-side phase machine decides
  // the plan. Loss stays on device (d_loss()).
  void forward_backward(const StepInputs& in, int B, int S, cudaStream_t s,
                        mimose_step_report* rep);
  void optimizer_step(float grad_scale, cudaStream_t s);
  // native bucketed gradient all-reduce during backward (nullptr detaches)
  void attach_dp(DataParallel* dp, int64_t bucket_bytes);
  const std::vector<Bucket>& dp_buckets() const { return buckets_; }

  // host inputs -> staged H2D -> forward_backward (+ hook + optimizer) -> loss D2H
  void step_host(const int32_t* tokens, const int32_t* types, const int32_t* labels, int B,
                 int S, int do_optimizer, cudaStream_t s, mimose_step_report* rep,
                 bool sync = true);
  // loss of a host-input step (blocks until that step's read-back landed)
  float loss(int64_t iter);

  void set_forced_plan(const int* ids, int n, int active);
  void set_grad_hook(mimose_grad_hook fn, void* user) {
    hook_ = fn;
    hook_user_ = user;
  }

  // introspection
  float* params_f32() const { return p32_; }
  void* params_bf16() const { return p16_; }
  float* grads() const { return g32_; }
  int64_t num_params() const { return nparam_; }
  float* d_loss() const { return d_loss_; }
  float* d_logits() const { return d_logits_; }
  const mimose::ModelSpec& spec() const { return spec_; }
  const mimose::CollectorState& collector() const { return cstate_; }
  const mimose::EstimatorModel& estimator() const { return est_; }
  bool trained() const { return trained_; }
  const mimose::PlanCache& cache() const { return cache_; }
  const mimose::SchedulerConfig& sched() const { return sched_; }
  const std::deque<mimose_step_report>& history() const { return history_; }
  int64_t constant_bytes() const { return constant_bytes_; }
  int64_t reserve_bytes() const { return sched_.effective_reserve(); }
  int param_count() const { return static_cast<int>(param_names_.size()); }
  void param_info(int i, const char** name, int64_t* off, int64_t* n) const;
  // bytes outside the planner-managed units that can be live at once; with
  // n_dropped >= 0 the retained outputs of exactly that many dropped units,
  // else of every unit
  int64_t extras_bytes(int S, int n_dropped = -1) const;
  // a unit's checkpoint boundary: its output (+ post-LN: the output
  // LayerNorm's {mean, rstd}, which its LN backward reads with the output)
  int64_t unit_out_bytes(int S) const {
    return (2LL * H_ + (post_ln() ? 8 : 0)) * t_.batch * S;
  }
  bool post_ln() const { return m_.arch != MIMOSE_ARCH_GPT2; }
  int64_t head_bytes(int S) const;
  int64_t block_work_bytes(int S) const;
  int64_t nonunit_bytes(int S) const;
  // peak residency of an iteration under `plan`, as this executor runs it
  int64_t replay_peak(const mimose::CheckpointPlan& plan, int64_t x) const;
  // FFN-half unit u whose attention half is dropped too (half units only)
  bool pair_dropped(int u, const std::vector<char>& d) const {
    return half_ && u % 2 == 1 && d[static_cast<size_t>(u)] && d[static_cast<size_t>(u) - 1];
  }
  int64_t dtr_headroom(int S) const;
  // the run so far in the reference's report schema (harness.hpp:57-118):
  // per-iteration rows with MEASURED peak bytes and device milliseconds
  mimose::SimReport report();

 private:
  ParamRef add_param(const std::string& name, int64_t n, bool decay, std::vector<ParamRef*>& fix);

  void build_params();
  void init_params(cudaStream_t s);
  void build_spec();

  // unit executor. Checkpoint units are whole blocks (ckpt_unit 0, the
  // reference's layer granularity) or block halves (ckpt_unit 1: unit 2l =
  // attention half of block l, 2l + 1 = its FFN half). A unit forward with
  // save == nullptr keeps only its output; the backward consumes dy (and the
  // pre-LN attention-branch gradient *aux handed from an FFN half) and the
  // saved set, and returns the gradient of the unit input.
 public:
  int units() const { return half_ ? 2 * L_ : L_; }
  int unit_block(int u) const { return half_ ? u / 2 : u; }
  // lean == true: recompute of a dropped unit whose boundary (output + its
  // statistics, unit_out_bytes) this step still holds: only the tensors its
  // backward reads are regenerated - the final projection GEMM and LayerNorm
  // that produced the (retained) output are skipped
  void unit_fwd(int u, const void* in, void* out, UnitSave* save, const StepGeo& g,
                cudaStream_t s, bool lean = false);
  void* unit_bwd(int u, const void* in, UnitSave& sv, void* dy, void** aux, const StepGeo& g,
                 cudaStream_t s);
  // boundary records of the current step: unit output and (post-LN) its
  // LayerNorm statistics, from the unit's forward until its backward
  bool has_boundary(int u, const void* out) const {
    return u >= 0 && u < units() && bnd_out_[static_cast<size_t>(u)] == out && out != nullptr;
  }
  void drop_boundary(int u);
  void clear_boundaries();
  void free_save(UnitSave& sv);
  void* take(int64_t bytes, int tag);
  void drop(void*& p);

 private:
  // st_out: post-LN output LayerNorm statistics buffer (or null); lean: skip
  // the output projection (+ LN) - the output already exists
  void attn_half_fwd(int l, const void* h, void* h1, AttnSave* save, void* st_out, bool lean,
                     const StepGeo& g, cudaStream_t s);
  void ffn_half_fwd(int l, const void* h1, void* y, FfnSave* save, void* st_out, bool lean,
                    const StepGeo& g, cudaStream_t s);
  // y / y_st (h1 / h1_st): the half's output and its LN statistics (post-LN)
  void* ffn_half_bwd(int l, const void* h1, const void* y, const void* y_st, FfnSave& sv,
                     void* dy, void** da, const StepGeo& g, cudaStream_t s);
  void* attn_half_bwd(int l, const void* h, void* h1, void* h1_st, bool own_h1, AttnSave& sv,
                      void* dh1, void* da, const StepGeo& g, cudaStream_t s);
  void* attn_fwd(int l, const void* x, AttnSave* save, const StepGeo& g, cudaStream_t s);
  void* attn_bwd(int l, AttnSave& sv, void* dctx, const StepGeo& g, cudaStream_t s);
  bool ffn_deriv() const;
  int fused_attn(int S) const;
  bool save_pd() const;
  void* head_fwd_bwd(const StepInputs& in, const void* hidden, const StepGeo& g, cudaStream_t s);

 public:
  // model ends, used by forward_backward and the layer-level C ABI
  StepGeo geometry(int B, int S, int64_t step) const;
  void* embed_fwd(const StepInputs& in, const StepGeo& g, EmbedSave& es, cudaStream_t s);
  void* head_block(const StepInputs& in, const void* last, const StepGeo& g, cudaStream_t s);
  void embed_bwd(const StepInputs& in, const StepGeo& g, EmbedSave& es, void* h0, void* dy,
                 cudaStream_t s);
  int64_t iter() const { return iter_; }
  // pre-LN attention-branch gradient between an FFN half's and its attention
  // half's backward when driven unit by unit through the C ABI
  void* pending_aux_ = nullptr;

 private:
  int label_count(int B, int S) const;
 public:
  void device_labels(StepInputs& in, int B, int S, cudaStream_t s);
  void release_device_labels(StepInputs& in);

 private:
  // phase machine (reference harness.hpp:215-296)
  enum class Mode { Plain, Collect, AllLayers, Planned };
  Mode decide(int64_t x, mimose::CheckpointPlan& plan, mimose_step_report* rep);
  void refit(mimose_step_report* rep);

  mimose_ctx* ctx_;
  mimose_model_cfg m_;
  mimose_train_cfg t_;
  int H_, nh_, F_, L_;
  bool half_ = false;  // checkpoint units = block halves

  float* p32_ = nullptr;
  void* p16_ = nullptr;
  float* g32_ = nullptr;
  float* am_ = nullptr;
  float* av_ = nullptr;
  int64_t nparam_ = 0;
  std::vector<char> param_decay_;
  uint8_t* decay_chunk_ = nullptr;
  std::vector<int64_t> unit_off_;  // gradient units: embeddings, layers, head (+ end)
  DataParallel* dp_ = nullptr;     // not owned
  std::vector<Bucket> buckets_;
  void dp_unit_done(int unit, cudaStream_t s);
  std::vector<std::string> param_names_;
  std::vector<ParamRef> param_refs_;
  ParamRef word_, pos_, type_, eln_g_, eln_b_, wp_, bp_, wc_, bc_;
  ParamRef fln_g_, fln_b_, qaw_, qab_, mlmw_, mlmb_, mlm_g_, mlm_beta_, decb_;
  std::vector<LayerParams> lp_;

  float* ln_partial_ = nullptr;
  float* col_partial_ = nullptr;
  float* norm_partial_ = nullptr;
  float* norm2_ = nullptr;
  void* wgrad_ws_ = nullptr;  // split-K partials of the weight-gradient GEMMs
  int64_t wgrad_ws_bytes_ = 0;
  float* d_loss_ = nullptr;
  float* d_logits_ = nullptr;
  static constexpr int kLossRing = 4;
  float* h_loss_ = nullptr;  // pinned ring of read-back losses
  cudaEvent_t loss_ev_[kLossRing] = {};
  int64_t loss_iter_[kLossRing] = {};

  // double-buffered pinned staging for host inputs
  int32_t* h_stage_[2] = {nullptr, nullptr};
  cudaEvent_t stage_ev_[2] = {};
  bool stage_used_[2] = {false, false};
  int64_t stage_elems_ = 0;

  std::vector<cudaEvent_t> ev_;  // 2 per layer (collector timing)
  // side stream: flash attention keep bits generated during the QKV GEMM
  cudaStream_t side_ = nullptr;
  cudaEvent_t side_ev_[2] = {};

  mimose::ModelSpec spec_;
  // spec_ with the FITTED activation polynomials (unvalidated): the replay
  // (simulate_iteration) that checks a plan's true peak before it runs
  mimose::ModelSpec sim_spec_;
  mimose::SchedulerConfig sched_;
  mimose::CollectorConfig ccfg_;
  mimose::CollectorState cstate_;
  mimose::EstimatorModel est_;
  mimose::PlanCache cache_;
  bool trained_ = false;
  int64_t iter_ = 0;
  int adam_t_ = 0;
  int64_t constant_bytes_ = 0;
  // per-iteration rows (bounded: the oldest are dropped past kHistoryCap) and
  // their device milliseconds, resolved lazily from a fixed ring of event
  // pairs recorded on the step's stream (-1 = not resolved yet)
  static constexpr size_t kHistoryCap = size_t(1) << 18;
  static constexpr int kEvRing = 16;
  std::deque<mimose_step_report> history_;
  std::deque<float> history_ms_;
  int64_t history_first_ = 0;  // iter of history_.front()
  cudaEvent_t step_ev_[kEvRing][2] = {};
  int64_t step_ev_iter_[kEvRing] = {};
  void resolve_step_ms(int slot);
  mimose_step_report* history_row(int64_t iter);
  // reserve the plan of each input size was generated with (cache entries)
  std::map<int64_t, int64_t> plan_reserve_;

  // exception safety: arena blocks taken during a step are tracked and
  // released if the step throws (budget breach, bad input), so a failed step
  // does not shrink the arena for the next one
  bool in_step_ = false;
  std::unordered_set<void*> step_live_;
  std::vector<void*> bnd_out_, bnd_st_;  // per unit: retained output / its LN statistics
  friend struct StepScope;
 public:
  void begin_step();
  void end_step(bool ok);
 private:

  bool forced_active_ = false;
  std::vector<int> forced_;

  mimose_grad_hook hook_ = nullptr;
  void* hook_user_ = nullptr;
};

// Counting sort of token ids (stable): perm lists positions grouped by id
// (ascending position inside a group), seg[u]..seg[u+1] delimits group u,
// uid[u] is its id. Returns the number of distinct ids.
int build_token_tables(const int32_t* tokens, int64_t T, int V, int32_t* perm, int32_t* seg,
                       int32_t* uid);

}  // namespace mimose_rt
