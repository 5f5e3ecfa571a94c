// Layer executor + Mimose training loop; see trainer.hpp.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <set>
#include <stdexcept>

#include "ops.hpp"
#include "ops_attn.hpp"
#include "ops_mem.hpp"
#include "trainer.hpp"
#include "prof.hpp"

namespace mimose_rt {

using bf16raw = uint16_t;  // bf16 storage viewed from host code (pointer arithmetic only)
using mimose_ops::GemmCall;
using mimose_ops::MatView;

namespace {

constexpr int64_t kAlignElems = 64;  // 256 B (fp32) / 128 B (bf16) per tensor

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

int round8(int v) { return (v + 7) / 8 * 8; }

MatView mat(const void* p, int64_t rows, int64_t cols, int64_t ld) {
  MatView v;
  v.ptr = p;
  v.rows = rows;
  v.cols = cols;
  v.ld = ld;
  return v;
}

// per-head [B][nh][S][64] view into a row-major [T][row_ld] buffer
MatView head_view(const void* base, int64_t part_off, int S, int64_t row_ld) {
  MatView v;
  v.ptr = static_cast<const bf16raw*>(base) + part_off;
  v.rows = S;
  v.cols = 64;
  v.ld = row_ld;
  v.bs1 = 64;
  v.bs2 = (int64_t)S * row_ld;
  return v;
}

// [B][nh][S][S] score view with row pitch ld
MatView sq_view(const void* base, int S, int ld, int nh) {
  MatView v;
  v.ptr = base;
  v.rows = S;
  v.cols = S;
  v.ld = ld;
  v.bs1 = (int64_t)S * ld;
  v.bs2 = (int64_t)nh * S * ld;
  return v;
}

void run_gemm(const GemmCall& c, cudaStream_t s) { ck(mimose_ops::gemm(c, s), "gemm"); }

// Y[T,N] = X[T,K] W[N,K]^T (+bias) ; epilogue variants
GemmCall linear_call(const void* X, const void* W, int64_t T, int N, int K, void* Y, int epi,
                     const float* bias) {
  GemmCall c;
  c.M = (int)T;
  c.N = N;
  c.K = K;
  c.A = mat(X, T, K, K);
  c.B = mat(W, N, K, K);
  c.epi = epi;
  c.out = Y;
  c.bias = bias;
  c.ldo = N;
  return c;
}

// dX[T,K] = dY[T,N] W[N,K] (+ aux)
GemmCall dgrad_call(const void* dY, const void* W, int64_t T, int N, int K, void* dX, int epi,
                    const void* aux) {
  GemmCall c;
  c.M = (int)T;
  c.N = K;
  c.K = N;
  c.A = mat(dY, T, N, N);
  c.B = mat(W, N, K, K);  // rows = reduction dim -> MN-major
  c.b_mn = true;
  c.epi = epi;
  c.out = dX;
  c.aux = aux;
  c.ldo = K;
  return c;
}

// dW[N,K] (fp32) = dY[T,N]^T X[T,K]; split-K over T into `ws` when it helps
void* g_wgrad_ws = nullptr;
int64_t g_wgrad_ws_bytes = 0;
GemmCall wgrad_call(const void* dY, const void* X, int64_t T, int N, int K, float* dW) {
  GemmCall c;
  c.M = N;
  c.N = K;
  c.K = (int)T;
  c.A = mat(dY, T, N, N);
  c.a_mn = true;
  c.B = mat(X, T, K, K);
  c.b_mn = true;
  c.epi = mimose_ops::kEpiF32;
  c.out = dW;
  c.ldo = K;
  c.workspace = g_wgrad_ws;
  c.workspace_bytes = g_wgrad_ws_bytes;
  return c;
}

uint64_t stream_id(uint64_t step, int layer, int site) {
  return (step << 20) | (static_cast<uint64_t>(layer & 0xFFFF) << 4) | static_cast<uint64_t>(site);
}

enum Site { kSiteAttnProbs = 0, kSiteAttnOut = 1, kSiteFfnOut = 2, kSiteEmbed = 3, kSitePool = 4 };

}  // namespace

// ------------------------------------------------------------------ tables
int build_token_tables(const int32_t* tokens, int64_t T, int V, int32_t* perm, int32_t* seg,
                       int32_t* uid) {
  std::vector<int32_t> count(static_cast<size_t>(V) + 1, 0);
  for (int64_t i = 0; i < T; ++i) {
    const int32_t t = tokens[i];
    if (t < 0 || t >= V) throw std::runtime_error("token id out of range");
    count[t + 1] += 1;
  }
  for (int v = 0; v < V; ++v) count[v + 1] += count[v];
  std::vector<int32_t> next(count.begin(), count.end() - 1);
  for (int64_t i = 0; i < T; ++i) perm[next[tokens[i]]++] = static_cast<int32_t>(i);
  int nu = 0;
  for (int v = 0; v < V; ++v) {
    if (count[v + 1] > count[v]) {
      seg[nu] = count[v];
      uid[nu] = v;
      ++nu;
    }
  }
  seg[nu] = static_cast<int32_t>(T);
  return nu;
}

// ------------------------------------------------------------------ setup
void* Trainer::take(int64_t bytes, int tag) {
  void* p = ctx_->arena.alloc(bytes, tag);
  if (p != nullptr && in_step_) step_live_.insert(p);
  if (p == nullptr) {
    const auto& st = ctx_->arena.stats();
    throw std::runtime_error("budget exceeded: request " + std::to_string(bytes) + " B with " +
                             std::to_string(st.reserved) + " B live of " +
                             std::to_string(st.budget) + " B (largest free " +
                             std::to_string(st.largest_free) + " B)");
  }
  return p;
}

void Trainer::drop(void*& p) {
  if (p != nullptr) {
    if (!ctx_->arena.free(p)) throw std::runtime_error("arena free of unknown pointer");
    if (in_step_) step_live_.erase(p);
    p = nullptr;
  }
}

Trainer::Trainer(mimose_ctx* ctx, const mimose_model_cfg& m, const mimose_train_cfg& t)
    : ctx_(ctx), m_(m), t_(t) {
  H_ = m.hidden;
  nh_ = m.heads;
  F_ = m.ffn;
  L_ = m.layers;
  if (t.ckpt_unit != 0 && t.ckpt_unit != 1) throw std::runtime_error("ckpt_unit must be 0 (block) or 1 (half)");
  if (t.attn_fused != 0 && t.attn_fused != 2 && t.attn_fused != 3)
    throw std::runtime_error("attn_fused must be 0 (GEMM + softmax), 2 (fused scores) or 3 (flash)");
  half_ = t.ckpt_unit == 1;
  if (units() > 64) throw std::runtime_error("at most 64 checkpoint units (layers <= 32 with half units)");
  if (H_ % 256 || H_ > 1024 || H_ / nh_ != 64 || F_ % 64 || L_ < 1 || L_ > 64)
    throw std::runtime_error("unsupported model shape (need hidden % 256 == 0, <= 1024, head dim 64)");
  if (m.arch != MIMOSE_ARCH_BERT && m.arch != MIMOSE_ARCH_GPT2) throw std::runtime_error("unknown arch");
  if (m.head < MIMOSE_HEAD_MC || m.head > MIMOSE_HEAD_MLM) throw std::runtime_error("unknown head");
  if (m.type_vocab < 0 || m.type_vocab > 2) throw std::runtime_error("type_vocab must be 0, 1 or 2");
  if (m.head == MIMOSE_HEAD_MC && (m.num_choices < 1 || t.batch % m.num_choices))
    throw std::runtime_error("batch must be a multiple of num_choices");
  if (m.vocab < 2) throw std::runtime_error("bad vocab");
  if (m.pad_token_id < -1 || m.pad_token_id >= m.vocab) throw std::runtime_error("bad pad_token_id");
  if (t.seq_min < 1 || t.seq_max < t.seq_min || t.seq_max > m.max_pos || round8(t.seq_max) > 2048)
    throw std::runtime_error("bad sequence range");

  build_params();
  cudaStream_t s = nullptr;
  init_params(s);

  // persistent scratch for the deterministic two-stage reductions
  const int64_t Tmax = (int64_t)t.batch * t.seq_max;
  const int lnb = mimose_ops::ln_bwd_blocks((int)Tmax);
  ln_partial_ = static_cast<float*>(take((int64_t)lnb * 3 * H_ * 4, kTagOther));
  col_partial_ = static_cast<float*>(take(mimose_ops::colsum_scratch_bytes(), kTagOther));
  norm_partial_ = static_cast<float*>(take((int64_t)mimose_ops::sumsq_blocks() * 4, kTagOther));
  {
    // split-K workspace for the weight-gradient GEMMs (largest need over the shapes)
    const int h = H_, f = F_;
    int64_t ws = 0;
    const int v = (m.head == MIMOSE_HEAD_LM || m.head == MIMOSE_HEAD_MLM) ? m.vocab : h;
    const int shapes[5][2] = {{h, f}, {f, h}, {3 * h, h}, {h, h}, {v, h}};
    for (const auto& sh : shapes)
      ws = std::max(ws, mimose_ops::splitk_workspace_bytes(sh[0], sh[1], (int)Tmax));
    wgrad_ws_bytes_ = ws;
    wgrad_ws_ = ws > 0 ? take(ws, kTagOther) : nullptr;
  }
  norm2_ = static_cast<float*>(take(4, kTagOther));
  d_loss_ = static_cast<float*>(take(4, kTagOther));
  // MC: one logit per sequence ; QA: start / end logit per token
  d_logits_ = static_cast<float*>(
      take((m.head == MIMOSE_HEAD_QA ? 2 * Tmax : (int64_t)t.batch) * 4, kTagOther));
  ck(cudaMallocHost(&h_loss_, kLossRing * sizeof(float)), "cudaMallocHost");
  for (int j = 0; j < kLossRing; ++j) {
    ck(cudaEventCreateWithFlags(&loss_ev_[j], cudaEventDisableTiming), "event");
    loss_iter_[j] = -1;
  }
  stage_elems_ = 8 * Tmax + 2 * t.batch + 8;
  for (int k = 0; k < 2; ++k) {
    ck(cudaMallocHost(&h_stage_[k], stage_elems_ * sizeof(int32_t)), "cudaMallocHost");
    ck(cudaEventCreateWithFlags(&stage_ev_[k], cudaEventDisableTiming), "event");
  }
  ev_.resize(2 * static_cast<size_t>(units()));
  bnd_out_.assign(static_cast<size_t>(units()), nullptr);
  bnd_st_.assign(static_cast<size_t>(units()), nullptr);
  for (auto& e : ev_) ck(cudaEventCreate(&e), "cudaEventCreate");
  for (int k = 0; k < kEvRing; ++k) {
    ck(cudaEventCreate(&step_ev_[k][0]), "cudaEventCreate");
    ck(cudaEventCreate(&step_ev_[k][1]), "cudaEventCreate");
    step_ev_iter_[k] = -1;
  }
  ck(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking), "cudaStreamCreate");
  for (auto& e : side_ev_) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  ck(cudaStreamSynchronize(s), "init sync");

  constant_bytes_ = ctx_->arena.stats().requested;
  build_spec();
}

mimose::SimReport Trainer::report() {
  mimose::SimReport rep;
  rep.planner = t_.planner == MIMOSE_PLANNER_NONE     ? mimose::PlannerChoice::None
                : t_.planner == MIMOSE_PLANNER_STATIC ? mimose::PlannerChoice::StaticMax
                : t_.planner == MIMOSE_PLANNER_DTR    ? mimose::PlannerChoice::Dtr
                                                      : mimose::PlannerChoice::Mimose;
  rep.budget_bytes = sched_.budget_bytes;
  rep.reserve_bytes = sched_.effective_reserve();
  rep.iterations = static_cast<int64_t>(history_.size());
  for (int k = 0; k < kEvRing; ++k) resolve_step_ms(k);
  std::set<int64_t> distinct;
  for (size_t i = 0; i < history_.size(); ++i) {
    const mimose_step_report& h = history_[i];
    mimose::IterationRow row;
    row.iter = h.iter;
    row.x = h.x;
    row.planner = rep.planner;
    row.cache_hit = h.cache_hit != 0;
    row.peak_bytes = h.peak_reserved;  // measured (arena), not simulated
    row.iteration_ms = std::max(0.f, history_ms_[i]);
    // recompute cost from the measured per-block forward-time model
    double rc = 0.0;
    for (const auto& l : spec_.layers)
      if (l.id < 64 && ((h.dropped_mask_lo >> l.id) & 1u)) rc += l.forward_ms(h.x);
    row.recompute_ms = rc;
    row.sheltered = h.phase == MIMOSE_PHASE_COLLECT || h.phase == MIMOSE_PHASE_SHELTERED ||
                    h.phase == MIMOSE_PHASE_FALLBACK;
    row.plan_size = h.plan_size;
    row.insufficient = h.insufficient != 0;
    distinct.insert(h.x);
    const double plain = mimose::detail::plain_iteration_ms(spec_, h.x);
    if (row.sheltered) {
      rep.sheltered_iterations += 1;
      rep.collector_overhead_ms += row.iteration_ms - plain;
    }
    if (h.phase == MIMOSE_PHASE_FALLBACK) rep.fallback_sheltered_iterations += 1;
    if (row.peak_bytes > rep.budget_bytes) rep.oom_risk_iterations += 1;
    if (row.insufficient) rep.insufficient_budget_iterations += 1;
    if (h.fit_order >= 0) {
      rep.fit_order = h.fit_order;
      if (rep.fit_at_iter < 0) rep.fit_at_iter = h.iter;
    }
    rep.planner_wall_ms += h.plan_us / 1000.0;
    rep.fit_wall_ms += h.fit_us / 1000.0;
    rep.total_time_ms += row.iteration_ms;
    rep.recompute_total_ms += row.recompute_ms;
    rep.plain_total_ms += plain;
    rep.mean_peak_bytes += static_cast<double>(row.peak_bytes);
    rep.rows.push_back(row);
  }
  rep.collector_iterations = cstate_.collected_iterations;
  rep.cache_hits = cache_.hits;
  rep.cache_misses = cache_.misses;
  rep.planner_invocations = cache_.misses;
  rep.distinct_sizes = static_cast<int64_t>(distinct.size());
  if (rep.iterations > 0) {
    const double n = static_cast<double>(rep.iterations);
    rep.mean_peak_bytes /= n;
    rep.plain_iteration_ms = rep.plain_total_ms / n;
    if (rep.plain_iteration_ms > 0.0) {
      rep.overhead_iterations =
          (rep.collector_overhead_ms + rep.planner_wall_ms + rep.fit_wall_ms) /
          rep.plain_iteration_ms;
      rep.slowdown_vs_plain = rep.total_time_ms / rep.plain_total_ms;
    }
  }
  return rep;
}

Trainer::~Trainer() {
  for (auto& e : step_ev_)
    for (cudaEvent_t ev : e)
      if (ev) cudaEventDestroy(ev);
  for (auto& e : ev_) cudaEventDestroy(e);
  for (auto& e : side_ev_)
    if (e) cudaEventDestroy(e);
  if (side_) cudaStreamDestroy(side_);
  if (h_loss_) cudaFreeHost(h_loss_);
  for (int k = 0; k < 2; ++k) {
    if (h_stage_[k]) cudaFreeHost(h_stage_[k]);
    if (stage_ev_[k]) cudaEventDestroy(stage_ev_[k]);
  }
  for (int j = 0; j < kLossRing; ++j)
    if (loss_ev_[j]) cudaEventDestroy(loss_ev_[j]);
  // arena memory is released with the context
}

ParamRef Trainer::add_param(const std::string& name, int64_t n, bool decay,
                            std::vector<ParamRef*>& fix) {
  (void)fix;
  ParamRef r;
  r.n = n;
  r.off = nparam_;
  nparam_ += (n + kAlignElems - 1) / kAlignElems * kAlignElems;
  param_names_.push_back(name);
  param_refs_.push_back(r);
  param_decay_.push_back(decay ? 1 : 0);
  return r;
}

// Parameter names follow oracle/bert_ref.py param_shapes (HF BERT / GPT-2
// tensors with fused QKV). Tied LM / MLM decoders reuse embeddings.word.
// Layout: contiguous gradient units in forward order - [embeddings]
// [layer 0] ... [layer L-1] [final LN + head] - so that the backward finishes
// them back to front and the data-parallel all-reduce can ship each bucket
// while earlier layers are still differentiating. Weight decay is a
// per-64-element chunk flag (tensors are 64-aligned).
void Trainer::build_params() {
  std::vector<ParamRef*> fix;
  const int64_t H = H_, F = F_;
  const bool bert = m_.arch == MIMOSE_ARCH_BERT;
  lp_.resize(L_);
  unit_off_.clear();
  unit_off_.push_back(nparam_);
  word_ = add_param("embeddings.word", (int64_t)m_.vocab * H, true, fix);
  pos_ = add_param("embeddings.position", (int64_t)m_.max_pos * H, true, fix);
  if (m_.type_vocab > 0) type_ = add_param("embeddings.token_type", (int64_t)m_.type_vocab * H, true, fix);
  if (bert) {
    eln_g_ = add_param("embeddings.ln.weight", H, false, fix);
    eln_b_ = add_param("embeddings.ln.bias", H, false, fix);
  }
  for (int l = 0; l < L_; ++l) {
    unit_off_.push_back(nparam_);
    const std::string p = "layer." + std::to_string(l) + ".";
    lp_[l].wqkv = add_param(p + "attn.qkv.weight", 3 * H * H, true, fix);
    lp_[l].wo = add_param(p + "attn.out.weight", H * H, true, fix);
    lp_[l].w1 = add_param(p + "ffn.in.weight", F * H, true, fix);
    lp_[l].w2 = add_param(p + "ffn.out.weight", H * F, true, fix);
    lp_[l].bqkv = add_param(p + "attn.qkv.bias", 3 * H, false, fix);
    lp_[l].bo = add_param(p + "attn.out.bias", H, false, fix);
    lp_[l].ln1_g = add_param(p + "attn.ln.weight", H, false, fix);
    lp_[l].ln1_b = add_param(p + "attn.ln.bias", H, false, fix);
    lp_[l].b1 = add_param(p + "ffn.in.bias", F, false, fix);
    lp_[l].b2 = add_param(p + "ffn.out.bias", H, false, fix);
    lp_[l].ln2_g = add_param(p + "ffn.ln.weight", H, false, fix);
    lp_[l].ln2_b = add_param(p + "ffn.ln.bias", H, false, fix);
  }
  unit_off_.push_back(nparam_);
  if (!bert) {
    fln_g_ = add_param("final_ln.weight", H, false, fix);
    fln_b_ = add_param("final_ln.bias", H, false, fix);
  }
  switch (m_.head) {
    case MIMOSE_HEAD_MC:
      wp_ = add_param("pooler.weight", H * H, true, fix);
      bp_ = add_param("pooler.bias", H, false, fix);
      wc_ = add_param("classifier.weight", H, true, fix);
      bc_ = add_param("classifier.bias", 1, false, fix);
      break;
    case MIMOSE_HEAD_QA:
      qaw_ = add_param("qa.weight", 2 * H, true, fix);
      qab_ = add_param("qa.bias", 2, false, fix);
      break;
    case MIMOSE_HEAD_MLM:
      mlmw_ = add_param("mlm.transform.weight", H * H, true, fix);
      mlmb_ = add_param("mlm.transform.bias", H, false, fix);
      mlm_g_ = add_param("mlm.ln.weight", H, false, fix);
      mlm_beta_ = add_param("mlm.ln.bias", H, false, fix);
      decb_ = add_param("mlm.decoder.bias", m_.vocab, false, fix);
      break;
    default: break;
  }
  unit_off_.push_back(nparam_);

  p32_ = static_cast<float*>(take(nparam_ * 4, kTagParam));
  p16_ = take(nparam_ * 2, kTagParam);
  g32_ = static_cast<float*>(take(nparam_ * 4, kTagGrad));
  am_ = static_cast<float*>(take(nparam_ * 4, kTagOptim));
  av_ = static_cast<float*>(take(nparam_ * 4, kTagOptim));
  // decay flag per 64-element chunk
  std::vector<uint8_t> chunk(static_cast<size_t>(nparam_ / kAlignElems), 0);
  for (size_t i = 0; i < param_refs_.size(); ++i)
    if (param_decay_[i])
      for (int64_t c = param_refs_[i].off / kAlignElems;
           c < (param_refs_[i].off + param_refs_[i].n + kAlignElems - 1) / kAlignElems; ++c)
        chunk[static_cast<size_t>(c)] = 1;
  decay_chunk_ = static_cast<uint8_t*>(take(static_cast<int64_t>(chunk.size()) + 64, kTagParam));
  ck(cudaMemcpy(decay_chunk_, chunk.data(), chunk.size(), cudaMemcpyHostToDevice), "memcpy");
}

// attn_fused: 0 = QK^T GEMM + softmax kernels; 2 = single-row fused kernels
// (attn_sm100.cuh: S <= 512, causal too; longer rows: the GEMM + softmax
// pair); 3 = flash attention
// (flash_sm100.cuh: no S x S tensor at all -- the block saves one fp32
// log-sum-exp per row and, with dropout, one keep bit per score)
// Dropped-out attention probabilities Pd are saved by default. With
// MIMOSE_SAVE_PD=0 the backward regenerates them from the saved P with the
// same Philox stream (bit-identical values), trading a 4 B/score elementwise
// pass for one S x S tensor per kept block. Measured: at a budget defined as a
// fraction of the no-checkpoint peak the smaller peak shrinks the budget too,
// so regeneration lowered samples/s (GPT-2 298 -> 275, RoBERTa-large 707 ->
// 660); it pays only under a fixed absolute budget.
bool Trainer::save_pd() const {
  static const bool keep = [] {
    const char* e = std::getenv("MIMOSE_SAVE_PD");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return keep && m_.attn_dropout > 0.f;
}

// FFN1's GEMM saves GELU'(u) instead of the pre-activation u when the kept
// FFN half also keeps g = GELU(u) (u's only other reader is the u-only
// regeneration of g): the forward epilogue derives GELU' from the same erfc /
// exponential as GELU, and the backward's dGELU GEMM becomes a plain product
// (light epilogue, CTA pair). Same bytes saved. MIMOSE_FFN_DERIV=0: save u.
bool Trainer::ffn_deriv() const {
  static const bool on = [] {
    const char* e = std::getenv("MIMOSE_FFN_DERIV");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on && t_.ffn_regen_g == 0;
}

// The forward, the backward and the byte model (block_work_bytes) all ask
// this one function, so they always agree on the path for a given S.
int Trainer::fused_attn(int S) const {
  if (t_.attn_fused == 2 && mimose_ops::attn_fused_supported(S)) return 2;
  if (t_.attn_fused == 3 && mimose_ops::flash_supported(S)) return 3;
  return 0;
}

void Trainer::init_params(cudaStream_t s) {
  ck(cudaMemsetAsync(p32_, 0, nparam_ * 4, s), "memset");
  ck(cudaMemsetAsync(g32_, 0, nparam_ * 4, s), "memset");
  ck(cudaMemsetAsync(am_, 0, nparam_ * 4, s), "memset");
  ck(cudaMemsetAsync(av_, 0, nparam_ * 4, s), "memset");
  uint64_t k = 0;
  auto normal = [&](const ParamRef& r) {
    ck(mimose_ops::init_normal(p32_ + r.off, r.n, 0.f, m_.init_std, m_.seed, 0xA000 + (k++), s),
       "init_normal");
  };
  auto ones = [&](const ParamRef& r) {
    std::vector<float> v(static_cast<size_t>(r.n), 1.f);
    ck(cudaMemcpy(p32_ + r.off, v.data(), r.n * 4, cudaMemcpyHostToDevice), "memcpy");
  };
  auto maybe = [&](const ParamRef& r, bool one) {
    if (r.n == 0) return;
    if (one) ones(r);
    else normal(r);
  };
  normal(word_);
  normal(pos_);
  maybe(type_, false);
  for (auto& l : lp_) {
    normal(l.wqkv);
    normal(l.wo);
    normal(l.w1);
    normal(l.w2);
    ones(l.ln1_g);
    ones(l.ln2_g);
  }
  maybe(wp_, false);
  maybe(wc_, false);
  maybe(qaw_, false);
  maybe(mlmw_, false);
  maybe(eln_g_, true);
  maybe(fln_g_, true);
  maybe(mlm_g_, true);
  ck(mimose_ops::f32_to_bf16(p32_, p16_, nparam_, s), "f32_to_bf16");
}

// Peak bytes the task head (and the GPT-2 final LayerNorm) holds at once,
// mirroring head_fwd_bwd's allocation order. MLM is sized for every token
// masked (the count is only known per step).
int64_t Trainer::head_bytes(int S) const {
  const int64_t B = t_.batch, T = B * S, H = H_;
  const int64_t act = 2 * T * H;
  const int64_t Vp = (m_.vocab + 63) / 64 * 64;
  int64_t head = 0;
  switch (m_.head) {
    case MIMOSE_HEAD_MC: head = act + 2 * (2 * B * H); break;
    case MIMOSE_HEAD_QA:
      head = act + 8 * T + 8 * B + (int64_t)mimose_ops::qa_row_blocks((int)T) * (2 * H + 2) * 4;
      break;
    case MIMOSE_HEAD_LM: head = act + 2 * T * Vp + 4 * T; break;
    default: head = 6 * act + 8 * T + 2 * T * Vp + 4 * T; break;
  }
  if (m_.arch == MIMOSE_ARCH_GPT2) head += 2 * act + 8 * T;  // xf, stats, d(final LN)
  return head + 64 * 1024;
}

// Worst extra live set of one unit's backward above its saved set and the
// incoming gradient: transients allocated minus saved tensors already
// released, replayed in ffn_half_bwd / attn_half_bwd / attn_bwd's exact
// allocation order (a saved tensor freed early is reused by later
// transients, so summing every transient would over-reserve by ~3x at
// S = 512). Whole-block units replay both halves back to back; half units
// take the larger of the two. Also covers the forward's transient score
// buffer of the unfused attention path.
int64_t Trainer::block_work_bytes(int S) const {
  const int64_t B = t_.batch, T = B * S, H = H_, F = F_;
  const int64_t ld = round8(S);
  const int64_t quad = B * nh_ * (int64_t)S * ld * 2;
  const int64_t act = 2 * T * H, fact = 2 * T * F, qkv3 = 2 * T * 3 * H, st = 8 * T;
  const bool pre = m_.arch == MIMOSE_ARCH_GPT2;
  const bool hid = m_.hidden_dropout > 0.f;
  const int64_t pd = m_.attn_dropout > 0.f ? quad : 0;
  const int fused = fused_attn(S);
  const bool flash = fused == 3;
  const int64_t lse = 4 * B * nh_ * (int64_t)S;
  const int64_t kmask = m_.attn_dropout > 0.f ? 4 * B * nh_ * (int64_t)S * ((S + 31) / 32) : 0;
  int64_t live = 0, peak = 0;
  auto take_b = [&](int64_t n) { live += n; peak = std::max(peak, live); };
  auto drop_b = [&](int64_t n) { live -= n; };
  const bool regen = t_.ffn_regen_g != 0;
  auto g_use = [&] {  // the W2 gradient's g: saved, or regenerated then freed
    if (regen) take_b(fact);
    drop_b(fact);
  };
  auto ffn = [&] {  // ffn_half_bwd: dy live -> dh1 (+ da) live
    if (pre) {
      if (hid) take_b(act);                     // df
      g_use(); take_b(fact);                    // g -> du
      if (hid) drop_b(act);                     // df
      drop_b(fact);                             // u
      take_b(act); drop_b(act);                 // dh1, x2
      if (hid) take_b(act);                     // da
      take_b(act);                              // dx2
      drop_b(fact); drop_b(act); drop_b(act);   // du, dx2, dy
      drop_b(st);                               // st2
    } else {
      take_b(act); if (hid) take_b(act);        // dres (dz2), df
      drop_b(act);                              // dy (LN2 backward reads y, st: boundary)
      g_use(); take_b(fact);                    // g -> du
      if (hid) drop_b(act);                     // df
      drop_b(fact);                             // u
      take_b(act);                              // dh1
      drop_b(fact); drop_b(act);                // du, dres
    }
  };
  auto attn = [&] {  // attn_half_bwd: dh1 (+ da) live -> dx live
    if (!pre) {
      take_b(act); if (hid) take_b(act);        // dz1, da
      drop_b(act);                              // dh1 (LN1 backward reads h1, st)
      if (!half_) { drop_b(act); drop_b(st); }  // block-internal h1, st1
    }
    if (!flash) drop_b(act);                    // ctx
    take_b(act);                                // dctx
    if (hid) drop_b(act);                       // da
    if (flash) {
      take_b(qkv3); take_b(lse);                // dqkv, D = rowsum(dO o O)
      drop_b(lse); drop_b(act); drop_b(lse);    // D, dctx, saved lse
      drop_b(kmask); drop_b(qkv3); drop_b(act); // keep bits, qkv, ctx
    } else {
      take_b(qkv3);                             // dqkv
      if (!save_pd()) take_b(pd);               // regenerated Pd (0 without dropout)
      drop_b(pd);                               // Pd (saved or regenerated) after dV
      take_b(quad);                             // dP
      drop_b(act); drop_b(quad);                // dctx, P
      drop_b(quad); drop_b(qkv3);               // dP, qkv
    }
    take_b(act);                                // dx
    if (pre) {
      take_b(act);                              // dx1
      drop_b(qkv3); drop_b(act); drop_b(act);   // dqkv, x1, dx1
      drop_b(st); drop_b(act);                  // st1, dh1
    } else {
      drop_b(qkv3); drop_b(act);                // dqkv, dz1
    }
  };
  int64_t work = 0;
  if (half_) {
    live = peak = act;                          // dy
    ffn();
    work = peak;
    live = peak = act + (pre && hid ? act : 0); // dh1 (+ da)
    attn();
    work = std::max(work, peak);
  } else {
    live = peak = act;                          // dy
    ffn();
    if (pre) drop_b(act);                       // h1 (block-internal, saved; post-LN: after LN1')
    attn();
    work = peak;
  }
  // forward: the unfused path's score buffer lives next to the unit's saves
  const int64_t fwd = fused ? 0 : quad;
  return std::max(work, fwd);
}

// Bytes outside the planner-managed units that can be live at once: inputs
// + token tables, embedding saves (z0, stats, h0), head tensors and one
// unit's backward workspace.
int64_t Trainer::nonunit_bytes(int S) const {
  const int64_t B = t_.batch, T = B * S, H = H_;
  const int64_t act = 2 * T * H;
  const int64_t inputs = 4 * (7 * T + 2 * B + 8);
  const int64_t embed = m_.arch == MIMOSE_ARCH_BERT ? 2 * act + 8 * T : act;
  return inputs + embed + head_bytes(S) + block_work_bytes(S);
}

// ... plus the retained outputs of n_dropped dropped units (every unit when
// n_dropped < 0: the scheduler's excess formula credits a dropped unit with
// its whole a(x), but the unit keeps its output, simulator.hpp:131-135).
int64_t Trainer::extras_bytes(int S, int n_dropped) const {
  const int n = n_dropped < 0 ? units() : n_dropped;
  return nonunit_bytes(S) + (int64_t)n * unit_out_bytes(S);
}

// Bytes that appear only transiently after the forward (head + one unit's
// backward workspace) plus a 2 % fragmentation margin: what the reactive
// evictor must leave free.
int64_t Trainer::dtr_headroom(int S) const {
  return head_bytes(S) + block_work_bytes(S) + ctx_->arena.stats().budget / 50;
}

void Trainer::build_spec() {
  const int64_t H = H_, F = F_;
  const double B = t_.batch;
  spec_ = mimose::ModelSpec{};
  spec_.constant_footprint = constant_bytes_;
  spec_.input_min = (int64_t)t_.batch * t_.seq_min;
  spec_.input_max = (int64_t)t_.batch * t_.seq_max;
  const bool flash = t_.attn_fused == 3;
  // attention-half quadratic term: P (+ Pd) for the materialised paths, the
  // keep bits (1 bit per score) for flash attention; flash adds 4 B per row
  // (lse)
  const double p_quad = flash ? (m_.attn_dropout > 0.f ? nh_ / (8.0 * B) : 0.0)
                              : (save_pd() ? 2.0 : 1.0) * nh_ * 2.0 / B;
  const double lin_extra = flash ? 4.0 * nh_ : 0.0;
  // prior a(x) per token: attention half qkv + ctx (+ x1 + st1 pre-LN) + output
  // h1 (+ its LN statistics post-LN); FFN half u + g (+ x2 + st2 pre-LN) +
  // output y (+ statistics post-LN)
  const bool pre = m_.arch == MIMOSE_ARCH_GPT2;
  const double attn_lin = static_cast<double>(pre ? 12 * H + 8 : 10 * H + 8) + lin_extra;
  const double ffn_lin =
      static_cast<double>((t_.ffn_regen_g ? 2 : 4) * F + (pre ? 4 * H + 8 : 2 * H + 8));
  for (int u = 0; u < units(); ++u) {
    const bool attn_part = !half_ || u % 2 == 0;
    const bool ffn_part = !half_ || u % 2 == 1;
    const double quad = attn_part ? p_quad : 0.0;
    mimose::LayerSpec ls;
    ls.id = u;
    ls.position = u;
    ls.stage_id = unit_block(u);
    // flash attention without dropout saves nothing quadratic: a(x) is linear
    ls.category = quad > 0.0 ? mimose::LayerCategory::QuadraticStructure
                             : mimose::LayerCategory::ImplicitReduction;
    ls.activation_coeffs = {0.0, (attn_part ? attn_lin : 0.0) + (ffn_part ? ffn_lin : 0.0), quad};
    ls.boundary_coeffs = {0.0, static_cast<double>(2 * H + (pre ? 0 : 8))};
    ls.forward_time_coeffs = {0.01, 1e-6};
    spec_.layers.push_back(ls);
  }
  mimose::validate_model(spec_);
  sim_spec_ = spec_;

  sched_ = mimose::SchedulerConfig{};
  sched_.budget_bytes = ctx_->arena.stats().budget;
  const int64_t margin = sched_.budget_bytes * 3 / 100;  // 3% fragmentation margin
  sched_.reserve_bytes = t_.reserve_bytes >= 0 ? t_.reserve_bytes : extras_bytes(t_.seq_max) + margin;
  if (sched_.reserve_bytes >= sched_.budget_bytes) sched_.reserve_bytes = sched_.budget_bytes - 1;
  sched_.bucket_tolerance = t_.bucket_tolerance;
  sched_.cache_tolerance = t_.cache_tolerance;
  sched_.excess_includes_constant = true;
  ccfg_.max_sheltered_iters = t_.max_sheltered_iters;
  ccfg_.collect_new_sizes_always = t_.collect_new_sizes_always != 0;
}

void Trainer::param_info(int i, const char** name, int64_t* off, int64_t* n) const {
  if (i < 0 || i >= param_count()) throw std::runtime_error("param index out of range");
  *name = param_names_[i].c_str();
  *off = param_refs_[i].off;
  *n = param_refs_[i].n;
}

void Trainer::set_forced_plan(const int* ids, int n, int active) {
  forced_active_ = active != 0;
  forced_.assign(ids, ids + (ids ? n : 0));
}

// ------------------------------------------------------------ attention
// qkv = x Wqkv^T + bqkv ; P = softmax(q k^T / 8 [causal]) ; Pd = dropout(P) ;
// ctx = Pd v (head-interleaved [T, H]). Saved tensors go to *save when kept.
void* Trainer::attn_fwd(int l, const void* x, AttnSave* save, const StepGeo& g, cudaStream_t s) {
  const LayerParams& P = lp_[l];
  const int64_t T = g.T, H = H_;
  const int S = g.S, ld = g.ld, nh = nh_;
  auto* W = static_cast<bf16raw*>(p16_);
  const bool keep = save != nullptr;
  const int act_tag = keep ? kTagAct : kTagTransient;
  const int64_t quad = (int64_t)g.B * nh * S * ld * 2;

  const bool flash = fused_attn(S) == 3;
  // flash keep bits: generated on the side stream while the QKV GEMM runs
  // (they depend only on the Philox stream and the shape)
  const auto fdrop =
      mimose_ops::make_dropout(m_.attn_dropout, m_.seed, stream_id(g.step, l, kSiteAttnProbs));
  void* kmask = flash && m_.attn_dropout > 0.f
                    ? take(4 * (int64_t)g.B * nh * S * ((S + 31) / 32), act_tag)
                    : nullptr;
  // (serialised on the main stream while the kernel profiler records, so
  // every kernel's event time is its own)
  const bool overlap = kmask != nullptr && !mimose_ops::prof_on();
  if (overlap) {
    ck(cudaEventRecord(side_ev_[0], s), "cudaEventRecord");
    ck(cudaStreamWaitEvent(side_, side_ev_[0], 0), "cudaStreamWaitEvent");
  }
  auto keep_bits = [&](cudaStream_t st) {
    ck(mimose_ops::flash_keep_mask(static_cast<uint32_t*>(kmask), S, ld, nh, g.B, fdrop,
                                   m_.causal != 0, st),
       "flash_keep_mask");
  };
  if (kmask != nullptr && !overlap) keep_bits(s);
  void* qkv = take(T * 3 * H * 2, act_tag);
  run_gemm(linear_call(x, W + P.wqkv.off, T, 3 * (int)H, (int)H, qkv, mimose_ops::kEpiBf16,
                       p32_ + P.bqkv.off),
           s);
  if (overlap) {
    // enqueued after the GEMM: its persistent CTAs take the SMs first and the
    // ALU-bound keep-bit blocks fill the thread slots they leave (launched
    // first, the keep-bit grid held every slot and the GEMM waited for it)
    keep_bits(side_);
    ck(cudaEventRecord(side_ev_[1], side_), "cudaEventRecord");
  }
  if (flash) {
    // flash: ctx plus one fp32 log-sum-exp per row (and keep bits) instead of P / Pd
    if (overlap) ck(cudaStreamWaitEvent(s, side_ev_[1], 0), "cudaStreamWaitEvent");
    void* lse = take(4 * (int64_t)g.B * nh * S, act_tag);
    void* ctx = take(T * H * 2, act_tag);
    ck(mimose_ops::flash_fwd(head_view(qkv, 0, S, 3 * H), head_view(qkv, H, S, 3 * H),
                             head_view(qkv, 2 * H, S, 3 * H), ctx, H, static_cast<float*>(lse),
                             static_cast<uint32_t*>(kmask), S, ld, nh, g.B, 0.125f, fdrop,
                             m_.causal != 0, s),
       "flash_fwd");
    if (keep) {
      save->qkv = qkv; save->lse = lse; save->mask = kmask;
    } else {
      drop(qkv); drop(lse); drop(kmask);
    }
    return ctx;
  }
  void* Pm = take(quad, act_tag);
  // Pd: only the P V operand unless saved (save_pd); the backward regenerates it
  void* Pd = m_.attn_dropout > 0.f ? take(quad, save_pd() ? act_tag : kTagTransient) : nullptr;
  const auto pdrop = mimose_ops::make_dropout(m_.attn_dropout, m_.seed, stream_id(g.step, l, kSiteAttnProbs));
  const int fused = fused_attn(S);
  if (fused == 2) {
    // fused, whole key row in TMEM
    ck(mimose_ops::attn_scores_fwd(head_view(qkv, 0, S, 3 * H), head_view(qkv, H, S, 3 * H), Pm,
                                   Pd, S, ld, nh, g.B, 0.125f, pdrop, s, m_.causal != 0),
       "attn_scores_fwd");
  } else {
    // scores = q k^T / sqrt(64), batched over (head, sequence); then softmax
    void* sc = take(quad, kTagTransient);
    GemmCall c;
    c.M = S; c.N = S; c.K = 64; c.nb1 = nh; c.nb2 = g.B;
    c.A = head_view(qkv, 0, S, 3 * H);
    c.B = head_view(qkv, H, S, 3 * H);
    c.epi = mimose_ops::kEpiBf16;
    c.out = sc; c.ldo = ld; c.obs1 = (int64_t)S * ld; c.obs2 = (int64_t)nh * S * ld;
    c.alpha = 0.125f;
    c.causal_tiles = m_.causal != 0;  // the softmax never reads keys above the diagonal
    run_gemm(c, s);
    ck(mimose_ops::softmax_fwd(sc, Pm, Pd, (int64_t)g.B * nh * S, S, ld, pdrop, s, m_.causal != 0),
       "softmax_fwd");
    drop(sc);
  }
  // ctx = Pd V, written head-interleaved into [T, H]
  void* ctx = take(T * H * 2, act_tag);
  {
    GemmCall c;
    c.M = S; c.N = 64; c.K = S; c.nb1 = nh; c.nb2 = g.B;
    c.A = sq_view(Pd ? Pd : Pm, S, ld, nh);
    c.B = head_view(qkv, 2 * H, S, 3 * H);
    c.b_mn = true;
    c.epi = mimose_ops::kEpiBf16;
    c.out = ctx; c.ldo = H; c.obs1 = 64; c.obs2 = (int64_t)S * H;
    c.causal_k = m_.causal ? 1 : 0;  // keys j <= query i only
    run_gemm(c, s);
  }
  if (!(keep && save_pd())) {
    drop(Pd);
    Pd = nullptr;
  }
  if (keep) {
    save->qkv = qkv; save->P = Pm; save->Pd = Pd;
  } else {
    drop(qkv);
    drop(Pm);
  }
  return ctx;
}

// Attention backward from dctx (consumed) through the saved qkv / P / Pd
// (freed); returns dqkv [T, 3H].
void* Trainer::attn_bwd(int l, AttnSave& sv, void* dctx, const StepGeo& g, cudaStream_t s) {
  const int64_t T = g.T, H = H_;
  const int S = g.S, ld = g.ld, nh = nh_;
  const int64_t quad = (int64_t)g.B * nh * S * ld * 2;
  // dPd = dctx V^T ; dV = Pd^T dctx ; dS = softmax'(dP) ; dQ = dS K ; dK = dS^T Q
  void* dqkv = take(T * 3 * H * 2, kTagTransient);
  if (fused_attn(S) == 3) {
    const auto fdrop =
        mimose_ops::make_dropout(m_.attn_dropout, m_.seed, stream_id(g.step, l, kSiteAttnProbs));
    void* dvec = take(4 * (int64_t)g.B * nh * S, kTagTransient);
    ck(mimose_ops::flash_bwd(head_view(sv.qkv, 0, S, 3 * H), head_view(sv.qkv, H, S, 3 * H),
                             head_view(sv.qkv, 2 * H, S, 3 * H), sv.ctx, dctx, H,
                             static_cast<const float*>(sv.lse),
                             static_cast<const uint32_t*>(sv.mask), static_cast<float*>(dvec),
                             dqkv, S, ld, nh, g.B, 0.125f, fdrop, m_.causal != 0, s),
       "flash_bwd");
    drop(dvec);
    drop(dctx);
    drop(sv.lse);
    drop(sv.mask);
    drop(sv.qkv);
    return dqkv;
  }
  const auto pdrop = mimose_ops::make_dropout(m_.attn_dropout, m_.seed, stream_id(g.step, l, kSiteAttnProbs));
  if (sv.Pd == nullptr && m_.attn_dropout > 0.f) {
    // regenerate Pd = keep * P / (1 - p) from the saved P (same Philox
    // stream and element index as the forward: bit-identical)
    sv.Pd = take(quad, kTagTransient);
    ck(mimose_ops::dropout_apply(sv.P, sv.Pd, quad / 2, pdrop, s), "dropout_apply");
  }
  {
    GemmCall c;
    c.M = S; c.N = 64; c.K = S; c.nb1 = nh; c.nb2 = g.B;
    c.A = sq_view(sv.Pd ? sv.Pd : sv.P, S, ld, nh);
    c.a_mn = true;
    c.B = head_view(dctx, 0, S, H);
    c.b_mn = true;
    c.epi = mimose_ops::kEpiBf16;
    c.causal_k = m_.causal ? 2 : 0;  // dV_j: queries i >= key j only
    c.out = static_cast<bf16raw*>(dqkv) + 2 * H;
    c.ldo = 3 * H; c.obs1 = 64; c.obs2 = (int64_t)S * 3 * H;
    run_gemm(c, s);
  }
  const int fused = fused_attn(S);
  drop(sv.Pd);
  sv.Pd = nullptr;
  void* dP = take(quad, kTagTransient);
  if (fused == 2) {
    // fused: dPd stays in TMEM; softmax backward in the epilogue writes dS
    ck(mimose_ops::attn_scores_bwd(head_view(dctx, 0, S, H), head_view(sv.qkv, 2 * H, S, 3 * H),
                                   sv.P, dP, S, ld, nh, g.B, 0.125f, pdrop, s),
       "attn_scores_bwd");
  } else {
    // causal: P is exactly 0 above the diagonal, so softmax' gives dS = 0 there
    GemmCall c;
    c.M = S; c.N = S; c.K = 64; c.nb1 = nh; c.nb2 = g.B;
    c.A = head_view(dctx, 0, S, H);
    c.B = head_view(sv.qkv, 2 * H, S, 3 * H);
    c.epi = mimose_ops::kEpiBf16;
    c.out = dP; c.ldo = ld; c.obs1 = (int64_t)S * ld; c.obs2 = (int64_t)nh * S * ld;
    c.causal_tiles = m_.causal != 0;
    run_gemm(c, s);
    ck(mimose_ops::softmax_bwd(sv.P, dP, (int64_t)g.B * nh * S, S, ld, pdrop, 0.125f, s,
                               m_.causal != 0),
       "softmax_bwd");
  }
  drop(dctx);
  drop(sv.P);
  {
    GemmCall c;  // dQ = dS K
    c.M = S; c.N = 64; c.K = S; c.nb1 = nh; c.nb2 = g.B;
    c.A = sq_view(dP, S, ld, nh);
    c.B = head_view(sv.qkv, H, S, 3 * H);
    c.b_mn = true;
    c.epi = mimose_ops::kEpiBf16;
    c.out = dqkv; c.ldo = 3 * H; c.obs1 = 64; c.obs2 = (int64_t)S * 3 * H;
    c.causal_k = m_.causal ? 1 : 0;  // keys j <= query i
    run_gemm(c, s);
    // dK = dS^T Q
    c.A = sq_view(dP, S, ld, nh);
    c.a_mn = true;
    c.causal_k = m_.causal ? 2 : 0;  // queries i >= key j
    c.B = head_view(sv.qkv, 0, S, 3 * H);
    c.out = static_cast<bf16raw*>(dqkv) + H;
    run_gemm(c, s);
  }
  drop(dP);
  drop(sv.qkv);
  return dqkv;
}

// ------------------------------------------------------------ block halves
// Each transformer block is two halves.
//   BERT (post-LN)   attention  z1 = h + drop(attn(h) Wo + bo), h1 = LN1(z1)
//                    FFN        z2 = h1 + drop(gelu(h1 W1 + b1) W2 + b2), y = LN2(z2)
//                    (residual + dropout + LN in one row pass after each GEMM)
//   GPT-2 (pre-LN)   attention  x1 = LN1(h), h1 = h + drop(attn(x1) Wo + bo)
//                    FFN        x2 = LN2(h1), y = h1 + drop(gelu(x2 W1 + b1) W2 + b2)
//                    (residual + dropout in the epilogue of the GEMM ending each half)
// Saved sets: attention {qkv, lse (+ keep bits) | P (+ Pd), ctx (, x1, st1
// pre-LN)}, FFN {u, g (, x2, st2 pre-LN)}. Post-LN halves keep no LN input:
// the LN backward takes x-hat from the LN OUTPUT (the unit's output, kept as
// its boundary anyway) and rstd from the output statistics st_out, which the
// boundary keeps too (8 B per token). So a dropped unit's recompute (lean)
// stops before the output projection: attention = QKV GEMM + flash, FFN =
// the FFN1 GEMM - the projection GEMM and LN that made the retained output
// are not rerun (pre-LN likewise: the residual epilogue GEMM is skipped).
void Trainer::attn_half_fwd(int l, const void* h, void* h1, AttnSave* save, void* st_out,
                            bool lean, const StepGeo& g, cudaStream_t s) {
  const LayerParams& P = lp_[l];
  const int64_t T = g.T, H = H_;
  auto* W = static_cast<bf16raw*>(p16_);
  const bool keep = save != nullptr;
  const int act_tag = keep ? kTagAct : kTagTransient;
  const bool pre = m_.arch == MIMOSE_ARCH_GPT2;
  const auto attn_out_drop =
      mimose_ops::make_dropout(m_.hidden_dropout, m_.seed, stream_id(g.step, l, kSiteAttnOut));
  void* x1 = nullptr;
  void* st1 = nullptr;
  const void* ain = h;
  if (pre) {
    x1 = take(T * H * 2, act_tag);
    st1 = keep ? take(T * 8, act_tag) : nullptr;
    mimose_ops::LnFwdArgs la;
    la.rows = (int)T; la.br = h;
    la.gamma = p32_ + P.ln1_g.off; la.beta = p32_ + P.ln1_b.off; la.eps = m_.ln_eps;
    la.stats = st1; la.y = x1;
    ck(mimose_ops::add_ln_fwd(la, (int)H, s), "add_ln_fwd");
    ain = x1;
  }
  void* ctx = attn_fwd(l, ain, save, g, s);
  if (pre && !keep) drop(x1);
  if (lean) {  // recompute: h1 (and its statistics) are retained
    save->ctx = ctx;
    save->z1 = x1;
    save->st1 = st1;
    return;
  }
  if (pre) {
    // output projection with the residual + branch dropout in the epilogue
    GemmCall c = linear_call(ctx, W + P.wo.off, T, (int)H, (int)H, h1, mimose_ops::kEpiBf16,
                             p32_ + P.bo.off);
    c.aux = h;
    c.drop = attn_out_drop;
    run_gemm(c, s);
    if (!keep) drop(ctx);
  } else {
    // post-LN: the projection stays a light-epilogue GEMM; residual, branch
    // dropout and LN1 in one row pass (Philox in the GEMM epilogue measured
    // slower: the K = H projection is epilogue-bound, 29 -> 43 us at S = 288)
    void* a = take(T * H * 2, kTagTransient);
    run_gemm(linear_call(ctx, W + P.wo.off, T, (int)H, (int)H, a, mimose_ops::kEpiBf16,
                         p32_ + P.bo.off),
             s);
    if (!keep) drop(ctx);
    st1 = st_out;
    mimose_ops::LnFwdArgs la;
    la.rows = (int)T; la.res = h; la.br = a; la.br_drop = attn_out_drop;
    la.gamma = p32_ + P.ln1_g.off; la.beta = p32_ + P.ln1_b.off; la.eps = m_.ln_eps;
    la.stats = st1; la.y = h1;
    ck(mimose_ops::add_ln_fwd(la, (int)H, s), "add_ln_fwd");
    drop(a);
  }
  if (keep) {
    save->ctx = ctx;
    save->z1 = x1;
    if (pre) save->st1 = st1;
  }
}

void Trainer::ffn_half_fwd(int l, const void* h1, void* y, FfnSave* save, void* st_out,
                           bool lean, const StepGeo& g, cudaStream_t s) {
  const LayerParams& P = lp_[l];
  const int64_t T = g.T, H = H_, F = F_;
  auto* W = static_cast<bf16raw*>(p16_);
  const bool keep = save != nullptr;
  const int act_tag = keep ? kTagAct : kTagTransient;
  const bool pre = m_.arch == MIMOSE_ARCH_GPT2;
  const auto ffn_out_drop =
      mimose_ops::make_dropout(m_.hidden_dropout, m_.seed, stream_id(g.step, l, kSiteFfnOut));
  void* x2 = nullptr;
  void* st2 = nullptr;
  const void* fin = h1;
  if (pre) {
    x2 = take(T * H * 2, act_tag);
    st2 = keep ? take(T * 8, act_tag) : nullptr;
    mimose_ops::LnFwdArgs la;
    la.rows = (int)T; la.br = h1;
    la.gamma = p32_ + P.ln2_g.off; la.beta = p32_ + P.ln2_b.off; la.eps = m_.ln_eps;
    la.stats = st2; la.y = x2;
    ck(mimose_ops::add_ln_fwd(la, (int)H, s), "add_ln_fwd");
    fin = x2;
  }
  const bool regen = t_.ffn_regen_g != 0;
  void* u = take(T * F * 2, act_tag);
  void* gg = take(T * F * 2, regen ? kTagTransient : act_tag);
  {
    GemmCall c = linear_call(fin, W + P.w1.off, T, (int)F, (int)H, u, mimose_ops::kEpiBiasGelu,
                             p32_ + P.b1.off);
    c.out2 = gg;
    c.gelu_tanh = m_.gelu_tanh;
    c.gelu_deriv = ffn_deriv();
    run_gemm(c, s);
  }
  if (!keep) {
    drop(u);
    if (pre) drop(x2);
  }
  if (lean) {  // recompute: y (and its statistics) are retained
    if (regen) drop(gg);
    save->z2 = x2;
    save->st2 = st2;
    save->u = u;
    save->g = gg;
    return;
  }
  if (pre) {
    // y = h1 + dropout(g W2^T + b2): residual + dropout in the GEMM epilogue
    GemmCall c = linear_call(gg, W + P.w2.off, T, (int)H, (int)F, y, mimose_ops::kEpiBf16,
                             p32_ + P.b2.off);
    c.aux = h1;
    c.drop = ffn_out_drop;
    run_gemm(c, s);
    if (!keep || regen) drop(gg);
  } else {
    void* f = take(T * H * 2, kTagTransient);
    run_gemm(linear_call(gg, W + P.w2.off, T, (int)H, (int)F, f, mimose_ops::kEpiBf16,
                         p32_ + P.b2.off),
             s);
    if (!keep || regen) drop(gg);
    mimose_ops::LnFwdArgs la;
    la.rows = (int)T; la.res = h1; la.br = f; la.br_drop = ffn_out_drop;
    la.gamma = p32_ + P.ln2_g.off; la.beta = p32_ + P.ln2_b.off; la.eps = m_.ln_eps;
    la.stats = st_out; la.y = y;
    ck(mimose_ops::add_ln_fwd(la, (int)H, s), "add_ln_fwd");
    drop(f);
  }
  if (keep) {
    save->z2 = x2;
    save->st2 = st2;
    save->u = u;
    save->g = gg;
  }
}

void Trainer::unit_fwd(int u, const void* in, void* out, UnitSave* save, const StepGeo& g,
                       cudaStream_t s, bool lean) {
  if (u < 0 || u >= units()) throw std::runtime_error("unit index out of range");
  if (lean && (save == nullptr || !has_boundary(u, out)))
    throw std::runtime_error("unit_fwd: lean recompute needs the unit's boundary of this step");
  if (save != nullptr) save->live = true;
  // a full forward (re)writes the unit's boundary: output + output LN statistics
  void* st = nullptr;
  if (!lean) {
    drop_boundary(u);
    if (post_ln()) st = take(g.T * 8, kTagBoundary);
    bnd_out_[static_cast<size_t>(u)] = out;
    bnd_st_[static_cast<size_t>(u)] = st;
  }
  if (half_) {
    if (u % 2 == 0) attn_half_fwd(u / 2, in, out, save ? &save->a : nullptr, st, lean, g, s);
    else ffn_half_fwd(u / 2, in, out, save ? &save->f : nullptr, st, lean, g, s);
    return;
  }
  // whole block: h1 is block-internal, so even a lean recompute runs the
  // attention half in full (h1 + its statistics into the saved set); only the
  // FFN half stops before its output projection
  void* h1 = take(g.T * H_ * 2, save ? kTagAct : kTagTransient);
  void* st1 = save && post_ln() ? take(g.T * 8, kTagAct) : nullptr;
  attn_half_fwd(u, in, h1, save ? &save->a : nullptr, st1, false, g, s);
  if (save != nullptr && post_ln()) save->a.st1 = st1;
  ffn_half_fwd(u, h1, out, save ? &save->f : nullptr, st, lean, g, s);
  if (save != nullptr) save->h1 = h1;
  else drop(h1);
}

void Trainer::drop_boundary(int u) {
  const auto k = static_cast<size_t>(u);
  drop(bnd_st_[k]);
  bnd_out_[k] = nullptr;
}

// (step failure: the step scope already returned the blocks to the arena)
void Trainer::clear_boundaries() {
  std::fill(bnd_out_.begin(), bnd_out_.end(), nullptr);
  std::fill(bnd_st_.begin(), bnd_st_.end(), nullptr);
}

void Trainer::free_save(UnitSave& sv) {
  AttnSave& a = sv.a;
  FfnSave& f = sv.f;
  drop(a.qkv); drop(a.P); drop(a.Pd); drop(a.ctx); drop(a.z1); drop(a.st1); drop(a.lse);
  drop(a.mask);
  drop(f.z2); drop(f.st2); drop(f.u); drop(f.g);
  drop(sv.h1);
  sv.live = false;
}

// ----------------------------------------------------------- half backward
// FFN half: consumes dy (grad of y) and the saved set, returns d h1. Pre-LN
// blocks also return (*da) the attention branch's dropped-out gradient and
// accumulate dbo: both come out of LN2's backward, which already reads d h1.
void* Trainer::ffn_half_bwd(int l, const void* h1, const void* y, const void* y_st, FfnSave& sv,
                            void* dy, void** da_out, const StepGeo& g, cudaStream_t s) {
  const LayerParams& P = lp_[l];
  const int64_t T = g.T, H = H_, F = F_;
  auto* W = static_cast<bf16raw*>(p16_);
  float* G = g32_;
  const bool hid_drop = m_.hidden_dropout > 0.f;
  const bool pre = m_.arch == MIMOSE_ARCH_GPT2;
  const auto attn_out_drop =
      mimose_ops::make_dropout(m_.hidden_dropout, m_.seed, stream_id(g.step, l, kSiteAttnOut));
  const auto ffn_out_drop =
      mimose_ops::make_dropout(m_.hidden_dropout, m_.seed, stream_id(g.step, l, kSiteFfnOut));
  *da_out = nullptr;
  void* dres = nullptr;  // gradient reaching h1 through the residual
  void* df = nullptr;    // gradient of the FFN output (after the branch dropout)
  if (pre) {
    dres = dy;  // y = h1 + drop(f)
    if (hid_drop) {
      df = take(T * H * 2, kTagTransient);
      ck(mimose_ops::dropout_apply(dy, df, T * H, ffn_out_drop, s), "dropout_apply");
    }
    ck(mimose_ops::colsum(df ? df : dy, (int)T, (int)H, H, nullptr, 1, col_partial_, G + P.b2.off, s),
       "colsum");
  } else {
    dres = take(T * H * 2, kTagTransient);  // dz2
    df = hid_drop ? take(T * H * 2, kTagTransient) : nullptr;
    // x-hat from the LN output y (the unit's boundary) and its rstd
    mimose_ops::LnBwdArgs a;
    a.rows = (int)T; a.dy = dy; a.z = y; a.stats = y_st; a.gamma = p32_ + P.ln2_g.off;
    a.beta = p32_ + P.ln2_b.off;
    a.dz = dres; a.dbr = df; a.br_drop = ffn_out_drop;
    a.partial = ln_partial_;
    ck(mimose_ops::ln_bwd(a, (int)H, G + P.ln2_g.off, G + P.ln2_b.off, G + P.b2.off, s), "ln_bwd");
    drop(dy);
  }
  void* dfp = df ? df : (pre ? dy : dres);
  // FFN2: dW2 = df^T g ; du = (df W2) * gelu'(u)
  if (sv.g == nullptr) {  // u-only save: regenerate g (bit-identical to the forward's)
    sv.g = take(T * F * 2, kTagTransient);
    ck(mimose_ops::gelu_regen(sv.u, sv.g, T * F, m_.gelu_tanh != 0, s), "gelu_regen");
  }
  run_gemm(wgrad_call(dfp, sv.g, T, (int)H, (int)F, G + P.w2.off), s);
  drop(sv.g);
  void* du = take(T * F * 2, kTagTransient);
  {
    GemmCall c = dgrad_call(dfp, W + P.w2.off, T, (int)H, (int)F, du, mimose_ops::kEpiDGelu, sv.u);
    c.gelu_tanh = m_.gelu_tanh;
    c.gelu_deriv = ffn_deriv();  // sv.u holds GELU'(u)
    run_gemm(c, s);
  }
  drop(df);
  drop(sv.u);
  // FFN1: dW1 = du^T (FFN input); db1 = du^T 1 summed by the same GEMM from
  // its staged du tiles (no second pass over du)
  {
    GemmCall c = wgrad_call(du, pre ? sv.z2 : h1, T, (int)F, (int)H, G + P.w1.off);
    c.rowsum = G + P.b1.off;
    run_gemm(c, s);
  }
  void* dh1 = take(T * H * 2, kTagTransient);
  if (pre) {
    drop(sv.z2);
    void* da = hid_drop ? take(T * H * 2, kTagTransient) : nullptr;
    // dx2 = du W1 ; d h1 = LN2'(dx2) + dy ; da = drop'(d h1), dbo
    void* dx2 = take(T * H * 2, kTagTransient);
    run_gemm(dgrad_call(du, W + P.w1.off, T, (int)F, (int)H, dx2, mimose_ops::kEpiBf16, nullptr), s);
    drop(du);
    mimose_ops::LnBwdArgs a;
    a.rows = (int)T; a.dy = dx2; a.z = h1; a.stats = sv.st2; a.gamma = p32_ + P.ln2_g.off;
    a.dres = dres;
    a.dz = dh1; a.dbr = da; a.br_drop = attn_out_drop;
    a.partial = ln_partial_;
    ck(mimose_ops::ln_bwd(a, (int)H, G + P.ln2_g.off, G + P.ln2_b.off, G + P.bo.off, s), "ln_bwd");
    drop(dx2);
    drop(dy);
    drop(sv.st2);
    *da_out = da;
  } else {
    // d h1 = du W1 + dz2 (residual)
    run_gemm(dgrad_call(du, W + P.w1.off, T, (int)F, (int)H, dh1, mimose_ops::kEpiBf16, dres), s);
    drop(du);
    drop(dres);
  }
  return dh1;
}

// Attention half: consumes d h1 (and, pre-LN, the FFN half's da), returns
// d h (grad of the block input).
void* Trainer::attn_half_bwd(int l, const void* h, void* h1, void* h1_st, bool own_h1,
                             AttnSave& sv, void* dh1, void* da, const StepGeo& g, cudaStream_t s) {
  const LayerParams& P = lp_[l];
  const int64_t T = g.T, H = H_;
  auto* W = static_cast<bf16raw*>(p16_);
  float* G = g32_;
  const bool hid_drop = m_.hidden_dropout > 0.f;
  const bool pre = m_.arch == MIMOSE_ARCH_GPT2;
  const auto attn_out_drop =
      mimose_ops::make_dropout(m_.hidden_dropout, m_.seed, stream_id(g.step, l, kSiteAttnOut));
  void* dz1 = nullptr;  // post-LN: gradient reaching h through the residual
  if (!pre) {
    // LN1 backward (+ attention-output dropout, dbo)
    dz1 = take(T * H * 2, kTagTransient);
    da = hid_drop ? take(T * H * 2, kTagTransient) : nullptr;
    // x-hat from the LN output h1 and its rstd (whole-block units own the
    // block-internal h1 and its statistics: released right here)
    mimose_ops::LnBwdArgs a;
    a.rows = (int)T; a.dy = dh1; a.z = h1; a.stats = h1_st; a.gamma = p32_ + P.ln1_g.off;
    a.beta = p32_ + P.ln1_b.off;
    a.dz = dz1; a.dbr = da; a.br_drop = attn_out_drop;
    a.partial = ln_partial_;
    ck(mimose_ops::ln_bwd(a, (int)H, G + P.ln1_g.off, G + P.ln1_b.off, G + P.bo.off, s), "ln_bwd");
    drop(dh1);
    if (own_h1) {
      drop(h1);
      drop(h1_st);
    }
  }
  void* dap = da ? da : (pre ? dh1 : dz1);
  // output projection: dWo = da^T ctx ; dctx = da Wo
  run_gemm(wgrad_call(dap, sv.ctx, T, (int)H, (int)H, G + P.wo.off), s);
  // flash attention reads ctx in attn_bwd (rowsum(dP o P) = dO . ctx)
  const int fused = fused_attn(g.S);
  if (fused != 3) drop(sv.ctx);
  void* dctx = take(T * H * 2, kTagTransient);
  run_gemm(dgrad_call(dap, W + P.wo.off, T, (int)H, (int)H, dctx, mimose_ops::kEpiBf16, nullptr), s);
  drop(da);
  void* dqkv = attn_bwd(l, sv, dctx, g, s);
  if (fused == 3) drop(sv.ctx);
  // QKV projection: dWqkv = dqkv^T xin, dbqkv = dqkv^T 1 (row sums of the
  // GEMM's staged dqkv tiles)
  {
    GemmCall c = wgrad_call(dqkv, pre ? sv.z1 : h, T, 3 * (int)H, (int)H, G + P.wqkv.off);
    c.rowsum = G + P.bqkv.off;
    run_gemm(c, s);
  }
  void* dx = take(T * H * 2, kTagTransient);
  if (pre) {
    // dx1 = dqkv Wqkv ; dx = LN1'(dx1) + d h1
    void* dx1 = take(T * H * 2, kTagTransient);
    run_gemm(dgrad_call(dqkv, W + P.wqkv.off, T, 3 * (int)H, (int)H, dx1, mimose_ops::kEpiBf16, nullptr), s);
    drop(dqkv);
    drop(sv.z1);
    mimose_ops::LnBwdArgs a;
    a.rows = (int)T; a.dy = dx1; a.z = h; a.stats = sv.st1; a.gamma = p32_ + P.ln1_g.off;
    a.dres = dh1;
    a.dz = dx;
    a.partial = ln_partial_;
    ck(mimose_ops::ln_bwd(a, (int)H, G + P.ln1_g.off, G + P.ln1_b.off, nullptr, s), "ln_bwd");
    drop(dx1);
    drop(sv.st1);
    drop(dh1);
  } else {
    // dx = dqkv Wqkv + dz1 (residual)
    run_gemm(dgrad_call(dqkv, W + P.wqkv.off, T, 3 * (int)H, (int)H, dx, mimose_ops::kEpiBf16, dz1), s);
    drop(dqkv);
    drop(dz1);
  }
  return dx;
}

// The unit's boundary (output + post-LN statistics, bnd_out_ / bnd_st_) must
// still be held: its LN backward reads them; the statistics are released
// here, the output by the caller.
void* Trainer::unit_bwd(int u, const void* in, UnitSave& sv, void* dy, void** aux,
                        const StepGeo& g, cudaStream_t s) {
  if (u < 0 || u >= units()) throw std::runtime_error("unit index out of range");
  const auto k = static_cast<size_t>(u);
  if (post_ln() && bnd_out_[k] == nullptr)
    throw std::runtime_error("unit_bwd: the unit's output (boundary) is not held");
  void* out = bnd_out_[k];
  void* ost = bnd_st_[k];
  sv.live = false;
  void* dx = nullptr;
  if (half_) {
    if (u % 2 == 1) {
      dx = ffn_half_bwd(u / 2, in, out, ost, sv.f, dy, aux, g, s);
    } else {
      void* da = *aux;
      *aux = nullptr;
      dx = attn_half_bwd(u / 2, in, out, ost, false, sv.a, dy, da, g, s);
    }
  } else {
    void* da = nullptr;
    void* dh1 = ffn_half_bwd(u, sv.h1, out, ost, sv.f, dy, &da, g, s);
    if (post_ln()) {
      // the attention half's LN backward reads h1: it releases h1 / st1
      dx = attn_half_bwd(u, in, sv.h1, sv.a.st1, true, sv.a, dh1, da, g, s);
      sv.h1 = nullptr;
      sv.a.st1 = nullptr;
    } else {
      drop(sv.h1);
      dx = attn_half_bwd(u, in, nullptr, nullptr, false, sv.a, dh1, da, g, s);
    }
  }
  drop_boundary(u);
  return dx;
}
// ------------------------------------------------------------ replay
// Peak residency of one iteration under `plan` as THIS executor runs it:
// the reference's iteration semantics (simulate_iteration, simulator.hpp:
// 104-160: a dropped unit's forward transient a(x), then its own output o(x)
// kept; recompute +(a - o) right before its backward; the backward frees
// a(x)) plus the half-unit rule - a block whose two halves are both dropped
// keeps only the FFN half's output and recomputes its attention half (whole
// a(x), output included) right before the FFN half. a(x) is the fitted
// polynomial (sim_spec_), o(x) the unit output.
int64_t Trainer::replay_peak(const mimose::CheckpointPlan& plan, int64_t x) const {
  const int U = units();
  const double xd = static_cast<double>(x);
  std::vector<int64_t> a(U), o(U);
  std::vector<char> d(U, 0), rec(U, 0);
  for (int u = 0; u < U; ++u) {
    a[u] = mimose::round_bytes(sim_spec_.layers[static_cast<size_t>(u)].activation_at(xd));
    o[u] = mimose::round_bytes(sim_spec_.layers[static_cast<size_t>(u)].boundary_at(xd));
  }
  for (int id : plan.dropped_layers)
    if (id >= 0 && id < U) d[id] = 1;
  int64_t res = sim_spec_.constant_footprint, peak = res;
  for (int u = 0; u < U; ++u) {
    if (d[u]) {
      peak = std::max(peak, res + a[u]);
      res += o[u];
      if (pair_dropped(u, d)) res -= o[u - 1];
    } else {
      res += a[u];
      peak = std::max(peak, res);
    }
  }
  for (int u = U - 1; u >= 0; --u) {
    if (d[u] && !rec[u]) {
      if (pair_dropped(u, d)) {
        res += a[u - 1];
        rec[u - 1] = 1;
        peak = std::max(peak, res);
      }
      res += a[u] - o[u];
      rec[u] = 1;
      peak = std::max(peak, res);
    }
    res -= a[u];
  }
  return peak;
}

// ------------------------------------------------------------ phase machine
void Trainer::refit(mimose_step_report* rep) {
  const int order = std::min(t_.estimator_order, cstate_.distinct_sizes() - 1);
  const auto t0 = std::chrono::steady_clock::now();
  est_ = mimose::fit(cstate_.samples, order);
  const auto t1 = std::chrono::steady_clock::now();
  if (rep) {
    rep->fit_us += std::chrono::duration<double, std::micro>(t1 - t0).count();
    rep->fit_order = order;
  }
  // the plan cache is kept across refits, as the reference harness does
  // measured profile -> model document (activation coefficients = the fit
  // padded to order 2 when possible, forward time = per-layer linear fit)
  sim_spec_ = spec_;
  for (auto& ls : sim_spec_.layers) {
    const auto& c = est_.per_layer_coeffs.at(ls.id);
    std::array<double, 3> a{0, 0, 0};
    for (size_t k = 0; k < c.size() && k < 3; ++k) a[k] = c[k];
    ls.activation_coeffs = a;
  }
  for (auto& ls : spec_.layers) {
    const auto& c = est_.per_layer_coeffs.at(ls.id);
    std::array<double, 3> a{0, 0, 0};
    for (size_t k = 0; k < c.size() && k < 3; ++k) a[k] = c[k];
    double sx = 0, sy = 0, sxx = 0, sxy = 0;
    int n = 0;
    for (const auto& smp : cstate_.samples) {
      if (smp.layer_id != ls.id) continue;
      const double x = static_cast<double>(smp.input_size), yv = smp.measured_forward_ms;
      sx += x; sy += yv; sxx += x * x; sxy += x * yv; ++n;
    }
    double t1c = 0.0, t0c = n ? sy / n : 0.01;
    if (n >= 2 && (n * sxx - sx * sx) > 0) {
      t1c = (n * sxy - sx * sy) / (n * sxx - sx * sx);
      t0c = (sy - t1c * sx) / n;
    }
    // keep the document valid (validate_model invariants) if the fit is odd
    mimose::ModelSpec trial = spec_;
    for (auto& tl : trial.layers)
      if (tl.id == ls.id) {
        tl.activation_coeffs = a;
        tl.forward_time_coeffs = {t0c, t1c};
      }
    try {
      mimose::validate_model(trial);
      spec_ = trial;
    } catch (const mimose::Error&) {
    }
  }
}

Trainer::Mode Trainer::decide(int64_t x, mimose::CheckpointPlan& plan, mimose_step_report* rep) {
  plan = mimose::CheckpointPlan{};
  plan.source_input_size = x;
  if (forced_active_) {
    plan.dropped_layers = forced_;
    plan.normalize();
    return Mode::Plain;
  }
  switch (t_.planner) {
    case MIMOSE_PLANNER_NONE:
    case MIMOSE_PLANNER_DTR:
      return Mode::Plain;
    case MIMOSE_PLANNER_ALL:
      for (int u = 0; u < units(); ++u) plan.dropped_layers.push_back(u);
      return Mode::Plain;
    default:
      // MIMOSE and STATIC share the sheltered collection and the fit; the
      // static planner (reference baselines.hpp:20-23 static_max_plan) then
      // provisions every step for the largest input instead of this one
      break;
  }
  const bool unseen = cstate_.seen_sizes.count(x) == 0;
  if (!trained_) {
    if (mimose::should_collect(cstate_, x, iter_, ccfg_)) return Mode::Collect;
    if (iter_ < ccfg_.max_sheltered_iters) return Mode::AllLayers;
    if (unseen && cstate_.distinct_sizes() < t_.estimator_order + 1) {
      rep->phase = MIMOSE_PHASE_FALLBACK;
      return Mode::Collect;
    }
    refit(rep);
    trained_ = true;
  }
  if (ccfg_.collect_new_sizes_always && unseen) return Mode::Collect;
  // Reserve for this input size (reserve_per_size, default). The scheduler
  // bounds the END-OF-FORWARD residency of the kept units
  // (scheduler.hpp:125-126); what it does not see scales with S: inputs,
  // embedding and head tensors, one unit's backward workspace, a 3 %
  // fragmentation margin (nonunit_bytes), and what the plan itself adds -
  // the retained outputs of dropped units, their forward transients and the
  // recompute before their backward. The latter is measured with the
  // reference's own iteration replay (simulate_iteration, simulator.hpp:104)
  // over the FITTED a(x): the reserve is raised by the replay's overshoot
  // and the size re-planned until the plan fits (a fixed point, a few
  // generate_plan calls of ~1 us). The plan cache is keyed by x and each
  // entry keeps the reserve it was generated with, so a hit replays exactly.
  mimose::SchedulerConfig sc = sched_;
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t xp = t_.planner == MIMOSE_PLANNER_STATIC ? spec_.input_max : x;
  if (t_.reserve_bytes < 0 && t_.reserve_per_size) {
    const int64_t budget = sched_.budget_bytes;
    const auto known = plan_reserve_.find(xp);
    if (known != plan_reserve_.end() && cache_.entries.count(xp)) {
      sc.reserve_bytes = known->second;
    } else {
      const int64_t fixed = nonunit_bytes(static_cast<int>(xp / t_.batch)) + budget * 3 / 100;
      int64_t R = std::min<int64_t>(fixed, budget - 1);
      for (int it = 0; it <= units() + 1; ++it) {
        sc.reserve_bytes = R;
        const mimose::CheckpointPlan trial = mimose::generate_plan(est_, spec_, xp, sc);
        if (trial.insufficient_budget) break;
        const int64_t over = replay_peak(trial, xp) + fixed - budget;
        if (over <= 0 || R >= budget - 1) break;
        R = std::min<int64_t>(R + over, budget - 1);
      }
      sc.reserve_bytes = R;
    }
  }
  rep->reserve_bytes = sc.effective_reserve();
  auto [p, hit] = mimose::lookup_or_plan(cache_, est_, spec_, xp, sc);
  const auto t1 = std::chrono::steady_clock::now();
  rep->plan_us = std::chrono::duration<double, std::micro>(t1 - t0).count();
  if (!hit) {
    cache_.entries[xp].generated_at_iter = iter_;
    p.generated_at_iter = iter_;
    plan_reserve_[xp] = sc.reserve_bytes;
  }
  rep->cache_hit = hit ? 1 : 0;
  rep->predicted_kept = mimose::detail::estimated_kept_bytes(est_, spec_, p, xp);
  plan = p;
  return Mode::Planned;
}

// ------------------------------------------------------------------- heads
// Forward + loss + backward of the task head on `hidden` ([T, H] final hidden
// states); returns d hidden (bf16 [T, H], caller frees). Loss -> d_loss_.
void* Trainer::head_fwd_bwd(const StepInputs& in, const void* hidden, const StepGeo& g,
                            cudaStream_t s) {
  const int64_t T = g.T, H = H_;
  const int B = g.B, S = g.S;
  auto* W = static_cast<bf16raw*>(p16_);
  float* G = g32_;
  void* dh = take(T * H * 2, kTagTransient);
  if (m_.head == MIMOSE_HEAD_MC) {
    // pooled = tanh(cls Wp^T + bp) -> dropout -> logits -> CE over choices
    void* pre = take((int64_t)B * H * 2, kTagTransient);
    {
      GemmCall c;
      c.M = B; c.N = (int)H; c.K = (int)H;
      c.A = mat(hidden, B, H, (int64_t)S * H);  // row 0 of every sequence
      c.B = mat(W + wp_.off, H, H, H);
      c.epi = mimose_ops::kEpiBf16;
      c.out = pre; c.ldo = H; c.bias = p32_ + bp_.off;
      run_gemm(c, s);
    }
    void* dpre = take((int64_t)B * H * 2, kTagTransient);
    ck(mimose_ops::mc_head(pre, B, (int)H, m_.num_choices, p32_ + wc_.off, p32_ + bc_.off,
                           in.labels,
                           mimose_ops::make_dropout(m_.hidden_dropout, m_.seed,
                                                    stream_id(g.step, L_, kSitePool)),
                           d_loss_, d_logits_, dpre, G + wc_.off, G + bc_.off, s),
       "mc_head");
    drop(pre);
    ck(cudaMemsetAsync(dh, 0, T * H * 2, s), "memset");
    GemmCall c;  // dWp = dpre^T cls
    c.M = (int)H; c.N = (int)H; c.K = B;
    c.A = mat(dpre, B, H, H);
    c.a_mn = true;
    c.B = mat(hidden, B, H, (int64_t)S * H);
    c.b_mn = true;
    c.epi = mimose_ops::kEpiF32;
    c.out = G + wp_.off; c.ldo = H;
    run_gemm(c, s);
    ck(mimose_ops::colsum(dpre, B, (int)H, H, nullptr, 1, col_partial_, G + bp_.off, s), "colsum");
    GemmCall d = dgrad_call(dpre, W + wp_.off, B, (int)H, (int)H, dh, mimose_ops::kEpiBf16, nullptr);
    d.ldo = (int64_t)S * H;  // dcls -> rows s = 0
    run_gemm(d, s);
    drop(dpre);
    return dh;
  }
  if (m_.head == MIMOSE_HEAD_QA) {
    float* dl = static_cast<float*>(take(T * 2 * 4, kTagTransient));
    float* parts = static_cast<float*>(take((int64_t)2 * B * 4, kTagTransient));
    ck(mimose_ops::qa_head(hidden, B, S, (int)H, p32_ + qaw_.off, p32_ + qab_.off, in.labels,
                           d_logits_, dl, parts, s),
       "qa_head");
    ck(mimose_ops::sum_f32(parts, 2 * B, 1.f, d_loss_, s), "sum_f32");
    float* qpart = static_cast<float*>(
        take((int64_t)mimose_ops::qa_row_blocks((int)T) * (2 * H + 2) * 4, kTagTransient));
    ck(mimose_ops::qa_head_bwd(hidden, dl, (int)T, (int)H, p32_ + qaw_.off, dh, qpart,
                               G + qaw_.off, G + qab_.off, s),
       "qa_head_bwd");
    void* q = qpart;
    drop(q);
    void* v = dl;
    drop(v);
    v = parts;
    drop(v);
    return dh;
  }
  // tied vocabulary decoders
  const int V = m_.vocab;
  const int Vp = (V + 63) / 64 * 64;
  const bool mlm = m_.head == MIMOSE_HEAD_MLM;
  const int rows = mlm ? in.n_mask : (int)T;
  const float inv = 1.f / static_cast<float>(std::max(1, mlm ? in.n_mask : in.n_valid));
  void* xm = nullptr;    // MLM: gathered masked rows
  void* ut = nullptr;    // MLM transform pre-activation
  void* gt = nullptr;    // MLM transform GELU output (LN input)
  void* stt = nullptr;   // MLM LN stats
  const void* dec_in = hidden;
  if (mlm) {
    if (rows == 0) throw std::runtime_error("MLM step without masked positions");
    xm = take((int64_t)rows * H * 2, kTagTransient);
    ck(mimose_ops::gather_rows(hidden, in.mask_pos, rows, (int)H, xm, s), "gather_rows");
    ut = take((int64_t)rows * H * 2, kTagTransient);
    gt = take((int64_t)rows * H * 2, kTagTransient);
    GemmCall c = linear_call(xm, W + mlmw_.off, rows, (int)H, (int)H, ut, mimose_ops::kEpiBiasGelu,
                             p32_ + mlmb_.off);
    c.out2 = gt;
    c.gelu_tanh = m_.gelu_tanh;
    run_gemm(c, s);
    void* t = take((int64_t)rows * H * 2, kTagTransient);
    stt = take((int64_t)rows * 8, kTagTransient);
    mimose_ops::LnFwdArgs la;
    la.rows = rows; la.br = gt;
    la.gamma = p32_ + mlm_g_.off; la.beta = p32_ + mlm_beta_.off; la.eps = m_.ln_eps;
    la.stats = stt; la.y = t;
    ck(mimose_ops::add_ln_fwd(la, (int)H, s), "add_ln_fwd");
    dec_in = t;
  }
  void* logits = take((int64_t)rows * Vp * 2, kTagTransient);
  {
    GemmCall c = linear_call(dec_in, W + word_.off, rows, V, (int)H, logits, mimose_ops::kEpiBf16,
                             mlm ? p32_ + decb_.off : nullptr);
    c.ldo = Vp;
    run_gemm(c, s);
  }
  float* lrows = static_cast<float*>(take((int64_t)rows * 4, kTagTransient));
  ck(mimose_ops::ce_rows(logits, rows, V, Vp, mlm ? in.mask_lab : in.labels, inv, lrows, s),
     "ce_rows");
  ck(mimose_ops::sum_f32(lrows, rows, inv, d_loss_, s), "sum_f32");
  void* lr = lrows;
  drop(lr);
  // logits now hold dlogits (bf16, already scaled by 1 / count)
  if (mlm)
    ck(mimose_ops::colsum(logits, rows, Vp, Vp, nullptr, 1, col_partial_, G + decb_.off, s),
       "colsum");
  {
    // tied decoder weight gradient written in full (the embedding scatter adds to it)
    GemmCall c;
    c.M = V; c.N = (int)H; c.K = rows;
    c.A = mat(logits, rows, V, Vp);
    c.a_mn = true;
    c.B = mat(dec_in, rows, H, H);
    c.b_mn = true;
    c.epi = mimose_ops::kEpiF32;
    c.out = G + word_.off; c.ldo = H;
    c.workspace = g_wgrad_ws;
    c.workspace_bytes = g_wgrad_ws_bytes;
    run_gemm(c, s);
  }
  void* ddec = mlm ? take((int64_t)rows * H * 2, kTagTransient) : dh;
  {
    GemmCall c;  // d dec_in = dlogits Wword
    c.M = rows; c.N = (int)H; c.K = V;
    c.A = mat(logits, rows, V, Vp);
    c.B = mat(W + word_.off, V, H, H);
    c.b_mn = true;
    c.epi = mimose_ops::kEpiBf16;
    c.out = ddec; c.ldo = H;
    run_gemm(c, s);
  }
  drop(logits);
  if (!mlm) return dh;
  // MLM transform backward: LN, GELU, dense; scatter to the masked positions
  void* dg = take((int64_t)rows * H * 2, kTagTransient);
  {
    mimose_ops::LnBwdArgs a;
    a.rows = rows; a.dy = ddec; a.z = gt; a.stats = stt; a.gamma = p32_ + mlm_g_.off;
    a.dz = dg;
    a.partial = ln_partial_;
    ck(mimose_ops::ln_bwd(a, (int)H, G + mlm_g_.off, G + mlm_beta_.off, nullptr, s), "ln_bwd");
  }
  void* dtv = const_cast<void*>(dec_in);
  drop(dtv);
  drop(ddec);
  drop(stt);
  drop(gt);
  void* du = take((int64_t)rows * H * 2, kTagTransient);
  ck(mimose_ops::dgelu_apply(dg, ut, du, (int64_t)rows * H, m_.gelu_tanh != 0, s), "dgelu_apply");
  drop(dg);
  drop(ut);
  ck(mimose_ops::colsum(du, rows, (int)H, H, nullptr, 1, col_partial_, G + mlmb_.off, s), "colsum");
  run_gemm(wgrad_call(du, xm, rows, (int)H, (int)H, G + mlmw_.off), s);
  void* dxm = take((int64_t)rows * H * 2, kTagTransient);
  run_gemm(dgrad_call(du, W + mlmw_.off, rows, (int)H, (int)H, dxm, mimose_ops::kEpiBf16, nullptr), s);
  drop(du);
  drop(xm);
  ck(cudaMemsetAsync(dh, 0, T * H * 2, s), "memset");
  ck(mimose_ops::scatter_rows(dxm, in.mask_pos, rows, (int)H, dh, s), "scatter_rows");
  drop(dxm);
  return dh;
}

// ------------------------------------------------------------------- step
// ------------------------------------------------------ model ends
// Embeddings: BERT z0 = word + pos (+ type), h0 = dropout(LN(z0)); GPT-2
// h0 = dropout(word + pos) (no LayerNorm). Returns h0; z0 / stats saved.
void* Trainer::embed_fwd(const StepInputs& in, const StepGeo& g, EmbedSave& es, cudaStream_t s) {
  const int64_t T = g.T, H = H_;
  auto* W = static_cast<bf16raw*>(p16_);
  const bool bert = m_.arch == MIMOSE_ARCH_BERT;
  es.z0 = bert ? take(T * H * 2, kTagAct) : nullptr;
  es.st0 = bert ? take(T * 8, kTagAct) : nullptr;
  void* h0 = take(T * H * 2, kTagAct);
  mimose_ops::LnFwdArgs la;
  la.rows = (int)T;
  la.skip_ln = !bert;
  la.gamma = bert ? p32_ + eln_g_.off : nullptr;
  la.beta = bert ? p32_ + eln_b_.off : nullptr;
  la.eps = m_.ln_eps;
  la.z = es.z0; la.stats = es.st0; la.y = h0;
  la.out_drop = mimose_ops::make_dropout(m_.hidden_dropout, m_.seed, stream_id(g.step, L_, kSiteEmbed));
  ck(mimose_ops::embed_ln_fwd(la, (int)H, in.tokens, m_.type_vocab > 0 ? in.types : nullptr,
                              W + word_.off, W + pos_.off,
                              m_.type_vocab > 0 ? W + type_.off : nullptr, g.S, s),
     "embed_ln_fwd");
  return h0;
}

// Final LayerNorm (pre-LN / GPT-2) + task head forward, loss (-> d_loss_),
// head backward; returns the gradient of the last unit's output.
void* Trainer::head_block(const StepInputs& in, const void* last, const StepGeo& g,
                          cudaStream_t s) {
  const int64_t T = g.T, H = H_;
  float* G = g32_;
  if (m_.arch == MIMOSE_ARCH_BERT) return head_fwd_bwd(in, last, g, s);
  void* xf = take(T * H * 2, kTagAct);
  void* stf = take(T * 8, kTagAct);
  mimose_ops::LnFwdArgs la;
  la.rows = (int)T; la.br = last;
  la.gamma = p32_ + fln_g_.off; la.beta = p32_ + fln_b_.off; la.eps = m_.ln_eps;
  la.stats = stf; la.y = xf;
  ck(mimose_ops::add_ln_fwd(la, (int)H, s), "add_ln_fwd");
  void* dy = head_fwd_bwd(in, xf, g, s);
  void* dl = take(T * H * 2, kTagTransient);
  mimose_ops::LnBwdArgs a;
  a.rows = (int)T; a.dy = dy; a.z = last; a.stats = stf; a.gamma = p32_ + fln_g_.off;
  a.dz = dl;
  a.partial = ln_partial_;
  ck(mimose_ops::ln_bwd(a, (int)H, G + fln_g_.off, G + fln_b_.off, nullptr, s), "ln_bwd");
  drop(dy);
  drop(xf);
  drop(stf);
  return dl;
}

// Embedding backward: consumes dy (grad of h0), h0 and the saves.
void Trainer::embed_bwd(const StepInputs& in, const StepGeo& g, EmbedSave& es, void* h0, void* dy,
                        cudaStream_t s) {
  const int64_t T = g.T, H = H_;
  float* G = g32_;
  const bool bert = m_.arch == MIMOSE_ARCH_BERT;
  const bool tied = m_.head == MIMOSE_HEAD_LM || m_.head == MIMOSE_HEAD_MLM;
  if (!tied) ck(cudaMemsetAsync(G + word_.off, 0, word_.n * 4, s), "memset");
  ck(cudaMemsetAsync(G + pos_.off, 0, pos_.n * 4, s), "memset");
  void* de = take(T * H * 2, kTagTransient);
  const auto edrop = mimose_ops::make_dropout(m_.hidden_dropout, m_.seed, stream_id(g.step, L_, kSiteEmbed));
  if (bert) {
    mimose_ops::LnBwdArgs a;
    a.rows = (int)T; a.dy = dy; a.z = es.z0; a.stats = es.st0; a.gamma = p32_ + eln_g_.off;
    a.in_drop = edrop;
    a.dz = de;
    a.partial = ln_partial_;
    ck(mimose_ops::ln_bwd(a, (int)H, G + eln_g_.off, G + eln_b_.off, nullptr, s), "ln_bwd");
  } else {
    ck(mimose_ops::dropout_apply(dy, de, T * H, edrop, s), "dropout_apply");
  }
  drop(dy);
  drop(es.z0); drop(es.st0); drop(h0);
  // tied decoders (LM / MLM) already wrote their [V, H] weight gradient: add
  ck(mimose_ops::embed_word_grad(de, (int)H, in.perm, in.seg, in.uid, in.n_unique, G + word_.off, s,
                                 tied, m_.pad_token_id),
     "embed_word_grad");
  ck(mimose_ops::embed_pos_grad(de, g.B, g.S, (int)H, G + pos_.off, s), "embed_pos_grad");
  if (m_.type_vocab > 0)
    ck(mimose_ops::colsum(de, (int)T, (int)H, H, m_.type_vocab == 2 ? in.types : nullptr,
                          m_.type_vocab, col_partial_, G + type_.off, s),
       "colsum");
  drop(de);
}

StepGeo Trainer::geometry(int B, int S, int64_t step) const {
  if (B != t_.batch) throw std::runtime_error("batch differs from the configured batch");
  if (S < t_.seq_min || S > t_.seq_max) throw std::runtime_error("sequence length outside range");
  StepGeo g;
  g.B = B;
  g.S = S;
  g.ld = round8(S);
  g.T = (int64_t)B * S;
  g.step = static_cast<uint64_t>(step);
  g_wgrad_ws = wgrad_ws_;
  g_wgrad_ws_bytes = wgrad_ws_bytes_;
  return g;
}

void Trainer::forward_backward(const StepInputs& in, int B, int S, cudaStream_t s,
                               mimose_step_report* rep) {
  const StepGeo g = geometry(B, S, iter_);
  const int64_t x = g.T;
  const int64_t T = g.T, H = H_;
  const int U = units();

  const auto host_t0 = std::chrono::steady_clock::now();
  mimose_step_report local{};
  mimose_step_report* r = rep ? rep : &local;
  std::memset(r, 0, sizeof(*r));
  r->iter = iter_;
  r->x = x;
  r->batch = B;
  r->seq = S;
  r->fit_order = -1;
  r->budget = ctx_->arena.stats().budget;
  r->phase = MIMOSE_PHASE_PLAIN;

  mimose::CheckpointPlan plan;
  const Mode mode = decide(x, plan, r);
  if (mode == Mode::Collect && r->phase != MIMOSE_PHASE_FALLBACK) r->phase = MIMOSE_PHASE_COLLECT;
  if (mode == Mode::AllLayers) r->phase = MIMOSE_PHASE_SHELTERED;
  if (mode == Mode::Planned) r->phase = MIMOSE_PHASE_PLANNED;
  // an insufficient_budget plan already holds every unit
  // (scheduler.hpp:153-156): it runs all-dropped and the arena decides
  std::vector<char> dropped(U, 0);
  if (mode == Mode::Collect || mode == Mode::AllLayers) {
    std::fill(dropped.begin(), dropped.end(), 1);
  } else {
    for (int id : plan.dropped_layers)
      if (id >= 0 && id < U) dropped[id] = 1;
  }
  for (int u = 0; u < U; ++u)
    if (dropped[u]) {
      r->plan_size += 1;
      if (u < 64) r->dropped_mask_lo |= (uint64_t)1 << u;
    }
  r->insufficient = plan.insufficient_budget ? 1 : 0;
  if (mode != Mode::Planned)
    r->predicted_kept = constant_bytes_;  // informational only

  ctx_->arena.reset_peak();
  const int slot = static_cast<int>(iter_ % kEvRing);
  resolve_step_ms(slot);
  ck(cudaEventRecord(step_ev_[slot][0], s), "event");

  for (int u = 0; u < U; ++u) drop_boundary(u);  // (none left by a finished step)
  EmbedSave es;
  void* h0 = embed_fwd(in, g, es, s);

  // ---- checkpoint units (blocks or block halves)
  std::vector<void*> out(U, nullptr);
  std::vector<UnitSave> saves(U);
  std::vector<int64_t> measured(U, 0);
  const bool collect = mode == Mode::Collect;
  // ---- DTR-style reactive eviction (reference baselines.hpp:62-159) on the
  // real arena: before a unit needs a_u(x) more bytes than fit under the
  // budget minus the backward headroom, evict the resident saved set that
  // maximises staleness * bytes / forward_ms down to its boundary output.
  const bool dtr = t_.planner == MIMOSE_PLANNER_DTR && !forced_active_;
  int64_t tick = 0;
  std::vector<int64_t> last_use(U, 0);
  const int64_t dtr_room = ctx_->arena.stats().budget - dtr_headroom(S);
  auto need_of = [&](int u) {
    const auto& ls = spec_.layers[static_cast<size_t>(u)];
    return static_cast<int64_t>(ls.activation_at(static_cast<double>(x)));
  };
  auto evict_until = [&](int64_t need, int upto) {
    while (ctx_->arena.stats().reserved + need > dtr_room) {
      int victim = -1;
      double best = -1.0;
      for (int j = 0; j < upto; ++j) {
        if (dropped[j] || !saves[j].live) continue;
        const double ms = std::max(1e-3, spec_.layers[static_cast<size_t>(j)].forward_ms(x));
        const double score = static_cast<double>(tick - last_use[j]) *
                             static_cast<double>(std::max<int64_t>(measured[j], 1)) / ms;
        if (score > best) {
          best = score;
          victim = j;
        }
      }
      if (victim < 0) return;  // nothing left to evict: the arena decides
      free_save(saves[victim]);
      dropped[victim] = 1;
      r->plan_size += 1;
      if (victim < 64) r->dropped_mask_lo |= (uint64_t)1 << victim;
    }
  };
  for (int u = 0; u < U; ++u) {
    const void* hin = u == 0 ? h0 : out[u - 1];
    if (dtr) {
      ++tick;
      evict_until(need_of(u), u);
      last_use[u] = tick;
    }
    if (collect) {
      // measuring pass: full save set; the arena's requested-bytes delta is
      // the unit's activation footprint a_u(x) (output included), then
      // everything but the output (the checkpoint boundary) is released.
      const int64_t before = ctx_->arena.stats().requested;
      ck(cudaEventRecord(ev_[2 * u], s), "event");
      out[u] = take(T * H * 2, kTagBoundary);
      unit_fwd(u, hin, out[u], &saves[u], g, s);
      ck(cudaEventRecord(ev_[2 * u + 1], s), "event");
      measured[u] = ctx_->arena.stats().requested - before;
      free_save(saves[u]);
    } else if (dropped[u]) {
      out[u] = take(T * H * 2, kTagBoundary);
      unit_fwd(u, hin, out[u], nullptr, g, s);
    } else {
      const int64_t before = ctx_->arena.stats().requested;
      out[u] = take(T * H * 2, kTagAct);
      unit_fwd(u, hin, out[u], &saves[u], g, s);
      measured[u] = ctx_->arena.stats().requested - before;
    }
    // both halves of a block dropped: its FFN half's output is the only
    // boundary kept; h1 is regenerated with the attention half's recompute
    // right before the FFN half's (see the backward loop and replay_peak)
    if (pair_dropped(u, dropped) && !dtr) {
      drop_boundary(u - 1);
      drop(out[u - 1]);
    }
  }
  // memory-prediction error on the kept units (allocator-measured a_u(x))
  if (trained_) {
    double sum = 0.0, mx = 0.0;
    int n = 0;
    for (int u = 0; u < U; ++u) {
      if (dropped[u] || measured[u] <= 0) continue;
      const double pred = static_cast<double>(mimose::predict(est_, u, x));
      const double err = std::abs(pred - static_cast<double>(measured[u])) / static_cast<double>(measured[u]);
      sum += err;
      mx = std::max(mx, err);
      ++n;
    }
    r->pred_layers = n;
    r->pred_err_mean = n ? sum / n : 0.0;
    r->pred_err_max = mx;
  }

  // ---- final LayerNorm (pre-LN / GPT-2) and the task head (forward + backward)
  void* dy = head_block(in, out[U - 1], g, s);
  dp_unit_done(L_ + 1, s);

  // ---- backward through the units (recompute dropped ones first)
  void* aux = nullptr;  // pre-LN attention-branch gradient handed FFN half -> attention half
  for (int u = U - 1; u >= 0; --u) {
    if (dtr) {
      ++tick;
      if (dropped[u]) evict_until(need_of(u) - 2 * T * H, u);
      last_use[u] = tick;
    }
    if (dropped[u] && !saves[u].live) {
      if (out[u - (u > 0 ? 1 : 0)] == nullptr) {
        // the attention half of a doubly-dropped block first (regenerates h1)
        const void* ha = u == 1 ? h0 : out[u - 2];
        out[u - 1] = take(T * H * 2, kTagBoundary);
        unit_fwd(u - 1, ha, out[u - 1], &saves[u - 1], g, s);
      }
      // recompute, same kernels and Philox streams as the forward, of what
      // the backward reads (the retained output is not regenerated)
      unit_fwd(u, u == 0 ? h0 : out[u - 1], out[u], &saves[u], g, s, /*lean=*/true);
    }
    void* dx = unit_bwd(u, u == 0 ? h0 : out[u - 1], saves[u], dy, &aux, g, s);
    // a block's parameters are final once its attention half is done
    if (!half_ || u % 2 == 0) dp_unit_done(unit_block(u) + 1, s);
    drop(out[u]);
    dy = dx;
  }

  // ---- embedding backward
  embed_bwd(in, g, es, h0, dy, s);
  dp_unit_done(0, s);

  r->host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0)
                   .count();
  const auto& st = ctx_->arena.stats();
  r->peak_requested = st.peak_requested;
  r->peak_reserved = st.peak_reserved;

  // ---- commit collector measurements (reference collector.hpp:129-184)
  if (collect) {
    ck(cudaEventSynchronize(ev_[2 * U - 1]), "event sync");
    const bool fresh = cstate_.seen_sizes.count(x) == 0;
    for (int u = 0; u < U && fresh; ++u) {
      float ms = 0.f;
      ck(cudaEventElapsedTime(&ms, ev_[2 * u], ev_[2 * u + 1]), "event elapsed");
      mimose::CollectedSample smp;
      smp.layer_id = u;
      smp.input_size = x;
      smp.measured_activation_bytes = measured[u];
      smp.measured_forward_ms = ms;
      smp.valid = true;  // units are flat: no nested checkpoint scopes to filter
      cstate_.samples.push_back(smp);
    }
    cstate_.seen_sizes.insert(x);
    cstate_.collected_iterations += 1;
    if (trained_ && ccfg_.collect_new_sizes_always) refit(r);
  }
  ck(cudaEventRecord(step_ev_[slot][1], s), "event");
  step_ev_iter_[slot] = iter_;
  history_.push_back(*r);
  history_ms_.push_back(-1.f);
  while (history_.size() > kHistoryCap) {
    history_.pop_front();
    history_ms_.pop_front();
    history_first_ += 1;
  }
  iter_ += 1;
}

// Device milliseconds of the step recorded in ring slot `slot` -> its
// history row (the ring is recycled every kEvRing steps).
void Trainer::resolve_step_ms(int slot) {
  const int64_t it = step_ev_iter_[slot];
  if (it < 0) return;
  step_ev_iter_[slot] = -1;
  float ms = 0.f;
  ck(cudaEventSynchronize(step_ev_[slot][1]), "event");
  ck(cudaEventElapsedTime(&ms, step_ev_[slot][0], step_ev_[slot][1]), "event");
  const int64_t k = it - history_first_;
  if (k >= 0 && k < static_cast<int64_t>(history_ms_.size())) history_ms_[static_cast<size_t>(k)] = ms;
}

mimose_step_report* Trainer::history_row(int64_t iter) {
  const int64_t k = iter - history_first_;
  if (k < 0 || k >= static_cast<int64_t>(history_.size())) return nullptr;
  return &history_[static_cast<size_t>(k)];
}

// Step scope: arena blocks taken while a step runs are tracked; a step that
// throws (budget breach, bad input, CUDA error) releases them, so the next
// step starts from the post-constructor arena state.
void Trainer::begin_step() {
  step_live_.clear();
  in_step_ = true;
}

void Trainer::end_step(bool ok) {
  in_step_ = false;
  if (!ok) {
    for (void* p : step_live_) ctx_->arena.free(p);
    clear_boundaries();
    // the event slot of the failed step is recorded-but-unfinished at most
    for (int k = 0; k < kEvRing; ++k)
      if (step_ev_iter_[k] == iter_) step_ev_iter_[k] = -1;
  }
  step_live_.clear();
}

void Trainer::attach_dp(DataParallel* dp, int64_t bucket_bytes) {
  dp_ = dp;
  buckets_.clear();
  if (dp_ != nullptr) buckets_ = plan_buckets(unit_off_, std::max<int64_t>(bucket_bytes / 4, 1));
}

// Gradient unit `unit` is final on stream s: ship the bucket that ends here.
void Trainer::dp_unit_done(int unit, cudaStream_t s) {
  if (dp_ == nullptr) return;
  for (const Bucket& b : buckets_)
    if (b.after_unit == unit) dp_->allreduce_after(g32_ + b.begin, b.end - b.begin, s);
}

// With a native DP communicator attached the gradients were summed across
// ranks during backward: wait for the last bucket and average (1 / world).
void Trainer::optimizer_step(float grad_scale, cudaStream_t s) {
  if (dp_ != nullptr) {
    dp_->join(s);
    grad_scale /= static_cast<float>(dp_->world());
  }
  adam_t_ += 1;
  mimose_ops::AdamWArgs a;
  a.lr = t_.lr;
  a.beta1 = t_.beta1;
  a.beta2 = t_.beta2;
  a.eps = t_.adam_eps;
  a.weight_decay = t_.weight_decay;
  a.max_grad_norm = t_.max_grad_norm;
  a.grad_scale = grad_scale;
  a.bc1 = 1.f - std::pow(t_.beta1, (float)adam_t_);
  a.bc2 = 1.f - std::pow(t_.beta2, (float)adam_t_);
  if (a.max_grad_norm > 0.f) ck(mimose_ops::grad_norm2(g32_, nparam_, norm_partial_, norm2_, s), "grad_norm2");
  ck(mimose_ops::adamw(p32_, am_, av_, g32_, p16_, nparam_, decay_chunk_, norm2_, a, s), "adamw");
}

// Checks host labels against the head's layout; for MLM writes the masked
// row indices / labels to pos/lab and returns their count, for LM returns the
// number of labelled positions.
static int check_labels(const mimose_model_cfg& m, const int32_t* lb, int n, int S,
                        int32_t* pos, int32_t* lab) {
  int cnt = 0;
  for (int q = 0; q < n; ++q) {
    const int32_t v = lb[q];
    switch (m.head) {
      case MIMOSE_HEAD_MC:
        if (v < 0 || v >= m.num_choices) throw std::runtime_error("label out of range");
        break;
      case MIMOSE_HEAD_QA:
        if (v < 0 || v >= S) throw std::runtime_error("span label out of range");
        break;
      default:
        if (v < -1 || v >= m.vocab) throw std::runtime_error("token label out of range");
        if (v >= 0) {
          if (pos) {
            pos[cnt] = q;
            lab[cnt] = v;
          }
          ++cnt;
        }
    }
  }
  return cnt;
}

// Device-resident labels of the token heads: the loss normaliser (LM) and
// the masked-row list (MLM) are host quantities, so the labels are read back
// once (the stream is synchronised) and the MLM row list is uploaded.
void Trainer::device_labels(StepInputs& in, int B, int S, cudaStream_t s) {
  if (m_.head != MIMOSE_HEAD_LM && m_.head != MIMOSE_HEAD_MLM) return;
  const int64_t T = (int64_t)B * S;
  std::vector<int32_t> lb(static_cast<size_t>(T)), pos(static_cast<size_t>(2 * T));
  ck(cudaMemcpyAsync(lb.data(), in.labels, T * 4, cudaMemcpyDeviceToHost, s), "D2H labels");
  ck(cudaStreamSynchronize(s), "label sync");
  const bool mlm = m_.head == MIMOSE_HEAD_MLM;
  const int cnt = check_labels(m_, lb.data(), (int)T, S, mlm ? pos.data() : nullptr,
                               mlm ? pos.data() + T : nullptr);
  in.n_valid = cnt;
  if (!mlm || cnt == 0) return;
  std::memmove(pos.data() + cnt, pos.data() + T, cnt * 4);
  auto* d = static_cast<int32_t*>(take((int64_t)2 * cnt * 4 + 64, kTagInput));
  ck(cudaMemcpyAsync(d, pos.data(), (int64_t)2 * cnt * 4, cudaMemcpyHostToDevice, s), "H2D rows");
  ck(cudaStreamSynchronize(s), "label sync");
  in.mask_pos = d;
  in.mask_lab = d + cnt;
  in.n_mask = cnt;
}

void Trainer::release_device_labels(StepInputs& in) {
  if (in.mask_pos == nullptr) return;
  void* p = const_cast<int32_t*>(in.mask_pos);
  drop(p);
  in.mask_pos = in.mask_lab = nullptr;
}

int Trainer::label_count(int B, int S) const {
  switch (m_.head) {
    case MIMOSE_HEAD_MC: return B / m_.num_choices;
    case MIMOSE_HEAD_QA: return 2 * B;
    default: return B * S;
  }
}

void Trainer::step_host(const int32_t* tokens, const int32_t* types, const int32_t* labels, int B,
                        int S, int do_optimizer, cudaStream_t s, mimose_step_report* rep,
                        bool sync) {
  const int64_t T = (int64_t)B * S;
  const int Q = label_count(B, S);
  const bool mlm = m_.head == MIMOSE_HEAD_MLM;
  if (7 * T + Q + 1 > stage_elems_) throw std::runtime_error("staging buffer too small");
  // double-buffered pinned staging: wait for the H2D that last read this slot
  const int k = static_cast<int>(iter_ & 1);
  if (stage_used_[k]) ck(cudaEventSynchronize(stage_ev_[k]), "staging wait");
  int32_t* tk = h_stage_[k];
  int32_t* ty = tk + T;
  int32_t* lb = ty + T;
  int32_t* pm = lb + Q;
  int32_t* sg = pm + T;
  int32_t* ui = sg + T + 1;
  std::memcpy(tk, tokens, T * 4);
  if (types && m_.type_vocab > 0) std::memcpy(ty, types, T * 4);
  else std::memset(ty, 0, T * 4);
  std::memcpy(lb, labels, Q * 4);
  for (int64_t i = 0; i < T; ++i)
    if (ty[i] < 0 || ty[i] >= std::max(1, m_.type_vocab)) throw std::runtime_error("token type out of range");
  const int nu = build_token_tables(tk, T, m_.vocab, pm, sg, ui);
  // contiguous upload (uid packed right after seg, MLM rows after uid)
  std::memmove(sg + nu + 1, ui, nu * 4);
  int32_t* mp = sg + nu + 1 + nu;
  const int cnt = check_labels(m_, lb, Q, S, mlm ? mp : nullptr, mlm ? mp + T : nullptr);
  if (mlm) std::memmove(mp + cnt, mp + T, cnt * 4);
  const int64_t n_in = 2 * T + Q + T + (nu + 1) + nu + (mlm ? 2 * cnt : 0);
  int32_t* d = static_cast<int32_t*>(take(n_in * 4 + 64, kTagInput));
  ck(cudaMemcpyAsync(d, h_stage_[k], n_in * 4, cudaMemcpyHostToDevice, s), "H2D inputs");
  ck(cudaEventRecord(stage_ev_[k], s), "event");
  stage_used_[k] = true;
  StepInputs in;
  in.tokens = d;
  in.types = d + T;
  in.labels = d + 2 * T;
  in.perm = d + 2 * T + Q;
  in.seg = in.perm + T;
  in.uid = in.seg + nu + 1;
  in.n_unique = nu;
  in.n_valid = cnt;
  if (mlm) {
    in.mask_pos = in.uid + nu;
    in.mask_lab = in.mask_pos + cnt;
    in.n_mask = cnt;
  }
  const int64_t this_iter = iter_;
  forward_backward(in, B, S, s, rep);
  void* dv = d;
  drop(dv);
  if (do_optimizer) {
    if (hook_) {
      // the hook sees final gradients: bucketed all-reduces still in flight
      // on the communicator's stream are joined first (the optimizer's own
      // join then has nothing left to wait for)
      if (dp_ != nullptr) dp_->join(s);
      hook_(hook_user_, g32_, nparam_, s);
    }
    optimizer_step(1.f, s);
  }
  // loss read-back into a pinned ring slot (read later by loss(iter) or now)
  const int j = static_cast<int>(this_iter % kLossRing);
  if (loss_iter_[j] >= 0) ck(cudaEventSynchronize(loss_ev_[j]), "loss slot wait");
  ck(cudaMemcpyAsync(h_loss_ + j, d_loss_, sizeof(float), cudaMemcpyDeviceToHost, s), "D2H loss");
  ck(cudaEventRecord(loss_ev_[j], s), "event");
  loss_iter_[j] = this_iter;
  if (sync) {
    const float v = loss(this_iter);
    if (rep) rep->loss = v;
  }
}

float Trainer::loss(int64_t iter) {
  const int j = static_cast<int>(iter % kLossRing);
  if (iter < 0 || loss_iter_[j] != iter)
    throw std::runtime_error("loss of iteration " + std::to_string(iter) + " is not available");
  ck(cudaEventSynchronize(loss_ev_[j]), "loss wait");
  const float v = h_loss_[j];
  if (mimose_step_report* h = history_row(iter)) h->loss = v;
  return v;
}

}  // namespace mimose_rt

// =================================================================== C ABI
using mimose_capi::fail;
using mimose_rt::Trainer;

struct mimose_trainer {
  Trainer* impl = nullptr;
};
struct mimose_dp {
  mimose_rt::DataParallel* impl = nullptr;
};
struct mimose_saved {
  bool embed = false;
  mimose_rt::UnitSave unit;
  mimose_rt::EmbedSave emb;
};

namespace {
template <typename Fn>
int guarded(const char* what, Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::exception& e) {
    return fail(std::string(what) + ": " + e.what());
  }
}
// one training step inside the trainer's step scope (see begin_step)
template <typename Fn>
void in_step(Trainer* t, Fn&& fn) {
  t->begin_step();
  try {
    fn();
  } catch (...) {
    t->end_step(false);
    throw;
  }
  t->end_step(true);
}
char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}
}  // namespace

extern "C" {

int mimose_trainer_create(mimose_ctx* ctx, const mimose_model_cfg* m, const mimose_train_cfg* t,
                          mimose_trainer** out) {
  if (!ctx || !m || !t || !out) return fail("mimose_trainer_create: null argument");
  return guarded("mimose_trainer_create", [&] {
    auto* tr = new mimose_trainer();
    try {
      tr->impl = new Trainer(ctx, *m, *t);
    } catch (...) {
      delete tr;
      throw;
    }
    *out = tr;
  });
}

int mimose_trainer_destroy(mimose_trainer* tr) {
  if (tr) {
    delete tr->impl;
    delete tr;
  }
  return 0;
}

int mimose_trainer_step(mimose_trainer* tr, const int32_t* tokens, const int32_t* types,
                        const int32_t* labels, int batch, int seq, void* stream,
                        mimose_step_report* rep) {
  return guarded("mimose_trainer_step", [&] {
    in_step(tr->impl, [&] {
      tr->impl->step_host(tokens, types, labels, batch, seq, 1, static_cast<cudaStream_t>(stream), rep);
    });
  });
}

int mimose_trainer_step_async(mimose_trainer* tr, const int32_t* tokens, const int32_t* types,
                              const int32_t* labels, int batch, int seq, void* stream,
                              mimose_step_report* rep) {
  return guarded("mimose_trainer_step_async", [&] {
    in_step(tr->impl, [&] {
      tr->impl->step_host(tokens, types, labels, batch, seq, 1, static_cast<cudaStream_t>(stream),
                          rep, /*sync=*/false);
    });
  });
}

int mimose_trainer_loss(mimose_trainer* tr, int64_t iter, float* loss) {
  return guarded("mimose_trainer_loss", [&] { *loss = tr->impl->loss(iter); });
}

int mimose_trainer_forward_backward(mimose_trainer* tr, const int32_t* tokens,
                                    const int32_t* types, const int32_t* labels, int batch,
                                    int seq, void* stream, mimose_step_report* rep) {
  return guarded("mimose_trainer_forward_backward", [&] {
    in_step(tr->impl, [&] {
      tr->impl->step_host(tokens, types, labels, batch, seq, 0, static_cast<cudaStream_t>(stream), rep);
    });
  });
}

int mimose_trainer_step_device(mimose_trainer* tr, const int32_t* tokens, const int32_t* types,
                               const int32_t* labels, const int32_t* perm, const int32_t* seg,
                               const int32_t* uid, int n_unique, int batch, int seq,
                               int do_optimizer, void* stream, mimose_step_report* rep) {
  return guarded("mimose_trainer_step_device", [&] {
    mimose_rt::StepInputs in;
    in.tokens = tokens; in.types = types; in.labels = labels;
    in.perm = perm; in.seg = seg; in.uid = uid; in.n_unique = n_unique;
    auto s = static_cast<cudaStream_t>(stream);
    in_step(tr->impl, [&] {
      tr->impl->device_labels(in, batch, seq, s);
      tr->impl->forward_backward(in, batch, seq, s, rep);
      tr->impl->release_device_labels(in);
    });
    if (do_optimizer) tr->impl->optimizer_step(1.f, s);
  });
}

int mimose_trainer_optimizer_step(mimose_trainer* tr, float grad_scale, void* stream) {
  return guarded("mimose_trainer_optimizer_step", [&] {
    tr->impl->optimizer_step(grad_scale, static_cast<cudaStream_t>(stream));
  });
}

int mimose_trainer_force_plan(mimose_trainer* tr, const int* ids, int n, int active) {
  return guarded("mimose_trainer_force_plan", [&] { tr->impl->set_forced_plan(ids, n, active); });
}

int mimose_trainer_set_grad_hook(mimose_trainer* tr, mimose_grad_hook fn, void* user) {
  tr->impl->set_grad_hook(fn, user);
  return 0;
}

int mimose_trainer_buffers(mimose_trainer* tr, float** p32, void** p16, float** g32, int64_t* n,
                           float** d_loss, float** d_logits) {
  if (p32) *p32 = tr->impl->params_f32();
  if (p16) *p16 = tr->impl->params_bf16();
  if (g32) *g32 = tr->impl->grads();
  if (n) *n = tr->impl->num_params();
  if (d_loss) *d_loss = tr->impl->d_loss();
  if (d_logits) *d_logits = tr->impl->d_logits();
  return 0;
}

int mimose_trainer_param_count(mimose_trainer* tr) { return tr->impl->param_count(); }

int mimose_trainer_param_info(mimose_trainer* tr, int i, const char** name, int64_t* offset,
                              int64_t* numel) {
  return guarded("mimose_trainer_param_info", [&] { tr->impl->param_info(i, name, offset, numel); });
}

int mimose_trainer_sync_params(mimose_trainer* tr, void* stream) {
  return guarded("mimose_trainer_sync_params", [&] {
    mimose_rt::ck(mimose_ops::f32_to_bf16(tr->impl->params_f32(), tr->impl->params_bf16(),
                                          tr->impl->num_params(), static_cast<cudaStream_t>(stream)),
                  "f32_to_bf16");
  });
}

int mimose_trainer_samples_csv(mimose_trainer* tr, char** out) {
  return guarded("mimose_trainer_samples_csv", [&] {
    std::ostringstream os;
    mimose::write_samples_csv(tr->impl->collector().samples, os);
    *out = dup_string(os.str());
  });
}

int mimose_trainer_estimator_text(mimose_trainer* tr, char** out) {
  return guarded("mimose_trainer_estimator_text", [&] {
    *out = dup_string(mimose::estimator_to_string(tr->impl->estimator()));
  });
}

int mimose_trainer_model_text(mimose_trainer* tr, char** out) {
  return guarded("mimose_trainer_model_text", [&] {
    *out = dup_string(mimose::model_to_string(tr->impl->spec()));
  });
}

int mimose_trainer_report(mimose_trainer* tr, char** summary, char** csv) {
  return guarded("mimose_trainer_report", [&] {
    const mimose::SimReport rep = tr->impl->report();
    std::ostringstream s, c;
    mimose::write_report_summary(rep, s);
    mimose::write_report_csv(rep, c);
    *summary = dup_string(s.str());
    *csv = dup_string(c.str());
  });
}

int mimose_trainer_info(mimose_trainer* tr, int64_t* constant_bytes, int64_t* reserve_bytes,
                        int64_t* budget, int* trained, int64_t* cache_hits,
                        int64_t* cache_misses) {
  if (constant_bytes) *constant_bytes = tr->impl->constant_bytes();
  if (reserve_bytes) *reserve_bytes = tr->impl->reserve_bytes();
  if (budget) *budget = tr->impl->sched().budget_bytes;
  if (trained) *trained = tr->impl->trained() ? 1 : 0;
  if (cache_hits) *cache_hits = tr->impl->cache().hits;
  if (cache_misses) *cache_misses = tr->impl->cache().misses;
  return 0;
}

void mimose_free_string(char* s) { std::free(s); }

int mimose_build_token_tables(const int32_t* tokens, int64_t T, int vocab, int32_t* perm,
                              int32_t* seg, int32_t* uid, int* n_unique) {
  return guarded("mimose_build_token_tables", [&] {
    *n_unique = mimose_rt::build_token_tables(tokens, T, vocab, perm, seg, uid);
  });
}

int mimose_dp_unique_id(void* out128) {
  if (!out128) return fail("mimose_dp_unique_id: null argument");
  return guarded("mimose_dp_unique_id", [&] { mimose_rt::DataParallel::unique_id(out128); });
}

int mimose_dp_create(int device, const void* uid, int rank, int world, mimose_dp** out) {
  if (!uid || !out) return fail("mimose_dp_create: null argument");
  return guarded("mimose_dp_create", [&] {
    auto* dp = new mimose_dp();
    try {
      dp->impl = new mimose_rt::DataParallel(device, uid, rank, world);
    } catch (...) {
      delete dp;
      throw;
    }
    *out = dp;
  });
}

// ------------------------------------------------------- layer-level ABI
static mimose_rt::StepInputs io_inputs(const mimose_layer_io* io) {
  mimose_rt::StepInputs in;
  in.tokens = io->tokens; in.types = io->types; in.labels = io->labels;
  in.perm = io->perm; in.seg = io->seg; in.uid = io->uid; in.n_unique = io->n_unique;
  return in;
}

int mimose_trainer_units(mimose_trainer* tr, int* n_units) {
  if (!tr || !n_units) return fail("mimose_trainer_units: null argument");
  *n_units = tr->impl->units();
  return 0;
}

int mimose_embed_fwd(mimose_trainer* tr, const mimose_layer_io* io, void** h0,
                     mimose_saved** saved, void* stream) {
  if (!tr || !io || !h0 || !saved) return fail("mimose_embed_fwd: null argument");
  return guarded("mimose_embed_fwd", [&] {
    Trainer* t = tr->impl;
    const auto g = t->geometry(io->batch, io->seq, io->step);
    auto* sv = new mimose_saved();
    sv->embed = true;
    try {
      *h0 = t->embed_fwd(io_inputs(io), g, sv->emb, static_cast<cudaStream_t>(stream));
    } catch (...) {
      delete sv;
      throw;
    }
    *saved = sv;
  });
}

int mimose_layer_fwd(mimose_trainer* tr, int unit, const mimose_layer_io* io, const void* x_in,
                     void* x_out, mimose_saved** saved, void* stream) {
  if (!tr || !io || !x_in || !x_out) return fail("mimose_layer_fwd: null argument");
  return guarded("mimose_layer_fwd", [&] {
    Trainer* t = tr->impl;
    const auto g = t->geometry(io->batch, io->seq, io->step);
    if (saved == nullptr) {
      t->unit_fwd(unit, x_in, x_out, nullptr, g, static_cast<cudaStream_t>(stream));
      return;
    }
    auto* sv = new mimose_saved();
    try {
      t->unit_fwd(unit, x_in, x_out, &sv->unit, g, static_cast<cudaStream_t>(stream));
    } catch (...) {
      t->free_save(sv->unit);
      delete sv;
      throw;
    }
    *saved = sv;
  });
}

int mimose_layer_recompute(mimose_trainer* tr, int unit, const mimose_layer_io* io,
                           const void* x_in, void* x_out, mimose_saved** saved, void* stream) {
  if (!tr || !io || !x_in || !x_out || !saved) return fail("mimose_layer_recompute: null argument");
  return guarded("mimose_layer_recompute", [&] {
    Trainer* t = tr->impl;
    const auto g = t->geometry(io->batch, io->seq, io->step);
    auto* sv = new mimose_saved();
    try {
      t->unit_fwd(unit, x_in, x_out, &sv->unit, g, static_cast<cudaStream_t>(stream), true);
    } catch (...) {
      t->free_save(sv->unit);
      delete sv;
      throw;
    }
    *saved = sv;
  });
}

int mimose_layer_release(mimose_trainer* tr, int unit) {
  if (!tr || unit < 0 || unit >= tr->impl->units()) return fail("mimose_layer_release: bad argument");
  return guarded("mimose_layer_release", [&] { tr->impl->drop_boundary(unit); });
}

int mimose_layer_bwd(mimose_trainer* tr, int unit, const mimose_layer_io* io, const void* x_in,
                     mimose_saved* saved, void* dy, void** dx, void* stream) {
  if (!tr || !io || !x_in || !saved || saved->embed || !dy || !dx)
    return fail("mimose_layer_bwd: bad argument");
  return guarded("mimose_layer_bwd", [&] {
    Trainer* t = tr->impl;
    const auto g = t->geometry(io->batch, io->seq, io->step);
    *dx = t->unit_bwd(unit, x_in, saved->unit, dy, &t->pending_aux_, g,
                      static_cast<cudaStream_t>(stream));
    delete saved;
  });
}

int mimose_head_fwd_bwd(mimose_trainer* tr, const mimose_layer_io* io, const void* last,
                        void** dlast, void* stream) {
  if (!tr || !io || !last || !dlast) return fail("mimose_head_fwd_bwd: null argument");
  return guarded("mimose_head_fwd_bwd", [&] {
    Trainer* t = tr->impl;
    auto s = static_cast<cudaStream_t>(stream);
    auto in = io_inputs(io);
    t->device_labels(in, io->batch, io->seq, s);
    const auto g = t->geometry(io->batch, io->seq, io->step);
    try {
      *dlast = t->head_block(in, last, g, s);
    } catch (...) {
      t->release_device_labels(in);
      throw;
    }
    t->release_device_labels(in);
  });
}

int mimose_embed_bwd(mimose_trainer* tr, const mimose_layer_io* io, mimose_saved* saved,
                     void* h0, void* dh0, void* stream) {
  if (!tr || !io || !saved || !saved->embed || !h0 || !dh0)
    return fail("mimose_embed_bwd: bad argument");
  return guarded("mimose_embed_bwd", [&] {
    Trainer* t = tr->impl;
    const auto g = t->geometry(io->batch, io->seq, io->step);
    t->embed_bwd(io_inputs(io), g, saved->emb, h0, dh0, static_cast<cudaStream_t>(stream));
    delete saved;
  });
}

int mimose_saved_free(mimose_trainer* tr, mimose_saved* saved) {
  if (!tr || !saved) return 0;
  return guarded("mimose_saved_free", [&] {
    if (saved->embed) {
      tr->impl->drop(saved->emb.z0);
      tr->impl->drop(saved->emb.st0);
    } else {
      tr->impl->free_save(saved->unit);
    }
    delete saved;
  });
}

int mimose_adamw_step(mimose_trainer* tr, float grad_scale, void* stream) {
  return mimose_trainer_optimizer_step(tr, grad_scale, stream);
}

int mimose_event_create(void** ev) {
  if (!ev) return fail("mimose_event_create: null argument");
  return guarded("mimose_event_create", [&] {
    cudaEvent_t e = nullptr;
    mimose_rt::ck(cudaEventCreate(&e), "cudaEventCreate");
    *ev = e;
  });
}

int mimose_event_record(void* ev, void* stream) {
  return guarded("mimose_event_record", [&] {
    mimose_rt::ck(cudaEventRecord(static_cast<cudaEvent_t>(ev), static_cast<cudaStream_t>(stream)),
                  "cudaEventRecord");
  });
}

int mimose_event_elapsed(void* start, void* end, float* ms) {
  if (!ms) return fail("mimose_event_elapsed: null argument");
  return guarded("mimose_event_elapsed", [&] {
    mimose_rt::ck(cudaEventSynchronize(static_cast<cudaEvent_t>(end)), "cudaEventSynchronize");
    mimose_rt::ck(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(start),
                                       static_cast<cudaEvent_t>(end)),
                  "cudaEventElapsedTime");
  });
}

int mimose_event_destroy(void* ev) {
  if (ev) cudaEventDestroy(static_cast<cudaEvent_t>(ev));
  return 0;
}

int mimose_dp_create_custom(int device, int rank, int world, mimose_dp_reduce_fn fn, void* user,
                            mimose_dp** out) {
  if (!fn || !out) return fail("mimose_dp_create_custom: null argument");
  return guarded("mimose_dp_create_custom", [&] {
    auto* dp = new mimose_dp();
    try {
      dp->impl = new mimose_rt::DataParallel(device, rank, world, fn, user);
    } catch (...) {
      delete dp;
      throw;
    }
    *out = dp;
  });
}

int mimose_dp_device_bytes(mimose_dp* dp, int64_t* out) {
  if (!dp || !out) return fail("mimose_dp_device_bytes: null argument");
  *out = dp->impl->device_bytes();
  return 0;
}

int mimose_dp_destroy(mimose_dp* dp) {
  if (!dp) return 0;
  return guarded("mimose_dp_destroy", [&] {
    delete dp->impl;
    delete dp;
  });
}

int mimose_dp_allreduce(mimose_dp* dp, void* buf, int64_t n, int dtype, int op, void* stream) {
  if (!dp || (!buf && n > 0)) return fail("mimose_dp_allreduce: null argument");
  return guarded("mimose_dp_allreduce", [&] {
    dp->impl->allreduce(buf, n, dtype, op, static_cast<cudaStream_t>(stream));
  });
}

int mimose_trainer_attach_dp(mimose_trainer* tr, mimose_dp* dp, int64_t bucket_bytes) {
  if (!tr) return fail("mimose_trainer_attach_dp: null trainer");
  return guarded("mimose_trainer_attach_dp", [&] {
    tr->impl->attach_dp(dp ? dp->impl : nullptr, bucket_bytes);
  });
}

static void write_triples(const std::vector<mimose_rt::Bucket>& b, int64_t* out, int cap, int* n) {
  *n = static_cast<int>(b.size());
  for (int i = 0; i < cap && i < static_cast<int>(b.size()); ++i) {
    out[3 * i] = b[static_cast<size_t>(i)].after_unit;
    out[3 * i + 1] = b[static_cast<size_t>(i)].begin;
    out[3 * i + 2] = b[static_cast<size_t>(i)].end;
  }
}

int mimose_trainer_dp_buckets(mimose_trainer* tr, int64_t* triples, int cap, int* n) {
  if (!tr || !n || (cap > 0 && !triples)) return fail("mimose_trainer_dp_buckets: null argument");
  write_triples(tr->impl->dp_buckets(), triples, cap, n);
  return 0;
}

int mimose_dp_plan_buckets(const int64_t* unit_off, int n_units, int64_t bucket_elems,
                           int64_t* triples, int cap, int* n) {
  if (!unit_off || !n || n_units < 0 || (cap > 0 && !triples))
    return fail("mimose_dp_plan_buckets: bad argument");
  return guarded("mimose_dp_plan_buckets", [&] {
    std::vector<int64_t> off(unit_off, unit_off + n_units + 1);
    for (int u = 0; u < n_units; ++u)
      if (off[static_cast<size_t>(u) + 1] < off[static_cast<size_t>(u)])
        throw std::runtime_error("unit offsets must be non-decreasing");
    write_triples(mimose_rt::plan_buckets(off, std::max<int64_t>(bucket_elems, 1)), triples, cap, n);
  });
}

}  // extern "C"
