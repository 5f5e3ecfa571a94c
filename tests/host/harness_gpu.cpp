// Compiled C++ host of the reference's training loop over the two C ABIs.
//
// Reproduces the Mimose branch of reference proj/include/mimose/harness.hpp:
// 215-296 - sheltered collection window, conservative all-units iterations for
// sizes already seen inside the window, fallback collection while fewer than
// order + 1 sizes are known, the reduced-order fit, then the responsive
// lookup_or_plan per iteration (and every-new-size collection + refit) - with
// the two simulated iterations it makes (collect_iteration, collector.hpp:115,
// and simulate_iteration, simulator.hpp:104, at harness.hpp:189,196,221,231,
// 240,265,286) replaced by REAL GPU iterations driven unit by unit through
// include/mimose_cuda.h (mimose_embed_* / mimose_layer_* / mimose_head_* /
// mimose_adamw_step / mimose_event_*), and the planner reached only through
// include/mimose_planner.h (mimose_planner_fit, mimose_planner_session_*).
// The collector's bytes are the arena's requested-bytes delta around each
// unit's measuring forward (mimose_mem_stats_get), its times CUDA events.
//
// usage: harness_gpu CONFIG STEPS > rows
//   CONFIG: "key value" lines (model / train config, budget, device)
//   STEPS : binary [n][B] then per step [S][tokens B*S][types B*S][n_lab][labels]
// prints per iteration: iter x phase cache_hit insufficient mask_hex loss_bits_hex
// then "estimator" and the final estimator dump (estimator.hpp:182 format).
#include <cuda_runtime.h>

#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "mimose_cuda.h"
#include "mimose_planner.h"

namespace {

void die(const char* what, const char* msg) {
  std::fprintf(stderr, "%s: %s\n", what, msg ? msg : "");
  std::exit(2);
}
void ck(int rc, const char* what) {
  if (rc != 0) die(what, mimose_last_error());
}
void pk(int rc, const char* what) {
  if (rc != 0) die(what, mimose_planner_last_error());
}
void cu(cudaError_t e, const char* what) {
  if (e != cudaSuccess) die(what, cudaGetErrorString(e));
}

struct Step {
  int S = 0;
  std::vector<int32_t> tokens, types, labels;
};

struct Sample {
  int layer;
  int64_t x, bytes;
  float ms;
};

}  // namespace

int main(int argc, char** argv) {
  if (argc != 3) die("usage", "harness_gpu CONFIG STEPS");
  std::map<std::string, double> kv;
  {
    std::ifstream in(argv[1]);
    std::string k;
    double v;
    while (in >> k >> v) kv[k] = v;
  }
  auto I = [&](const char* k) { return static_cast<int>(kv.at(k)); };

  mimose_model_cfg m{};
  m.layers = I("layers"); m.hidden = I("hidden"); m.heads = I("heads"); m.ffn = I("ffn");
  m.vocab = I("vocab"); m.max_pos = I("max_pos"); m.type_vocab = I("type_vocab");
  m.num_choices = I("num_choices");
  m.hidden_dropout = static_cast<float>(kv.at("hidden_dropout"));
  m.attn_dropout = static_cast<float>(kv.at("attn_dropout"));
  m.ln_eps = static_cast<float>(kv.at("ln_eps"));
  m.init_std = static_cast<float>(kv.at("init_std"));
  m.seed = static_cast<uint64_t>(kv.at("seed"));
  m.arch = I("arch"); m.head = I("head"); m.causal = I("causal"); m.gelu_tanh = I("gelu_tanh");
  m.pad_token_id = I("pad_token_id");
  mimose_train_cfg t{};
  t.planner = 1;  // the trainer's own planner stays idle: this host plans
  t.batch = I("batch"); t.seq_min = I("seq_min"); t.seq_max = I("seq_max");
  t.reserve_bytes = -1; t.bucket_tolerance = kv.at("bucket_tolerance");
  t.cache_tolerance = kv.at("cache_tolerance");
  t.max_sheltered_iters = I("max_sheltered_iters");
  t.collect_new_sizes_always = I("collect_new_sizes_always");
  t.estimator_order = I("estimator_order");
  t.lr = static_cast<float>(kv.at("lr")); t.beta1 = 0.9f; t.beta2 = 0.999f; t.adam_eps = 1e-8f;
  t.weight_decay = 0.01f; t.max_grad_norm = 1.f;
  t.attn_fused = I("attn_fused"); t.reserve_per_size = 0; t.ckpt_unit = I("ckpt_unit");
  const int64_t budget = static_cast<int64_t>(kv.at("budget"));

  // steps
  std::vector<Step> steps;
  int B = 0;
  {
    std::ifstream in(argv[2], std::ios::binary);
    int32_t n = 0, b = 0;
    in.read(reinterpret_cast<char*>(&n), 4);
    in.read(reinterpret_cast<char*>(&b), 4);
    B = b;
    for (int i = 0; i < n; ++i) {
      Step s;
      int32_t S = 0, nl = 0;
      in.read(reinterpret_cast<char*>(&S), 4);
      s.S = S;
      s.tokens.resize(static_cast<size_t>(B) * S);
      s.types.resize(static_cast<size_t>(B) * S);
      in.read(reinterpret_cast<char*>(s.tokens.data()), 4 * s.tokens.size());
      in.read(reinterpret_cast<char*>(s.types.data()), 4 * s.types.size());
      in.read(reinterpret_cast<char*>(&nl), 4);
      s.labels.resize(nl);
      in.read(reinterpret_cast<char*>(s.labels.data()), 4 * nl);
      steps.push_back(std::move(s));
    }
  }

  cu(cudaSetDevice(I("device")), "cudaSetDevice");
  mimose_ctx* ctx = nullptr;
  ck(mimose_ctx_create(I("device"), budget, &ctx), "ctx");
  mimose_trainer* tr = nullptr;
  ck(mimose_trainer_create(ctx, &m, &t, &tr), "trainer");
  int U = 0;
  ck(mimose_trainer_units(tr, &U), "units");
  int64_t constant = 0, reserve = 0, bgt = 0, hits = 0, misses = 0;
  int trained_flag = 0;
  ck(mimose_trainer_info(tr, &constant, &reserve, &bgt, &trained_flag, &hits, &misses), "info");
  char* model_text = nullptr;
  ck(mimose_trainer_model_text(tr, &model_text), "model text");
  float* d_loss = nullptr;
  ck(mimose_trainer_buffers(tr, nullptr, nullptr, nullptr, nullptr, &d_loss, nullptr), "buffers");
  cudaStream_t s = nullptr;
  cu(cudaStreamCreate(&s), "stream");
  std::vector<void*> ev(2 * static_cast<size_t>(U));
  for (auto& e : ev) ck(mimose_event_create(&e), "event");

  mimose_sched_cfg sc{};
  sc.budget_bytes = bgt;
  sc.reserve_bytes = reserve;
  sc.bucket_tolerance = t.bucket_tolerance;
  sc.cache_tolerance = t.cache_tolerance;
  sc.excess_includes_constant = 1;

  // collector state (collector.hpp:96-103) and planner state
  std::set<int64_t> seen;
  std::vector<Sample> samples;
  bool trained = false;
  std::string est_text;
  mimose_plan_session* session = nullptr;
  const int order_cfg = t.estimator_order;
  const int window = t.max_sheltered_iters;
  const bool every_new = t.collect_new_sizes_always != 0;
  const bool half = t.ckpt_unit == 1;

  auto refit = [&]() {
    const int order = std::min(order_cfg, static_cast<int>(seen.size()) - 1);
    std::ostringstream csv;
    csv << "layer_id,input_size,bytes,ms,valid\n";
    for (const Sample& sm : samples) {
      char buf[64];
      std::snprintf(buf, sizeof buf, "%.9g", static_cast<double>(sm.ms));
      csv << sm.layer << ',' << sm.x << ',' << sm.bytes << ',' << buf << ",1\n";
    }
    char* e = nullptr;
    pk(mimose_planner_fit(csv.str().c_str(), order, &e), "fit");
    est_text = e;
    mimose_planner_free(e);
    if (session == nullptr)
      pk(mimose_planner_session_create(est_text.c_str(), model_text, &sc, &session), "session");
    else
      pk(mimose_planner_session_set_estimator(session, est_text.c_str()), "set estimator");
  };

  for (size_t it = 0; it < steps.size(); ++it) {
    const Step& st = steps[it];
    const int S = st.S;
    const int64_t T = static_cast<int64_t>(B) * S;
    const int64_t x = T;
    const bool unseen = seen.count(x) == 0;
    // ---- the phase machine (harness.hpp:215-296)
    enum { kCollect, kSheltered, kFallback, kPlanned } phase = kPlanned;
    bool decided = false;
    if (!trained) {
      if ((unseen && static_cast<int64_t>(it) < window) || (every_new && unseen)) {
        phase = kCollect;  // should_collect (collector.hpp:190-196)
        decided = true;
      } else if (static_cast<int64_t>(it) < window) {
        phase = kSheltered;
        decided = true;
      } else if (unseen && static_cast<int>(seen.size()) < order_cfg + 1) {
        phase = kFallback;
        decided = true;
      } else {
        refit();
        trained = true;
      }
    }
    uint64_t mask = 0;
    int insufficient = 0, hit = 0;
    if (!decided) {
      if (every_new && unseen) {
        phase = kCollect;
      } else {
        phase = kPlanned;
        pk(mimose_planner_session_plan(session, x, -1, &mask, 1, &insufficient, &hit), "plan");
      }
    }
    const bool collect = phase == kCollect || phase == kFallback;
    std::vector<char> dropped(U, 1);
    if (phase == kPlanned)
      for (int u = 0; u < U; ++u) dropped[u] = (mask >> u) & 1u;

    // ---- inputs into the arena
    std::vector<int32_t> perm(T), seg(T + 1), uid(T);
    int nu = 0;
    ck(mimose_build_token_tables(st.tokens.data(), T, m.vocab, perm.data(), seg.data(), uid.data(),
                                 &nu), "token tables");
    const int64_t nin = 2 * T + static_cast<int64_t>(st.labels.size()) + T + (nu + 1) + nu + 8;
    void* din = nullptr;
    ck(mimose_alloc(ctx, nin * 4, 6, &din), "alloc inputs");
    int32_t* d = static_cast<int32_t*>(din);
    mimose_layer_io io{};
    io.tokens = d;
    io.types = d + T;
    io.labels = d + 2 * T;
    io.perm = io.labels + st.labels.size();
    io.seg = io.perm + T;
    io.uid = io.seg + nu + 1;
    io.n_unique = nu;
    io.batch = B;
    io.seq = S;
    io.step = static_cast<int64_t>(it);
    cu(cudaMemcpyAsync(const_cast<int32_t*>(io.tokens), st.tokens.data(), 4 * T, cudaMemcpyHostToDevice, s), "h2d");
    cu(cudaMemcpyAsync(const_cast<int32_t*>(io.types), st.types.data(), 4 * T, cudaMemcpyHostToDevice, s), "h2d");
    cu(cudaMemcpyAsync(const_cast<int32_t*>(io.labels), st.labels.data(), 4 * st.labels.size(),
                       cudaMemcpyHostToDevice, s), "h2d");
    cu(cudaMemcpyAsync(const_cast<int32_t*>(io.perm), perm.data(), 4 * T, cudaMemcpyHostToDevice, s), "h2d");
    cu(cudaMemcpyAsync(const_cast<int32_t*>(io.seg), seg.data(), 4 * (nu + 1), cudaMemcpyHostToDevice, s), "h2d");
    cu(cudaMemcpyAsync(const_cast<int32_t*>(io.uid), uid.data(), 4 * nu, cudaMemcpyHostToDevice, s), "h2d");

    // ---- forward
    void* h0 = nullptr;
    mimose_saved* esave = nullptr;
    ck(mimose_embed_fwd(tr, &io, &h0, &esave, s), "embed fwd");
    std::vector<void*> out(U, nullptr);
    std::vector<mimose_saved*> sv(U, nullptr);
    std::vector<int64_t> measured(U, 0);
    for (int u = 0; u < U; ++u) {
      const void* in = u == 0 ? h0 : out[u - 1];
      if (collect) {
        // measuring pass: full save set, arena requested-bytes delta, then
        // only the output (the checkpoint boundary) is kept (collector.hpp:138-156)
        mimose_mem_stats a{}, b{};
        ck(mimose_mem_stats_get(ctx, &a), "stats");
        ck(mimose_event_record(ev[2 * u], s), "event");
        ck(mimose_alloc(ctx, 2 * T * m.hidden, 4, &out[u]), "alloc out");
        ck(mimose_layer_fwd(tr, u, &io, in, out[u], &sv[u], s), "layer fwd");
        ck(mimose_event_record(ev[2 * u + 1], s), "event");
        ck(mimose_mem_stats_get(ctx, &b), "stats");
        measured[u] = b.requested - a.requested;
        ck(mimose_saved_free(tr, sv[u]), "saved free");
        sv[u] = nullptr;
      } else if (dropped[u]) {
        ck(mimose_alloc(ctx, 2 * T * m.hidden, 4, &out[u]), "alloc out");
        ck(mimose_layer_fwd(tr, u, &io, in, out[u], nullptr, s), "layer fwd (no save)");
      } else {
        ck(mimose_alloc(ctx, 2 * T * m.hidden, 3, &out[u]), "alloc out");
        ck(mimose_layer_fwd(tr, u, &io, in, out[u], &sv[u], s), "layer fwd");
      }
      // half units: a block whose attention AND FFN halves are both dropped
      // keeps only the FFN half's output (the executor's rule, see
      // Trainer::replay_peak); h1 is regenerated before the FFN half's recompute
      if (half && u % 2 == 1 && (collect || (dropped[u] && dropped[u - 1]))) {
        ck(mimose_layer_release(tr, u - 1), "release h1");
        ck(mimose_free(ctx, out[u - 1]), "free h1");
        out[u - 1] = nullptr;
      }
    }
    void* dy = nullptr;
    ck(mimose_head_fwd_bwd(tr, &io, out[U - 1], &dy, s), "head");
    // ---- backward (dropped units recomputed right before their backward)
    for (int u = U - 1; u >= 0; --u) {
      if (u > 0 && out[u - 1] == nullptr) {  // h1 of a doubly-dropped block
        ck(mimose_alloc(ctx, 2 * T * m.hidden, 4, &out[u - 1]), "alloc h1");
        ck(mimose_layer_fwd(tr, u - 1, &io, u == 1 ? h0 : out[u - 2], out[u - 1], &sv[u - 1], s),
           "recompute attention half");
      }
      const void* in = u == 0 ? h0 : out[u - 1];
      if (sv[u] == nullptr) ck(mimose_layer_recompute(tr, u, &io, in, out[u], &sv[u], s), "recompute");
      void* dx = nullptr;
      ck(mimose_layer_bwd(tr, u, &io, in, sv[u], dy, &dx, s), "layer bwd");
      ck(mimose_free(ctx, out[u]), "free out");
      dy = dx;
    }
    ck(mimose_embed_bwd(tr, &io, esave, h0, dy, s), "embed bwd");
    ck(mimose_adamw_step(tr, 1.f, s), "adamw");
    float loss = 0.f;
    cu(cudaMemcpyAsync(&loss, d_loss, 4, cudaMemcpyDeviceToHost, s), "d2h loss");
    cu(cudaStreamSynchronize(s), "sync");
    ck(mimose_free(ctx, din), "free inputs");

    // ---- collector commit (collector.hpp:129-184)
    if (collect && unseen) {
      for (int u = 0; u < U; ++u) {
        float ms = 0.f;
        ck(mimose_event_elapsed(ev[2 * u], ev[2 * u + 1], &ms), "elapsed");
        samples.push_back({u, x, measured[u], ms});
      }
      seen.insert(x);
      if (trained && every_new) refit();
    }
    uint32_t bits = 0;
    std::memcpy(&bits, &loss, 4);
    static const char* names[] = {"collect", "sheltered", "fallback-collect", "planned"};
    const unsigned long long shown =
        phase == kPlanned ? mask : (U >= 64 ? ~0ull : ((1ull << U) - 1));
    std::printf("%zu %" PRId64 " %s %d %d %llx %08x\n", it, x, names[phase], hit, insufficient,
                shown, bits);
  }
  std::printf("estimator\n%s", est_text.c_str());
  for (auto& e : ev) mimose_event_destroy(e);
  if (session) mimose_planner_session_destroy(session);
  mimose_free_string(model_text);
  mimose_trainer_destroy(tr);
  mimose_ctx_destroy(ctx);
  return 0;
}
