// mimose_gpu: the reference's command-line front end (reference
// proj/tools/mimose_main.cpp) driving REAL B200 training runs instead of the
// simulator. Same subcommand names, flag names / meanings and exit codes
// (0 ok, 1 error, 2 infeasible: mimose_main.cpp:22-24, report_exit_code), and
// the reports come out of the reference's own writers (harness.hpp:339-379)
// via mimose_trainer_report:
//
//   run           one experiment: --planner, --budget, --reserve, --bucket-tol,
//                 --cache-tol, --sheltered-iters, --collect-new-sizes, --order,
//                 --seed, --iters, --dist, --batch-multiplier, --out, --format
//   compare       grid over --budgets x --planners (mimose_main.cpp cmd_compare
//                 CSV columns)
//   fit           sheltered GPU collection over the workload's distinct sizes,
//                 then fit(); --dump-estimator / --dump-samples / --order
//   gen-workload  the seeded size sequence (workload.hpp sample_workload)
//
// Differences, all forced by running hardware instead of a replay:
//   * --model names a model preset (small4-h256, bert-base-mc, roberta-base-qa,
//     roberta-large-qa, gpt2-medium-lm, bert-large-mlm) or a file of
//     "key value" lines (mimose_model_cfg fields, starting from BERT-base);
//     the per-layer byte / time polynomials are MEASURED, not read.
//   * a size unit is one token position (sequence length S), and
//     --batch-multiplier is the number of sequences per step B, so the
//     planner's input size is x = B * S elements exactly as in the reference.
//   * --budget is the device arena (a hard cap); 0 = 90 % of free memory.
//     --reserve also takes "auto" (one measured reserve for every size);
//     without --reserve the reserve is sized per input size. An explicit
//     byte reserve below the real transients lets steps fail (exit 2).
//   * simulate / plan operate on .model documents only (no device work): use
//     the reference CLI over include/mimose (the headers are drop-in).
//   * extra flags: --device, --attn flash|materialised, --ckpt-unit block|half,
//     --dump-model / --dump-estimator / --dump-samples (GPU-measured profile
//     in the reference's text formats, model_spec.hpp:268, estimator.hpp:182,
//     collector.hpp:198), --data-seed.
#include <cuda_runtime.h>

#include <cctype>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <random>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "mimose_cuda.h"
#include "mimose_planner.h"

namespace {

constexpr int kOk = 0, kError = 1, kInfeasible = 2;

struct Fail : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// the budget cannot hold even the constant footprint (weights, gradients,
// AdamW state): the reference's "insufficient budget" outcome, exit code 2
struct Infeasible : Fail {
  using Fail::Fail;
};

void ck(int rc, const char* what) {
  if (rc != 0) throw Fail(std::string(what) + ": " + mimose_last_error());
}
void pk(int rc, const char* what) {
  if (rc != 0) throw Fail(std::string(what) + ": " + mimose_planner_last_error());
}

std::string take(char* s) {
  std::string r = s ? s : "";
  mimose_free_string(s);
  return r;
}

// byte quantities as the reference CLI accepts them: a number with an
// optional k / m / g / t (or ki / mi / ...) suffix in powers of 1024 and an
// optional trailing 'b'; rounded to the nearest byte (model_spec round_bytes)
int64_t parse_bytes(const std::string& text) {
  if (text.empty()) throw Fail("empty byte quantity");
  char* end = nullptr;
  const double v = std::strtod(text.c_str(), &end);
  if (end == text.c_str()) throw Fail("bad byte quantity: '" + text + "'");
  std::string suf;
  for (const char* p = end; *p; ++p) suf += static_cast<char>(std::tolower(*p));
  if (!suf.empty() && suf.back() == 'b') suf.pop_back();
  static const std::map<std::string, int> pow1024 = {
      {"", 0}, {"k", 1}, {"ki", 1}, {"m", 2}, {"mi", 2}, {"g", 3}, {"gi", 3}, {"t", 4}, {"ti", 4}};
  const auto it = pow1024.find(suf);
  if (it == pow1024.end()) throw Fail("bad byte suffix: '" + text + "'");
  return static_cast<int64_t>(std::llround(v * std::pow(1024.0, it->second)));
}

std::vector<std::string> split(const std::string& s, char sep = ',') {
  std::vector<std::string> out;
  std::string cur;
  std::istringstream in(s);
  while (std::getline(in, cur, sep))
    if (!cur.empty()) out.push_back(cur);
  return out;
}

// ------------------------------------------------------------ options
struct Opts {
  std::string model = "bert-base-mc", budget = "0", reserve, planner = "mimose";
  uint64_t seed = 1;
  int64_t iters = 2000;
  std::string dist = "uniform:30:332";
  int64_t batch_multiplier = 32;
  std::string out, format = "csv";
  int sheltered_iters = 10;
  bool collect_new_sizes = false;
  double bucket_tol = 0.10, cache_tol = 0.0;
  int order = 2;
  // fit / compare
  std::string dump_estimator, dump_samples, dump_model, budgets,
      planners = "mimose,static-max,dtr,none";
  // GPU-only
  int device = 0;
  std::string attn = "flash", ckpt_unit = "half";
  uint64_t data_seed = 0;
  bool data_seed_set = false;
};

// flags each subcommand accepts (mimose_main.cpp:254-319 + the GPU extras)
const std::map<std::string, std::set<std::string>> kFlags = {
    {"run", {"--model", "--planner", "--out", "--format", "--noise", "--noise-seed",
             "--sheltered-iters", "--collect-new-sizes", "--dtr-eviction-cost", "--order",
             "--budget", "--reserve", "--bucket-tol", "--cache-tol", "--excess-includes-constant",
             "--seed", "--iters", "--dist", "--batch-multiplier", "--device", "--attn",
             "--ckpt-unit", "--dump-model", "--dump-estimator", "--dump-samples", "--data-seed"}},
    {"compare", {"--model", "--budgets", "--planners", "--out", "--noise", "--noise-seed",
                 "--sheltered-iters", "--dtr-eviction-cost", "--budget", "--reserve",
                 "--bucket-tol", "--cache-tol", "--excess-includes-constant", "--seed", "--iters",
                 "--dist", "--batch-multiplier", "--device", "--attn", "--ckpt-unit",
                 "--data-seed"}},
    {"fit", {"--model", "--dump-estimator", "--dump-samples", "--noise", "--noise-seed", "--order",
             "--seed", "--iters", "--dist", "--batch-multiplier", "--device", "--attn",
             "--ckpt-unit", "--budget", "--data-seed", "--dump-model"}},
    {"gen-workload", {"--out", "--seed", "--iters", "--dist", "--batch-multiplier"}},
};

void usage(std::ostream& o) {
  o << "mimose_gpu: input-aware checkpointing, real B200 training runs\n"
       "usage: mimose_gpu {run|compare|fit|gen-workload} [--flag value ...]\n"
       "  (reference flags: see proj/tools/mimose_main.cpp; --model = preset or key/value "
       "file)\n";
}

Opts parse(const std::string& cmd, int argc, char** argv) {
  Opts o;
  const auto& allowed = kFlags.at(cmd);
  for (int i = 2; i < argc; ++i) {
    std::string f = argv[i], v;
    const auto eq = f.find('=');
    if (eq != std::string::npos) {
      v = f.substr(eq + 1);
      f = f.substr(0, eq);
    }
    if (!allowed.count(f)) throw Fail("unknown option for '" + cmd + "': " + f);
    if (f == "--collect-new-sizes") {  // flag
      o.collect_new_sizes = true;
      continue;
    }
    if (eq == std::string::npos) {
      if (i + 1 >= argc) throw Fail("option " + f + " needs a value");
      v = argv[++i];
    }
    auto num = [&](auto& dst) {
      std::istringstream in(v);
      if (!(in >> dst) || !in.eof()) throw Fail("bad value for " + f + ": '" + v + "'");
    };
    if (f == "--model") o.model = v;
    else if (f == "--planner") o.planner = v;
    else if (f == "--out") o.out = v;
    else if (f == "--format") o.format = v;
    else if (f == "--sheltered-iters") num(o.sheltered_iters);
    else if (f == "--order") num(o.order);
    else if (f == "--budget") o.budget = v;
    else if (f == "--reserve") o.reserve = v;
    else if (f == "--bucket-tol") num(o.bucket_tol);
    else if (f == "--cache-tol") num(o.cache_tol);
    else if (f == "--seed") num(o.seed);
    else if (f == "--iters") num(o.iters);
    else if (f == "--dist") o.dist = v;
    else if (f == "--batch-multiplier") num(o.batch_multiplier);
    else if (f == "--budgets") o.budgets = v;
    else if (f == "--planners") o.planners = v;
    else if (f == "--dump-estimator") o.dump_estimator = v;
    else if (f == "--dump-samples") o.dump_samples = v;
    else if (f == "--dump-model") o.dump_model = v;
    else if (f == "--device") num(o.device);
    else if (f == "--attn") o.attn = v;
    else if (f == "--ckpt-unit") o.ckpt_unit = v;
    else if (f == "--data-seed") { num(o.data_seed); o.data_seed_set = true; }
    else if (f == "--noise" || f == "--noise-seed" || f == "--dtr-eviction-cost") {
      // simulator knobs: measurements are real, eviction decisions are timed
      double x;
      num(x);
      if (f == "--noise" && x != 0.0)
        std::cerr << "note: --noise ignored (collector samples are measured)\n";
    } else if (f == "--excess-includes-constant") {
      if (v != "1" && v != "true")
        throw Fail("--excess-includes-constant: the GPU planner always includes the constant");
    }
  }
  if (o.iters < 0) throw Fail("--iters must be >= 0");
  if (o.batch_multiplier < 1) throw Fail("--batch-multiplier must be >= 1");
  if (o.format != "csv" && o.format != "summary")
    throw Fail("unknown report format '" + o.format + "'");
  if (!o.data_seed_set) o.data_seed = o.seed;
  return o;
}

// ------------------------------------------------------------ models
mimose_model_cfg bert_base() {
  mimose_model_cfg m{};
  m.layers = 12; m.hidden = 768; m.heads = 12; m.ffn = 3072; m.vocab = 30522; m.max_pos = 512;
  m.type_vocab = 2; m.num_choices = 4; m.hidden_dropout = 0.1f; m.attn_dropout = 0.1f;
  m.ln_eps = 1e-12f; m.init_std = 0.02f; m.seed = 1234; m.arch = MIMOSE_ARCH_BERT;
  m.head = MIMOSE_HEAD_MC; m.causal = 0; m.gelu_tanh = 0; m.pad_token_id = 0;
  return m;
}

// the BASELINE presets (paper_2209_02478_b200/trainer.py PRESETS)
mimose_model_cfg model_of(const std::string& name) {
  mimose_model_cfg m = bert_base();
  auto big = [&] { m.layers = 24; m.hidden = 1024; m.heads = 16; m.ffn = 4096; };
  if (name == "bert-base-mc") return m;
  if (name == "small4-h256") {
    m.layers = 4; m.hidden = 256; m.heads = 4; m.ffn = 1024;
    return m;
  }
  if (name == "roberta-base-qa" || name == "roberta-large-qa") {
    if (name == "roberta-large-qa") big();
    m.vocab = 50265; m.max_pos = 514; m.type_vocab = 1; m.ln_eps = 1e-5f; m.head = MIMOSE_HEAD_QA;
    return m;
  }
  if (name == "gpt2-medium-lm") {
    big();
    m.vocab = 50257; m.max_pos = 1024; m.type_vocab = 0; m.ln_eps = 1e-5f;
    m.arch = MIMOSE_ARCH_GPT2; m.head = MIMOSE_HEAD_LM; m.causal = 1; m.gelu_tanh = 1;
    m.pad_token_id = -1;
    return m;
  }
  if (name == "bert-large-mlm") {
    big();
    m.max_pos = 2048; m.head = MIMOSE_HEAD_MLM;
    return m;
  }
  // a file of "key value" lines over the BERT-base defaults
  std::ifstream in(name);
  if (!in) throw Fail("unknown model preset and unreadable file: '" + name + "'");
  std::string k;
  double v;
  while (in >> k >> v) {
    if (k == "layers") m.layers = (int)v;
    else if (k == "hidden") m.hidden = (int)v;
    else if (k == "heads") m.heads = (int)v;
    else if (k == "ffn") m.ffn = (int)v;
    else if (k == "vocab") m.vocab = (int)v;
    else if (k == "max_pos") m.max_pos = (int)v;
    else if (k == "type_vocab") m.type_vocab = (int)v;
    else if (k == "num_choices") m.num_choices = (int)v;
    else if (k == "hidden_dropout") m.hidden_dropout = (float)v;
    else if (k == "attn_dropout") m.attn_dropout = (float)v;
    else if (k == "ln_eps") m.ln_eps = (float)v;
    else if (k == "init_std") m.init_std = (float)v;
    else if (k == "seed") m.seed = (uint64_t)v;
    else if (k == "arch") m.arch = (int)v;
    else if (k == "head") m.head = (int)v;
    else if (k == "causal") m.causal = (int)v;
    else if (k == "gelu_tanh") m.gelu_tanh = (int)v;
    else if (k == "pad_token_id") m.pad_token_id = (int)v;
    else throw Fail("model file: unknown key '" + k + "'");
  }
  return m;
}

int planner_id(const std::string& p) {
  if (p == "mimose") return MIMOSE_PLANNER_MIMOSE;
  if (p == "static-max") return MIMOSE_PLANNER_STATIC;
  if (p == "dtr") return MIMOSE_PLANNER_DTR;
  if (p == "none") return MIMOSE_PLANNER_NONE;
  throw Fail("unknown planner '" + p + "'");
}

// ------------------------------------------------------------ workload + data
// sizes in units (S), reference sampler (workload.hpp:63) with multiplier 1
std::vector<int64_t> sizes_of(const Opts& o) {
  std::vector<int64_t> s(static_cast<size_t>(o.iters));
  if (o.iters > 0)
    pk(mimose_planner_sample_workload(o.dist.c_str(), 1, o.iters, o.seed, s.data()),
       "sample_workload");
  return s;
}

struct Batch {
  std::vector<int32_t> tok, typ, lab;
};

// synthetic task batch with the head's label layout (trainer.py synthetic_task_batch)
Batch make_batch(std::mt19937_64& g, const mimose_model_cfg& m, int B, int S) {
  Batch b;
  const size_t T = static_cast<size_t>(B) * S;
  b.tok.resize(T);
  b.typ.assign(T, 0);
  std::uniform_int_distribution<int32_t> tok(0, m.vocab - 1);
  for (auto& t : b.tok) t = tok(g);
  if (m.head == MIMOSE_HEAD_MC) {
    if (m.type_vocab > 1)
      for (int i = 0; i < B; ++i) {
        const int cut = std::uniform_int_distribution<int>(1, S > 1 ? S - 1 : 1)(g);
        for (int s = cut; s < S; ++s) b.typ[(size_t)i * S + s] = 1;
      }
    b.lab.resize(B / m.num_choices);
    for (auto& l : b.lab) l = std::uniform_int_distribution<int32_t>(0, m.num_choices - 1)(g);
  } else if (m.head == MIMOSE_HEAD_QA) {
    b.lab.resize(2 * (size_t)B);
    for (int i = 0; i < B; ++i) {
      const int st = std::uniform_int_distribution<int>(0, S - 1)(g);
      b.lab[2 * i] = st;
      b.lab[2 * i + 1] = std::min(S - 1, st + std::uniform_int_distribution<int>(0, 7)(g));
    }
  } else if (m.head == MIMOSE_HEAD_LM) {
    b.lab.assign(T, -1);
    for (int i = 0; i < B; ++i)
      for (int s = 0; s + 1 < S; ++s) b.lab[(size_t)i * S + s] = b.tok[(size_t)i * S + s + 1];
  } else {
    b.lab.assign(T, -1);
    std::bernoulli_distribution pick(0.15);
    for (size_t t = 0; t < T; ++t)
      if (pick(g)) b.lab[t] = b.tok[t];
    const size_t one = std::uniform_int_distribution<size_t>(0, T - 1)(g);
    b.lab[one] = b.tok[one];
  }
  return b;
}

// ------------------------------------------------------------ one GPU run
struct RunOut {
  std::string summary, csv, estimator, samples, model;
  int64_t failed = 0;
};

std::string summary_field(const std::string& summary, const std::string& key) {
  std::istringstream in(summary);
  std::string line;
  while (std::getline(in, line))
    if (line.rfind(key + ": ", 0) == 0) return line.substr(key.size() + 2);
  return "";
}

int64_t budget_bytes(const Opts& o) {
  const int64_t b = parse_bytes(o.budget);
  if (b > 0) return b;
  size_t free_b = 0, total = 0;
  if (cudaSetDevice(o.device) != cudaSuccess || cudaMemGetInfo(&free_b, &total) != cudaSuccess)
    throw Fail("cannot query device memory for --budget 0");
  return static_cast<int64_t>(0.9 * static_cast<double>(free_b));
}

RunOut run_gpu(const Opts& o, const std::string& planner, const std::string& budget_text,
               bool collect_all_sizes_only = false) {
  Opts local = o;
  local.budget = budget_text;
  const int64_t budget = budget_bytes(local);
  const mimose_model_cfg m = model_of(o.model);
  const std::vector<int64_t> sizes = sizes_of(o);
  const int B = static_cast<int>(o.batch_multiplier);
  if (m.head == MIMOSE_HEAD_MC && B % m.num_choices != 0)
    throw Fail("--batch-multiplier must be a multiple of num_choices for a multiple-choice head");
  // the model's input range is the distribution's [LO, HI] (the last two
  // fields of uniform:LO:HI | normal:MU:SIGMA:LO:HI | powerlaw:ALPHA:LO:HI),
  // as the reference requires of a workload (run_experiment range check)
  const std::vector<std::string> df = split(o.dist, ':');
  if (df.size() < 3) throw Fail("bad distribution '" + o.dist + "'");
  const int smin = std::atoi(df[df.size() - 2].c_str()), smax = std::atoi(df.back().c_str());
  if (smin < 1 || smax < smin) throw Fail("bad distribution range '" + o.dist + "'");
  if (smax > m.max_pos) throw Fail("workload size exceeds the model's position table");

  mimose_train_cfg t{};
  t.planner = planner_id(planner);
  t.batch = B;
  t.seq_min = smin;
  t.seq_max = smax;
  // --reserve BYTES: the scheduler reserve for every size, as the reference;
  // --reserve auto: one automatic reserve (the backward's transients and the
  // S-dependent extras measured at the largest size) for every size;
  // no --reserve: the trainer sizes an automatic reserve per input size
  t.reserve_bytes = (o.reserve.empty() || o.reserve == "auto") ? -1 : parse_bytes(o.reserve);
  t.reserve_per_size = o.reserve.empty() ? 1 : 0;
  t.bucket_tolerance = o.bucket_tol;
  t.cache_tolerance = o.cache_tol;
  t.max_sheltered_iters = collect_all_sizes_only ? (int)o.iters : o.sheltered_iters;
  t.collect_new_sizes_always = o.collect_new_sizes ? 1 : 0;
  t.estimator_order = o.order;
  t.lr = 5e-5f; t.beta1 = 0.9f; t.beta2 = 0.999f; t.adam_eps = 1e-8f; t.weight_decay = 0.01f;
  t.max_grad_norm = 1.f;
  if (o.attn != "flash" && o.attn != "materialised") throw Fail("--attn flash|materialised");
  t.attn_fused = o.attn == "flash" ? 3 : 2;
  if (o.ckpt_unit != "half" && o.ckpt_unit != "block") throw Fail("--ckpt-unit half|block");
  t.ckpt_unit = o.ckpt_unit == "half" ? 1 : 0;
  t.ffn_regen_g = 0;

  mimose_ctx* ctx = nullptr;
  mimose_trainer* tr = nullptr;
  RunOut out;
  cudaStream_t stream = nullptr;
  try {
    ck(mimose_ctx_create(o.device, budget, &ctx), "mimose_ctx_create");
    if (mimose_trainer_create(ctx, &m, &t, &tr) != 0) {
      const std::string e = mimose_last_error();
      if (e.find("budget exceeded") != std::string::npos)
        throw Infeasible("budget below the constant footprint: " + e);
      throw Fail("mimose_trainer_create: " + e);
    }
    if (cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking) != cudaSuccess)
      throw Fail("cudaStreamCreate");
    std::mt19937_64 g(o.data_seed);
    for (int64_t s : sizes) {
      const Batch b = make_batch(g, m, B, static_cast<int>(s));
      mimose_step_report rep{};
      if (mimose_trainer_step(tr, b.tok.data(), b.typ.data(), b.lab.data(), B,
                              static_cast<int>(s), stream, &rep) != 0) {
        const std::string e = mimose_last_error();
        // a step the arena could not hold: nothing recorded (the trainer
        // released its blocks), counted here; any other failure is an error
        if (e.find("budget exceeded") == std::string::npos)
          throw Fail("mimose_trainer_step (S=" + std::to_string(s) + "): " + e);
        ++out.failed;
        std::cerr << "step failed (S=" << s << "): " << e << "\n";
      }
    }
    char *sum = nullptr, *csv = nullptr, *txt = nullptr;
    ck(mimose_trainer_report(tr, &sum, &csv), "mimose_trainer_report");
    out.summary = take(sum);
    out.csv = take(csv);
    if (mimose_trainer_estimator_text(tr, &txt) == 0) out.estimator = take(txt);
    if (mimose_trainer_samples_csv(tr, &txt) == 0) out.samples = take(txt);
    if (mimose_trainer_model_text(tr, &txt) == 0) out.model = take(txt);
  } catch (...) {
    if (tr) mimose_trainer_destroy(tr);
    if (ctx) mimose_ctx_destroy(ctx);
    if (stream) cudaStreamDestroy(stream);
    throw;
  }
  mimose_trainer_destroy(tr);
  mimose_ctx_destroy(ctx);
  cudaStreamDestroy(stream);
  return out;
}

void write_text(const std::string& path, const std::string& text) {
  std::ofstream f(path);
  if (!f) throw Fail("cannot write output file: " + path);
  f << text;
  if (!f) throw Fail("failed while writing: " + path);
}

int exit_code_of(const RunOut& r) {
  const auto n = [&](const char* k) {
    const std::string v = summary_field(r.summary, k);
    return v.empty() ? 0LL : std::atoll(v.c_str());
  };
  return (n("oom_risk_iterations") > 0 || n("insufficient_budget_iterations") > 0 || r.failed > 0)
             ? kInfeasible
             : kOk;
}

void dumps(const Opts& o, const RunOut& r) {
  if (!o.dump_model.empty()) write_text(o.dump_model, r.model);
  if (!o.dump_estimator.empty()) write_text(o.dump_estimator, r.estimator);
  if (!o.dump_samples.empty()) write_text(o.dump_samples, r.samples);
}

int cmd_run(const Opts& o) {
  const RunOut r = run_gpu(o, o.planner, o.budget);
  const std::string& text = o.format == "csv" ? r.csv : r.summary;
  if (o.out.empty()) std::cout << text;
  else write_text(o.out, text);
  dumps(o, r);
  if (r.failed) std::cerr << "failed_iterations: " << r.failed << "\n";
  return exit_code_of(r);
}

int cmd_compare(const Opts& o) {
  std::ostringstream out;
  out << "planner,budget_bytes,total_time_ms,mean_peak_bytes,recompute_total_ms,"
         "planner_invocations,collector_iterations,cache_hits,oom_risk_iterations,"
         "insufficient_budget_iterations,overhead_iterations\n";
  int code = kOk;
  const auto budgets = split(o.budgets);
  if (budgets.empty()) throw Fail("--budgets is required");
  for (const auto& b : budgets)
    for (const auto& p : split(o.planners)) {
      RunOut r;
      try {
        r = run_gpu(o, p, b);
      } catch (const Infeasible& e) {
        // this cell's budget cannot hold the model: an empty row, exit 2
        std::cerr << "infeasible (" << p << ", " << b << "): " << e.what() << "\n";
        out << p << ',' << parse_bytes(b) << ",,,,,,,,,\n";
        code = kInfeasible;
        continue;
      }
      const auto f = [&](const char* k) { return summary_field(r.summary, k); };
      out << p << ',' << f("budget_bytes") << ',' << f("total_time_ms") << ','
          << f("mean_peak_bytes") << ',' << f("recompute_total_ms") << ','
          << f("planner_invocations") << ',' << f("collector_iterations") << ','
          << f("cache_hits") << ',' << f("oom_risk_iterations") << ','
          << f("insufficient_budget_iterations") << ',' << f("overhead_iterations") << '\n';
      code = std::max(code, exit_code_of(r));
    }
  if (o.out.empty()) std::cout << out.str();
  else write_text(o.out, out.str());
  return code;
}

// collect (every distinct size measured in a sheltered pass) + fit: the
// reference fit subcommand over the GPU-measured samples
int cmd_fit(const Opts& o) {
  const RunOut r = run_gpu(o, "mimose", o.budget, /*collect_all_sizes_only=*/true);
  if (!o.dump_samples.empty()) write_text(o.dump_samples, r.samples);
  char* est = nullptr;
  pk(mimose_planner_fit(r.samples.c_str(), o.order, &est), "fit");
  const std::string e = est ? est : "";
  mimose_planner_free(est);
  if (!o.dump_estimator.empty()) write_text(o.dump_estimator, e);
  else std::cout << e;
  if (!o.dump_model.empty()) write_text(o.dump_model, r.model);
  const std::vector<int64_t> sz = sizes_of(o);
  const std::set<int64_t> distinct(sz.begin(), sz.end());
  std::cerr << "collected_iterations: " << summary_field(r.summary, "collector_iterations") << "\n"
            << "distinct_sizes: " << distinct.size() << "\n";
  return kOk;
}

int cmd_gen_workload(const Opts& o) {
  std::vector<int64_t> x(static_cast<size_t>(o.iters));
  if (o.iters > 0)
    pk(mimose_planner_sample_workload(o.dist.c_str(), o.batch_multiplier, o.iters, o.seed,
                                      x.data()),
       "sample_workload");
  std::ostringstream out;
  for (int64_t v : x) out << v << '\n';
  if (o.out.empty()) std::cout << out.str();
  else write_text(o.out, out.str());
  return kOk;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage(std::cerr);
    return kError;
  }
  const std::string cmd = argv[1];
  if (cmd == "--help" || cmd == "-h") {
    usage(std::cout);
    return kOk;
  }
  if (cmd == "simulate" || cmd == "plan") {
    std::cerr << "'" << cmd << "' replays a .model document without device work: use the "
                 "reference CLI over include/mimose (drop-in headers)\n";
    return kError;
  }
  if (!kFlags.count(cmd)) {
    std::cerr << "unknown subcommand '" << cmd << "'\n";
    usage(std::cerr);
    return kError;
  }
  try {
    const Opts o = parse(cmd, argc, argv);
    if (cmd == "run") return cmd_run(o);
    if (cmd == "compare") return cmd_compare(o);
    if (cmd == "fit") return cmd_fit(o);
    return cmd_gen_workload(o);
  } catch (const Infeasible& e) {
    std::cerr << "infeasible: " << e.what() << "\n";
    return kInfeasible;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kError;
  }
}
