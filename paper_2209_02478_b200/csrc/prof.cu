// Per-launch kernel profiler (see prof.hpp).
#include <cstring>
#include <string>
#include <vector>

#include "prof.hpp"

namespace mimose_ops {

namespace {

struct Rec {
  const char* cls;
  std::string desc;
  double flops, bytes;
};

struct Profiler {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;  // pooled, never freed
  std::vector<Rec> rec;
} g;

}  // namespace

void prof_enable(bool on) {
  g.on = on;
  g.rec.clear();
}

bool prof_on() { return g.on; }

int prof_begin(const char* cls, const std::string& desc, double flops, double bytes,
               cudaStream_t s) {
  const size_t i = g.rec.size();
  if (i == g.ev.size()) {
    std::pair<cudaEvent_t, cudaEvent_t> e;
    cudaEventCreate(&e.first);
    cudaEventCreate(&e.second);
    g.ev.push_back(e);
  }
  g.rec.push_back(Rec{cls, desc, flops, bytes});
  cudaEventRecord(g.ev[i].first, s);
  return static_cast<int>(i);
}

void prof_end(int idx, cudaStream_t s) { cudaEventRecord(g.ev[idx].second, s); }

static float rec_ms(size_t i, cudaError_t* err) {
  cudaError_t e = cudaEventSynchronize(g.ev[i].second);
  float m = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&m, g.ev[i].first, g.ev[i].second);
  if (e != cudaSuccess && err != nullptr) *err = e;
  return m;
}

std::string prof_csv() {
  std::string out = "class,desc,flops,bytes,ms\n";
  for (size_t i = 0; i < g.rec.size(); ++i) {
    const float m = rec_ms(i, nullptr);
    out += std::string(g.rec[i].cls) + ",\"" + g.rec[i].desc + "\"," +
           std::to_string(g.rec[i].flops) + "," + std::to_string(g.rec[i].bytes) + "," +
           std::to_string(m) + "\n";
  }
  return out;
}

cudaError_t prof_read(const char* prefix, double* flops, double* bytes, double* ms,
                      int64_t* launches) {
  cudaError_t err = cudaSuccess;
  double f = 0, b = 0, t = 0;
  int64_t n = 0;
  const size_t pl = std::strlen(prefix);
  for (size_t i = 0; i < g.rec.size(); ++i) {
    if (std::strncmp(g.rec[i].cls, prefix, pl) != 0) continue;
    t += rec_ms(i, &err);
    f += g.rec[i].flops;
    b += g.rec[i].bytes;
    ++n;
  }
  *flops = f;
  *bytes = b;
  *ms = t;
  *launches = n;
  return err;
}

}  // namespace mimose_ops
