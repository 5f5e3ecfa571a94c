// Per-launch kernel profiler (roofline evidence). While enabled, every
// instrumented launch is bracketed by CUDA events on the stream it is issued
// on and tagged with its kernel class and ALGORITHMIC work: flops for the
// tensor-bound GEMMs, bytes that must cross HBM at least once for the
// memory-bound stages (DESIGN.md §2 lists the per-unit figures). Off by
// default: a disabled scope costs one branch.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace mimose_ops {

void prof_enable(bool on);
bool prof_on();
// opens a record; returns its index or -1 when profiling is off
int prof_begin(const char* cls, const std::string& desc, double flops, double bytes,
               cudaStream_t s);
void prof_end(int idx, cudaStream_t s);
// "class,desc,flops,bytes,ms" per launch (synchronises on the events)
std::string prof_csv();
// summed flops / bytes / ms / launches over records whose class starts with `prefix`
cudaError_t prof_read(const char* prefix, double* flops, double* bytes, double* ms,
                      int64_t* launches);

struct ProfScope {
  int idx;
  cudaStream_t s;
  ProfScope(const char* cls, double flops, double bytes, cudaStream_t st,
            const std::string& desc = std::string())
      : idx(prof_on() ? prof_begin(cls, desc, flops, bytes, st) : -1), s(st) {}
  ~ProfScope() {
    if (idx >= 0) prof_end(idx, s);
  }
  ProfScope(const ProfScope&) = delete;
  ProfScope& operator=(const ProfScope&) = delete;
};

}  // namespace mimose_ops
