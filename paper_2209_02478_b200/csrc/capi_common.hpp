// Shared definitions behind the opaque C handles.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "allocator.hpp"

struct mimose_ctx {
  int device = 0;
  mimose_rt::DeviceArena arena;
};

namespace mimose_capi {
int fail(const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
}  // namespace mimose_capi
