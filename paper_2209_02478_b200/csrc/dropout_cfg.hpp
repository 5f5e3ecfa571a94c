// Counter-based dropout configuration shared by host launchers and kernels.
#pragma once

#include <cstdint>

namespace mimose_dev {

struct DropoutCfg {
  uint64_t seed = 0;
  uint64_t stream = 0;
  uint32_t threshold = 0;  // keep iff 16-bit rand >= threshold; 0 disables dropout
  float scale = 1.f;       // 1 / (1 - p)
};

}  // namespace mimose_dev
