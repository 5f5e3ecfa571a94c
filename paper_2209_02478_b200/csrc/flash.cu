// Host side of the flash-attention kernels (flash_sm100.cuh).
#include <cuda.h>
#include <cuda_runtime.h>

#include "flash_sm100.cuh"
#include "ops.hpp"
#include "ops_attn.hpp"
#include "prof.hpp"

namespace mimose_ops {

namespace {

int flash_sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

template <typename Kern>
cudaError_t launch_flash(Kern kern, int smem, int threads, int tiles, const CUtensorMap& a,
                         const CUtensorMap& b, const CUtensorMap& c,
                         const mimose_dev::FlashParams& p, cudaStream_t s, bool& configured) {
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int grid = tiles < flash_sm_count() ? tiles : flash_sm_count();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a, b, c, p);
  if (e != cudaSuccess) return e;
  count_launch();
  return cudaGetLastError();
}

}  // namespace

bool flash_supported(int S) { return S >= 1 && S <= 8192; }

cudaError_t flash_fwd(const MatView& q, const MatView& k, const MatView& v, void* ctx,
                      int64_t ctx_ld, float* lse, int S, int ld, int nh, int B, float alpha,
                      const mimose_dev::DropoutCfg& drop, bool causal, cudaStream_t s) {
  if (!flash_supported(S) || (ctx_ld * 2) % 16 || (reinterpret_cast<uintptr_t>(ctx) & 15))
    return cudaErrorInvalidValue;
  const double nz = (double)nh * B;
  const double pairs = causal ? 0.5 * S * (double)(S + 1) : (double)S * S;
  // QK^T and P V; q, k, v read, ctx + lse written
  ProfScope prof("attn_flash_fwd", 4.0 * 64 * pairs * nz, nz * (8.0 * S * 64 + 4.0 * S), s);
  CUtensorMap tq, tk, tv;
  if (!make_operand_map(&tq, q, nh, B, 128) || !make_operand_map(&tk, k, nh, B, 128) ||
      !make_operand_map(&tv, v, nh, B, 64))
    return cudaErrorInvalidValue;
  mimose_dev::FlashParams p{};
  p.S = S; p.nh = nh; p.B = B; p.ld = ld;
  p.sc = alpha * 1.4426950408889634f;
  p.drop = drop;
  p.causal = causal ? 1 : 0;
  p.ctx = static_cast<__nv_bfloat16*>(ctx);
  p.ctx_ld = ctx_ld;
  p.lse = lse;
  static bool configured = false;
  using Cfg = mimose_dev::FlashFwdCfg;
  return launch_flash(mimose_dev::flash_fwd_kernel, Cfg::kSmemBytes, Cfg::kThreads,
                      ((S + 127) / 128) * nh * B, tq, tk, tv, p, s, configured);
}

}  // namespace mimose_ops
