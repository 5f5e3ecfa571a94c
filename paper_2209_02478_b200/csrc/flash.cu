// Host side of the flash-attention kernels (flash_sm100.cuh).
#include <cuda.h>
#include <cuda_runtime.h>

#include "flash_sm100.cuh"
#include "ops.hpp"
#include "ops_attn.hpp"
#include "prof.hpp"

#include <algorithm>
#include <cstdlib>
#include <string>

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
  const int grid = tiles;  // callers cap it at the resident CTAs
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

template <typename Kern>
cudaError_t launch_flash5(Kern kern, int smem, int threads, int tiles, const CUtensorMap& a,
                          const CUtensorMap& b, const CUtensorMap& c, const CUtensorMap& d,
                          const CUtensorMap& e5, const mimose_dev::FlashParams& p,
                          cudaStream_t s, bool& configured) {
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int grid = tiles;  // callers cap it at the resident CTAs
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
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a, b, c, d, e5, p);
  if (e != cudaSuccess) return e;
  count_launch();
  return cudaGetLastError();
}

}  // namespace

bool flash_supported(int S) { return S >= 1 && S <= 8192; }

cudaError_t flash_fwd(const MatView& q, const MatView& k, const MatView& v, void* ctx,
                      int64_t ctx_ld, float* lse, uint32_t* mask, int S, int ld, int nh, int B,
                      float alpha, const mimose_dev::DropoutCfg& drop, bool causal,
                      cudaStream_t s) {
  if (!flash_supported(S) || (ctx_ld * 2) % 16 || (reinterpret_cast<uintptr_t>(ctx) & 15))
    return cudaErrorInvalidValue;
  const double nz = (double)nh * B;
  const double pairs = causal ? 0.5 * S * (double)(S + 1) : (double)S * S;
  // QK^T and P V; q, k, v read, ctx + lse written
  const int mw = (S + 31) / 32;
  const bool with_mask = drop.threshold != 0;
  if (with_mask && mask == nullptr) return cudaErrorInvalidValue;
  ProfScope prof("attn_flash_fwd", 4.0 * 64 * pairs * nz,
                 nz * (8.0 * S * 64 + 4.0 * S + (with_mask ? 4.0 * S * mw : 0.0)), s);
  // key block: 64 (two CTAs per SM) unless MIMOSE_FLASH_KB=128
  static const int kb = [] {
    const char* e = std::getenv("MIMOSE_FLASH_KB");
    return e != nullptr && std::atoi(e) == 128 ? 128 : 64;
  }();
  CUtensorMap tq, tk, tv;
  if (!make_operand_map(&tq, q, nh, B, 128) || !make_operand_map(&tk, k, nh, B, kb) ||
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
  p.mask = with_mask ? mask : nullptr;
  p.mw = mw;
  const int tiles = ((S + 127) / 128) * nh * B;
  if (kb == 128) {
    using Cfg = mimose_dev::FlashFwdCfg<128>;
    static bool configured[2] = {false, false};
    return launch_flash(with_mask ? mimose_dev::flash_fwd_kernel<128, true>
                                  : mimose_dev::flash_fwd_kernel<128, false>,
                        Cfg::kSmemBytes, Cfg::kThreads, std::min(tiles, flash_sm_count()), tq, tk,
                        tv, p, s, configured[with_mask]);
  }
  using Cfg = mimose_dev::FlashFwdCfg<64>;
  static bool configured[2] = {false, false};
  return launch_flash(with_mask ? mimose_dev::flash_fwd_kernel<64, true>
                                : mimose_dev::flash_fwd_kernel<64, false>,
                      Cfg::kSmemBytes, Cfg::kThreads, std::min(tiles, 2 * flash_sm_count()), tq, tk,
                      tv, p, s, configured[with_mask]);
}

cudaError_t flash_keep_mask(uint32_t* mask, int S, int ld, int nh, int B,
                            const mimose_dev::DropoutCfg& drop, bool causal, cudaStream_t s) {
  if (drop.threshold == 0) return cudaSuccess;
  if (mask == nullptr || !flash_supported(S) || ld % 8 != 0) return cudaErrorInvalidValue;
  const int mw = (S + 31) / 32;
  if ((int64_t)B * nh * S * mw >= (int64_t(1) << 32)) return cudaErrorInvalidValue;
  ProfScope prof("attn_flash_mask", 0.0, (double)nh * B * 4.0 * S * mw, s);
  const int64_t n = (int64_t)B * nh * S * mw;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 16 * flash_sm_count());
  mimose_dev::flash_keep_mask_kernel<<<blocks, 256, 0, s>>>(
      drop.seed, drop.stream, drop.threshold, (uint32_t)((int64_t)B * nh * S), S, ld, mw, causal ? 1 : 0,
      mask);
  count_launch();
  return cudaGetLastError();
}

cudaError_t flash_bwd(const MatView& q, const MatView& k, const MatView& v, const void* ctx,
                      const void* dctx, int64_t ctx_ld, const float* lse, const uint32_t* mask,
                      float* dvec, void* dqkv, int S, int ld, int nh, int B, float alpha,
                      const mimose_dev::DropoutCfg& drop, bool causal, cudaStream_t s) {
  if (!flash_supported(S) || (ctx_ld * 2) % 16 || (drop.threshold != 0 && mask == nullptr))
    return cudaErrorInvalidValue;
  const double nz = (double)nh * B;
  const double pairs = causal ? 0.5 * S * (double)(S + 1) : (double)S * S;
  const int mw = (S + 31) / 32;
  MatView dov;
  dov.ptr = dctx;
  dov.rows = S;
  dov.cols = 64;
  dov.ld = ctx_ld;
  dov.bs1 = 64;
  dov.bs2 = (int64_t)S * ctx_ld;
  MatView cv = dov;
  cv.ptr = ctx;
  CUtensorMap tq, tk, tv, to, tc, tk64, tv64;
  if (!make_operand_map(&tq, q, nh, B, 128) || !make_operand_map(&tk, k, nh, B, 128) ||
      !make_operand_map(&tv, v, nh, B, 128) || !make_operand_map(&to, dov, nh, B, 128) ||
      !make_operand_map(&tc, cv, nh, B, 128) || !make_operand_map(&tk64, k, nh, B, 64) ||
      !make_operand_map(&tv64, v, nh, B, 64))
    return cudaErrorInvalidValue;
  mimose_dev::FlashParams p{};
  p.S = S; p.nh = nh; p.B = B; p.ld = ld;
  p.sc = alpha * 1.4426950408889634f;
  p.drop = drop;
  p.causal = causal ? 1 : 0;
  p.ctx_ld = ctx_ld;
  p.lse = const_cast<float*>(lse);
  p.mask = const_cast<uint32_t*>(mask);
  p.mw = mw;
  p.dvec = dvec;
  p.dqkv = static_cast<__nv_bfloat16*>(dqkv);
  p.ds_scale = alpha;
  using CfgQ = mimose_dev::FlashBwdCfg<1, 64>;
  using CfgKV = mimose_dev::FlashBwdCfg<0, 128>;
  const int items = ((S + 127) / 128) * nh * B;
  const double mbytes = drop.threshold != 0 ? 4.0 * S * mw : 0.0;
  {
    // S, dPd recomputed; dQ accumulated: 3 MMAs per block pair; also
    // D = dO . O per row (dO, O tiles read once per query block)
    ProfScope prof("attn_flash_bwd_q", 6.0 * 64 * pairs * nz,
                   nz * (10.0 * S * 64 + 8.0 * S + mbytes + 2.0 * S * 64), s);
    static bool configured = false;
    cudaError_t e = launch_flash5(mimose_dev::flash_bwd_kernel<1, 64>, CfgQ::kSmemBytes,
                                  CfgQ::kThreads, std::min(items, 2 * flash_sm_count()), tq,
                                  tk64, tv64, to, tc, p, s, configured);
    if (e != cudaSuccess) return e;
  }

  {
    // S, dPd recomputed; dV, dK accumulated: 4 MMAs per (query, key) block pair
    ProfScope prof("attn_flash_bwd_kv", 8.0 * 64 * pairs * nz,
                   nz * (8.0 * S * 64 + 8.0 * S + mbytes + 4.0 * S * 64), s);
    static bool configured = false;
    return launch_flash5(mimose_dev::flash_bwd_kernel<0, 128>, CfgKV::kSmemBytes,
                         CfgKV::kThreads, std::min(items, flash_sm_count()), tq, tk, tv, to, to,
                         p, s, configured);
  }
}

}  // namespace mimose_ops

#ifdef MIMOSE_FLASH_TRACE
extern "C" int mimose_debug_flash_trace(void* dst) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(dst, mimose_dev::g_flash_trace, 4096 * 8);
  return 0;
}
#endif
