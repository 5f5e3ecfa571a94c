// Host side of the fused attention-score kernels (attn_sm100.cuh).
#include <cuda.h>
#include <cuda_runtime.h>

#include "attn_sm100.cuh"
#include "ops.hpp"
#include "ops_attn.hpp"
#include "prof.hpp"

namespace mimose_ops {

namespace {

int attn_sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

template <int NC, bool BWD>
cudaError_t launch(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& o1,
                   const CUtensorMap& o2, const mimose_dev::AttnParams& p, cudaStream_t s) {
  using Cfg = mimose_dev::AttnCfg<NC>;
  auto kern = mimose_dev::attn_scores_kernel<NC, BWD>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int tiles = ((p.S + 127) / 128) * p.nh * p.B;
  const int grid = tiles < attn_sm_count() ? tiles : attn_sm_count();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(Cfg::kThreads);
  cfg.dynamicSmemBytes = Cfg::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a, b, o1, o2, p);
  if (e != cudaSuccess) return e;
  count_launch();
  return cudaGetLastError();
}


}  // namespace

bool attn_fused_supported(int S) { return S >= 1 && S <= 512; }

cudaError_t attn_scores_fwd(const MatView& q, const MatView& k, void* P, void* Pd, int S, int ld,
                            int nh, int B, float alpha, const mimose_dev::DropoutCfg& drop,
                            cudaStream_t s, bool causal) {
  if (!attn_fused_supported(S)) return cudaErrorInvalidValue;
  const double nz = (double)nh * B;
  // Q, K read; P (+ Pd) written
  ProfScope prof("attn_fused_fwd", 2.0 * S * (double)S * 64 * nz,
                 nz * (4.0 * S * 64 + 2.0 * S * (double)ld * (Pd != nullptr ? 2 : 1)), s);
  CUtensorMap ta, tb, t1, t2;
  if (!make_operand_map(&ta, q, nh, B, 128) || !make_operand_map(&tb, k, nh, B, 256))
    return cudaErrorInvalidValue;
  if (!make_output_map(&t1, P, S, S, ld, (int64_t)S * ld, (int64_t)nh * S * ld, nh, B, 32, true))
    return cudaErrorInvalidValue;
  if (Pd != nullptr &&
      !make_output_map(&t2, Pd, S, S, ld, (int64_t)S * ld, (int64_t)nh * S * ld, nh, B, 32, true))
    return cudaErrorInvalidValue;
  if (Pd == nullptr) t2 = t1;
  mimose_dev::AttnParams p{};
  p.S = S; p.ld = ld; p.nh = nh; p.B = B;
  p.alpha = alpha;
  p.drop = drop;
  p.store_pd = Pd != nullptr;
  p.causal = causal ? 1 : 0;
  return S <= 256 ? launch<256, false>(ta, tb, t1, t2, p, s) : launch<512, false>(ta, tb, t1, t2, p, s);
}

cudaError_t attn_scores_bwd(const MatView& dout, const MatView& v, const void* P, void* dS, int S,
                            int ld, int nh, int B, float ds_scale,
                            const mimose_dev::DropoutCfg& drop, cudaStream_t s) {
  if (!attn_fused_supported(S)) return cudaErrorInvalidValue;
  const double nz = (double)nh * B;
  // dO, V, P read; dS written
  ProfScope prof("attn_fused_bwd", 2.0 * S * (double)S * 64 * nz,
                 nz * (4.0 * S * 64 + 4.0 * S * (double)S), s);
  CUtensorMap ta, tb, t1;
  if (!make_operand_map(&ta, dout, nh, B, 128) || !make_operand_map(&tb, v, nh, B, 256))
    return cudaErrorInvalidValue;
  if (!make_output_map(&t1, dS, S, S, ld, (int64_t)S * ld, (int64_t)nh * S * ld, nh, B, 32, true))
    return cudaErrorInvalidValue;
  mimose_dev::AttnParams p{};
  p.S = S; p.ld = ld; p.nh = nh; p.B = B;
  p.ds_scale = ds_scale;
  p.drop = drop;
  p.P = static_cast<const __nv_bfloat16*>(P);
  return S <= 256 ? launch<256, true>(ta, tb, t1, t1, p, s) : launch<512, true>(ta, tb, t1, t1, p, s);
}

}  // namespace mimose_ops
