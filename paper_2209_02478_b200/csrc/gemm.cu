// Host side of the sm_100a GEMM: tensor-map encoding (driver entry point,
// no -lcuda link dependency), tile-width heuristic, persistent launch.
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <mutex>
#include <utility>
#include <vector>

#include "gemm_sm100.cuh"
#include "ops.hpp"

namespace mimose_ops {

namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

std::atomic<uint64_t> g_launches{0};

// optional per-launch event bracketing (roofline evidence)
struct GemmProfile {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  std::vector<double> flops;
  size_t used = 0;
} g_prof;

EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeFn>(nullptr);
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

int sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// 4-D map (cols, rows, nb1, nb2) over a bf16 view with a {64, box_rows} box,
// 128-byte swizzle, zero fill out of bounds.
bool make_map(CUtensorMap* map, const MatView& v, int nb1, int nb2, uint32_t box_rows) {
  EncodeFn fn = encode_fn();
  if (fn == nullptr) return false;
  const uint64_t esz = 2;
  cuuint64_t dims[4] = {(cuuint64_t)v.cols, (cuuint64_t)v.rows, (cuuint64_t)nb1,
                        (cuuint64_t)nb2};
  uint64_t plane = (uint64_t)v.ld * (uint64_t)v.rows * esz;
  plane = (plane + 15) & ~uint64_t(15);
  cuuint64_t strides[3] = {(cuuint64_t)(v.ld * esz),
                           (cuuint64_t)(nb1 > 1 ? v.bs1 * esz : plane),
                           (cuuint64_t)(nb2 > 1 ? v.bs2 * esz : plane)};
  cuuint32_t box[4] = {64, box_rows, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(v.ptr), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, int EPI>
cudaError_t launch_t(const CUtensorMap& ta, const CUtensorMap& tb,
                     const mimose_dev::GemmParams& p, int grid, cudaStream_t stream) {
  using Cfg = mimose_dev::GemmCfg<BN>;
  auto kern = mimose_dev::gemm_bf16_tn_kernel<BN, EPI>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  kern<<<grid, mimose_dev::kGemmThreads, Cfg::kSmemBytes, stream>>>(ta, tb, p);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <int BN>
cudaError_t launch_bn(int epi, const CUtensorMap& ta, const CUtensorMap& tb,
                      const mimose_dev::GemmParams& p, int grid, cudaStream_t s) {
  switch (epi) {
    case kEpiBf16: return launch_t<BN, mimose_dev::kEpiBf16>(ta, tb, p, grid, s);
    case kEpiBiasGelu: return launch_t<BN, mimose_dev::kEpiBiasGelu>(ta, tb, p, grid, s);
    case kEpiDGelu: return launch_t<BN, mimose_dev::kEpiDGelu>(ta, tb, p, grid, s);
    case kEpiF32: return launch_t<BN, mimose_dev::kEpiF32>(ta, tb, p, grid, s);
  }
  return cudaErrorInvalidValue;
}

int pick_bn(const GemmCall& c) {
  if (c.force_bn) return c.force_bn;
  if (c.N <= 64) return 64;
  const int64_t batches = (int64_t)c.nb1 * c.nb2;
  const int64_t tm = (c.M + 127) / 128;
  const int64_t t256 = tm * ((c.N + 255) / 256) * batches;
  if (c.N > 128 && t256 >= 2 * sm_count()) return 256;
  return 128;
}

}  // namespace

uint64_t launch_count() { return g_launches.load(); }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

cudaError_t gemm(const GemmCall& c, cudaStream_t stream) {
  if (c.M <= 0 || c.N <= 0 || c.K <= 0 || c.nb1 <= 0 || c.nb2 <= 0) return cudaErrorInvalidValue;
  if ((c.A.ld * 2) % 16 || (c.B.ld * 2) % 16) return cudaErrorInvalidValue;
  if ((reinterpret_cast<uintptr_t>(c.A.ptr) & 15) || (reinterpret_cast<uintptr_t>(c.B.ptr) & 15))
    return cudaErrorMisalignedAddress;
  const int bn = pick_bn(c);
  CUtensorMap ta, tb;
  if (!make_map(&ta, c.A, c.nb1, c.nb2, c.a_mn ? 64u : 128u)) return cudaErrorInvalidValue;
  if (!make_map(&tb, c.B, c.nb1, c.nb2, c.b_mn ? 64u : (uint32_t)bn))
    return cudaErrorInvalidValue;

  mimose_dev::GemmParams p{};
  p.M = c.M; p.N = c.N; p.K = c.K; p.nb1 = c.nb1; p.nb2 = c.nb2;
  p.a_mn = c.a_mn; p.b_mn = c.b_mn;
  p.out = c.out; p.out2 = c.out2;
  p.aux = reinterpret_cast<const __nv_bfloat16*>(c.aux);
  p.bias = c.bias;
  p.ldo = c.ldo; p.obs1 = c.obs1; p.obs2 = c.obs2;
  p.alpha = c.alpha; p.beta = c.beta;
  {
    const int64_t vel = c.epi == kEpiF32 ? 4 : 8;  // elements per 16 bytes
    auto al = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    p.vec = (c.ldo % vel == 0) && (c.obs1 % vel == 0) && (c.obs2 % vel == 0) && al(c.out) &&
            (c.out2 == nullptr || al(c.out2)) && (c.aux == nullptr || al(c.aux));
  }

  const int64_t tiles = (int64_t)((c.M + 127) / 128) * ((c.N + bn - 1) / bn) * c.nb1 * c.nb2;
  const int grid = (int)(tiles < sm_count() ? tiles : sm_count());
  std::pair<cudaEvent_t, cudaEvent_t>* pe = nullptr;
  if (g_prof.on) {
    if (g_prof.used == g_prof.ev.size()) {
      std::pair<cudaEvent_t, cudaEvent_t> e;
      cudaEventCreate(&e.first);
      cudaEventCreate(&e.second);
      g_prof.ev.push_back(e);
    }
    pe = &g_prof.ev[g_prof.used++];
    g_prof.flops.push_back(2.0 * c.M * (double)c.N * c.K * c.nb1 * c.nb2);
    cudaEventRecord(pe->first, stream);
  }
  cudaError_t err = cudaErrorInvalidValue;
  switch (bn) {
    case 64: err = launch_bn<64>(c.epi, ta, tb, p, grid, stream); break;
    case 128: err = launch_bn<128>(c.epi, ta, tb, p, grid, stream); break;
    case 256: err = launch_bn<256>(c.epi, ta, tb, p, grid, stream); break;
  }
  if (pe != nullptr) cudaEventRecord(pe->second, stream);
  return err;
}

void gemm_profile_enable(bool on) {
  g_prof.on = on;
  g_prof.used = 0;
  g_prof.flops.clear();
}

cudaError_t gemm_profile_read(double* flops, double* ms, int64_t* launches) {
  double f = 0.0, t = 0.0;
  for (size_t i = 0; i < g_prof.used; ++i) {
    cudaError_t e = cudaEventSynchronize(g_prof.ev[i].second);
    if (e != cudaSuccess) return e;
    float m = 0.f;
    e = cudaEventElapsedTime(&m, g_prof.ev[i].first, g_prof.ev[i].second);
    if (e != cudaSuccess) return e;
    t += m;
    f += g_prof.flops[i];
  }
  *flops = f;
  *ms = t;
  *launches = (int64_t)g_prof.used;
  return cudaSuccess;
}

}  // namespace mimose_ops
