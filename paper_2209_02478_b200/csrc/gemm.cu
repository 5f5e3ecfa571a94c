// Host side of the sm_100a GEMM: tensor-map encoding (driver entry point,
// no -lcuda link dependency), tile-width heuristic, persistent launch.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include <string>
#include <utility>
#include <vector>

#include "gemm_sm100.cuh"
#include "ops.hpp"
#include "ops_attn.hpp"
#include "prof.hpp"

namespace mimose_ops {

namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

std::atomic<uint64_t> g_launches{0};

}  // namespace

// PDL for the tcgen05 kernels (MIMOSE_PDL=0 disables, for A/B timing)
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MIMOSE_PDL");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}

namespace {


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

// 4-D map (cols, rows, nb1, nb2) with a {box_cols, box_rows} box, 128-byte
// swizzle, zero fill out of bounds. esz 2 = bf16, 4 = fp32.
struct MapKey {
  const void* ptr;
  int64_t rows, cols, ld, bs1, bs2;
  int nb1, nb2;
  uint32_t box_cols, box_rows;
  int esz;
  bool sw64;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && rows == o.rows && cols == o.cols && ld == o.ld && bs1 == o.bs1 &&
           bs2 == o.bs2 && nb1 == o.nb1 && nb2 == o.nb2 && box_cols == o.box_cols &&
           box_rows == o.box_rows && esz == o.esz && sw64 == o.sw64;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    uint64_t h = reinterpret_cast<uintptr_t>(k.ptr);
    auto mix = [&h](uint64_t v) { h ^= v + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2); };
    mix(k.rows); mix(k.cols); mix(k.ld); mix(k.bs1); mix(k.bs2); mix(k.nb1); mix(k.nb2);
    mix(k.box_cols); mix(k.box_rows); mix(k.esz); mix(k.sw64);
    return static_cast<size_t>(h);
  }
};
// Encoded tensor maps are pure functions of their arguments; the executor
// re-issues the same views every step (arena addresses repeat), so encoding
// is cached on the host.
std::unordered_map<MapKey, CUtensorMap, MapKeyHash>& map_cache() {
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> c;
  return c;
}

bool make_map_uncached(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                       int64_t bs1, int64_t bs2, int nb1, int nb2, uint32_t box_cols,
                       uint32_t box_rows, int esz, bool sw64);

bool make_map_t(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                int64_t bs1, int64_t bs2, int nb1, int nb2, uint32_t box_cols, uint32_t box_rows,
                int esz, bool sw64 = false) {
  const MapKey key{ptr, rows, cols, ld, nb1 > 1 ? bs1 : 0, nb2 > 1 ? bs2 : 0, nb1, nb2,
                   box_cols, box_rows, esz, sw64};
  auto& cache = map_cache();
  auto it = cache.find(key);
  if (it != cache.end()) {
    *map = it->second;
    return true;
  }
  if (!make_map_uncached(map, ptr, rows, cols, ld, bs1, bs2, nb1, nb2, box_cols, box_rows, esz,
                         sw64))
    return false;
  if (cache.size() > 16384) cache.clear();
  cache.emplace(key, *map);
  return true;
}

bool make_map_uncached(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                       int64_t bs1, int64_t bs2, int nb1, int nb2, uint32_t box_cols,
                       uint32_t box_rows, int esz, bool sw64) {
  EncodeFn fn = encode_fn();
  if (fn == nullptr) return false;
  cuuint64_t dims[4] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)nb1, (cuuint64_t)nb2};
  uint64_t plane = (uint64_t)ld * (uint64_t)rows * esz;
  plane = (plane + 15) & ~uint64_t(15);
  cuuint64_t strides[3] = {(cuuint64_t)(ld * esz), (cuuint64_t)(nb1 > 1 ? bs1 * esz : plane),
                           (cuuint64_t)(nb2 > 1 ? bs2 * esz : plane)};
  cuuint32_t box[4] = {box_cols, box_rows, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                  4, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  sw64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_map(CUtensorMap* map, const MatView& v, int nb1, int nb2, uint32_t box_rows) {
  return make_map_t(map, v.ptr, v.rows, v.cols, v.ld, v.bs1, v.bs2, nb1, nb2, 64, box_rows, 2);
}

template <int BN, int EPI, int EW, int CG = 1>
cudaError_t launch_t(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& td,
                     const CUtensorMap& td2, const mimose_dev::GemmParams& p, int grid,
                     cudaStream_t stream) {
  using Cfg = mimose_dev::GemmCfg<BN, EPI, EW, CG>;
  auto kern = mimose_dev::gemm_bf16_tn_kernel<BN, EPI, EW, CG>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  // programmatic dependent launch (the kernel calls pdl_wait() before its
  // first dependent access) + cluster (2, 1, 1) for CTA pairs; `grid` counts CTAs
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(Cfg::kThreads);
  cfg.dynamicSmemBytes = Cfg::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if constexpr (CG > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = CG;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ta, tb, td, td2, p);
  if (e != cudaSuccess) return e;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

// CTA-pair (cta_group::2) launches: BN = 256 only
cudaError_t launch_pair(int epi, int ew, const CUtensorMap& ta, const CUtensorMap& tb,
                        const CUtensorMap& td, const CUtensorMap& td2,
                        const mimose_dev::GemmParams& p, int grid, cudaStream_t s) {
  using namespace mimose_dev;
  switch (epi) {
    case kEpiBf16: return launch_t<256, kEpiBf16, 8, 2>(ta, tb, td, td2, p, grid, s);
    case kEpiBiasGelu: return launch_t<256, kEpiBiasGelu, 16, 2>(ta, tb, td, td2, p, grid, s);
    case kEpiDGelu: return launch_t<256, kEpiDGelu, 16, 2>(ta, tb, td, td2, p, grid, s);
    case kEpiF32: return launch_t<256, kEpiF32, 8, 2>(ta, tb, td, td2, p, grid, s);
  }
  (void)ew;
  return cudaErrorInvalidValue;
}

template <int BN>
cudaError_t launch_bn(int epi, int ew, const CUtensorMap& ta, const CUtensorMap& tb,
                      const CUtensorMap& td, const CUtensorMap& td2,
                      const mimose_dev::GemmParams& p, int grid, cudaStream_t s) {
  using namespace mimose_dev;
  switch (epi) {
    case kEpiBf16:
      return ew == 16 ? launch_t<BN, kEpiBf16, 16>(ta, tb, td, td2, p, grid, s)
                      : launch_t<BN, kEpiBf16, 8>(ta, tb, td, td2, p, grid, s);
    case kEpiBiasGelu:
      return ew == 16 ? launch_t<BN, kEpiBiasGelu, 16>(ta, tb, td, td2, p, grid, s)
                      : launch_t<BN, kEpiBiasGelu, 8>(ta, tb, td, td2, p, grid, s);
    case kEpiDGelu:
      return ew == 16 ? launch_t<BN, kEpiDGelu, 16>(ta, tb, td, td2, p, grid, s)
                      : launch_t<BN, kEpiDGelu, 8>(ta, tb, td, td2, p, grid, s);
    case kEpiF32: return launch_t<BN, kEpiF32, 8>(ta, tb, td, td2, p, grid, s);
  }
  return cudaErrorInvalidValue;
}

// epilogue warps: 16 for the GELU / dGELU epilogues (math-bound: FFN1
// 549 -> 742 TFLOP/s, dGELU 638 -> 802), 8 otherwise (the write-bound
// attention contractions measured slower with 16). MIMOSE_GEMM_EW
// (8 / 16) overrides for A/B timing.
// CTA pair (cta_group::2, 256 x 256 tiles over two SMs): halves the B-operand
// traffic per SM and deepens the smem pipeline (6 stages of 32 KB). Used for
// unbatched, un-split GEMMs with >= 2 row blocks whose epilogue is light
// (K >= 768 projections and data gradients: 1090 -> 1250 TFLOP/s at K = 3072).
// MIMOSE_GEMM_CG=1/2 forces (A/B timing); force_cg in the call overrides.
// MIMOSE_AUX_TMA=0: aux rows through per-thread loads (A/B timing)
bool aux_tma_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MIMOSE_AUX_TMA");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}

int pick_cg(const GemmCall& c, int bn) {
  static const int forced = [] {
    const char* e = std::getenv("MIMOSE_GEMM_CG");
    return e != nullptr ? std::atoi(e) : 0;
  }();
  if (bn != 256 || c.nb1 * c.nb2 != 1 || c.M <= 128) return 1;
  if (c.force_cg == 1 || c.force_cg == 2) return c.force_cg;
  if (forced == 1 || forced == 2) return forced;
  // the dGELU epilogue (aux tile in, one output) is the slower side of its
  // pipeline, and the pair's joint accumulator release costs it (852 -> 794
  // TFLOP/s); the GELU GEMM's mainloop is the slower side and the pair's
  // halved B traffic helps it (887 -> 909)
  // (with the derivative saved by the forward, dGELU is a plain product: light)
  if (c.epi == kEpiDGelu && !c.gelu_deriv) return 1;
  return 2;
}

int pick_ew(const GemmCall& c, int bn) {
  static const int forced = [] {
    const char* e = std::getenv("MIMOSE_GEMM_EW");
    return e != nullptr ? std::atoi(e) : 0;
  }();
  if (c.epi == kEpiF32 || bn < 128) return 8;  // 16 warps need >= 32 columns each
  if (c.force_ew == 8 || c.force_ew == 16) return c.force_ew;
  if (forced == 8 || forced == 16) return forced;
  return (c.epi == kEpiBiasGelu || c.epi == kEpiDGelu) ? 16 : 8;
}

int pick_bn(const GemmCall& c) {
  if (c.force_bn) return c.force_bn;
  if (c.epi == kEpiBiasGelu || c.epi == kEpiDGelu) {  // A/B knob for the GELU epilogues
    static const int gelu_bn = [] {
      const char* e = std::getenv("MIMOSE_GELU_BN");
      return e != nullptr ? std::atoi(e) : 0;
    }();
    if (gelu_bn == 128 || gelu_bn == 256) return gelu_bn;
  }
  if (c.N <= 64) return 64;
  const int64_t batches = (int64_t)c.nb1 * c.nb2;
  const int64_t tm = (c.M + 127) / 128;
  // fp32 (weight-gradient) GEMMs with a split-K workspace: take the widest
  // tile and let split-K fill the machine
  if (c.epi == kEpiF32 && c.workspace != nullptr && c.N >= 256 && batches == 1) return 256;
  // widest tile that still gives >= 2 waves (the epilogue skips padded
  // column chunks, so padding costs only idle MMA slots)
  const int64_t t256 = tm * ((c.N + 255) / 256) * batches;
  if (c.N > 128 && t256 >= 2 * sm_count()) return 256;
  // light-epilogue unbatched GEMMs run 256-wide tiles on CTA pairs (see
  // pick_cg): take them whenever the pair grid is not clearly worse-filled
  // than the 128-wide single-SM grid (pair tiles are ~1.3x faster per flop)
  if (c.N > 128 && batches == 1 && c.M > 128 && (c.epi != kEpiDGelu || c.gelu_deriv) &&
      c.force_cg != 1) {
    const int64_t pairs = sm_count() / 2;
    const int64_t tp = ((c.M + 255) / 256) * ((c.N + 255) / 256);
    const int64_t t128 = tm * ((c.N + 127) / 128);
    auto eff = [](int64_t t, int64_t slots) {
      const int64_t w = (t + slots - 1) / slots;
      return (double)t / (double)(w * slots);
    };
    if (1.3 * eff(tp, pairs) >= eff(t128, sm_count())) return 256;
  }
  return 128;
}

// rs_out[m] = sum_p rs[p * M + m], p = 0 .. nparts - 1 in order (row-sum partials)
__device__ __forceinline__ void rowsum_parts(const float* __restrict__ rs, int nparts, int M,
                                             float* __restrict__ rs_out) {
  for (long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x; m < M;
       m += (long long)gridDim.x * blockDim.x) {
    float acc = rs[m];
    for (int q = 1; q < nparts; ++q) acc += rs[(long long)q * M + m];
    rs_out[m] = acc;
  }
}
__global__ void rowsum_reduce_kernel(const float* __restrict__ rs, int nparts, int M,
                                     float* __restrict__ rs_out) {
  rowsum_parts(rs, nparts, M, rs_out);
}

// out[m][n] (ld) = sum_s ws[s][m][n] (+ beta * out), fixed summation order;
// with rs_out: rs_out[m] = sum of the rs_parts row-sum partials after the
// [splits][M][N] block
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int splits, int M, int N,
                                     float* __restrict__ out, long long ldo, float beta,
                                     float* __restrict__ rs_out, int rs_parts) {
  const long long total = (long long)M * N;
  if (rs_out != nullptr) rowsum_parts(ws + (long long)splits * total, rs_parts, M, rs_out);
  const bool v4 = (N % 4 == 0) && (ldo % 4 == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  if (v4 && ldo == N) {
    // dense output: linear index, no row / column division
    const long long n4 = total / 4;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
         i += (long long)gridDim.x * blockDim.x) {
      // every split's partial (<= 8) loaded before the in-order sum: the
      // loads overlap instead of one dependent round trip per split
      float4 t[8];
#pragma unroll
      for (int s = 0; s < 8; ++s)
        if (s < splits) t[s] = __ldcs(reinterpret_cast<const float4*>(ws + (long long)s * total) + i);
      float4 acc = t[0];
#pragma unroll
      for (int s = 1; s < 8; ++s)
        if (s < splits) {
          acc.x += t[s].x; acc.y += t[s].y; acc.z += t[s].z; acc.w += t[s].w;
        }
      for (int s = 8; s < splits; ++s) {  // forced split counts above 8
        const float4 u = reinterpret_cast<const float4*>(ws + (long long)s * total)[i];
        acc.x += u.x; acc.y += u.y; acc.z += u.z; acc.w += u.w;
      }
      float4* o = reinterpret_cast<float4*>(out) + i;
      if (beta != 0.f) {
        const float4 old = *o;
        acc.x += beta * old.x; acc.y += beta * old.y; acc.z += beta * old.z; acc.w += beta * old.w;
      }
      *o = acc;
    }
  } else if (v4) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total / 4;
         i += (long long)gridDim.x * blockDim.x) {
      const long long e = i * 4;
      const long long m = e / N, n = e % N;
      float4 acc = reinterpret_cast<const float4*>(ws)[i];
      for (int s = 1; s < splits; ++s) {
        const float4 t = reinterpret_cast<const float4*>(ws + (long long)s * total)[i];
        acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
      }
      float4* o = reinterpret_cast<float4*>(out + m * ldo + n);
      if (beta != 0.f) {
        const float4 old = *o;
        acc.x += beta * old.x; acc.y += beta * old.y; acc.z += beta * old.z; acc.w += beta * old.w;
      }
      *o = acc;
    }
  } else {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
      const long long m = e / N, n = e % N;
      float acc = ws[e];
      for (int s = 1; s < splits; ++s) acc += ws[(long long)s * total + e];
      float* o = out + m * ldo + n;
      *o = acc + (beta != 0.f ? beta * *o : 0.f);
    }
  }
}


}  // namespace

bool make_operand_map(CUtensorMap* map, const MatView& v, int nb1, int nb2, uint32_t box_rows) {
  return make_map(map, v, nb1, nb2, box_rows);
}

bool make_output_map(CUtensorMap* map, void* ptr, int64_t rows, int64_t cols, int64_t ld,
                     int64_t bs1, int64_t bs2, int nb1, int nb2, uint32_t box_cols, bool sw64) {
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * 2) % 16) return false;
  return make_map_t(map, ptr, rows, cols, ld, bs1, bs2, nb1, nb2, box_cols, 32, 2, sw64);
}

// split-K count by a small cost model: mainloop time ~ waves * k-blocks per
// split (one k-block of a 128x256 tile per SM or a 256x256 pair tile per pair:
// ~0.45 us measured at the sustained clocks, tools/bench_gemm.py --splitk;
// the nominal 0.27 us made the model under-weight an extra wave and pick 2
// splits for the 2304 x 768 QKV weight gradient, 66 us, where 5 run 62),
// plus writing and re-reading the fp32 partials at HBM speed. Keeps >= 8
// k-blocks per split.
int pick_split_k(int M, int N, int K, int bn, int cg) {
  const int64_t tiles = (int64_t)((M + 128 * cg - 1) / (128 * cg)) * ((N + bn - 1) / bn);
  const int64_t slots = sm_count() / cg;
  const int kb = (K + 63) / 64;
  const double t_kb = 0.45e-6 * bn / 256.0, hbm = 6.0e12;
  auto cost = [&](int s) {
    const int64_t waves = (tiles * s + slots - 1) / slots;
    const double main = (double)waves * ((kb + s - 1) / s) * t_kb;
    return main + (s > 1 ? (double)s * M * N * 8.0 / hbm : 0.0);
  };
  int best = 1;
  double best_cost = cost(1);
  for (int s = 2; s <= 8; ++s) {
    if (kb / s < 8) break;  // keep >= 8 k-blocks per split
    const double c = cost(s);
    if (c < 0.97 * best_cost) {
      best = s;
      best_cost = c;
    }
  }
  return best;
}

int64_t splitk_workspace_bytes(int M, int N, int K) {
  GemmCall c;
  c.M = M; c.N = N; c.K = K; c.epi = kEpiF32;
  int dummy = 0;
  c.workspace = &dummy;  // "a workspace will be provided"
  const int bn = pick_bn(c);
  int s = pick_split_k(M, N, K, bn, pick_cg(c, bn));
  // split-K partials + [splits][tiles_n <= N / 64][M] row-sum partials (one
  // per column tile)
  return (int64_t)s * M * ((s > 1 ? N : 0) + (N + 63) / 64) * 4;
}

// g = GELU(u) over bf16 elements, with the GEMM epilogue's own device
// functions (gemm_sm100.cuh gelu_fast / gelu_tanh_f on the bf16 value): the
// regenerated g is bit-identical to the one the bias+GELU epilogue produced.
__global__ void gelu_regen_kernel(const __nv_bfloat16* __restrict__ u, __nv_bfloat16* __restrict__ g,
                                  int64_t n8, int tanh_form) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 raw = __ldcs(reinterpret_cast<const uint4*>(u) + i);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(&raw);
    uint4 out;
    uint32_t* o = reinterpret_cast<uint32_t*>(&out);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float a = __uint_as_float(w[q] << 16), b = __uint_as_float(w[q] & 0xFFFF0000u);
      o[q] = tanh_form ? mimose_dev::pack_bf16x2(mimose_dev::gelu_tanh_f(a), mimose_dev::gelu_tanh_f(b))
                       : [&] {
                           const float2 g = mimose_dev::gelu_fast2(make_float2(a, b));
                           return mimose_dev::pack_bf16x2(g.x, g.y);
                         }();
    }
    reinterpret_cast<uint4*>(g)[i] = out;
  }
}

cudaError_t gelu_regen(const void* u, void* g, int64_t n, bool tanh_form, cudaStream_t s) {
  if (n % 8) return cudaErrorInvalidValue;
  ProfScope prof("mem_gelu_regen", 0, 4.0 * n, s);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n8 = n / 8;
  const int blocks = (int)std::min<int64_t>((n8 + 255) / 256, 8LL * sms);
  gelu_regen_kernel<<<blocks, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(u),
                                           static_cast<__nv_bfloat16*>(g), n8, tanh_form ? 1 : 0);
  count_launch();
  return cudaGetLastError();
}

uint64_t launch_count() { return g_launches.load(); }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

cudaError_t gemm(const GemmCall& c, cudaStream_t stream) {
  if (c.M <= 0 || c.N <= 0 || c.K <= 0 || c.nb1 <= 0 || c.nb2 <= 0) return cudaErrorInvalidValue;
  if ((c.A.ld * 2) % 16 || (c.B.ld * 2) % 16) return cudaErrorInvalidValue;
  if ((reinterpret_cast<uintptr_t>(c.A.ptr) & 15) || (reinterpret_cast<uintptr_t>(c.B.ptr) & 15))
    return cudaErrorMisalignedAddress;
  const int bn = pick_bn(c);
  int ew = pick_ew(c, bn);
  const int cg = pick_cg(c, bn);
  if (cg == 2) ew = (c.epi == kEpiBiasGelu || c.epi == kEpiDGelu) ? 16 : 8;  // launch_pair
  if (c.rowsum != nullptr &&
      (c.epi != kEpiF32 || !c.a_mn || c.nb1 != 1 || c.nb2 != 1 || c.causal_k != 0 || c.causal_tiles))
    return cudaErrorInvalidValue;
  int splits = 1;
  if (c.epi == kEpiF32 && c.nb1 == 1 && c.nb2 == 1 && c.workspace != nullptr && c.split_k != 1 &&
      c.N % 4 == 0 && (reinterpret_cast<uintptr_t>(c.workspace) & 15) == 0) {
    splits = c.split_k > 1 ? c.split_k : pick_split_k(c.M, c.N, c.K, bn, cg);
    const int kb = (c.K + 63) / 64;
    if (splits > kb) splits = kb;
    const int64_t per_split = (int64_t)c.M * c.N * 4;
    while (splits > 1 && splits * per_split > c.workspace_bytes) --splits;
  }
  CUtensorMap ta, tb;
  if (!make_map(&ta, c.A, c.nb1, c.nb2, c.a_mn ? 64u : 128u)) return cudaErrorInvalidValue;
  if (!make_map(&tb, c.B, c.nb1, c.nb2, c.b_mn ? 64u : (uint32_t)(bn / cg)))
    return cudaErrorInvalidValue;

  mimose_dev::GemmParams p{};
  p.M = c.M; p.N = c.N; p.K = c.K; p.nb1 = c.nb1; p.nb2 = c.nb2;
  p.a_mn = c.a_mn; p.b_mn = c.b_mn;
  p.out = c.out; p.out2 = c.out2;
  p.aux = reinterpret_cast<const __nv_bfloat16*>(c.aux);
  p.bias = c.bias;
  p.ldo = c.ldo; p.obs1 = c.obs1; p.obs2 = c.obs2;
  p.alpha = c.alpha; p.beta = c.beta;
  p.gelu_tanh = c.gelu_tanh;
  p.gelu_deriv = c.gelu_deriv;
  p.drop = c.drop;
  p.causal_tiles = c.causal_tiles ? 1 : 0;
  p.causal_k = c.causal_k;
  if (c.causal_k != 0 && splits > 1) return cudaErrorInvalidValue;
  p.rowsum = c.rowsum;
  if (c.drop.threshold != 0 && (c.epi != kEpiBf16 || c.nb1 != 1 || c.nb2 != 1 || c.N % 8 != 0))
    return cudaErrorInvalidValue;  // dropout index = row * ldo + col, 8-column groups
  {
    const int64_t vel = c.epi == kEpiF32 ? 4 : 8;  // elements per 16 bytes
    auto al = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    p.vec = (c.ldo % vel == 0) && (c.obs1 % vel == 0) && (c.obs2 % vel == 0) && al(c.out) &&
            (c.out2 == nullptr || al(c.out2)) && (c.aux == nullptr || al(c.aux));
  }
  {
    // every split must own >= 1 k-block (an empty split would never signal
    // its accumulator): recompute the split count from the per-split depth
    const int kb = (c.K + 63) / 64;
    const int kbps = (kb + splits - 1) / splits;
    splits = (kb + kbps - 1) / kbps;
    p.kb_per_split = kbps;
  }
  p.splits = splits;
  // row sums: every column tile of a row block sums 1 / tiles_n of the
  // k-blocks into its own partial (balanced: with one tile per CTA the first
  // column tiles alone would set the kernel time) when the workspace holds
  // [splits][tiles_n][M] partials after the split-K block; else the first
  // column tile sums all, per split
  int rs_parts = 1;
  float* rs_ws = nullptr;
  if (c.rowsum != nullptr) {
    const int tiles_n = (c.N + bn - 1) / bn;
    const int64_t base = splits > 1 ? (int64_t)splits * c.M * c.N : 0;
    if (tiles_n > 1 && c.workspace != nullptr &&
        (base + (int64_t)splits * tiles_n * c.M) * 4 <= c.workspace_bytes)
      rs_parts = tiles_n;
    if (splits > 1 || rs_parts > 1) {
      if ((base + (int64_t)splits * rs_parts * c.M) * 4 > c.workspace_bytes)
        return cudaErrorInvalidValue;
      rs_ws = static_cast<float*>(c.workspace) + base;
      p.rowsum = rs_ws;
    }
  }
  p.rs_parts = rs_parts;
  // output through TMA when the view is addressable (16 B pitch / batch strides)
  CUtensorMap td{}, td2{};
  if (splits > 1) {
    // partials: workspace viewed as [splits][M][N] fp32, split index = batch 1
    // fp32 chunk: 32 columns (128 B) -- every tile width here has >= 128 B halves
    if (!make_map_t(&td, c.workspace, c.M, c.N, c.N, (int64_t)c.M * c.N, 0, splits, 1, 32, 32, 4))
      return cudaErrorInvalidValue;
    p.tma_store = 1;
    p.beta = 0.f;
  } else {
    const int esz = c.epi == kEpiF32 ? 4 : 2;
    const int cb = mimose_dev::gemm_chunk_bytes(bn, c.epi, ew);  // GemmCfg::kChunkBytes
    const uint32_t cw = cb / esz;
    const bool sw64 = cb == 64;
    auto al = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    // MIMOSE_GEMM_DIRECT_STORE=1: per-thread stores everywhere (compute-sanitizer
    // initcheck does not track TMA bulk stores, so their outputs would read as
    // uninitialised downstream)
    static const bool force_direct = [] {
      const char* e = std::getenv("MIMOSE_GEMM_DIRECT_STORE");
      return e != nullptr && std::atoi(e) != 0;
    }();
    bool ok = !c.direct_store && !force_direct && !(c.epi == kEpiF32 && c.beta != 0.f) && al(c.out) &&
              (c.ldo * esz) % 16 == 0 && (c.nb1 == 1 || (c.obs1 * esz) % 16 == 0) &&
              (c.nb2 == 1 || (c.obs2 * esz) % 16 == 0) &&
              (c.epi != kEpiBiasGelu || (c.out2 != nullptr && al(c.out2)));
    ok = ok && make_map_t(&td, c.out, c.M, c.N, c.ldo, c.obs1, c.obs2, c.nb1, c.nb2, cw, 32, esz,
                          sw64);
    if (ok && c.epi == kEpiBiasGelu)
      ok = make_map_t(&td2, c.out2, c.M, c.N, c.ldo, c.obs1, c.obs2, c.nb1, c.nb2, cw, 32, esz,
                      sw64);
    p.tma_store = ok ? 1 : 0;
    // aux (dGELU input / residual) tiles by TMA into the staging buffers: same
    // addressing as the output, so the same box and swizzle
    if (ok && c.aux != nullptr && (c.epi == kEpiDGelu || c.epi == kEpiBf16) && al(c.aux) &&
        aux_tma_enabled())
      p.aux_tma = make_map_t(&td2, const_cast<void*>(c.aux), c.M, c.N, c.ldo, c.obs1, c.obs2,
                             c.nb1, c.nb2, cw, 32, esz, sw64) ? 1 : 0;
  }

  const int64_t tiles = (int64_t)((c.M + 128 * cg - 1) / (128 * cg)) * ((c.N + bn - 1) / bn) *
                        c.nb1 * c.nb2 * splits;
  // CTAs (cg = 1) or CTA pairs (cg = 2) resident at once (64-wide tiles: two per SM)
  const int slots =
      sm_count() * ((bn == 64 && ew == 8 && c.epi == kEpiBf16 && cg == 1) ? 2 : 1) / cg;
  const int grid = (int)(tiles < slots ? tiles : slots) * cg;
  // roofline record: algorithmic flops 2*M*N*K*batch; algorithmic bytes =
  // operands read once + outputs (and epilogue side inputs) once. Batched
  // (per-head) views are the materialised-attention contractions.
  const double nb = (double)c.nb1 * c.nb2;
  const double osz = c.epi == kEpiF32 ? 4.0 : 2.0;
  double gbytes = nb * (2.0 * c.M * c.K + 2.0 * c.N * c.K + osz * c.M * c.N);
  if (c.epi == kEpiBiasGelu) gbytes += nb * 2.0 * c.M * c.N;       // second output (u, g)
  if (c.aux != nullptr) gbytes += nb * 2.0 * c.M * c.N;             // residual / GELU input
  if (c.epi == kEpiF32 && c.beta != 0.f) gbytes += nb * 4.0 * c.M * c.N;
  std::string gdesc;
  if (prof_on())
    gdesc = std::to_string(c.M) + " " + std::to_string(c.N) + " " + std::to_string(c.K) + " " +
            std::to_string(c.nb1 * c.nb2) + " bn" + std::to_string(bn) + " amn" +
            std::to_string((int)c.a_mn) + " bmn" + std::to_string((int)c.b_mn) + " epi" +
            std::to_string(c.epi) + " ew" + std::to_string(ew) + " cg" + std::to_string(cg) +
            " splits" + std::to_string(splits) + " grid" +
            std::to_string(grid);
  ProfScope prof(nb > 1 ? "gemm_attn" : "gemm_dense", 2.0 * c.M * (double)c.N * c.K * nb, gbytes,
                 stream, gdesc);
  cudaError_t err = cudaErrorInvalidValue;
  switch (bn) {
    case 64: err = launch_bn<64>(c.epi, ew, ta, tb, td, td2, p, grid, stream); break;
    case 128: err = launch_bn<128>(c.epi, ew, ta, tb, td, td2, p, grid, stream); break;
    case 256:
      err = cg == 2 ? launch_pair(c.epi, ew, ta, tb, td, td2, p, grid, stream)
                    : launch_bn<256>(c.epi, ew, ta, tb, td, td2, p, grid, stream);
      break;
  }
  if (err == cudaSuccess && splits > 1) {
    splitk_reduce_kernel<<<4 * sm_count(), 256, 0, stream>>>(
        static_cast<const float*>(c.workspace), splits, c.M, c.N, static_cast<float*>(c.out),
        c.ldo, c.beta, c.rowsum, splits * rs_parts);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    err = cudaGetLastError();
  } else if (err == cudaSuccess && rs_ws != nullptr) {
    rowsum_reduce_kernel<<<(c.M + 255) / 256, 256, 0, stream>>>(rs_ws, rs_parts, c.M, c.rowsum);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    err = cudaGetLastError();
  }
  return err;
}

void gemm_profile_enable(bool on) { prof_enable(on); }

std::string gemm_profile_csv() { return prof_csv(); }

cudaError_t gemm_profile_read(double* flops, double* ms, int64_t* launches) {
  double bytes = 0.0;
  return prof_read("gemm", flops, &bytes, ms, launches);
}

}  // namespace mimose_ops

#ifdef MIMOSE_GEMM_TRACE
extern "C" int mimose_debug_trace(void* dst, int n, int clear) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(dst, mimose_dev::g_gemm_trace, n * 8);
  if (clear) {
    static unsigned long long z[1 << 15];
    cudaMemcpyToSymbol(mimose_dev::g_gemm_trace, z, sizeof(z));
  }
  return 0;
}
#endif
