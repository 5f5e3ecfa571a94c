// Persistent warp-specialised bf16 GEMM for sm_100a:
//   TMA (128B-swizzled tiles) -> smem ring (mbarrier full/empty) ->
//   tcgen05.mma (one elected thread, fp32 accumulators in TMEM, double
//   buffered) -> tcgen05.ld epilogue (bias / GELU / dGELU / residual / fp32)
//   -> swizzled smem staging -> TMA bulk tensor store.
//
//   D[z][m][n] = sum_k A[z][m][k] * B[z][n][k]
//
// Either operand may be K-major (k contiguous) or MN-major (m/n contiguous),
// which is what lets the same kernel run forward (X W^T), data-gradient
// (dY W) and weight-gradient (dY^T X) contractions plus every batched
// attention contraction (QK^T, PV, dO V^T, P^T dO, dS K, dS^T Q) without a
// transpose pass. Batched operands are addressed through 4-D tensor maps
// (cols, rows, batch1, batch2), so per-head views into the fused QKV buffer
// need no copies. The output is written through a 4-D tensor map as well
// (full 128-byte lines, clipped at the M/N edges by the TMA unit); views the
// TMA cannot address (unaligned pitch, fp32 read-modify-write) fall back to
// per-thread vector stores.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "ptx_sm100.cuh"

namespace mimose_dev {

enum EpiKind : int {
  kEpiBf16 = 0,      // out(bf16) = alpha*acc + bias (+ aux)
  kEpiBiasGelu = 1,  // out(bf16) = u = acc + bias ; out2(bf16) = gelu(u)
  kEpiDGelu = 2,     // out(bf16) = acc * gelu'(aux)
  kEpiF32 = 3,       // out(f32)  = alpha*acc + beta*out
};

struct GemmParams {
  int M, N, K;
  int nb1, nb2;             // batch = nb1 * nb2; z -> (z % nb1, z / nb1)
  int a_mn, b_mn;           // operand majors (0 = K-major, 1 = MN-major)
  void* out;                // bf16 or f32 depending on epilogue
  void* out2;               // bf16 (GELU output)
  const __nv_bfloat16* aux; // bf16, same addressing as out (dGELU input / residual)
  const float* bias;        // [N] or nullptr
  long long ldo, obs1, obs2;  // output strides in elements
  float alpha, beta;
  int vec;                  // 1 if 16-byte vector stores/loads are aligned (fallback path)
  int tma_store;            // 1: stage through smem + TMA store
  int splits;               // split-K factor (>1: fp32 partials, batch must be 1)
  int kb_per_split;         // k-blocks per split
  int gelu_tanh;            // GELU flavour of kEpiBiasGelu / kEpiDGelu: 0 erf, 1 tanh
  int gelu_deriv;           // kEpiBiasGelu: out = GELU'(u) instead of u (the backward's
                            // only use of u); kEpiDGelu: aux already holds GELU'(u), so
                            // the epilogue is a plain product
  DropoutCfg drop;          // kEpiBf16: dropout on (alpha*acc + bias) before adding aux
  int causal_tiles;         // batched S x S score GEMMs of a causal model: skip tiles
                            // whose columns (keys) all exceed their rows (queries)
  int aux_tma;              // 1: the aux tile arrives by TMA (map in the tmD2 slot) into
                            // the warp's staging buffers instead of per-row loads
  int causal_k;             // causal contractions over S: 1 = only k <= row contributes
                            // (P V, dS K), 2 = only k >= row (P^T dO, dS^T Q); the
                            // k-blocks outside are exact zeros and are skipped
  float* rowsum;            // kEpiF32, MN-major A: sums of A's rows over this split's K
                            // range (the bias gradient of a weight-gradient GEMM, dY^T 1,
                            // read from the staged dY tiles) -> rowsum[part * M + m]
  int rs_parts;             // 1: the first column tile of a row block sums every k-block
                            // (part = split); tiles_n: column tile tn sums the k-blocks
                            // kb0 + tn, + tiles_n, ... (part = split * tiles_n + tn)
};

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kSmemBudget = 227 * 1024;

// EW epilogue warps: EW / 4 per TMEM lane quarter, each owning BN / (EW / 4)
// accumulator columns. 8 (column halves) by default; 16 (column quarters)
// for the math-heavy GELU / dGELU epilogues and the write-bound attention
// contractions, which would otherwise leave the tensor pipe idle.
// warp 0 TMA, warp 1 MMA, EW epilogue warps; fp32 (weight-gradient) kernels
// add kRsWarps A-row-sum warps after the epilogue warps
constexpr int kRsWarps = 4;
constexpr int gemm_threads(int EW, int EPI = -1) {
  return 64 + 32 * EW + (EPI == kEpiF32 ? 32 * kRsWarps : 0);
}

// staged row chunk of one epilogue warp: 128 B (SWIZZLE_128B) or 64 B
// (SWIZZLE_64B) when the warp's column span is narrower than 128 B or when
// 16 warps share the register file (32-column chunks)
constexpr int gemm_chunk_bytes(int BN, int EPI, int EW) {
  return (EW == 16 && EPI != kEpiF32) ? 64
         : ((BN / (EW / 4)) * (EPI == kEpiF32 ? 4 : 2) >= 128 ? 128 : 64);
}

// CG = cta_group: 1 (one SM per 128 x BN tile) or 2 (a CTA pair per
// 256 x BN tile: each CTA loads its 128 A rows and half of the B rows, the
// leader issues the pair's MMAs, each CTA's TMEM holds its 128 output rows)
template <int BN, int EPI, int EW = 8, int CG = 1>
struct GemmCfg {
  static constexpr int kBRows = BN / CG;  // B rows staged per CTA
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = kBRows * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kNOut = EPI == kEpiBiasGelu ? 2 : 1;
  // the GELU epilogue's two outputs go through the same staging buffer one
  // after the other: one fewer buffer per warp buys a pipeline stage
  static constexpr int kEsz = EPI == kEpiF32 ? 4 : 2;
  static constexpr int kEpiWarps = EW;
  static constexpr int kColParts = EW / 4;
  static constexpr int kThreads = gemm_threads(EW, EPI);
  static constexpr int kChunkBytes = gemm_chunk_bytes(BN, EPI, EW);
  static constexpr int kChunkCols = kChunkBytes / kEsz;
  static constexpr int kBufBytes = 32 * kChunkBytes;  // 32 rows x one chunk
  // per epilogue warp: kBufs sets of kNOut buffers of 32 rows x kChunkBytes
  // (2 measured for plain outputs: attention unchanged, dense -4 %; the dGELU
  // epilogue takes 2 so both chunks' aux tiles are requested by TMA before
  // the accumulator is ready)
  static constexpr int kBufs = EPI == kEpiDGelu ? 2 : 1;
  static constexpr int kStagingBytes = EW * kBufs * kBufBytes;
  // TMEM accumulators: as many BN-column tiles as fit 512 columns (max 4), so
  // the MMA can run up to kAcc - 1 tiles ahead of the epilogue
  static constexpr int kAcc = (512 / BN) > 4 ? 4 : (512 / BN);
  // bias is read straight from global memory (uniform across the warp: one
  // L1 broadcast per float4) rather than staged per tile in shared memory
  static constexpr int kBiasBytes = 0;
  // row-sum warps' per-tile combine: [kRsWarps][128] floats after the barriers
  static constexpr int kRsBytes = EPI == kEpiF32 ? kRsWarps * 128 * 4 : 0;
  // 64-wide tiles (the streaming attention contractions, K = S) run two CTAs
  // per SM: two independent load / MMA / epilogue pipelines, each with half
  // the shared memory and TMEM
  static constexpr int kMinBlocks = (BN == 64 && EW == 8 && EPI == kEpiBf16 && CG == 1) ? 2 : 1;
  static constexpr int kStagesRaw =
      (kSmemBudget / kMinBlocks - 1024 - 512 - kStagingBytes - kBiasBytes - kRsBytes) / kStageBytes;
  // two-CTA-per-SM contractions measured fastest with 3 stages (S = 288
  // step, P.V / dV / dK / dQ: 2 stages 2.40 ms, 3 stages 2.12, 4 stages 2.69)
  static constexpr int kMaxStages = kMinBlocks == 2 ? 3 : 8;
  static constexpr int kStages = kStagesRaw > kMaxStages ? kMaxStages : kStagesRaw;
  static constexpr int kTmemCols = kAcc * BN;
  static constexpr int kSmemBytes =
      kStages * kStageBytes + kStagingBytes + kBiasBytes + 1024 + 512 + kRsBytes;
  static_assert(kStages >= 2, "not enough shared memory for a pipeline");
};

// erf(z) with |error| < 1.5e-7 (Abramowitz & Stegun 7.1.26), branch-free, and
// the e^{-z^2} it needs (reused by the GELU derivative). The GELU output is
// rounded to bf16 (rel. 2^-9), so this is exact for every purpose here while
// costing ~1/3 of erff.
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float erf_as(float z, float& ez2) {
  const float a = fabsf(z);
  const float t = rcp_approx(fmaf(0.3275911f, a, 1.0f));
  ez2 = ex2_approx(-1.4426950408889634f * z * z);
  float poly = fmaf(1.061405429f, t, -1.453152027f);
  poly = fmaf(poly, t, 1.421413741f);
  poly = fmaf(poly, t, -0.284496736f);
  poly = fmaf(poly, t, 0.254829592f);
  const float r = fmaf(-poly * t, ez2, 1.0f);
  return copysignf(r, z);
}

// Epilogue forms of GELU / GELU' (exact-erf GELU, the same A&S 7.1.26 erf
// with |error| < 1.5e-7), rearranged for instruction count: with
// a = |x| / sqrt 2, t = 1 / (1 + p a), e = 2^(-x^2 / (2 ln 2)) = e^{-x^2/2}
// and h = 0.5 * t * poly(t) * e = 0.5 * erfc(a):
//   Phi(x) = x >= 0 ? 1 - h : h,   GELU(x) = x Phi(x),
//   GELU'(x) = Phi(x) + x e / sqrt(2 pi).
// Evaluated on PAIRS with the paired f32x2 instructions (FFMA2 / FMUL2: the
// GELU / dGELU GEMM epilogues are issue-bound), 2 MUFU per element. Every
// caller (GEMM epilogues, the u-only regeneration kernel) uses these pair
// forms, so a regenerated g is bit-identical to the epilogue's.
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 gelu_half_erfc2(float2 x, float2& e) {
  const float2 ta = __ffma2_rn(f2(0.3275911f * 0.70710678118654752f),
                               make_float2(fabsf(x.x), fabsf(x.y)), f2(1.0f));
  const float2 t = make_float2(rcp_approx(ta.x), rcp_approx(ta.y));
  const float2 ea = __fmul2_rn(__fmul2_rn(f2(-0.72134752044448170f), x), x);  // -log2(e) / 2
  e = make_float2(ex2_approx(ea.x), ex2_approx(ea.y));
  // 0.5 * (A&S coefficients)
  float2 poly = __ffma2_rn(f2(0.5307027145f), t, f2(-0.7265760135f));
  poly = __ffma2_rn(poly, t, f2(0.7107068705f));
  poly = __ffma2_rn(poly, t, f2(-0.142248368f));
  poly = __ffma2_rn(poly, t, f2(0.127414796f));
  return __fmul2_rn(__fmul2_rn(poly, t), e);
}
__device__ __forceinline__ float2 gelu_fast2(float2 x) {
  float2 e;
  const float2 h = gelu_half_erfc2(x, e);
  const float2 xh = __fmul2_rn(x, h);
  const float2 d = __ffma2_rn(xh, f2(-1.0f), x);  // x - xh (the product by -1 is exact)
  return make_float2(x.x >= 0.f ? d.x : xh.x, x.y >= 0.f ? d.y : xh.y);
}
__device__ __forceinline__ float2 dgelu_fast2(float2 x) {
  float2 e;
  const float2 h = gelu_half_erfc2(x, e);
  const float2 omh = __ffma2_rn(h, f2(-1.0f), f2(1.0f));  // 1 - h
  const float2 cdf = make_float2(x.x >= 0.f ? omh.x : h.x, x.y >= 0.f ? omh.y : h.y);
  return __ffma2_rn(__fmul2_rn(x, f2(0.39894228040143268f)), e, cdf);
}
// GELU and GELU' of the same pair from one h / e evaluation (bit-identical to
// gelu_fast2 / dgelu_fast2: same operations on the same values)
__device__ __forceinline__ float2 gelu_both2(float2 x, float2& dg) {
  float2 e;
  const float2 h = gelu_half_erfc2(x, e);
  const float2 xh = __fmul2_rn(x, h);
  const float2 d = __ffma2_rn(xh, f2(-1.0f), x);
  const float2 omh = __ffma2_rn(h, f2(-1.0f), f2(1.0f));
  const float2 cdf = make_float2(x.x >= 0.f ? omh.x : h.x, x.y >= 0.f ? omh.y : h.y);
  dg = __ffma2_rn(__fmul2_rn(x, f2(0.39894228040143268f)), e, cdf);
  return make_float2(x.x >= 0.f ? d.x : xh.x, x.y >= 0.f ? d.y : xh.y);
}
__device__ __forceinline__ float gelu_fast(float x) { return gelu_fast2(make_float2(x, x)).x; }
__device__ __forceinline__ float dgelu_fast(float x) { return dgelu_fast2(make_float2(x, x)).x; }

#ifdef MIMOSE_GELU_ERFF  // libm erff variant (A/B timing only)
__device__ __forceinline__ float gelu_f(float x) {
  return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
}
__device__ __forceinline__ float dgelu_f(float x) {
  const float cdf = 0.5f * (1.0f + erff(x * 0.70710678118654752f));
  return cdf + x * 0.39894228040143268f * __expf(-0.5f * x * x);
}
#else
// exact-erf GELU: x * Phi(x) = 0.5 x (1 + erf(x / sqrt 2))
__device__ __forceinline__ float gelu_f(float x) {
  float e;
  return 0.5f * x * (1.0f + erf_as(x * 0.70710678118654752f, e));
}
// d/dx GELU = Phi(x) + x phi(x), phi(x) = e^{-x^2/2} / sqrt(2 pi)
__device__ __forceinline__ float dgelu_f(float x) {
  float e;
  const float cdf = 0.5f * (1.0f + erf_as(x * 0.70710678118654752f, e));
  return fmaf(x * 0.39894228040143268f, e, cdf);
}
#endif

// tanh-approximation GELU ("gelu_new", GPT-2): 0.5 x (1 + tanh(k0 (x + k1 x^3)))
__device__ __forceinline__ float tanh_approx(float x) {
  float r;
  asm("tanh.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float gelu_tanh_f(float x) {
  const float u = 0.7978845608028654f * fmaf(0.044715f * x, x * x, x);
  return 0.5f * x * (1.0f + tanh_approx(u));
}
__device__ __forceinline__ float dgelu_tanh_f(float x) {
  const float x2 = x * x;
  const float u = 0.7978845608028654f * fmaf(0.044715f * x, x2, x);
  const float t = tanh_approx(u);
  const float du = 0.7978845608028654f * fmaf(0.134145f, x2, 1.0f);
  return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * du;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
// GELU' rounded to bf16 before the dGELU product: the value the forward
// saves in gelu_deriv mode, so both modes give bit-identical gradients
__device__ __forceinline__ float2 bf16_round2(float2 x) {
  const uint32_t h = pack_bf16x2(x.x, x.y);
  return make_float2(__uint_as_float(h << 16), __uint_as_float(h & 0xFFFF0000u));
}
__device__ __forceinline__ float bf16_round(float x) { return bf16_round2(make_float2(x, x)).x; }

// Epilogue math on NV consecutive accumulator columns of one row (values in
// v, first column col0). `bias_t` points at this chunk's slice of the bias
// in global memory, p.bias + col0 (or is null); `aux_pre` holds the chunk's aux
// row prefetched before the TMEM load (or is null: load here). Results in v
// (and g for the GELU output).
template <int EPI, int NV>
__device__ __forceinline__ void epilogue_math(float (&v)[NV], float (&g)[NV], const GemmParams& p,
                                              long long obase, int col0, bool row_ok,
                                              const float* bias_t, const uint4* aux_pre) {
  if constexpr (EPI == kEpiBf16 || EPI == kEpiBiasGelu || EPI == kEpiF32) {
    if (p.alpha != 1.f) {
#pragma unroll
      for (int i = 0; i < NV; ++i) v[i] *= p.alpha;
    }
  }
  if constexpr (EPI == kEpiBf16 || EPI == kEpiBiasGelu) {
    if (bias_t != nullptr) {
      if (col0 + NV <= p.N && (reinterpret_cast<uintptr_t>(bias_t) & 15) == 0) {
#pragma unroll
        for (int q = 0; q < NV / 4; ++q) {
          const float4 b = __ldg(reinterpret_cast<const float4*>(bias_t) + q);  // warp-uniform
          const float2 lo = __fadd2_rn(make_float2(v[4 * q], v[4 * q + 1]), make_float2(b.x, b.y));
          const float2 hi = __fadd2_rn(make_float2(v[4 * q + 2], v[4 * q + 3]), make_float2(b.z, b.w));
          v[4 * q] = lo.x;
          v[4 * q + 1] = lo.y;
          v[4 * q + 2] = hi.x;
          v[4 * q + 3] = hi.y;
        }
      } else {
#pragma unroll
        for (int i = 0; i < NV; ++i)
          if (col0 + i < p.N) v[i] += __ldg(bias_t + i);
      }
    }
  }
  if constexpr (EPI == kEpiBf16) {
    // branch dropout (pre-LN residual: out = aux + dropout(x W^T + b))
    if (p.drop.threshold != 0) {
      // Philox blocks two groups at a time (round-major), keep predicates
      // straight from the words (same masks as dropout_mask8)
      const uint32_t thr_hi = p.drop.threshold << 16;
#pragma unroll
      for (int q = 0; q < NV / 8; q += 2) {
        uint64_t grp[2];
        uint32_t rnd[2][4];
#pragma unroll
        for (int u = 0; u < 2; ++u) grp[u] = ((uint64_t)obase + col0 + 8 * (q + u)) >> 3;
        philox_n<2>(p.drop.seed, p.drop.stream, grp, rnd);
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int e = 0; e < 8; ++e)
            v[8 * (q + u) + e] =
                philox_keep_w(rnd[u], e, thr_hi) ? v[8 * (q + u) + e] * p.drop.scale : 0.f;
      }
    }
  }
  if constexpr (EPI == kEpiBf16 || EPI == kEpiDGelu) {
    if (p.aux != nullptr && row_ok) {
      const __nv_bfloat16* ax = p.aux + obase + col0;
      if (aux_pre != nullptr || (p.vec && col0 + NV <= p.N)) {
#pragma unroll
        for (int q = 0; q < NV / 8; ++q) {
          const uint4 raw = aux_pre != nullptr ? aux_pre[q]
                                               : *reinterpret_cast<const uint4*>(ax + 8 * q);
          const __nv_bfloat16* av = reinterpret_cast<const __nv_bfloat16*>(&raw);
          if constexpr (EPI == kEpiBf16) {
#pragma unroll
            for (int i = 0; i < 8; ++i) v[8 * q + i] += __bfloat162float(av[i]);
          } else if (p.gelu_deriv) {
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
              const float2 r = __fmul2_rn(make_float2(v[8 * q + i], v[8 * q + i + 1]),
                                          make_float2(__bfloat162float(av[i]), __bfloat162float(av[i + 1])));
              v[8 * q + i] = r.x;
              v[8 * q + i + 1] = r.y;
            }
          } else if (p.gelu_tanh) {
#pragma unroll
            for (int i = 0; i < 8; ++i) v[8 * q + i] *= bf16_round(dgelu_tanh_f(__bfloat162float(av[i])));
          } else {
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
              const float2 d = bf16_round2(
                  dgelu_fast2(make_float2(__bfloat162float(av[i]), __bfloat162float(av[i + 1]))));
              const float2 r = __fmul2_rn(make_float2(v[8 * q + i], v[8 * q + i + 1]), d);
              v[8 * q + i] = r.x;
              v[8 * q + i + 1] = r.y;
            }
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          if (col0 + i < p.N) {
            const float a = __bfloat162float(ax[i]);
            if constexpr (EPI == kEpiBf16) v[i] += a;
            else v[i] *= p.gelu_deriv ? a : bf16_round(p.gelu_tanh ? dgelu_tanh_f(a) : dgelu_fast(a));
          }
        }
      }
    }
  }
  if constexpr (EPI == kEpiBiasGelu) {
    // GELU of the bf16-rounded pre-activation, so recompute and the saved u
    // agree bit for bit with what backward differentiates (round a pair with
    // one F2FP, widen back with two bit ops)
#pragma unroll
    for (int i = 0; i < NV; i += 2) {
      const uint32_t h = pack_bf16x2(v[i], v[i + 1]);
      v[i] = __uint_as_float(h << 16);
      v[i + 1] = __uint_as_float(h & 0xFFFF0000u);
    }
    if (p.gelu_deriv) {  // g = GELU(u), v = GELU'(u) from one erfc / exponential
      if (p.gelu_tanh) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          g[i] = gelu_tanh_f(v[i]);
          v[i] = dgelu_tanh_f(v[i]);
        }
      } else {
#pragma unroll
        for (int i = 0; i < NV; i += 2) {
          float2 d;
          const float2 r = gelu_both2(make_float2(v[i], v[i + 1]), d);
          g[i] = r.x;
          g[i + 1] = r.y;
          v[i] = d.x;
          v[i + 1] = d.y;
        }
      }
    } else if (p.gelu_tanh) {
#pragma unroll
      for (int i = 0; i < NV; ++i) g[i] = gelu_tanh_f(v[i]);
    } else {
#pragma unroll
      for (int i = 0; i < NV; i += 2) {
        const float2 r = gelu_fast2(make_float2(v[i], v[i + 1]));
        g[i] = r.x;
        g[i + 1] = r.y;
      }
    }
  }
}

// Pipeline trace (build with -DMIMOSE_GEMM_TRACE; tools/gemm_trace.py): CTA 0
// records SM clocks per tile -- MMA start / last issue / cycles waiting for
// operands, and per epilogue warp the accumulator wait and the release. Off
// by default: every GT / GT_CLK compiles to nothing.
#ifdef MIMOSE_GEMM_TRACE
__device__ unsigned long long g_gemm_trace[1 << 15];
__device__ __forceinline__ unsigned long long clk64() {
  unsigned long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}
#define GT(i, v) if (blockIdx.x == 0 && (i) < (1 << 15)) g_gemm_trace[i] = (v)
#define GT_CLK() clk64()
#else
#define GT(i, v)
#define GT_CLK() 0ull
#endif

template <int BN, int EPI, int EW, int CG>
__global__ void __launch_bounds__(gemm_threads(EW, EPI), (GemmCfg<BN, EPI, EW, CG>::kMinBlocks))
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmD,
                        const __grid_constant__ CUtensorMap tmD2, const GemmParams p) {
  using Cfg = GemmCfg<BN, EPI, EW, CG>;
  constexpr int S = Cfg::kStages;
  constexpr int kEpiWarps = EW;
  constexpr int kTileM = kBM * CG;  // output rows per (pair) tile
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kABytes;
  uint8_t* sD = smem + S * Cfg::kStageBytes;  // epilogue staging (1024-aligned)
  uint64_t* full = reinterpret_cast<uint64_t*>(sD + Cfg::kStagingBytes + Cfg::kBiasBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;             // [kAcc]
  uint64_t* tempty = tfull + Cfg::kAcc;    // [kAcc]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + Cfg::kAcc);
  uint64_t* abar = tempty + Cfg::kAcc + 1;  // [EW][kBufs] aux-tile arrivals
  uint64_t* rs_done = abar + kEpiWarps * Cfg::kBufs;  // [S] row-sum warps done with a stage
  float* rs_red = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 512);  // [4][128]
  static_assert((2 * S + 2 * Cfg::kAcc + 1 + EW * Cfg::kBufs + S) * 8 <= 512,
                "barrier block overflows its 512 B");
  const bool rowsum = EPI == kEpiF32 && p.rowsum != nullptr;

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;

  const int tiles_m = (p.M + kTileM - 1) / kTileM;
  const int tiles_n = (p.N + BN - 1) / BN;
  const int tiles_per_batch = tiles_m * tiles_n;
  const int num_tiles = tiles_per_batch * p.nb1 * p.nb2 * p.splits;
  const int num_kb = (p.K + kBK - 1) / kBK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (p.tma_store) {
      tma_prefetch(&tmD);
      if (EPI == kEpiBiasGelu || p.aux_tma) tma_prefetch(&tmD2);
    }
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < Cfg::kAcc; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps * CG);  // one arrive per epilogue warp (of both CTAs)
    }
    for (int i = 0; i < kEpiWarps * Cfg::kBufs; ++i) mbar_init(&abar[i], 1);
    for (int s = 0; s < S; ++s) mbar_init(&rs_done[s], kRsWarps);
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (CG == 2) tmem_alloc_2sm(tmem_slot, Cfg::kTmemCols);
    else tmem_alloc(tmem_slot, Cfg::kTmemCols);
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync_all();  // peer barriers initialised before any remote signal
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // inputs of this launch are complete from here on

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int it = 0;
      const uint32_t full_leader = CG == 2 ? mapa_rank(&full[0], 0) : 0u;
      for (int tile = blockIdx.x / CG; tile < num_tiles; tile += gridDim.x / CG) {
        const int zz = tile / tiles_per_batch;
        const int t_in = tile % tiles_per_batch;
        if (p.causal_tiles && (t_in % tiles_n) * BN >= (t_in / tiles_n) * kTileM + kTileM) continue;
        // n-fastest raster: the CTAs that run concurrently share one A row
        // block (read once from HBM) and cycle through B (weights, L2-resident)
        const int m0 = (t_in / tiles_n) * kTileM + (int)rank * kBM;
        const int n0 = (t_in % tiles_n) * BN + (int)rank * Cfg::kBRows;
        const int split = zz % p.splits, z = zz / p.splits;
        const int b1 = z % p.nb1, b2 = z / p.nb1;
        int kb0 = split * p.kb_per_split;
        int kb1 = min(num_kb, kb0 + p.kb_per_split);
        {
          const int mb = (t_in / tiles_n) * kTileM;
          if (p.causal_k == 1) kb1 = min(kb1, (mb + kTileM + kBK - 1) / kBK);
          if (p.causal_k == 2) kb0 = max(kb0, mb / kBK);
        }
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % S;
          const uint32_t ph = (it / S) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          if (rowsum) mbar_wait(&rs_done[s], ph ^ 1);  // the row-sum warp has read it too
          uint8_t* a_dst = sA + s * Cfg::kABytes;
          uint8_t* b_dst = sB + s * Cfg::kBBytes;
          const int k0 = kb * kBK;
          if constexpr (CG == 2) {
            // both CTAs' bytes complete on the leader's full[s]; only the
            // leader arms it (a peer's early complete_tx is absorbed: the
            // phase cannot flip before the leader's arrive)
            const uint32_t fb = full_leader + (uint32_t)(s * sizeof(uint64_t));
            if (leader) mbar_arrive_expect_tx(&full[s], CG * Cfg::kStageBytes);
            if (!p.a_mn) {
              tma_load_4d_2sm(&tmA, fb, a_dst, k0, m0, b1, b2);
            } else {
#pragma unroll
              for (int j = 0; j < kBM / 64; ++j)
                tma_load_4d_2sm(&tmA, fb, a_dst + j * 8192, m0 + 64 * j, k0, b1, b2);
            }
            if (!p.b_mn) {
              tma_load_4d_2sm(&tmB, fb, b_dst, k0, n0, b1, b2);
            } else {
#pragma unroll
              for (int j = 0; j < Cfg::kBRows / 64; ++j)
                tma_load_4d_2sm(&tmB, fb, b_dst + j * 8192, n0 + 64 * j, k0, b1, b2);
            }
          } else {
            mbar_arrive_expect_tx(&full[s], Cfg::kStageBytes);
            if (!p.a_mn) {
              tma_load_4d(&tmA, &full[s], a_dst, k0, m0, b1, b2);
            } else {
#pragma unroll
              for (int j = 0; j < kBM / 64; ++j)
                tma_load_4d(&tmA, &full[s], a_dst + j * 8192, m0 + 64 * j, k0, b1, b2);
            }
            if (!p.b_mn) {
              tma_load_4d(&tmB, &full[s], b_dst, k0, n0, b1, b2);
            } else {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j)
                tma_load_4d(&tmB, &full[s], b_dst + j * 8192, n0 + 64 * j, k0, b1, b2);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // (CTA pair: the leader alone issues the 256-row MMAs for both CTAs)
    if (CG == 1 || leader) {
    const uint32_t idesc = idesc_bf16_f32(kTileM, BN, p.a_mn != 0, p.b_mn != 0);
    // K-major: advance 16 elements = 32 B inside the 128 B swizzle row.
    // MN-major: advance 16 K-rows = 2048 B; LBO = 64 rows * 128 B between MN blocks.
    const uint32_t a_step = p.a_mn ? 2048u : 32u;
    const uint32_t b_step = p.b_mn ? 2048u : 32u;
    const uint32_t a_lbo = p.a_mn ? 8192u : 16u;
    const uint32_t b_lbo = p.b_mn ? 8192u : 16u;
    int it = 0, local = 0;  // local counts processed tiles only (accumulator phases)
    for (int tile = blockIdx.x / CG; tile < num_tiles; tile += gridDim.x / CG) {
      {
        const int t_in = tile % tiles_per_batch;
        if (p.causal_tiles && (t_in % tiles_n) * BN >= (t_in / tiles_n) * kTileM + kTileM) continue;
      }
      const int acc = local % Cfg::kAcc;
      const uint32_t aph = (local / Cfg::kAcc) & 1;
      const int split = (tile / tiles_per_batch) % p.splits;
      int kb_n = min(num_kb, (split + 1) * p.kb_per_split) - split * p.kb_per_split;
      if (p.causal_k != 0) {  // same k-block range as the producer
        const int t_in = tile % tiles_per_batch;
        const int mb = (t_in / tiles_n) * kTileM;
        int kb0 = split * p.kb_per_split;
        int kb1 = min(num_kb, kb0 + p.kb_per_split);
        if (p.causal_k == 1) kb1 = min(kb1, (mb + kTileM + kBK - 1) / kBK);
        if (p.causal_k == 2) kb0 = max(kb0, mb / kBK);
        kb_n = kb1 - kb0;
      }
      mbar_wait(&tempty[acc], aph ^ 1);
      tc_fence_after();
      if (lane == 0 && local < 64) GT(local * 8 + 0, GT_CLK());
      unsigned long long fw = 0;
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < kb_n; ++kb, ++it) {
        const int s = it % S;
        const uint32_t ph = (it / S) & 1;
        const unsigned long long w0 = GT_CLK();
        mbar_wait(&full[s], ph);
        fw += GT_CLK() - w0;
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a_addr = smem_u32(sA + s * Cfg::kABytes);
          const uint32_t b_addr = smem_u32(sB + s * Cfg::kBBytes);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t da = smem_desc_sw128(a_addr + kk * a_step, a_lbo, 1024);
            const uint64_t db = smem_desc_sw128(b_addr + kk * b_step, b_lbo, 1024);
            if constexpr (CG == 2) umma_bf16_2sm(d_tmem, da, db, idesc, (kb | kk) != 0 ? 1u : 0u);
            else umma_bf16(d_tmem, da, db, idesc, (kb | kk) != 0 ? 1u : 0u);
          }
          if constexpr (CG == 2) {
            umma_commit_2sm(&empty[s], 0x3);
            if (kb == kb_n - 1) umma_commit_2sm(&tfull[acc], 0x3);
          } else {
            umma_commit(&empty[s]);
            if (kb == kb_n - 1) umma_commit(&tfull[acc]);
          }
        }
        __syncwarp();
      }
      if (lane == 0 && local < 64) { GT(local * 8 + 1, GT_CLK()); GT(local * 8 + 2, fw); }
      ++local;
    }
    }
  } else if (EPI == kEpiF32 && warp >= 2 + EW) {
    // ------------------------------------------------------------ A row sums
    // (MN-major A = dY of a weight gradient: its rows' sums over K are the
    // bias gradient). The kRsWarps warps follow the producer's stage
    // sequence: a stage is read after the MMAs that consumed it completed
    // (empty[s]: the commit reaches both CTAs of a pair) and handed back to
    // the producer by rs_done[s]. Only the first column tile of each row
    // block sums. Warp rw takes K rows [16 rw, 16 rw + 16) of the stage;
    // lane l reads 16-byte chunk (l & 7) of 64-row block ((l >> 3) & 1) in
    // rows of parity (l >> 4): 2 rows x 128 values per load, conflict free.
    // Per tile: lanes l, l ^ 16 combine by shuffle, the warps through smem
    // in a fixed order (deterministic).
    if (rowsum) {
      const int rw = warp - 2 - EW;
      int it = 0;
      const int j = (lane >> 3) & 1, c = lane & 7, r0 = lane >> 4;
      for (int tile = blockIdx.x / CG; tile < num_tiles; tile += gridDim.x / CG) {
        const int zz = tile / tiles_per_batch;
        const int t_in = tile % tiles_per_batch;
        const int split = zz % p.splits;
        const int kb0 = split * p.kb_per_split;
        const int kb1 = min(num_kb, kb0 + p.kb_per_split);
        const int tn = t_in % tiles_n;
        const bool active = p.rs_parts > 1 || tn == 0;
        float2 acc[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[e] = make_float2(0.f, 0.f);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % S;
          const uint32_t ph = (it / S) & 1;
          mbar_wait(&empty[s], ph);
          if (active && (p.rs_parts == 1 || (kb - kb0) % p.rs_parts == tn)) {
            const uint32_t base = smem_u32(sA + s * Cfg::kABytes) + j * 8192;
            uint4 q[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int k = 16 * rw + 2 * i + r0;
              q[i] = ld_shared_v4(base + k * 128 + ((c ^ (k & 7)) << 4));
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const uint32_t w[4] = {q[i].x, q[i].y, q[i].z, q[i].w};
#pragma unroll
              for (int e = 0; e < 4; ++e)
                acc[e] = __fadd2_rn(acc[e], make_float2(__uint_as_float(w[e] << 16),
                                                        __uint_as_float(w[e] & 0xFFFF0000u)));
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&rs_done[s]);
        }
        if (active) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            acc[e].x += __shfl_xor_sync(0xffffffffu, acc[e].x, 16);
            acc[e].y += __shfl_xor_sync(0xffffffffu, acc[e].y, 16);
          }
          const int col = j * 64 + c * 8;  // this lane's 8 row-sum slots
          if (lane < 16) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              rs_red[rw * 128 + col + 2 * e] = acc[e].x;
              rs_red[rw * 128 + col + 2 * e + 1] = acc[e].y;
            }
          }
          asm volatile("bar.sync 1, %0;" ::"n"(32 * kRsWarps) : "memory");
          if (rw == 0 && lane < 16) {
            const int m = (t_in / tiles_n) * kTileM + (int)rank * kBM + col;
            const int part = p.rs_parts > 1 ? split * p.rs_parts + tn : split;
            float* dst = p.rowsum + (size_t)part * p.M + m;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              float v = rs_red[col + e];
#pragma unroll
              for (int w2 = 1; w2 < kRsWarps; ++w2) v += rs_red[w2 * 128 + col + e];
              if (m + e < p.M) dst[e] = v;
            }
          }
          asm volatile("bar.sync 1, %0;" ::"n"(32 * kRsWarps) : "memory");  // rs_red reusable
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 2;            // epilogue warp 0..EW-1
    const int quarter = warp & 3;       // TMEM lane quarter this warp may access
    const int part = ew >> 2;           // which column part of the tile
    constexpr int CB = Cfg::kChunkBytes;
    constexpr int CW = Cfg::kChunkCols;
    constexpr int NCH = CB / 16;        // 16-byte chunks per staged row
    uint8_t* wbuf = sD + ew * (Cfg::kBufs * Cfg::kBufBytes);
    int local = 0, chunk_seq = 0;
    const uint32_t tempty_leader = CG == 2 ? mapa_rank(&tempty[0], 0) : 0u;
    for (int tile = blockIdx.x / CG; tile < num_tiles; tile += gridDim.x / CG) {
      const int zz = tile / tiles_per_batch;
      const int t_in = tile % tiles_per_batch;
      if (p.causal_tiles && (t_in % tiles_n) * BN >= (t_in / tiles_n) * kTileM + kTileM) continue;
      const int m0 = (t_in / tiles_n) * kTileM + (int)rank * kBM;
      const int n0 = (t_in % tiles_n) * BN;
      const int split = zz % p.splits, z = zz / p.splits;
      // split-K partials are addressed as batch index b1 = split of the workspace
      const int b1 = p.splits > 1 ? split : z % p.nb1;
      const int b2 = p.splits > 1 ? 0 : z / p.nb1;
      const int acc = local % Cfg::kAcc;
      const uint32_t aph = (local / Cfg::kAcc) & 1;
      const float* tb = nullptr;  // this tile's bias slice (global)
      if constexpr (EPI == kEpiBf16 || EPI == kEpiBiasGelu) {
        if (p.bias != nullptr) tb = p.bias + n0;
      }
      const int c_begin = part * (BN / Cfg::kColParts), c_end = c_begin + BN / Cfg::kColParts;
      // aux tiles by TMA: request the first kBufs chunks now (the buffers are
      // free once every earlier store has read them), so the loads overlap
      // the wait for the accumulator
      const bool aux_tma = (EPI == kEpiBf16 || EPI == kEpiDGelu) && p.aux_tma;
      auto issue_aux = [&](int c, int seq) {
        uint64_t* bar = &abar[ew * Cfg::kBufs + seq % Cfg::kBufs];
        mbar_arrive_expect_tx(bar, Cfg::kBufBytes);
        tma_load_4d(&tmD2, bar, wbuf + (seq % Cfg::kBufs) * Cfg::kBufBytes, n0 + c,
                    m0 + quarter * 32, b1, b2);
      };
      if (aux_tma && lane == 0) {
        bulk_wait_read<0>();
        for (int k = 0; k < Cfg::kBufs; ++k) {
          const int c = c_begin + k * CW;
          if (c >= c_end || n0 + c >= p.N) break;
          issue_aux(c, chunk_seq + k);
        }
      }
      if (lane == 0 && local < 64) GT(4096 + (local * 16 + ew) * 2, GT_CLK());
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      if (lane == 0 && local < 64) GT(4096 + (local * 16 + ew) * 2 + 1, GT_CLK());

      const int row = m0 + quarter * 32 + static_cast<int>(lane);
      const bool row_ok = row < p.M;
      const long long obase = (long long)b2 * p.obs2 + (long long)b1 * p.obs1 +
                              (long long)row * p.ldo;
      const uint32_t t_row = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;

      if (p.tma_store) {
        // ---- staged path: TMEM -> regs -> swizzled smem -> TMA store
#pragma unroll 1
        for (int c = c_begin; c < c_end; c += CW, ++chunk_seq) {
          if (n0 + c >= p.N) break;
          uint8_t* sb = wbuf + (chunk_seq % Cfg::kBufs) * Cfg::kBufBytes;
          // the store that last used this buffer has read it (aux by TMA: the
          // buffer was freed before its load was issued)
          if (!aux_tma && lane == 0) bulk_wait_read<Cfg::kBufs - 1>();
          __syncwarp();
          float v[CW], g[CW];
          // issue the aux-row loads before waiting on TMEM so the two latencies overlap
          uint4 aux_pre[CW / 8];
          bool have_pre = false;
          const uint32_t rbase = smem_u32(sb) + lane * CB;
          const uint32_t sw = CB == 128 ? (lane & 7) : ((lane >> 1) & 3);
          if (aux_tma) {
            mbar_wait(&abar[ew * Cfg::kBufs + chunk_seq % Cfg::kBufs], (chunk_seq / Cfg::kBufs) & 1);
#pragma unroll
            for (int j = 0; j < NCH; ++j) aux_pre[j] = ld_shared_v4(rbase + ((j ^ sw) << 4));
            have_pre = true;
          } else if constexpr (EPI == kEpiBf16 || EPI == kEpiDGelu) {
            if (p.aux != nullptr && row_ok && p.vec && n0 + c + CW <= p.N) {
              const __nv_bfloat16* ax = p.aux + obase + n0 + c;
#pragma unroll
              for (int q = 0; q < CW / 8; ++q) aux_pre[q] = *reinterpret_cast<const uint4*>(ax + 8 * q);
              have_pre = true;
            }
          }
          {
            uint32_t r[32];
#pragma unroll
            for (int h = 0; h < CW / 32; ++h) {
              tmem_ld32_nowait(t_row + c + 32 * h, r);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) v[32 * h + i] = __uint_as_float(r[i]);
            }
          }
          epilogue_math<EPI, CW>(v, g, p, obase, n0 + c, row_ok, tb ? tb + c : nullptr,
                                 have_pre ? aux_pre : nullptr);
#pragma unroll
          for (int j = 0; j < NCH; ++j) {
            const uint32_t addr = rbase + ((j ^ sw) << 4);
            if constexpr (EPI == kEpiF32) {
              st_shared_v4(addr, __float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                           __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
            } else {
              st_shared_v4(addr, pack_bf16x2(v[8 * j], v[8 * j + 1]),
                           pack_bf16x2(v[8 * j + 2], v[8 * j + 3]),
                           pack_bf16x2(v[8 * j + 4], v[8 * j + 5]),
                           pack_bf16x2(v[8 * j + 6], v[8 * j + 7]));
            }
          }
          fence_async_shared();
          __syncwarp();
          if (lane == 0) {
            tma_store_4d(&tmD, sb, n0 + c, m0 + quarter * 32, b1, b2);
            bulk_commit();
            // the next chunk's aux tile into this buffer once the store has read it
            const int cn = c + Cfg::kBufs * CW;
            if (aux_tma && cn < c_end && n0 + cn < p.N) {
              bulk_wait_read<0>();
              issue_aux(cn, chunk_seq + Cfg::kBufs);
            }
          }
          if constexpr (EPI == kEpiBiasGelu) {
            // second output through the same buffer once the first store has read it
            if (lane == 0) bulk_wait_read<0>();
            __syncwarp();
#pragma unroll
            for (int j = 0; j < NCH; ++j)
              st_shared_v4(rbase + ((j ^ sw) << 4), pack_bf16x2(g[8 * j], g[8 * j + 1]),
                           pack_bf16x2(g[8 * j + 2], g[8 * j + 3]),
                           pack_bf16x2(g[8 * j + 4], g[8 * j + 5]),
                           pack_bf16x2(g[8 * j + 6], g[8 * j + 7]));
            fence_async_shared();
            __syncwarp();
            if (lane == 0) {
              tma_store_4d(&tmD2, sb, n0 + c, m0 + quarter * 32, b1, b2);
              bulk_commit();
            }
          }
        }
      } else {
        // ---- fallback: per-thread vector stores (pitch not TMA-addressable)
#pragma unroll 1
        for (int c = c_begin; c < c_end; c += 16) {
          float v[16], g[16];
          __syncwarp();
          tmem_ld16(t_row + c, v);
          const int col0 = n0 + c;
          if (row_ok && col0 < p.N) {
            const bool full16 = p.vec && col0 + 16 <= p.N;
            if constexpr (EPI == kEpiF32) {
              float* o = reinterpret_cast<float*>(p.out) + obase + col0;
#pragma unroll
              for (int i = 0; i < 16; ++i) v[i] *= p.alpha;
              if (full16) {
                float4* o4 = reinterpret_cast<float4*>(o);
                if (p.beta != 0.f) {
#pragma unroll
                  for (int q = 0; q < 4; ++q) {
                    float4 old = o4[q];
                    v[4 * q + 0] += p.beta * old.x;
                    v[4 * q + 1] += p.beta * old.y;
                    v[4 * q + 2] += p.beta * old.z;
                    v[4 * q + 3] += p.beta * old.w;
                  }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q)
                  o4[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
              } else {
                for (int i = 0; i < 16 && col0 + i < p.N; ++i)
                  o[i] = v[i] + (p.beta != 0.f ? p.beta * o[i] : 0.f);
              }
            } else {
              epilogue_math<EPI, 16>(v, g, p, obase, col0, row_ok, tb ? tb + c : nullptr,
                                     nullptr);
              __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + obase + col0;
              alignas(16) __nv_bfloat16 hv[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) hv[i] = __float2bfloat16_rn(v[i]);
              if (full16) {
                uint4* o4 = reinterpret_cast<uint4*>(o);
                o4[0] = reinterpret_cast<const uint4*>(hv)[0];
                o4[1] = reinterpret_cast<const uint4*>(hv)[1];
              } else {
                for (int i = 0; i < 16 && col0 + i < p.N; ++i) o[i] = hv[i];
              }
              if constexpr (EPI == kEpiBiasGelu) {
#pragma unroll
                for (int i = 0; i < 16; ++i) hv[i] = __float2bfloat16_rn(g[i]);
                __nv_bfloat16* o2 = reinterpret_cast<__nv_bfloat16*>(p.out2) + obase + col0;
                if (full16) {
                  uint4* o4 = reinterpret_cast<uint4*>(o2);
                  o4[0] = reinterpret_cast<const uint4*>(hv)[0];
                  o4[1] = reinterpret_cast<const uint4*>(hv)[1];
                } else {
                  for (int i = 0; i < 16 && col0 + i < p.N; ++i) o2[i] = hv[i];
                }
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0 && local < 64) GT(8192 + (local * 16 + ew), GT_CLK());
      if (lane == 0) {
        if constexpr (CG == 2) mbar_arrive_cluster(tempty_leader + (uint32_t)(acc * sizeof(uint64_t)));
        else mbar_arrive(&tempty[acc]);
      }
      ++local;
    }
    if (p.tma_store && lane == 0) bulk_wait<0>();
  }
  if constexpr (CG == 2) {
    // both CTAs done with TMEM and with every remote barrier before teardown
    tc_fence_before();
    cluster_sync_all();
    if (warp == 1) {
      tc_fence_after();
      tmem_dealloc_2sm(tmem_base, Cfg::kTmemCols);
    }
    return;
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
}

}  // namespace mimose_dev
