// Device helpers shared by the memory-bound kernels: counter-based dropout
// RNG, bf16 <-> fp32 vector packing, warp reductions.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "dropout_cfg.hpp"

namespace mimose_dev {

// ------------------------------------------------------------------ Philox
// Philox4x32-10 (Salmon et al., SC'11). Dropout masks are a pure function of
// (seed, stream, element index): recompute of a dropped layer and the
// sheltered measuring pass regenerate bit-identical masks without saving
// them (replaces the paper's RNG save/restore).
struct Philox {
  uint32_t r[4];
  __device__ __forceinline__ Philox(uint64_t seed, uint64_t stream, uint64_t group) {
    uint32_t c0 = (uint32_t)group, c1 = (uint32_t)(group >> 32);
    uint32_t c2 = (uint32_t)stream, c3 = (uint32_t)(stream >> 32);
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
      const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
      c0 = hi1 ^ c1 ^ k0;
      c1 = lo1;
      c2 = hi0 ^ c3 ^ k1;
      c3 = lo0;
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    r[0] = c0; r[1] = c1; r[2] = c2; r[3] = c3;
  }
};

// keep-mask bits for 8 consecutive elements starting at `idx` (idx % 8 == 0):
// one Philox call per 8 elements; element idx + e compares the 16-bit half
// (e & 1) of word (e >> 1) of Philox(seed, stream, idx >> 3) with the
// threshold round(p * 65536).
__device__ __forceinline__ uint32_t dropout_mask8(const DropoutCfg& d, uint64_t idx) {
  if (d.threshold == 0) return 0xFFu;
  const Philox a(d.seed, d.stream, idx >> 3);
  uint32_t m = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const uint32_t r16 = (a.r[e >> 1] >> (16 * (e & 1))) & 0xFFFFu;
    m |= (r16 >= d.threshold ? 1u : 0u) << e;
  }
  return m;
}

// N independent Philox4x32-10 blocks (same key, counters (stream, group[i]))
// computed round-major: the key schedule is evaluated once per round for all
// N blocks, and the N multiply chains interleave. Bit-identical to Philox.
template <int N>
__device__ __forceinline__ void philox_n(uint64_t seed, uint64_t stream, const uint64_t (&group)[N],
                                         uint32_t (&out)[N][4]) {
  uint32_t c0[N], c1[N], c2[N], c3[N];
#pragma unroll
  for (int n = 0; n < N; ++n) {
    c0[n] = (uint32_t)group[n];
    c1[n] = (uint32_t)(group[n] >> 32);
    c2[n] = (uint32_t)stream;
    c3[n] = (uint32_t)(stream >> 32);
  }
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int i = 0; i < 10; ++i) {
#pragma unroll
    for (int n = 0; n < N; ++n) {
      const uint64_t p0 = (uint64_t)0xD2511F53u * c0[n];
      const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2[n];
      c0[n] = (uint32_t)(p1 >> 32) ^ c1[n] ^ k0;
      c1[n] = (uint32_t)p1;
      c2[n] = (uint32_t)(p0 >> 32) ^ c3[n] ^ k1;
      c3[n] = (uint32_t)p0;
    }
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
#pragma unroll
  for (int n = 0; n < N; ++n) {
    out[n][0] = c0[n];
    out[n][1] = c1[n];
    out[n][2] = c2[n];
    out[n][3] = c3[n];
  }
}

// keep predicate from a raw Philox block (see philox_keep)
__device__ __forceinline__ bool philox_keep_w(const uint32_t (&r)[4], int e, uint32_t thr_hi) {
  const uint32_t w = r[e >> 1];
  return ((e & 1) ? w : (w << 16)) >= thr_hi;
}

// 2^x for x <= 0 (softmax exponentials): ex2.approx.ftz, no range fix-up
__device__ __forceinline__ float exp2_neg(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// keep predicate of element e (0..7) of a Philox group without building the
// 8-bit mask: the 16-bit half (e & 1) of word (e >> 1) is >= threshold
// <=> (word << 16) >= thr_hi (even e) / word >= thr_hi (odd e), with
// thr_hi = threshold << 16 (threshold 0 keeps everything). Same decision as
// dropout_mask8 bit e.
__device__ __forceinline__ bool philox_keep(const Philox& a, int e, uint32_t thr_hi) {
  const uint32_t w = a.r[e >> 1];
  return ((e & 1) ? w : (w << 16)) >= thr_hi;
}

// keep decision for a single element (head kernel)
__device__ __forceinline__ bool dropout_keep1(const DropoutCfg& d, uint64_t idx) {
  if (d.threshold == 0) return true;
  const Philox a(d.seed, d.stream, idx >> 3);
  const int e = static_cast<int>(idx & 7);
  return ((a.r[e >> 1] >> (16 * (e & 1))) & 0xFFFFu) >= d.threshold;
}

// ------------------------------------------------------------------ vectors
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&v)[8]) {
  const uint4 raw = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}

__device__ __forceinline__ void store8(__nv_bfloat16* p, const float (&v)[8]) {
  uint4 raw;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = raw;
}

// Round-trip through bf16 (value a kernel would observe after store + load).
__device__ __forceinline__ float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace mimose_dev
