// Memory-bound sm_100a kernels of the transformer step: residual + dropout +
// LayerNorm (fwd / bwd), embedding gather + LayerNorm, scaled softmax +
// dropout (fwd / bwd), deterministic column reductions, embedding gradients,
// multiple-choice head + cross-entropy, fused AdamW with global-norm clip.
//
// Rules every kernel here follows:
//   * 16-byte vector loads/stores, one warp per row, warp-shuffle reductions;
//   * no atomics: every reduction is two-stage in a fixed order, so a
//     recomputed (checkpointed) layer and a saved one produce bit-identical
//     gradients;
//   * dropout masks come from Philox(seed, stream, element) - never stored.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "ops.hpp"
#include "ops_mem.hpp"
#include "prof.hpp"

namespace mimose_dev {

using bf16 = __nv_bfloat16;

__device__ __forceinline__ void unpack8(const uint4& raw, float (&v)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}

// =====================================================================
// LayerNorm forward (one warp per row; VPL 8-element chunks per lane)
// =====================================================================
template <int VPL>
__device__ __forceinline__ void ln_row_finish(float (&z)[VPL][8], int row, int lane,
                                              const mimose_ops::LnFwdArgs& a) {
  constexpr int H = VPL * 256;
  if (a.skip_ln) {  // plain (residual) sum: y = dropout_out(z)
#pragma unroll
    for (int c = 0; c < VPL; ++c) {
      const int col = 8 * (lane + 32 * c);
      const uint64_t idx = (uint64_t)row * H + col;
      const uint32_t m = dropout_mask8(a.out_drop, idx);
      float y[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) y[e] = ((m >> e) & 1u) ? z[c][e] * a.out_drop.scale : 0.f;
      store8(static_cast<bf16*>(a.y) + idx, y);
    }
    return;
  }
  // z arrives already rounded to bf16 (what is saved is what is normalised);
  // row sums on paired f32x2 instructions (two independent chains each)
  float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < VPL; ++c)
#pragma unroll
    for (int e = 0; e < 8; e += 2) s2 = __fadd2_rn(s2, make_float2(z[c][e], z[c][e + 1]));
  const float mean = warp_sum(s2.x + s2.y) * (1.f / H);
  float2 q2 = make_float2(0.f, 0.f);
  const float2 nm2 = make_float2(-mean, -mean);
#pragma unroll
  for (int c = 0; c < VPL; ++c)
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      const float2 d = __fadd2_rn(make_float2(z[c][e], z[c][e + 1]), nm2);
      q2 = __ffma2_rn(d, d, q2);
    }
  const float var = warp_sum(q2.x + q2.y) * (1.f / H);
  const float rstd = rsqrtf(var + a.eps);
  if (a.stats != nullptr && lane == 0)
    reinterpret_cast<float2*>(a.stats)[row] = make_float2(mean, rstd);
#pragma unroll
  for (int c = 0; c < VPL; ++c) {
    const int col = 8 * (lane + 32 * c);
    const uint64_t idx = (uint64_t)row * H + col;
    float y[8], g[8], b[8];
    const float4* g4 = reinterpret_cast<const float4*>(a.gamma + col);
    const float4* b4 = reinterpret_cast<const float4*>(a.beta + col);
    *reinterpret_cast<float4*>(g) = g4[0];
    *reinterpret_cast<float4*>(g + 4) = g4[1];
    *reinterpret_cast<float4*>(b) = b4[0];
    *reinterpret_cast<float4*>(b + 4) = b4[1];
    const uint32_t m = dropout_mask8(a.out_drop, idx);
    const float2 rs2 = make_float2(rstd, rstd);
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      // (z - mean) * rstd * gamma + beta, paired
      const float2 xh = __fmul2_rn(__fadd2_rn(make_float2(z[c][e], z[c][e + 1]), nm2), rs2);
      const float2 v = __ffma2_rn(xh, make_float2(g[e], g[e + 1]), make_float2(b[e], b[e + 1]));
      y[e] = ((m >> e) & 1u) ? v.x * a.out_drop.scale : 0.f;
      y[e + 1] = ((m >> (e + 1)) & 1u) ? v.y * a.out_drop.scale : 0.f;
    }
    store8(static_cast<bf16*>(a.y) + idx, y);
  }
}

// z = res + dropout(branch); y = LN(z). Warp w of block b walks rows
// b * 8 + w, + gridDim * 8, ...; the next row's branch / residual loads are
// issued before the current row's reductions (register double-buffering).
template <int VPL, bool RES>
__global__ void __launch_bounds__(256, 2) add_ln_fwd_kernel(const mimose_ops::LnFwdArgs a) {
  constexpr int H = VPL * 256;
  const int lane = threadIdx.x & 31;
  const int stride = gridDim.x * 8;
  int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  uint4 br[VPL], rs[VPL], nbr[VPL], nrs[VPL];
  auto load = [&](int r, uint4 (&b)[VPL], uint4 (&q)[VPL]) {
#pragma unroll
    for (int c = 0; c < VPL; ++c) {
      const uint64_t idx = (uint64_t)r * H + 8 * (lane + 32 * c);
      b[c] = __ldcs(reinterpret_cast<const uint4*>(static_cast<const bf16*>(a.br) + idx));
      if constexpr (RES)
        q[c] = __ldcs(reinterpret_cast<const uint4*>(static_cast<const bf16*>(a.res) + idx));
    }
  };
  if (row < a.rows) load(row, br, rs);
  for (; row < a.rows; row += stride) {
    if (row + stride < a.rows) load(row + stride, nbr, nrs);
    float z[VPL][8];
    uint32_t rnd[VPL][4];
    if (a.br_drop.threshold != 0) {
      uint64_t grp[VPL];
#pragma unroll
      for (int c = 0; c < VPL; ++c) grp[c] = ((uint64_t)row * H + 8 * (lane + 32 * c)) >> 3;
      philox_n<VPL>(a.br_drop.seed, a.br_drop.stream, grp, rnd);
    } else {
#pragma unroll
      for (int c = 0; c < VPL; ++c) rnd[c][0] = rnd[c][1] = rnd[c][2] = rnd[c][3] = 0xFFFFFFFFu;
    }
    const uint32_t thr_hi = a.br_drop.threshold << 16;
#pragma unroll
    for (int c = 0; c < VPL; ++c) {
      const int col = 8 * (lane + 32 * c);
      const uint64_t idx = (uint64_t)row * H + col;
      float b[8];
      unpack8(br[c], b);
      float r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if constexpr (RES) unpack8(rs[c], r);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        z[c][e] = bf16r(r[e] + (philox_keep_w(rnd[c], e, thr_hi) ? b[e] * a.br_drop.scale : 0.f));
      if (a.z != nullptr) store8(static_cast<bf16*>(a.z) + idx, z[c]);
    }
    ln_row_finish<VPL>(z, row, lane, a);
#pragma unroll
    for (int c = 0; c < VPL; ++c) {
      br[c] = nbr[c];
      if constexpr (RES) rs[c] = nrs[c];
    }
  }
}

// z = word[tok] + pos[s] + type[tt]; y = dropout(LN(z))
template <int VPL>
__global__ void __launch_bounds__(256) embed_ln_fwd_kernel(const mimose_ops::LnFwdArgs a,
                                                          const int32_t* tok, const int32_t* tt,
                                                          const bf16* word, const bf16* pos,
                                                          const bf16* type, int S) {
  constexpr int H = VPL * 256;
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= a.rows) return;
  const int64_t w = tok[row];
  const int64_t t = tt != nullptr ? tt[row] : 0;
  const int64_t s = row % S;
  float z[VPL][8];
#pragma unroll
  for (int c = 0; c < VPL; ++c) {
    const int col = 8 * (lane + 32 * c);
    float x0[8], x1[8], x2[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    load8(word + w * H + col, x0);
    load8(pos + s * H + col, x1);
    if (type != nullptr) load8(type + t * H + col, x2);
#pragma unroll
    for (int e = 0; e < 8; ++e) z[c][e] = bf16r(x0[e] + x1[e] + x2[e]);
    if (a.z != nullptr) store8(static_cast<bf16*>(a.z) + (uint64_t)row * H + col, z[c]);
  }
  ln_row_finish<VPL>(z, row, lane, a);
}

// =====================================================================
// LayerNorm backward (+ dropout backward of the branch / of the input)
//   dy_eff = (dy + dy2) [* in-dropout mask]
//   dz     = rstd * (g - mean(g) - xhat * mean(g * xhat)),  g = dy_eff * gamma
//   dbr    = dz * branch-dropout mask * scale
// per-block partials: [3][H] = {sum dy_eff*xhat, sum dy_eff, sum dbr}
//
// Layout: a row is owned by TPR = H / 8 threads (one 16-byte chunk each, so
// a thread's column accumulators are 3 x 8 floats); a block holds G such row
// groups, each walking rows r = blockIdx * G + grp + k * gridDim * G. The
// next row's operands are loaded before the current row is reduced
// (register double-buffering), so every thread keeps two rows of loads in
// flight. Row reductions: warp shuffles, then (H > 256) one float2 per warp
// through a parity-buffered smem slot behind a per-group named barrier.
// Fixed row -> group assignment + fixed-order combines: deterministic.
// =====================================================================

template <int WPR>
struct LnBwdGeo {
  static constexpr int TPR = WPR * 32;
  static constexpr int H = TPR * 8;
  static constexpr int G = WPR == 1 ? 8 : (WPR == 2 ? 4 : 2);  // <= 256 threads, 2 blocks / SM
  static constexpr int THREADS = G * TPR;
  static constexpr int MINB = 2;  // resident blocks per SM (3 measured slower: spills)
};

struct LnBwdRaw {
  uint4 z, dy, dy2, dres;
};

template <bool DY2, bool DRES>
__device__ __forceinline__ void ln_bwd_load(const mimose_ops::LnBwdArgs& a, int64_t idx,
                                            LnBwdRaw& r) {
  r.z = __ldcs(reinterpret_cast<const uint4*>(static_cast<const bf16*>(a.z) + idx));
  r.dy = __ldcs(reinterpret_cast<const uint4*>(static_cast<const bf16*>(a.dy) + idx));
  if (DY2)
    r.dy2 = __ldcs(reinterpret_cast<const uint4*>(static_cast<const bf16*>(a.dy2) + idx));
  if (DRES)
    r.dres = __ldcs(reinterpret_cast<const uint4*>(static_cast<const bf16*>(a.dres) + idx));
}

template <int WPR, bool DY2, bool DRES>
__global__ void __launch_bounds__(LnBwdGeo<WPR>::THREADS, LnBwdGeo<WPR>::MINB)
    ln_bwd_kernel(const mimose_ops::LnBwdArgs a) {
  using Geo = LnBwdGeo<WPR>;
  constexpr int TPR = Geo::TPR, H = Geo::H, G = Geo::G;
  __shared__ float2 red[2][G][WPR];
  __shared__ float comb[G][3][H];
  const int grp = threadIdx.x / TPR;
  const int t = threadIdx.x % TPR;
  const int w = t >> 5, lane = t & 31;
  const int col = 8 * t;
  float gam[8];
  {
    const float4* g4 = reinterpret_cast<const float4*>(a.gamma + col);
    *reinterpret_cast<float4*>(gam) = g4[0];
    *reinterpret_cast<float4*>(gam + 4) = g4[1];
  }
  // output-based x-hat (a.beta set: the row holds y = x-hat * gamma + beta):
  // x-hat = y * (1 / gamma) - beta / gamma; a zero gamma column has no x-hat
  // (its gradient terms vanish with gamma; its gamma gradient reads 0)
  const bool from_y = a.beta != nullptr;
  float xa[8], xb[8];
  if (from_y) {
    float bet[8];
    const float4* b4 = reinterpret_cast<const float4*>(a.beta + col);
    *reinterpret_cast<float4*>(bet) = b4[0];
    *reinterpret_cast<float4*>(bet + 4) = b4[1];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      xa[e] = gam[e] != 0.f ? 1.f / gam[e] : 0.f;
      xb[e] = -bet[e] * xa[e];
    }
  }
  float acc_g[8], acc_b[8], acc_d[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc_g[e] = acc_b[e] = acc_d[e] = 0.f;

  const int64_t step = (int64_t)gridDim.x * G;
  int64_t row = (int64_t)blockIdx.x * G + grp;
  LnBwdRaw cur{}, nxt{};
  float2 st_cur = make_float2(0.f, 0.f), st_nxt = st_cur;
  if (row < a.rows) {
    ln_bwd_load<DY2, DRES>(a, row * H + col, cur);
    st_cur = reinterpret_cast<const float2*>(a.stats)[row];
  }
  // element index of this thread's chunk, advanced by a constant per row
  // (no 64-bit row * H products in the loop)
  int64_t idx = row * H + col;
  const int64_t didx = step * H;
  for (int it = 0; row < a.rows; row += step, ++it, idx += didx) {
    const int64_t nrow = row + step;
    if (nrow < a.rows) {  // prefetch the next row of this group
      ln_bwd_load<DY2, DRES>(a, idx + didx, nxt);
      st_nxt = reinterpret_cast<const float2*>(a.stats)[nrow];
    }
    float zz[8], dy[8];
    unpack8(cur.z, zz);
    unpack8(cur.dy, dy);
    if constexpr (DY2) {
      float d2[8];
      unpack8(cur.dy2, d2);
#pragma unroll
      for (int e = 0; e < 8; ++e) dy[e] += d2[e];
    }
    if (a.in_drop.threshold != 0) {
      const Philox ph(a.in_drop.seed, a.in_drop.stream, (uint64_t)idx >> 3);
      const uint32_t thr_hi = a.in_drop.threshold << 16;
#pragma unroll
      for (int e = 0; e < 8; ++e) dy[e] = philox_keep(ph, e, thr_hi) ? dy[e] * a.in_drop.scale : 0.f;
    }
    if (!from_y) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        xa[e] = st_cur.y;
        xb[e] = -st_cur.x * st_cur.y;
      }
    }
    // paired f32x2 math (FFMA2 / FMUL2 / FADD2) over the 8 columns:
    // x-hat, g = dy * gamma and the two row sums (two paired chains each)
    float xh[8], gg[8];
    float2 s1p = make_float2(0.f, 0.f), s2p = s1p;
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      const float2 x2 = __ffma2_rn(make_float2(zz[e], zz[e + 1]), make_float2(xa[e], xa[e + 1]),
                                   make_float2(xb[e], xb[e + 1]));
      const float2 g2 = __fmul2_rn(make_float2(dy[e], dy[e + 1]), make_float2(gam[e], gam[e + 1]));
      s1p = __fadd2_rn(s1p, g2);
      s2p = __ffma2_rn(g2, x2, s2p);
      xh[e] = x2.x; xh[e + 1] = x2.y;
      gg[e] = g2.x; gg[e + 1] = g2.y;
    }
    float s1 = s1p.x + s1p.y, s2 = s2p.x + s2p.y;
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if constexpr (WPR > 1) {
      if (lane == 0) red[it & 1][grp][w] = make_float2(s1, s2);
      asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "r"(TPR) : "memory");
      s1 = 0.f;
      s2 = 0.f;
#pragma unroll
      for (int k = 0; k < WPR; ++k) {
        const float2 v = red[it & 1][grp][k];
        s1 += v.x;
        s2 += v.y;
      }
    }
    const float mg = s1 * (1.f / H);
    const float mgx = s2 * (1.f / H);
    // dz = rstd * (g - mean(g) - x-hat * mean(g x-hat)); gamma / beta partials
    float dz[8];
    const float2 rs2 = make_float2(st_cur.y, st_cur.y), nmg2 = make_float2(-mg, -mg);
    const float2 nmgx2 = make_float2(-mgx, -mgx);
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      const float2 x2 = make_float2(xh[e], xh[e + 1]), d2 = make_float2(dy[e], dy[e + 1]);
      const float2 t2 = __ffma2_rn(x2, nmgx2, __fadd2_rn(make_float2(gg[e], gg[e + 1]), nmg2));
      const float2 z2 = __fmul2_rn(rs2, t2);
      dz[e] = z2.x; dz[e + 1] = z2.y;
      const float2 ag = __ffma2_rn(d2, x2, make_float2(acc_g[e], acc_g[e + 1]));
      const float2 ab = __fadd2_rn(make_float2(acc_b[e], acc_b[e + 1]), d2);
      acc_g[e] = ag.x; acc_g[e + 1] = ag.y;
      acc_b[e] = ab.x; acc_b[e + 1] = ab.y;
    }
    if constexpr (DRES) {
      float rr[8];
      unpack8(cur.dres, rr);
#pragma unroll
      for (int e = 0; e < 8; ++e) dz[e] += rr[e];
    }
    // one rounding pass: the stored bf16 dz, widened back with bit ops, is the
    // value the branch gradient starts from (same as bf16r(dz))
    uint4 dzp;
    {
      __nv_bfloat162* hp = reinterpret_cast<__nv_bfloat162*>(&dzp);
#pragma unroll
      for (int q = 0; q < 4; ++q) hp[q] = __floats2bfloat162_rn(dz[2 * q], dz[2 * q + 1]);
      *reinterpret_cast<uint4*>(static_cast<bf16*>(a.dz) + idx) = dzp;
    }
    float dzr[8];
    {
      const uint32_t* w = reinterpret_cast<const uint32_t*>(&dzp);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        dzr[2 * q] = __uint_as_float(w[q] << 16);
        dzr[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
      }
    }
    float db[8];
    if (a.br_drop.threshold != 0) {
      const Philox ph(a.br_drop.seed, a.br_drop.stream, (uint64_t)idx >> 3);
      const uint32_t thr_hi = a.br_drop.threshold << 16;
#pragma unroll
      for (int e = 0; e < 8; ++e)
        db[e] = philox_keep(ph, e, thr_hi) ? dzr[e] * a.br_drop.scale : 0.f;
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) db[e] = dzr[e] * a.br_drop.scale;
    }
    // the branch gradient rounded to bf16 once: the stored words, widened
    // back, are also what the bias gradient sums (= bf16r(db) before)
    uint4 dbp;
    {
      uint32_t* hw = reinterpret_cast<uint32_t*>(&dbp);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        __nv_bfloat162 h = __floats2bfloat162_rn(db[2 * q], db[2 * q + 1]);
        hw[q] = *reinterpret_cast<uint32_t*>(&h);
        const float2 r2 = make_float2(__uint_as_float(hw[q] << 16), __uint_as_float(hw[q] & 0xFFFF0000u));
        const float2 ad = __fadd2_rn(make_float2(acc_d[2 * q], acc_d[2 * q + 1]), r2);
        acc_d[2 * q] = ad.x;
        acc_d[2 * q + 1] = ad.y;
      }
    }
    if (a.dbr != nullptr) *reinterpret_cast<uint4*>(static_cast<bf16*>(a.dbr) + idx) = dbp;
    cur = nxt;
    st_cur = st_nxt;
  }
  // fixed-order combine of the G row groups -> partial[blockIdx.x][3][H]
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    comb[grp][0][col + e] = acc_g[e];
    comb[grp][1][col + e] = acc_b[e];
    comb[grp][2][col + e] = acc_d[e];
  }
  __syncthreads();
  float* out = a.partial + (size_t)blockIdx.x * 3 * H;
  for (int i = threadIdx.x; i < 3 * H; i += Geo::THREADS) {
    float s = 0.f;
#pragma unroll
    for (int g = 0; g < G; ++g) s += (&comb[g][0][0])[i];
    out[i] = s;
  }
}

// sum over blocks of partial[nblk][W] -> out segments. A block owns
// kRedCols columns with 256 / kRedCols row phases each; each thread sums its
// rows (b = y, y + P, ...) strictly in order, with up to 16 of those loads
// issued before any is added (the partials are L2-resident: the kernel is
// load-latency-bound -- 32 columns x 8 phases gave 72 blocks for W = 2304,
// half the SMs, ~5.7 us per launch); the phases are then combined in a fixed
// order (eight runs of P / 8, then the eight run sums): deterministic.
constexpr int kRedCols = 8;
__global__ void __launch_bounds__(256) reduce_partials_kernel(const float* __restrict__ partial,
                                                              int nblk, int W, int seg, float* o0,
                                                              float* o1, float* o2) {
  constexpr int CW = kRedCols, P = 256 / CW;
  __shared__ float red[P][CW + 1];
  const int x = threadIdx.x % CW, y = threadIdx.x / CW;
  const int i = blockIdx.x * CW + x;
  float s = 0.f;
  if (i < W) {
    constexpr int kU = 16;
    int b = y;
    for (; b + P * (kU - 1) < nblk; b += P * kU) {
      float v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = partial[(size_t)(b + P * u) * W + i];
#pragma unroll
      for (int u = 0; u < kU; ++u) s += v[u];
    }
    float v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) v[u] = b + P * u < nblk ? partial[(size_t)(b + P * u) * W + i] : 0.f;
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (b + P * u < nblk) s += v[u];
  }
  red[y][x] = s;
  __syncthreads();
  constexpr int R = P / 8;
  if (y < 8) {
    float t = red[y * R][x];
#pragma unroll
    for (int k = 1; k < R; ++k) t += red[y * R + k][x];
    red[y * R][x] = t;  // only this thread reads / writes rows y R .. y R + R - 1 of column x
  }
  __syncthreads();
  if (y == 0 && i < W) {
    float t = red[0][x];
#pragma unroll
    for (int k = 1; k < 8; ++k) t += red[k * R][x];
    const int k = i / seg, j = i % seg;
    float* o = k == 0 ? o0 : (k == 1 ? o1 : o2);
    if (o != nullptr) o[j] = t;
  }
}

// =====================================================================
// column sums of a bf16 matrix [rows][N] (ld) with optional 2-way grouping
// partial[blockIdx.y][G][N]
// =====================================================================
// G = 1: plain column sums (bias gradients); G = 2: split by a per-row group
// id (token-type gradients). Eight rows of 16-byte loads in flight per
// thread (issued before any is consumed); fixed summation order.
template <int G>
__global__ void __launch_bounds__(256) colsum_partial_kernel(const bf16* __restrict__ x, int rows,
                                                             int N, int64_t ld,
                                                             const int32_t* __restrict__ grp,
                                                             float* __restrict__ partial) {
  __shared__ float red[8][G][256];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int col = (blockIdx.x * 32 + tx) * 8;
  float acc[G][8] = {};
  if (col < N) {
    const int step = gridDim.y * 8;
    int r = blockIdx.y * 8 + ty;
    constexpr int kU = 8;
    for (; r + (kU - 1) * step < rows; r += kU * step) {
      uint4 raw[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u)
        raw[u] = __ldcs(reinterpret_cast<const uint4*>(x + (int64_t)(r + u * step) * ld + col));
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        float v[8];
        unpack8(raw[u], v);
        if constexpr (G == 1) {
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[0][e] += v[e];
        } else {
          const int g = grp[r + u * step];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            acc[0][e] += g == 0 ? v[e] : 0.f;
            acc[1][e] += g == 1 ? v[e] : 0.f;
          }
        }
      }
    }
    for (; r < rows; r += step) {
      float v[8];
      load8(x + (int64_t)r * ld + col, v);
      const int g = G == 2 ? grp[r] : 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        acc[0][e] += (G == 1 || g == 0) ? v[e] : 0.f;
        if constexpr (G == 2) acc[G - 1][e] += g == 1 ? v[e] : 0.f;
      }
    }
  }
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int e = 0; e < 8; ++e) red[ty][g][tx * 8 + e] = acc[g][e];
  __syncthreads();
  for (int i = threadIdx.x; i < G * 256; i += 256) {
    const int g = i / 256, c = i % 256;
    const int gc = blockIdx.x * 256 + c;
    if (gc >= N) continue;
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += red[w][g][c];
    partial[((size_t)blockIdx.y * G + g) * N + gc] = s;
  }
}

// =====================================================================
// scaled softmax + dropout over rows of S (row pitch ld, ld % 8 == 0)
//
// A group of L lanes owns one row (32 / L rows per warp); every lane issues
// all of its MAXC 16-byte loads before reducing, so each thread keeps up to
// MAXC loads in flight (rows here are only S <= 2048 elements long, one
// warp per row would leave most of the HBM pipe idle).
// =====================================================================
template <int L>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <int L>
__device__ __forceinline__ float group_max(float v) {
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}


// All loads of a lane are issued before any arithmetic; exp is evaluated once.
// Instruction economy (the kernel is issue-bound, not HBM-bound, once Philox
// is counted): whole 8-column chunks skip per-element bounds checks, the
// max is taken on raw scores and folded into one FFMA before ex2, and the
// keep predicates come straight from the Philox words (philox_keep).
template <int L, int MAXC>
__global__ void __launch_bounds__(256) softmax_fwd_kernel(const bf16* __restrict__ s_in,
                                                          bf16* __restrict__ p_out,
                                                          bf16* __restrict__ pd_out, int64_t rows,
                                                          int S, int ld, DropoutCfg drop,
                                                          int causal) {
  constexpr int R = 32 / L;
  constexpr float kLog2e = 1.4426950408889634f;
  const int lane = threadIdx.x & 31;
  const int sub = lane % L;
  const int64_t row = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * R + lane / L;
  const bool live = row < rows;
  const bf16* in = s_in + (live ? row : 0) * ld;
  // causal: keys j > query i (= row within its sequence) are masked out
  const int jmax = live ? (causal ? static_cast<int>(row % S) + 1 : S) : 0;
  uint4 raw[MAXC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c) {
    const int j0 = 8 * (sub + L * c);
    raw[c] = j0 < jmax ? __ldcs(reinterpret_cast<const uint4*>(in + j0)) : make_uint4(0, 0, 0, 0);
  }
  float v[MAXC][8];
  float mx = -INFINITY;
#pragma unroll
  for (int c = 0; c < MAXC; ++c) {
    const int j0 = 8 * (sub + L * c);
    unpack8(raw[c], v[c]);
    if (j0 + 8 <= jmax) {
#pragma unroll
      for (int e = 0; e < 8; ++e) mx = fmaxf(mx, v[c][e]);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        v[c][e] = j0 + e < jmax ? v[c][e] : -INFINITY;
        mx = fmaxf(mx, v[c][e]);
      }
    }
  }
  mx = group_max<L>(mx);
  const float nmx = -mx * kLog2e;  // exp(s - max) = 2^(s log2e - max log2e)
  float sum = 0.f;
#pragma unroll
  for (int c = 0; c < MAXC; ++c)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      v[c][e] = exp2_neg(fmaf(v[c][e], kLog2e, nmx));
      sum += v[c][e];
    }
  const float inv = 1.f / group_sum<L>(sum);
  if (!live) return;
  const uint32_t thr_hi = drop.threshold << 16;
  // chunks in pairs: one Philox key schedule per pair, two interleaved chains
#pragma unroll
  for (int c2 = 0; c2 < MAXC; c2 += 2) {
    constexpr int W = 2;
    uint32_t rnd[W][4];
    if (pd_out != nullptr) {
      uint64_t grp[W];
#pragma unroll
      for (int u = 0; u < W; ++u) grp[u] = ((uint64_t)row * ld + 8 * (sub + L * (c2 + u))) >> 3;
      philox_n<W>(drop.seed, drop.stream, grp, rnd);
    }
#pragma unroll
    for (int u = 0; u < W; ++u) {
      const int c = c2 + u;
      if (c >= MAXC) break;
      const int j0 = 8 * (sub + L * c);
      if (j0 >= ld) continue;
      float p[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) p[e] = bf16r(v[c][e] * inv);
      store8(p_out + row * ld + j0, p);
      if (pd_out != nullptr) {
        float pd[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) pd[e] = philox_keep_w(rnd[u], e, thr_hi) ? p[e] * drop.scale : 0.f;
        store8(pd_out + row * ld + j0, pd);
      }
    }
  }
}

// dS = P * (dP - sum_j dP_j P_j) * scale,  dP = dPd * mask * (1/(1-p)); in place over dPd
template <int L, int MAXC>
__global__ void __launch_bounds__(256, (MAXC > 4) ? 1 : 2) softmax_bwd_kernel(const bf16* __restrict__ P,
                                                          bf16* __restrict__ dpd, int64_t rows,
                                                          int S, int ld, DropoutCfg drop,
                                                          float scale, int causal) {
  constexpr int R = 32 / L;
  const int lane = threadIdx.x & 31;
  const int sub = lane % L;
  const int64_t row = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * R + lane / L;
  const bool live = row < rows;
  const int64_t base = (live ? row : 0) * ld;
  // causal: keys above the diagonal carry P = 0 and may hold unwritten dPd
  // (their score tiles were skipped): never read them
  const int jmax = live ? (causal ? static_cast<int>(row % S) + 1 : S) : 0;
  uint4 praw[MAXC], draw[MAXC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c) {
    const int j0 = 8 * (sub + L * c);
    const bool in = j0 < jmax;
    praw[c] = in ? __ldcs(reinterpret_cast<const uint4*>(P + base + j0)) : make_uint4(0, 0, 0, 0);
    draw[c] = in ? __ldcs(reinterpret_cast<const uint4*>(dpd + base + j0)) : make_uint4(0, 0, 0, 0);
  }
  // g = dP = dPd * keep * scale (0 outside the row); P is 0 outside (zero-filled loads)
  const uint32_t thr_hi = drop.threshold << 16;
  float g[MAXC][8];
  float dot = 0.f;
  uint32_t rnd[MAXC][4];
  {
    uint64_t grp[MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) grp[c] = ((uint64_t)row * ld + 8 * (sub + L * c)) >> 3;
    philox_n<MAXC>(drop.seed, drop.stream, grp, rnd);
  }
#pragma unroll
  for (int c = 0; c < MAXC; ++c) {
    const int j0 = 8 * (sub + L * c);
    float p[8], dp[8];
    unpack8(praw[c], p);
    unpack8(draw[c], dp);
    if (j0 + 8 <= jmax) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        g[c][e] = philox_keep_w(rnd[c], e, thr_hi) ? dp[e] * drop.scale : 0.f;
        dot += g[c][e] * p[e];
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        g[c][e] = (j0 + e < jmax && philox_keep_w(rnd[c], e, thr_hi)) ? dp[e] * drop.scale : 0.f;
        dot += g[c][e] * p[e];
      }
    }
  }
  dot = group_sum<L>(dot);
  if (!live) return;
#pragma unroll
  for (int c = 0; c < MAXC; ++c) {
    const int j0 = 8 * (sub + L * c);
    if (j0 >= ld) continue;
    float p[8], ds[8];
    unpack8(praw[c], p);
#pragma unroll
    for (int e = 0; e < 8; ++e) ds[e] = j0 + e < S ? p[e] * (g[c][e] - dot) * scale : 0.f;
    store8(dpd + base + j0, ds);
  }
}

// =====================================================================
// embedding gradients
// =====================================================================
// one warp per distinct token id: rows of `de` listed (ascending position)
// in perm[seg[u] .. seg[u+1]) are summed in order -> dword[id[u]]
__global__ void __launch_bounds__(256) embed_word_grad_kernel(const bf16* __restrict__ de, int H,
                                                              const int32_t* __restrict__ perm,
                                                              const int32_t* __restrict__ seg,
                                                              const int32_t* __restrict__ uid,
                                                              int n_unique,
                                                              float* __restrict__ dword,
                                                              int accumulate, int pad) {
  const int lane = threadIdx.x & 31;
  const int u = blockIdx.x * 8 + (threadIdx.x >> 5);
  // the padding row gets no embedding gradient (HF padding_idx); a tied
  // decoder's own gradient for it stays in place
  if (u >= n_unique || uid[u] == pad) return;
  const int b = seg[u], e = seg[u + 1];
  float* out = dword + (int64_t)uid[u] * H;
  for (int c0 = lane * 8; c0 < H; c0 += 256) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int k = b; k < e; ++k) {
      float v[8];
      load8(de + (int64_t)perm[k] * H + c0, v);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += v[i];
    }
    float4* o4 = reinterpret_cast<float4*>(out + c0);
    if (accumulate) {  // tied decoder: its weight gradient is already in place
      const float4 p0 = o4[0], p1 = o4[1];
      acc[0] = p0.x + acc[0]; acc[1] = p0.y + acc[1]; acc[2] = p0.z + acc[2]; acc[3] = p0.w + acc[3];
      acc[4] = p1.x + acc[4]; acc[5] = p1.y + acc[5]; acc[6] = p1.z + acc[6]; acc[7] = p1.w + acc[7];
    }
    o4[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    o4[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
}

// dpos[s] = sum_b de[b*S + s]
__global__ void embed_pos_grad_kernel(const bf16* __restrict__ de, int B, int S, int H,
                                      float* __restrict__ dpos) {
  const int s = blockIdx.x;
  for (int c0 = threadIdx.x * 8; c0 < H; c0 += blockDim.x * 8) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int b = 0; b < B; ++b) {
      float v[8];
      load8(de + ((int64_t)b * S + s) * H + c0, v);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += v[i];
    }
    float4* o4 = reinterpret_cast<float4*>(dpos + (int64_t)s * H + c0);
    o4[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    o4[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
}

// =====================================================================
// multiple-choice head: pooled = tanh(pre); logits = dropout(pooled).wc + bc;
// loss = mean_q CE(softmax over C choices); writes dpre (bf16), dwc, dbc
// Single CTA (B <= a few hundred rows).
// =====================================================================
__global__ void __launch_bounds__(1024) mc_head_kernel(const bf16* __restrict__ pre, int B, int H,
                                                       int C, const float* __restrict__ wc,
                                                       const float* __restrict__ bc,
                                                       const int32_t* __restrict__ labels,
                                                       DropoutCfg drop, float* __restrict__ loss,
                                                       float* __restrict__ logits_out,
                                                       bf16* __restrict__ dpre,
                                                       float* __restrict__ dwc,
                                                       float* __restrict__ dbc) {
  extern __shared__ float sh[];  // logits[B], dlogit[B]
  float* lg = sh;
  float* dl = sh + B;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // logits: one warp per row
  for (int b = warp; b < B; b += nw) {
    float s = 0.f;
    for (int c = lane; c < H; c += 32) {
      const uint64_t idx = (uint64_t)b * H + c;
      const bool keep = dropout_keep1(drop, idx);
      const float t = tanhf(__bfloat162float(pre[idx]));
      s += keep ? t * drop.scale * wc[c] : 0.f;
    }
    s = warp_sum(s);
    if (lane == 0) lg[b] = s + bc[0];
  }
  __syncthreads();
  const int Q = B / C;
  if (threadIdx.x == 0) {
    float tot = 0.f;
    for (int q = 0; q < Q; ++q) {
      float mx = -INFINITY;
      for (int c = 0; c < C; ++c) mx = fmaxf(mx, lg[q * C + c]);
      float se = 0.f;
      for (int c = 0; c < C; ++c) se += expf(lg[q * C + c] - mx);
      const float lse = mx + logf(se);
      tot += lse - lg[q * C + labels[q]];
      for (int c = 0; c < C; ++c) {
        const float pr = expf(lg[q * C + c] - lse);
        dl[q * C + c] = (pr - (c == labels[q] ? 1.f : 0.f)) / (float)Q;
      }
    }
    loss[0] = tot / (float)Q;
    float db = 0.f;
    for (int b = 0; b < B; ++b) db += dl[b];
    dbc[0] = db;
  }
  __syncthreads();
  if (logits_out != nullptr)
    for (int b = threadIdx.x; b < B; b += blockDim.x) logits_out[b] = lg[b];
  // dwc[c] = sum_b dl[b] * td[b,c] ; dpre = dl[b]*wc[c]*mask*scale*(1 - t^2)
  for (int c = threadIdx.x; c < H; c += blockDim.x) {
    float acc = 0.f;
    for (int b = 0; b < B; ++b) {
      const uint64_t idx = (uint64_t)b * H + c;
      const bool keep = dropout_keep1(drop, idx);
      const float t = tanhf(__bfloat162float(pre[idx]));
      acc += keep ? dl[b] * t * drop.scale : 0.f;
      const float dt = keep ? dl[b] * wc[c] * drop.scale : 0.f;
      dpre[idx] = __float2bfloat16_rn(dt * (1.f - t * t));
    }
    dwc[c] = acc;
  }
}

// =====================================================================
// optimizer: global grad-norm (two-stage) + fused AdamW
// =====================================================================
__global__ void __launch_bounds__(256) sumsq_partial_kernel(const float* __restrict__ g, int64_t n,
                                                            float* __restrict__ partial) {
  __shared__ float red[8];
  float s = 0.f;
  const int64_t n4 = n / 4;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = g4[i];
    s += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  if (blockIdx.x == 0)
    for (int64_t i = n4 * 4 + threadIdx.x; i < n; i += blockDim.x) s += g[i] * g[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    partial[blockIdx.x] = t;
  }
}

__global__ void sum_partials_kernel(const float* __restrict__ partial, int n, float* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += partial[i];
    out[0] = (float)s;
  }
}

__global__ void __launch_bounds__(256) adamw_kernel(float* __restrict__ p, float* __restrict__ m,
                                                    float* __restrict__ v,
                                                    const float* __restrict__ g,
                                                    bf16* __restrict__ p16, int64_t n,
                                                    const uint8_t* __restrict__ decay_chunk,
                                                    const float* __restrict__ norm2,
                                                    mimose_ops::AdamWArgs a) {
  float clip = 1.f;
  if (a.max_grad_norm > 0.f) {
    const float nrm = sqrtf(norm2[0]);
    clip = fminf(1.f, a.max_grad_norm / (nrm * a.grad_scale + 1e-6f));
  }
  const float gs = clip * a.grad_scale;
  // n is a multiple of 4; decay_chunk[e / 64] = 1 when element e belongs to a
  // decayed tensor (tensors are 64-element aligned)
  const int64_t n4 = n / 4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 pv = reinterpret_cast<const float4*>(p)[i];
    float4 mv = reinterpret_cast<const float4*>(m)[i];
    float4 vv = reinterpret_cast<const float4*>(v)[i];
    const float4 gv = reinterpret_cast<const float4*>(g)[i];
    const bool decay = decay_chunk[(4 * i) >> 6] != 0;
    float* pp = &pv.x;
    float* mp = &mv.x;
    float* vp = &vv.x;
    const float* gp = &gv.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float gi = gp[k] * gs;
      float pi = pp[k];
      if (decay) pi -= a.lr * a.weight_decay * pi;
      const float mi = a.beta1 * mp[k] + (1.f - a.beta1) * gi;
      const float vi = a.beta2 * vp[k] + (1.f - a.beta2) * gi * gi;
      mp[k] = mi;
      vp[k] = vi;
      pi -= a.lr * (mi / a.bc1) / (sqrtf(vi / a.bc2) + a.eps);
      pp[k] = pi;
    }
    reinterpret_cast<float4*>(p)[i] = pv;
    reinterpret_cast<float4*>(m)[i] = mv;
    reinterpret_cast<float4*>(v)[i] = vv;
    __nv_bfloat162 lo = __floats2bfloat162_rn(pv.x, pv.y), hi = __floats2bfloat162_rn(pv.z, pv.w);
    uint2 packed;
    packed.x = *reinterpret_cast<uint32_t*>(&lo);
    packed.y = *reinterpret_cast<uint32_t*>(&hi);
    reinterpret_cast<uint2*>(p16)[i] = packed;
  }
}

// deterministic N(mean, std) init: Box-Muller over Philox(seed, stream, i/2)
__global__ void init_normal_kernel(float* __restrict__ p, int64_t n, float mean, float std,
                                   uint64_t seed, uint64_t stream) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const Philox ph(seed, stream, (uint64_t)i >> 1);
    const int k = (int)(i & 1) * 2;
    const float u1 = ((float)(ph.r[k] >> 8) + 1.f) * (1.f / 16777216.f);  // (0, 1]
    const float u2 = (float)(ph.r[k + 1] >> 8) * (1.f / 16777216.f);
    p[i] = mean + std * sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
  }
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ in, bf16* __restrict__ out,
                                   int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn(in[i]);
}


// =====================================================================
// elementwise helpers, row gather / scatter, deterministic sums
// =====================================================================
__global__ void dropout_apply_kernel(const bf16* __restrict__ in, bf16* __restrict__ out,
                                     int64_t n8, DropoutCfg d) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v[8];
    load8(in + 8 * i, v);
    const uint32_t m = dropout_mask8(d, (uint64_t)(8 * i));
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = ((m >> e) & 1u) ? v[e] * d.scale : 0.f;
    store8(out + 8 * i, v);
  }
}

__device__ __forceinline__ float gelu_erf_grad(float x) {
  return 0.5f * (1.0f + erff(x * 0.70710678118654752f)) +
         x * 0.39894228040143268f * __expf(-0.5f * x * x);
}
__device__ __forceinline__ float gelu_tanh_grad(float x) {
  const float x2 = x * x;
  const float t = tanhf(0.7978845608028654f * fmaf(0.044715f * x, x2, x));
  return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * 0.7978845608028654f * fmaf(0.134145f, x2, 1.0f);
}

__global__ void dgelu_apply_kernel(const bf16* __restrict__ dg, const bf16* __restrict__ u,
                                   bf16* __restrict__ out, int64_t n8, int tanh_form) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    float a[8], x[8];
    load8(dg + 8 * i, a);
    load8(u + 8 * i, x);
#pragma unroll
    for (int e = 0; e < 8; ++e) a[e] *= tanh_form ? gelu_tanh_grad(x[e]) : gelu_erf_grad(x[e]);
    store8(out + 8 * i, a);
  }
}

// one warp per row
__global__ void gather_rows_kernel(const bf16* __restrict__ src, const int32_t* __restrict__ idx,
                                   int n, int H, bf16* __restrict__ dst, int scatter) {
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  const int64_t from = scatter ? r : idx[r];
  const int64_t to = scatter ? idx[r] : r;
  for (int c = lane * 8; c < H; c += 256)
    *reinterpret_cast<uint4*>(dst + to * H + c) = *reinterpret_cast<const uint4*>(src + from * H + c);
}

// single CTA, fixed order: out = scale * sum x
__global__ void __launch_bounds__(1024) sum_f32_kernel(const float* __restrict__ x, int n,
                                                       float scale, float* __restrict__ out) {
  __shared__ float red[1024];
  float acc = 0.f;
  for (int i = threadIdx.x; i < n; i += 1024) acc += x[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0] * scale;
}

// =====================================================================
// extractive-QA head (one CTA per sequence)
// =====================================================================
__global__ void __launch_bounds__(512) qa_head_kernel(const bf16* __restrict__ x, int S, int H,
                                                      const float* __restrict__ w,
                                                      const float* __restrict__ bias,
                                                      const int32_t* __restrict__ labels,
                                                      float inv_count,
                                                      float* __restrict__ logits,
                                                      float* __restrict__ dl,
                                                      float* __restrict__ loss_parts) {
  extern __shared__ float sh[];  // [2][S]
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int t = warp; t < S; t += nw) {
    const bf16* row = x + ((int64_t)b * S + t) * H;
    float s0 = 0.f, s1 = 0.f;
    for (int c = lane * 8; c < H; c += 256) {
      float v[8];
      load8(row + c, v);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        s0 += v[e] * w[c + e];
        s1 += v[e] * w[H + c + e];
      }
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    if (lane == 0) {
      sh[t] = s0 + bias[0];
      sh[S + t] = s1 + bias[1];
    }
  }
  __syncthreads();
  // two warps: k = 0 (start) and k = 1 (end) softmax / CE over the S positions
  if (warp < 2) {
    const int k = warp;
    float* lg = sh + k * S;
    float mx = -INFINITY;
    for (int t = lane; t < S; t += 32) mx = fmaxf(mx, lg[t]);
    mx = warp_max(mx);
    float se = 0.f;
    for (int t = lane; t < S; t += 32) se += expf(lg[t] - mx);
    se = warp_sum(se);
    const float lse = mx + logf(se);
    const int lab = labels[2 * b + k];
    for (int t = lane; t < S; t += 32) {
      const int64_t r = (int64_t)b * S + t;
      logits[2 * r + k] = lg[t];
      dl[2 * r + k] = (expf(lg[t] - lse) - (t == lab ? 1.f : 0.f)) * inv_count;
    }
    if (lane == 0) loss_parts[2 * b + k] = (lse - lg[lab]) * inv_count;
  }
}

// dx[t] = dl[t][0] * w0 + dl[t][1] * w1 ; partials of dW[k][h] = sum_t dl[t][k] x[t][h]
// and db[k] = sum_t dl[t][k] over row block blockIdx.y
__global__ void __launch_bounds__(256) qa_head_bwd_kernel(const bf16* __restrict__ x,
                                                          const float* __restrict__ dl, int T,
                                                          int H, const float* __restrict__ w,
                                                          bf16* __restrict__ dx,
                                                          float* __restrict__ partial) {
  const int W = 2 * H + 2;
  const int h = blockIdx.x * 256 + threadIdx.x;  // column (h < H) or bias slot
  float a0 = 0.f, a1 = 0.f;
  const int rows_per = (T + gridDim.y - 1) / gridDim.y;
  const int r0 = blockIdx.y * rows_per, r1 = min(T, r0 + rows_per);
  for (int t = r0; t < r1; ++t) {
    const float d0 = dl[2 * t], d1 = dl[2 * t + 1];
    if (h < H) {
      const float xv = __bfloat162float(x[(int64_t)t * H + h]);
      a0 += d0 * xv;
      a1 += d1 * xv;
      dx[(int64_t)t * H + h] = __float2bfloat16_rn(d0 * w[h] + d1 * w[H + h]);
    } else if (h == H) {
      a0 += d0;
      a1 += d1;
    }
  }
  float* out = partial + (size_t)blockIdx.y * W;
  if (h < H) {
    out[h] = a0;
    out[H + h] = a1;
  } else if (h == H) {
    out[2 * H] = a0;
    out[2 * H + 1] = a1;
  }
}

// =====================================================================
// row-wise softmax cross-entropy over a large vocabulary (one CTA per row)
// =====================================================================
__global__ void __launch_bounds__(512) ce_rows_kernel(bf16* __restrict__ logits, int V, int ld,
                                                      const int32_t* __restrict__ labels,
                                                      float grad_scale,
                                                      float* __restrict__ loss_rows) {
  __shared__ float red[32];
  const int64_t r = blockIdx.x;
  bf16* row = logits + r * ld;
  const int lab = labels[r];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  if (lab < 0) {  // ignored position: zero gradient row
    for (int c = tid * 8; c < ld; c += blockDim.x * 8)
      *reinterpret_cast<uint4*>(row + c) = make_uint4(0, 0, 0, 0);
    if (tid == 0) loss_rows[r] = 0.f;
    return;
  }
  // pass 1: max
  float mx = -INFINITY;
  for (int c = tid * 8; c < V; c += blockDim.x * 8) {
    float v[8];
    load8(row + c, v);
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (c + e < V) mx = fmaxf(mx, v[e]);
  }
  mx = warp_max(mx);
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = -INFINITY;
  for (int i = 0; i < nw; ++i) mx = fmaxf(mx, red[i]);
  __syncthreads();
  // pass 2: sum of exp
  float se = 0.f;
  for (int c = tid * 8; c < V; c += blockDim.x * 8) {
    float v[8];
    load8(row + c, v);
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (c + e < V) se += __expf(v[e] - mx);
  }
  se = warp_sum(se);
  if (lane == 0) red[warp] = se;
  __syncthreads();
  se = 0.f;
  for (int i = 0; i < nw; ++i) se += red[i];
  const float lse = mx + logf(se);
  const float target = __bfloat162float(row[lab]);
  __syncthreads();
  // pass 3: gradient in place
  for (int c = tid * 8; c < ld; c += blockDim.x * 8) {
    float v[8];
    load8(row + c, v);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int j = c + e;
      v[e] = j < V ? (__expf(v[e] - lse) - (j == lab ? 1.f : 0.f)) * grad_scale : 0.f;
    }
    store8(row + c, v);
  }
  if (tid == 0) loss_rows[r] = lse - target;
}
}  // namespace mimose_dev

// =====================================================================
// host launchers
// =====================================================================
namespace mimose_ops {

using mimose_dev::bf16;

namespace {
int grid_for(int64_t work, int per_block) { return (int)((work + per_block - 1) / per_block); }
int persistent_blocks() {
  static int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}
}  // namespace

// blocks of the LayerNorm backward: enough to fill two blocks per SM even for
// small token counts (GPT-2 at short S), at most two per SM; a function of
// `rows` only (deterministic partial layout)
int ln_bwd_blocks(int rows) {
  const int want = (rows + 7) / 8;
  const int cap = 2 * persistent_blocks();
  return want < 1 ? 1 : (want < cap ? want : cap);
}

cudaError_t add_ln_fwd(const LnFwdArgs& a, int H, cudaStream_t s) {
  const int want = grid_for(a.rows, 8), cap = 2 * persistent_blocks();
  const int g = want < cap ? want : cap;
  // bytes/row: branch (+ residual) read, z (if saved) + y written, stats
  const double rb = 2.0 * H * (1 + (a.res != nullptr) + (a.z != nullptr) + 1) +
                    (a.stats != nullptr ? 8 : 0);
  ProfScope prof(a.skip_ln ? "mem_add" : "mem_ln_fwd", 0, rb * a.rows, s);
  switch (H) {
    case 256:
      if (a.res) mimose_dev::add_ln_fwd_kernel<1, true><<<g, 256, 0, s>>>(a);
      else mimose_dev::add_ln_fwd_kernel<1, false><<<g, 256, 0, s>>>(a);
      break;
    case 512:
      if (a.res) mimose_dev::add_ln_fwd_kernel<2, true><<<g, 256, 0, s>>>(a);
      else mimose_dev::add_ln_fwd_kernel<2, false><<<g, 256, 0, s>>>(a);
      break;
    case 768:
      if (a.res) mimose_dev::add_ln_fwd_kernel<3, true><<<g, 256, 0, s>>>(a);
      else mimose_dev::add_ln_fwd_kernel<3, false><<<g, 256, 0, s>>>(a);
      break;
    case 1024:
      if (a.res) mimose_dev::add_ln_fwd_kernel<4, true><<<g, 256, 0, s>>>(a);
      else mimose_dev::add_ln_fwd_kernel<4, false><<<g, 256, 0, s>>>(a);
      break;
    default: return cudaErrorInvalidValue;
  }
  count_launch();
  return cudaGetLastError();
}

cudaError_t embed_ln_fwd(const LnFwdArgs& a, int H, const int32_t* tok, const int32_t* tt,
                         const void* word, const void* pos, const void* type, int S,
                         cudaStream_t s) {
  const int g = grid_for(a.rows, 8);
  ProfScope prof("mem_embed_ln_fwd", 0,
                 (2.0 * H * (3 + (a.z != nullptr)) + 8.0) * a.rows, s);
  auto w = static_cast<const bf16*>(word);
  auto p = static_cast<const bf16*>(pos);
  auto t = static_cast<const bf16*>(type);
  switch (H) {
    case 256: mimose_dev::embed_ln_fwd_kernel<1><<<g, 256, 0, s>>>(a, tok, tt, w, p, t, S); break;
    case 512: mimose_dev::embed_ln_fwd_kernel<2><<<g, 256, 0, s>>>(a, tok, tt, w, p, t, S); break;
    case 768: mimose_dev::embed_ln_fwd_kernel<3><<<g, 256, 0, s>>>(a, tok, tt, w, p, t, S); break;
    case 1024: mimose_dev::embed_ln_fwd_kernel<4><<<g, 256, 0, s>>>(a, tok, tt, w, p, t, S); break;
    default: return cudaErrorInvalidValue;
  }
  count_launch();
  return cudaGetLastError();
}

template <int WPR>
static cudaError_t ln_bwd_t(const LnBwdArgs& a, int nblk, cudaStream_t s) {
  constexpr int T = mimose_dev::LnBwdGeo<WPR>::THREADS;
  const bool d2 = a.dy2 != nullptr, dr = a.dres != nullptr;
  if (d2 && dr) mimose_dev::ln_bwd_kernel<WPR, true, true><<<nblk, T, 0, s>>>(a);
  else if (d2) mimose_dev::ln_bwd_kernel<WPR, true, false><<<nblk, T, 0, s>>>(a);
  else if (dr) mimose_dev::ln_bwd_kernel<WPR, false, true><<<nblk, T, 0, s>>>(a);
  else mimose_dev::ln_bwd_kernel<WPR, false, false><<<nblk, T, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t ln_bwd(const LnBwdArgs& a, int H, float* dgamma, float* dbeta, float* dbias,
                   cudaStream_t s) {
  const int nblk = ln_bwd_blocks(a.rows);
  // bytes/row: z, dy (+ dy2, + dres) read, stats, dz (+ dbr) written
  ProfScope prof("mem_ln_bwd", 0,
                 (2.0 * H * (3 + (a.dy2 != nullptr) + (a.dres != nullptr) + (a.dbr != nullptr)) +
                  8.0) * a.rows,
                 s);
  cudaError_t e;
  switch (H) {
    case 256: e = ln_bwd_t<1>(a, nblk, s); break;
    case 512: e = ln_bwd_t<2>(a, nblk, s); break;
    case 768: e = ln_bwd_t<3>(a, nblk, s); break;
    case 1024: e = ln_bwd_t<4>(a, nblk, s); break;
    default: return cudaErrorInvalidValue;
  }
  count_launch();
  if (e != cudaSuccess) return e;
  using mimose_dev::kRedCols;
  mimose_dev::reduce_partials_kernel<<<grid_for(3 * H, kRedCols), 256, 0, s>>>(
      a.partial, nblk, 3 * H, H, dgamma, dbeta, dbias);
  count_launch();
  return cudaGetLastError();
}

// 256-thread colsum_partial blocks resident per SM (36-40 registers, 8-16 KB smem)
constexpr int kColsumBlocksPerSm = 6;

int colsum_row_blocks(int rows, int N) {
  // one wave: a fixed 128 row blocks gave 1.1-1.5 waves at N = 2304 / 3072
  // (the second, partial wave ran on a fraction of the SMs) and under-filled
  // the machine at N = 768
  const int want = (rows + 31) / 32;
  const int ncol = (N + 255) / 256;
  const int fill = std::max(1, kColsumBlocksPerSm * persistent_blocks() / ncol);
  return std::max(1, std::min(want, fill));
}

int64_t colsum_scratch_bytes() {
  // rb * G * N <= kColsumBlocksPerSm * SMs * 256 * G for every N, G <= 2
  return (int64_t)kColsumBlocksPerSm * persistent_blocks() * 256 * 2 * 4 + 1024;
}

cudaError_t colsum(const void* x, int rows, int N, int64_t ld, const int32_t* groups, int G,
                   float* partial, float* out, cudaStream_t s) {
  if (N % 8 || ld % 8 || G < 1 || G > 2 || (G == 2 && groups == nullptr))
    return cudaErrorInvalidValue;
  const int rb = colsum_row_blocks(rows, N);
  ProfScope prof("mem_colsum", 0, 2.0 * rows * N, s);
  dim3 grid((N + 255) / 256, rb);
  if (G == 2 && groups != nullptr)
    mimose_dev::colsum_partial_kernel<2><<<grid, 256, 0, s>>>(static_cast<const bf16*>(x), rows, N,
                                                              ld, groups, partial);
  else
    mimose_dev::colsum_partial_kernel<1><<<grid, 256, 0, s>>>(static_cast<const bf16*>(x), rows, N,
                                                              ld, nullptr, partial);
  count_launch();
  using mimose_dev::kRedCols;
  mimose_dev::reduce_partials_kernel<<<grid_for((int64_t)G * N, kRedCols), 256, 0, s>>>(
      partial, rb, G * N, G * N, out, nullptr, nullptr);
  count_launch();
  return cudaGetLastError();
}

template <int L, int MAXC>
static void softmax_fwd_t(const bf16* in, bf16* p, bf16* pd, int64_t rows, int S, int ld,
                          const mimose_dev::DropoutCfg& d, cudaStream_t s, int causal) {
  const int64_t rows_per_block = 8 * (32 / L);
  const int g = (int)((rows + rows_per_block - 1) / rows_per_block);
  mimose_dev::softmax_fwd_kernel<L, MAXC><<<g, 256, 0, s>>>(in, p, pd, rows, S, ld, d, causal);
}
template <int L, int MAXC>
static void softmax_bwd_t(const bf16* p, bf16* dp, int64_t rows, int S, int ld,
                          const mimose_dev::DropoutCfg& d, float scale, cudaStream_t s, int causal) {
  const int64_t rows_per_block = 8 * (32 / L);
  const int g = (int)((rows + rows_per_block - 1) / rows_per_block);
  mimose_dev::softmax_bwd_kernel<L, MAXC><<<g, 256, 0, s>>>(p, dp, rows, S, ld, d, scale, causal);
}

// Dispatch: L lanes per row (8 for rows up to 512, 16 up to 1024, 32 up to
// 2048) and exactly MAXC = ceil(chunks / L) chunks per lane, so no lane runs
// fully predicated-off chunk slots.
#define MIMOSE_SOFTMAX_CASES(FN)                                                   \
  switch (maxc) {                                                                  \
    case 1: FN(1); break;                                                          \
    case 2: FN(2); break;                                                          \
    case 3: FN(3); break;                                                          \
    case 4: FN(4); break;                                                          \
    case 5: FN(5); break;                                                          \
    case 6: FN(6); break;                                                          \
    case 7: FN(7); break;                                                          \
    default: FN(8); break;                                                         \
  }

// lanes per row: 8 up to 256 columns, 16 up to 512, 32 beyond, so rows up to
// 1024 need <= 4 chunks per lane (the prefetching variants)
static bool softmax_geometry(int ld, int* L, int* maxc) {
  const int chunks = ld / 8;
  if (ld <= 512) *L = 8;
  else if (ld <= 1024) *L = 16;
  else if (ld <= 2048) *L = 32;
  else return false;
  *maxc = (chunks + *L - 1) / *L;
  return *maxc >= 1 && *maxc <= 8;
}

cudaError_t softmax_fwd(const void* scores, void* P, void* Pd, int64_t rows, int S, int ld,
                        const mimose_dev::DropoutCfg& d, cudaStream_t s, bool causal) {
  const int cz = causal ? 1 : 0;
  // scores read (live region), P and dropped P written over the row pitch
  ProfScope prof("mem_softmax_fwd", 0,
                 (double)rows * (2.0 * (causal ? 0.5 * (S + 1) : S) +
                                 2.0 * ld * (1 + (Pd != nullptr))),
                 s);
  auto in = static_cast<const bf16*>(scores);
  auto p = static_cast<bf16*>(P);
  auto pd = static_cast<bf16*>(Pd);
  int L = 0, maxc = 0;
  if (!softmax_geometry(ld, &L, &maxc)) return cudaErrorInvalidValue;
#define FWD8(M) softmax_fwd_t<8, M>(in, p, pd, rows, S, ld, d, s, cz)
#define FWD16(M) softmax_fwd_t<16, M>(in, p, pd, rows, S, ld, d, s, cz)
#define FWD32(M) softmax_fwd_t<32, M>(in, p, pd, rows, S, ld, d, s, cz)
  if (L == 8) { MIMOSE_SOFTMAX_CASES(FWD8) }
  else if (L == 16) { MIMOSE_SOFTMAX_CASES(FWD16) }
  else { MIMOSE_SOFTMAX_CASES(FWD32) }
#undef FWD8
#undef FWD16
#undef FWD32
  count_launch();
  return cudaGetLastError();
}

cudaError_t softmax_bwd(const void* P, void* dPd, int64_t rows, int S, int ld,
                        const mimose_dev::DropoutCfg& d, float scale, cudaStream_t s, bool causal) {
  const int cz = causal ? 1 : 0;
  ProfScope prof("mem_softmax_bwd", 0, (double)rows * 6.0 * S, s);  // P, dPd read; dS written
  auto p = static_cast<const bf16*>(P);
  auto dp = static_cast<bf16*>(dPd);
  int L = 0, maxc = 0;
  if (!softmax_geometry(ld, &L, &maxc)) return cudaErrorInvalidValue;
#define BWD8(M) softmax_bwd_t<8, M>(p, dp, rows, S, ld, d, scale, s, cz)
#define BWD16(M) softmax_bwd_t<16, M>(p, dp, rows, S, ld, d, scale, s, cz)
#define BWD32(M) softmax_bwd_t<32, M>(p, dp, rows, S, ld, d, scale, s, cz)
  if (L == 8) { MIMOSE_SOFTMAX_CASES(BWD8) }
  else if (L == 16) { MIMOSE_SOFTMAX_CASES(BWD16) }
  else { MIMOSE_SOFTMAX_CASES(BWD32) }
#undef BWD8
#undef BWD16
#undef BWD32
  count_launch();
  return cudaGetLastError();
}

cudaError_t embed_word_grad(const void* de, int H, const int32_t* perm, const int32_t* seg,
                            const int32_t* uid, int n_unique, float* dword, cudaStream_t s,
                            bool accumulate, int pad) {
  if (n_unique == 0) return cudaSuccess;
  mimose_dev::embed_word_grad_kernel<<<grid_for(n_unique, 8), 256, 0, s>>>(
      static_cast<const bf16*>(de), H, perm, seg, uid, n_unique, dword, accumulate ? 1 : 0, pad);
  count_launch();
  return cudaGetLastError();
}

cudaError_t embed_pos_grad(const void* de, int B, int S, int H, float* dpos, cudaStream_t s) {
  mimose_dev::embed_pos_grad_kernel<<<S, 128, 0, s>>>(static_cast<const bf16*>(de), B, S, H, dpos);
  count_launch();
  return cudaGetLastError();
}

cudaError_t mc_head(const void* pre, int B, int H, int C, const float* wc, const float* bc,
                    const int32_t* labels, const mimose_dev::DropoutCfg& d, float* loss,
                    float* logits, void* dpre, float* dwc, float* dbc, cudaStream_t s) {
  if (B % C) return cudaErrorInvalidValue;
  mimose_dev::mc_head_kernel<<<1, 1024, 2 * B * sizeof(float), s>>>(
      static_cast<const bf16*>(pre), B, H, C, wc, bc, labels, d, loss, logits,
      static_cast<bf16*>(dpre), dwc, dbc);
  count_launch();
  return cudaGetLastError();
}

int sumsq_blocks() { return 2 * persistent_blocks(); }

cudaError_t grad_norm2(const float* g, int64_t n, float* partial, float* out, cudaStream_t s) {
  const int nb = sumsq_blocks();
  ProfScope prof("mem_gradnorm", 0, 4.0 * n, s);
  mimose_dev::sumsq_partial_kernel<<<nb, 256, 0, s>>>(g, n, partial);
  count_launch();
  mimose_dev::sum_partials_kernel<<<1, 32, 0, s>>>(partial, nb, out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t adamw(float* p, float* m, float* v, const float* g, void* p16, int64_t n,
                  const uint8_t* decay_chunk, const float* norm2, const AdamWArgs& a,
                  cudaStream_t s) {
  ProfScope prof("mem_adamw", 0, 30.0 * n, s);  // p, m, v, g read; p, m, v, p16 written
  mimose_dev::adamw_kernel<<<4 * persistent_blocks(), 256, 0, s>>>(
      p, m, v, g, static_cast<bf16*>(p16), n, decay_chunk, norm2, a);
  count_launch();
  return cudaGetLastError();
}

cudaError_t init_normal(float* p, int64_t n, float mean, float std, uint64_t seed,
                        uint64_t stream, cudaStream_t s) {
  mimose_dev::init_normal_kernel<<<4 * persistent_blocks(), 256, 0, s>>>(p, n, mean, std, seed,
                                                                         stream);
  count_launch();
  return cudaGetLastError();
}

cudaError_t f32_to_bf16(const float* in, void* out, int64_t n, cudaStream_t s) {
  mimose_dev::f32_to_bf16_kernel<<<4 * persistent_blocks(), 256, 0, s>>>(
      in, static_cast<bf16*>(out), n);
  count_launch();
  return cudaGetLastError();
}

cudaError_t dropout_apply(const void* in, void* out, int64_t n, const DropoutCfg& d,
                          cudaStream_t s) {
  if (n % 8) return cudaErrorInvalidValue;
  ProfScope prof("mem_dropout", 0, 4.0 * n, s);
  mimose_dev::dropout_apply_kernel<<<4 * persistent_blocks(), 256, 0, s>>>(
      static_cast<const bf16*>(in), static_cast<bf16*>(out), n / 8, d);
  count_launch();
  return cudaGetLastError();
}

cudaError_t dgelu_apply(const void* dg, const void* u, void* out, int64_t n, bool tanh_form,
                        cudaStream_t s) {
  if (n % 8) return cudaErrorInvalidValue;
  ProfScope prof("mem_dgelu", 0, 6.0 * n, s);
  mimose_dev::dgelu_apply_kernel<<<4 * persistent_blocks(), 256, 0, s>>>(
      static_cast<const bf16*>(dg), static_cast<const bf16*>(u), static_cast<bf16*>(out), n / 8,
      tanh_form ? 1 : 0);
  count_launch();
  return cudaGetLastError();
}

cudaError_t gather_rows(const void* src, const int32_t* idx, int n, int H, void* dst,
                        cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  mimose_dev::gather_rows_kernel<<<grid_for(n, 8), 256, 0, s>>>(
      static_cast<const bf16*>(src), idx, n, H, static_cast<bf16*>(dst), 0);
  count_launch();
  return cudaGetLastError();
}

cudaError_t scatter_rows(const void* src, const int32_t* idx, int n, int H, void* dst,
                         cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  mimose_dev::gather_rows_kernel<<<grid_for(n, 8), 256, 0, s>>>(
      static_cast<const bf16*>(src), idx, n, H, static_cast<bf16*>(dst), 1);
  count_launch();
  return cudaGetLastError();
}

cudaError_t sum_f32(const float* x, int n, float scale, float* out, cudaStream_t s) {
  mimose_dev::sum_f32_kernel<<<1, 1024, 0, s>>>(x, n, scale, out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t qa_head(const void* x, int B, int S, int H, const float* w, const float* b,
                    const int32_t* labels, float* logits, float* dlogits, float* loss_parts,
                    cudaStream_t s) {
  mimose_dev::qa_head_kernel<<<B, 512, 2 * S * sizeof(float), s>>>(
      static_cast<const bf16*>(x), S, H, w, b, labels, 1.f / (2.f * B), logits, dlogits,
      loss_parts);
  count_launch();
  return cudaGetLastError();
}

int qa_row_blocks(int T) { return T < 64 ? 1 : 64; }

cudaError_t qa_head_bwd(const void* x, const float* dlogits, int T, int H, const float* w,
                        void* dx, float* partial, float* dW, float* db, cudaStream_t s) {
  const int rb = qa_row_blocks(T);
  dim3 grid((H + 1 + 255) / 256, rb);
  mimose_dev::qa_head_bwd_kernel<<<grid, 256, 0, s>>>(static_cast<const bf16*>(x), dlogits, T, H,
                                                      w, static_cast<bf16*>(dx), partial);
  count_launch();
  const int W = 2 * H + 2;
  using mimose_dev::kRedCols;
  mimose_dev::reduce_partials_kernel<<<grid_for(W, kRedCols), 256, 0, s>>>(partial, rb, W, 2 * H,
                                                                         dW, db, nullptr);
  count_launch();
  return cudaGetLastError();
}

cudaError_t ce_rows(void* logits, int rows, int V, int ld, const int32_t* labels,
                    float grad_scale, float* loss_rows, cudaStream_t s) {
  if (ld % 8) return cudaErrorInvalidValue;
  ProfScope prof("mem_ce_rows", 0, 4.0 * rows * (double)V, s);
  mimose_dev::ce_rows_kernel<<<rows, 512, 0, s>>>(static_cast<bf16*>(logits), V, ld, labels,
                                                  grad_scale, loss_rows);
  count_launch();
  return cudaGetLastError();
}

}  // namespace mimose_ops
