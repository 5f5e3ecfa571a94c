// Block-looped fused attention-score kernels for sm_100a: any S, optional
// causal mask. A 128-query tile walks its keys in 256-column blocks, each
// block one tcgen05 accumulator (two of them double-buffered in TMEM), twice:
//
//   forward   pass 0 (stats) : s = alpha Q K^T per block -> online row max m
//                              and sum l = sum 2^(s log2e - m)
//             pass 1 (output): the same block MMA again -> P = 2^(...) / l,
//                              Pd = dropout(P) (Philox), TMA-stored
//   backward  one pass        : dot_i = sum_j dP_ij P_ij = dO_i . ctx_i (ctx = Pd V,
//                              the forward output: no stats pass), then per
//                              block dPd = dO V^T -> dS = P * (g - dot) * scale,
//                              g = keep ? dPd / (1 - p) : 0 (Philox keep)
//
// The second MMA of a block costs 2 * 128 * 256 * 64 flops (K = 64), far less
// than keeping a whole S-wide row in TMEM: with two 256-column accumulators
// the next block's MMA always overlaps the current block's epilogue, for any
// S (the single-row kernel in attn_sm100.cuh needs all 512 columns once
// S > 256 and serialises MMA and epilogue). P / Pd / dS stay materialised:
// the reference's quadratic activation term (proj/models/bert12.model c2).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "attn_sm100.cuh"
#include "common.cuh"
#include "ptx_sm100.cuh"

namespace mimose_dev {

struct Attn2Params {
  int S, ld, nh, B;
  float alpha;                 // fwd: score scale (1/sqrt(d))
  float ds_scale;              // bwd: scale folded into dS (1/sqrt(d))
  DropoutCfg drop;
  const __nv_bfloat16* P;      // bwd: saved probabilities [B][nh][S][ld]
  const __nv_bfloat16* Pd;     // bwd: saved dropped probabilities (nullptr: no dropout)
  int store_pd;                // fwd: also store the dropped-out probabilities
  int causal;                  // key j > query i masked (GPT-2)
  // bwd: dO and the forward's attention output ctx = Pd V, head-interleaved
  // [B * S][tok_ld] bf16 (head h at columns 64 h): rowsum(dP o P) = dO . ctx
  const __nv_bfloat16* dO;
  const __nv_bfloat16* ctx;
  int tok_ld;
};

struct Attn2Cfg {
  static constexpr int kEW = 16;                   // epilogue warps
  static constexpr int kThreads = 64 + 32 * kEW;
  static constexpr int kKB = 256;                  // key columns per block (one accumulator)
  static constexpr int kQBytes = 128 * 64 * 2;     // query (dO) tile, double-buffered
  static constexpr int kKBytes = kKB * 64 * 2;     // key (V) block
  static constexpr int kKStages = 3;
  static constexpr int kBufBytes = 32 * 64;        // staging: 32 rows x 32 bf16 columns
  static constexpr int kStagingBytes = kEW * 2 * kBufBytes;
  static constexpr int kRedBytes = 2 * 2 * 4 * 128 * 4;  // [tile parity][m|l][part][row]
  static constexpr int kSmemBytes =
      2 * kQBytes + kKStages * kKBytes + kStagingBytes + kRedBytes + 1024 + 256;
};

template <bool BWD>
__global__ void __launch_bounds__(Attn2Cfg::kThreads, 1)
    attn2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmO1, const __grid_constant__ CUtensorMap tmO2,
                 const Attn2Params p) {
  using Cfg = Attn2Cfg;
  constexpr int KS = Cfg::kKStages;
  constexpr float kLog2e = 1.4426950408889634f;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;                                  // [2][16 KB]
  uint8_t* sK = sQ + 2 * Cfg::kQBytes;                 // [KS][32 KB]
  uint8_t* sD = sK + KS * Cfg::kKBytes;                // staging
  float* red = reinterpret_cast<float*>(sD + Cfg::kStagingBytes);
  uint64_t* qfull = reinterpret_cast<uint64_t*>(sD + Cfg::kStagingBytes + Cfg::kRedBytes);
  uint64_t* qempty = qfull + 2;
  uint64_t* kfull = qempty + 2;
  uint64_t* kempty = kfull + KS;
  uint64_t* tfull = kempty + KS;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const int tiles_m = (p.S + 127) / 128;
  const int num_tiles = tiles_m * p.nh * p.B;
  const int nkb = (p.S + Cfg::kKB - 1) / Cfg::kKB;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    tma_prefetch(&tmO1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&qfull[i], 1);
      mbar_init(&qempty[i], 1);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], Cfg::kEW);
    }
    for (int s = 0; s < KS; ++s) {
      mbar_init(&kfull[s], 1);
      mbar_init(&kempty[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // inputs of this launch are complete from here on

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int it_t = 0, it_k = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it_t) {
        const int z = tile / tiles_m;
        const int m0 = (tile % tiles_m) * 128;
        const int b1 = z % p.nh, b2 = z / p.nh;
        const int qb = it_t & 1;
        mbar_wait(&qempty[qb], ((it_t >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&qfull[qb], Cfg::kQBytes);
        tma_load_4d(&tmA, &qfull[qb], sQ + qb * Cfg::kQBytes, 0, m0, b1, b2);
        for (int pass = 0; pass < (BWD ? 1 : 2); ++pass)
          for (int kb = 0; kb < nkb; ++kb, ++it_k) {
            const int ks = it_k % KS;
            mbar_wait(&kempty[ks], ((it_k / KS) & 1) ^ 1);
            mbar_arrive_expect_tx(&kfull[ks], Cfg::kKBytes);
            tma_load_4d(&tmB, &kfull[ks], sK + ks * Cfg::kKBytes, 0, kb * Cfg::kKB, b1, b2);
          }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = idesc_bf16_f32(128, Cfg::kKB, false, false);
    int it_t = 0, it_k = 0, seq = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it_t) {
      const int qb = it_t & 1;
      mbar_wait(&qfull[qb], (it_t >> 1) & 1);
      tc_fence_after();
      for (int pass = 0; pass < (BWD ? 1 : 2); ++pass)
        for (int kb = 0; kb < nkb; ++kb, ++it_k, ++seq) {
          const int acc = seq & 1;
          mbar_wait(&tempty[acc], ((seq >> 1) & 1) ^ 1);
          tc_fence_after();
          const int ks = it_k % KS;
          mbar_wait(&kfull[ks], (it_k / KS) & 1);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_addr = smem_u32(sQ + qb * Cfg::kQBytes);
            const uint32_t b_addr = smem_u32(sK + ks * Cfg::kKBytes);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t da = smem_desc_sw128(a_addr + kk * 32, 16, 1024);
              const uint64_t db = smem_desc_sw128(b_addr + kk * 32, 16, 1024);
              umma_bf16(tmem_base + acc * Cfg::kKB, da, db, idesc, kk != 0 ? 1u : 0u);
            }
            umma_commit(&kempty[ks]);
            umma_commit(&tfull[acc]);
          }
          __syncwarp();
        }
      if (lane == 0) umma_commit(&qempty[qb]);
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 2;
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int part = ew >> 2;      // 64-column part of each 256-column block
    const int r_local = quarter * 32 + static_cast<int>(lane);
    uint8_t* wbuf = sD + ew * (2 * Cfg::kBufBytes);
    const uint32_t rbase = smem_u32(wbuf) + lane * 64;
    const uint32_t sw = (lane >> 1) & 3;  // SWIZZLE_64B: 16 B chunk j of row r at j ^ ((r >> 1) & 3)
    const uint32_t thr_hi = p.drop.threshold << 16;
    const float sc = p.alpha * kLog2e;
    int seq = 0, it_t = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it_t) {
      float* red_a = red + (it_t & 1) * 1024;  // [4][128] max / dot
      float* red_b = red_a + 512;              // [4][128] sum
      const int z = tile / tiles_m;
      const int m0 = (tile % tiles_m) * 128;
      const int b1 = z % p.nh, b2 = z / p.nh;
      const int i = m0 + r_local;  // query row within its sequence
      const bool row_ok = i < p.S;
      const int64_t grow = ((int64_t)z * p.S + (row_ok ? i : 0));  // row of the [B*nh*S][ld] view
      // valid keys of this row / of any row of this warp (warp-uniform skip)
      const int jmax = row_ok ? (p.causal ? min(p.S, i + 1) : p.S) : 0;
      const int wmax = p.causal ? min(p.S, m0 + quarter * 32 + 32) : p.S;
      const uint32_t t_lane = tmem_base + ((uint32_t)(quarter * 32) << 16) + part * 64;

      if constexpr (!BWD) {
        // ---- pass 0: online row max / sum over the key blocks
        float m_run = -INFINITY, l_run = 0.f;
        for (int kb = 0; kb < nkb; ++kb, ++seq) {
          const int acc = seq & 1;
          mbar_wait(&tfull[acc], (seq >> 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int h = 0; h < 2; ++h) {
            const int c = kb * Cfg::kKB + part * 64 + h * 32;
            if (c >= wmax) break;
            uint32_t r[32];
            tmem_ld32_nowait(t_lane + acc * Cfg::kKB + h * 32, r);
            tmem_wait_ld();
            float mc = -INFINITY;
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (c + e < jmax) mc = fmaxf(mc, __uint_as_float(r[e]));
            if (mc != -INFINITY) {
              const float m_new = fmaxf(m_run, mc * sc);
              float acc_l = 0.f;
#pragma unroll
              for (int e = 0; e < 32; ++e)
                acc_l += c + e < jmax ? ex2f(fmaf(__uint_as_float(r[e]), sc, -m_new)) : 0.f;
              l_run = (m_run != -INFINITY ? l_run * ex2f(m_run - m_new) : 0.f) + acc_l;
              m_run = m_new;
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        red_a[part * 128 + r_local] = m_run;
        red_b[part * 128 + r_local] = l_run;
        epi_bar();
        float m = red_a[r_local];
#pragma unroll
        for (int q = 1; q < 4; ++q) m = fmaxf(m, red_a[q * 128 + r_local]);
        float l = 0.f;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float mq = red_a[q * 128 + r_local];
          if (mq != -INFINITY) l += red_b[q * 128 + r_local] * ex2f(mq - m);
        }
        const float inv = l > 0.f ? 1.f / l : 0.f;
        const float nm = m != -INFINITY ? -m : 0.f;
        // ---- pass 1: P = 2^(s sc - m) / l, Pd = dropout(P) -> stage -> TMA store
        for (int kb = 0; kb < nkb; ++kb, ++seq) {
          const int acc = seq & 1;
          mbar_wait(&tfull[acc], (seq >> 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int h = 0; h < 2; ++h) {
            const int c = kb * Cfg::kKB + part * 64 + h * 32;
            if (c >= p.S) break;
            uint32_t r[32];
            if (c < wmax) {
              tmem_ld32_nowait(t_lane + acc * Cfg::kKB + h * 32, r);
              tmem_wait_ld();
            }
            if (lane == 0) bulk_wait_read<0>();
            __syncwarp();
            uint32_t rnd[2][4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (p.store_pd && (q & 1) == 0) {  // Philox for 16 columns at a time
                uint64_t grp[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) grp[u] = ((uint64_t)grow * p.ld + c + 8 * (q + u)) >> 3;
                philox_n<2>(p.drop.seed, p.drop.stream, grp, rnd);
              }
              float pv[8], dv[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const int col = c + 8 * q + e;
                pv[e] = col < jmax ? bf16r(ex2f(fmaf(__uint_as_float(r[8 * q + e]), sc, nm)) * inv)
                                   : 0.f;
              }
              const uint32_t addr = rbase + ((q ^ sw) << 4);
              st_shared_v4(addr, pack_bf16x2_(pv[0], pv[1]), pack_bf16x2_(pv[2], pv[3]),
                           pack_bf16x2_(pv[4], pv[5]), pack_bf16x2_(pv[6], pv[7]));
              if (p.store_pd) {
#pragma unroll
                for (int e = 0; e < 8; ++e)
                  dv[e] = philox_keep_w(rnd[q & 1], e, thr_hi) ? pv[e] * p.drop.scale : 0.f;
                st_shared_v4(addr + Cfg::kBufBytes, pack_bf16x2_(dv[0], dv[1]),
                             pack_bf16x2_(dv[2], dv[3]), pack_bf16x2_(dv[4], dv[5]),
                             pack_bf16x2_(dv[6], dv[7]));
              }
            }
            fence_async_shared();
            __syncwarp();
            if (lane == 0) {
              tma_store_4d(&tmO1, wbuf, c, m0 + quarter * 32, b1, b2);
              if (p.store_pd)
                tma_store_4d(&tmO2, wbuf + Cfg::kBufBytes, c, m0 + quarter * 32, b1, b2);
              bulk_commit();
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
      } else {
        // ---- dot_i = dO_i . ctx_i; each column part sums 16 of the 64 head dims
        {
          float d = 0.f;
          if (row_ok) {
            const int64_t trow = (int64_t)b2 * p.S + i;
            const __nv_bfloat16* a = p.dO + trow * p.tok_ld + b1 * 64 + part * 16;
            const __nv_bfloat16* c = p.ctx + trow * p.tok_ld + b1 * 64 + part * 16;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              float fa[8], fc[8];
              unpack_bf16x8(*reinterpret_cast<const uint4*>(a + 8 * q), fa);
              unpack_bf16x8(*reinterpret_cast<const uint4*>(c + 8 * q), fc);
#pragma unroll
              for (int e = 0; e < 8; ++e) d = fmaf(fa[e], fc[e], d);
            }
          }
          red_a[part * 128 + r_local] = d;
        }
        epi_bar();
        const float dot =
            (red_a[r_local] + red_a[128 + r_local]) + (red_a[256 + r_local] + red_a[384 + r_local]);
        const __nv_bfloat16* prow = p.P + grow * p.ld;
        // ---- dS = P * (g - dot) * scale, g = keep ? dPd / (1 - p) : 0
        for (int kb = 0; kb < nkb; ++kb, ++seq) {
          const int acc = seq & 1;
          // this block's P rows (both 32-column chunks) in flight while the MMA lands
          const int cb = kb * Cfg::kKB + part * 64;
          uint4 pr[2][4];
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int col = cb + h * 32 + 8 * q;
              pr[h][q] = col < jmax ? __ldcs(reinterpret_cast<const uint4*>(prow + col))
                                    : make_uint4(0, 0, 0, 0);
            }
          mbar_wait(&tfull[acc], (seq >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = cb + h * 32;
            if (c < p.S) {
              uint32_t r[32];
              if (c < wmax) {
                tmem_ld32_nowait(t_lane + acc * Cfg::kKB + h * 32, r);
                tmem_wait_ld();
              }
              if (lane == 0) bulk_wait_read<0>();
              __syncwarp();
              uint32_t rnd[2][4];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                if ((q & 1) == 0) {
                  uint64_t grp[2];
#pragma unroll
                  for (int u = 0; u < 2; ++u) grp[u] = ((uint64_t)grow * p.ld + c + 8 * (q + u)) >> 3;
                  philox_n<2>(p.drop.seed, p.drop.stream, grp, rnd);
                }
                float pf[8], ds[8];
                unpack_bf16x8(pr[h][q], pf);
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                  const bool in = c + 8 * q + e < jmax;
                  const float g = (in && philox_keep_w(rnd[q & 1], e, thr_hi))
                                      ? __uint_as_float(r[8 * q + e]) * p.drop.scale
                                      : 0.f;
                  ds[e] = in ? pf[e] * (g - dot) * p.ds_scale : 0.f;
                }
                st_shared_v4(rbase + ((q ^ sw) << 4), pack_bf16x2_(ds[0], ds[1]),
                             pack_bf16x2_(ds[2], ds[3]), pack_bf16x2_(ds[4], ds[5]),
                             pack_bf16x2_(ds[6], ds[7]));
              }
              fence_async_shared();
              __syncwarp();
              if (lane == 0) {
                tma_store_4d(&tmO1, wbuf, c, m0 + quarter * 32, b1, b2);
                bulk_commit();
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
      }
    }
    if (lane == 0) bulk_wait<0>();
  }

  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace mimose_dev
