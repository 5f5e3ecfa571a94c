// Fused attention-score kernels for sm_100a (S <= 512): the batched
// contraction runs on tcgen05 with the whole key row of a 128-query tile in
// TMEM (256 or 512 fp32 columns), and the softmax lives in the epilogue, so
// the S x S score matrix never round-trips through HBM.
//
//   forward : S = alpha * Q K^T  ->  P = softmax(S), Pd = dropout(P)   (P, Pd stored)
//   backward: dPd = dO V^T       ->  dS = P * (dP - rowsum(dP * P)) * scale,
//                                    dP = dPd * mask / (1 - p)           (dS stored)
//
// Row statistics: 16 epilogue warps split each row into four column parts
// (TMEM lane quarter x part); partial max / sum / dot are exchanged through
// shared memory behind a named barrier. Forward: pass 1 online row max / sum
// with the exponentials written back into TMEM (tcgen05.st) relative to the
// running max, pass 2 normalise (per-chunk max correction) + Philox dropout,
// so every score costs one ex2 and two TMEM reads. Backward:
// the keep masks of pass 1 stay in registers for pass 2. Output chunks (32
// columns) go through 64B-swizzled staging buffers and TMA bulk stores.
// The materialised P / Pd / dS keep the reference's quadratic activation term
// (reference proj/models/bert12.model c2) exactly as the unfused path does.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "ptx_sm100.cuh"

namespace mimose_dev {

struct AttnParams {
  int S, ld, nh, B;
  float alpha;                // fwd: score scale (1/sqrt(d))
  float ds_scale;             // bwd: scale folded into dS (1/sqrt(d))
  DropoutCfg drop;
  const __nv_bfloat16* P;     // bwd: saved probabilities [B][nh][S][ld]
  int store_pd;               // fwd: also store the dropped-out probabilities
  int causal;                 // fwd: keys j > query i masked (P = 0 there, so the
                              // backward needs no mask: dS = P * (...) = 0)
};

template <int NC>
struct AttnCfg {
  static constexpr int kEW = 16;                 // epilogue warps
  static constexpr int kThreads = 64 + 32 * kEW;
  static constexpr int kQ = NC / 4;              // accumulator columns per epilogue warp
  static constexpr int kABytes = 128 * 64 * 2;
  static constexpr int kBBytes = NC * 64 * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = NC == 512 ? 1 : 2;
  static constexpr int kAcc = NC == 512 ? 1 : 2;  // TMEM accumulators (512 columns total)
  static constexpr int kBufBytes = 32 * 64;       // 32 rows x 64 B (32 bf16 columns)
  static constexpr int kStagingBytes = kEW * 2 * kBufBytes;
  static constexpr int kRedBytes = 2 * 2 * 4 * 128 * 4;  // [tile parity][max|sum][part][row]
  static constexpr int kSmemBytes =
      kStages * kStageBytes + kStagingBytes + kRedBytes + 1024 + 256;
};

__device__ __forceinline__ float ex2f(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ uint32_t pack_bf16x2_(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void epi_bar() {
  asm volatile("bar.sync 1, 512;" ::: "memory");
}

__device__ __forceinline__ void unpack_bf16x8(const uint4& raw, float (&v)[8]) {
  const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __bfloat1622float2(h2[e]);
    v[2 * e] = f.x;
    v[2 * e + 1] = f.y;
  }
}

template <int NC, bool BWD>
__global__ void __launch_bounds__(AttnCfg<NC>::kThreads, 1)
    attn_scores_kernel(const __grid_constant__ CUtensorMap tmA,
                       const __grid_constant__ CUtensorMap tmB,
                       const __grid_constant__ CUtensorMap tmO1,
                       const __grid_constant__ CUtensorMap tmO2, const AttnParams p) {
  using Cfg = AttnCfg<NC>;
  constexpr int NS = Cfg::kStages;
  constexpr int NCH = NC / 128;  // 32-column chunks per column part
  constexpr float kLog2e = 1.4426950408889634f;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + NS * Cfg::kABytes;
  uint8_t* sD = smem + NS * Cfg::kStageBytes;
  float* red = reinterpret_cast<float*>(sD + Cfg::kStagingBytes);  // [2][2][4][128]
  uint64_t* full = reinterpret_cast<uint64_t*>(sD + Cfg::kStagingBytes + Cfg::kRedBytes);
  uint64_t* empty = full + NS;
  uint64_t* tfull = empty + NS;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const int tiles_m = (p.S + 127) / 128;
  const int num_tiles = tiles_m * p.nh * p.B;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    tma_prefetch(&tmO1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], Cfg::kEW);
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
      int it = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        const int z = tile / tiles_m;
        const int m0 = (tile % tiles_m) * 128;
        const int b1 = z % p.nh, b2 = z / p.nh;
        const int s = it % NS;
        const uint32_t ph = (it / NS) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], Cfg::kStageBytes);
        tma_load_4d(&tmA, &full[s], sA + s * Cfg::kABytes, 0, m0, b1, b2);
#pragma unroll
        for (int part = 0; part < NC / 256; ++part)
          tma_load_4d(&tmB, &full[s], sB + s * Cfg::kBBytes + part * 256 * 128, 0, part * 256, b1,
                      b2);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // MMA width trimmed to the key columns that exist (multiple of 16): keys
    // >= S are zero-filled by the TMA and never read, so computing them only
    // burns tensor cycles (and power) - e.g. S = 288 needs 256 + 32 columns
    auto n_eff = [&](int col0) {
      const int n = min(256, ((p.S - col0 + 15) / 16) * 16);
      return n < 16 ? 16 : n;
    };
    const uint32_t idesc = idesc_bf16_f32(128, n_eff(0), false, false);
    const uint32_t idesc_hi = idesc_bf16_f32(128, n_eff(256), false, false);
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int s = it % NS;
      const uint32_t ph = (it / NS) & 1;
      if constexpr (NC == 512) {
        // one 512-column accumulator released in two halves: the lower half
        // of tile i + 1 is computed while the epilogue still works through
        // the upper half of tile i (tfull / tempty index = half)
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t hph = it & 1;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          mbar_wait(&tempty[half], hph ^ 1);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_addr = smem_u32(sA + s * Cfg::kABytes);
            const uint32_t b_addr = smem_u32(sB + s * Cfg::kBBytes);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t da = smem_desc_sw128(a_addr + kk * 32, 16, 1024);
              const uint64_t db = smem_desc_sw128(b_addr + half * 256 * 128 + kk * 32, 16, 1024);
              umma_bf16(tmem_base + half * 256, da, db, half ? idesc_hi : idesc, kk != 0 ? 1u : 0u);
            }
            umma_commit(&tfull[half]);
            if (half == 1) umma_commit(&empty[s]);
          }
          __syncwarp();
        }
        continue;
      }
      const int acc = it % Cfg::kAcc;
      const uint32_t aph = (it / Cfg::kAcc) & 1;
      mbar_wait(&tempty[acc], aph ^ 1);
      tc_fence_after();
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t a_addr = smem_u32(sA + s * Cfg::kABytes);
        const uint32_t b_addr = smem_u32(sB + s * Cfg::kBBytes);
#pragma unroll
        for (int part = 0; part < NC / 256; ++part) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t da = smem_desc_sw128(a_addr + kk * 32, 16, 1024);
            const uint64_t db = smem_desc_sw128(b_addr + part * 256 * 128 + kk * 32, 16, 1024);
            umma_bf16(tmem_base + acc * NC + part * 256, da, db, idesc, kk != 0 ? 1u : 0u);
          }
        }
        umma_commit(&empty[s]);
        umma_commit(&tfull[acc]);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 2;
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int part = ew >> 2;      // column part 0..3
    const int r_local = quarter * 32 + static_cast<int>(lane);
    uint8_t* wbuf = sD + ew * (2 * Cfg::kBufBytes);
    const uint32_t rbase = smem_u32(wbuf) + lane * 64;
    const uint32_t sw = (lane >> 1) & 3;  // SWIZZLE_64B: 16 B chunk j of row r at j ^ ((r >> 1) & 3)
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      // row-statistic exchange buffers, double-buffered by tile parity so a
      // warp running ahead cannot overwrite what another has yet to read
      float* red_a = red + (it & 1) * 1024;  // [4][128] max / dot
      float* red_b = red_a + 512;            // [4][128] sum
      const int z = tile / tiles_m;
      const int m0 = (tile % tiles_m) * 128;
      const int b1 = z % p.nh, b2 = z / p.nh;
      const int acc = it % Cfg::kAcc;
      const uint32_t aph = (it / Cfg::kAcc) & 1;
      const int i = m0 + r_local;  // query row
      const bool row_ok = i < p.S;
      const int64_t grow = ((int64_t)z * p.S + (row_ok ? i : 0));  // row of the [B*nh*S][ld] view
      if constexpr (NC != 512) {
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
      }
      // NC = 512: half h of the row lands on tfull[h] and is released on
      // tempty[h]; chunks j = 0, 1 are the lower half, j = 2, 3 the upper
      auto half_wait = [&](int j) {
        if constexpr (NC == 512) {
          if (j == 0 || j == 2) {
            mbar_wait(&tfull[j >> 1], it & 1);
            tc_fence_after();
          }
        }
      };
      auto half_release = [&](int j) {
        if constexpr (NC == 512) {
          if (j == 1 || j == 3) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[j >> 1]);
          }
        }
      };
      // 32-column chunks are dealt round-robin to the 4 column parts (chunk
      // ch -> part ch % 4), so every warp gets within one chunk of S / 4
      // columns whatever S is
      const uint32_t t_row = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * NC;
      const uint32_t thr_hi = p.drop.threshold << 16;

      if constexpr (!BWD) {
        const int jmax = p.causal ? min(p.S, i + 1) : p.S;  // valid keys of this row
        // ---- pass 1 (online): per chunk, the running row max m of this part
        // and the running sum of 2^(s sc - m) (rescaled when m grows); the
        // exponentials go back into TMEM relative to the max current at that
        // chunk (mch[j]), corrected in pass 2 by 2^(mch[j] - m_row)
        const float sc = p.alpha * kLog2e;
        float m_run = -INFINITY, l_run = 0.f;
        float mch[NCH];
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          half_wait(j);
          mch[j] = -INFINITY;
          const int c = (part + 4 * j) * 32;
          if (c < p.S) {
            uint32_t r[32];
            tmem_ld32_nowait(t_row + c, r);
            tmem_wait_ld();
            float cm = -INFINITY;
            if (c + 32 <= jmax) {
#pragma unroll
              for (int e = 0; e < 32; ++e) cm = fmaxf(cm, __uint_as_float(r[e]));
            } else {
#pragma unroll
              for (int e = 0; e < 32; ++e)
                if (c + e < jmax) cm = fmaxf(cm, __uint_as_float(r[e]));
            }
            const float m_new = fmaxf(m_run, cm * sc);
            if (m_new != -INFINITY) {
              if (m_run != -INFINITY) l_run *= ex2f(m_run - m_new);
              const float nm = -m_new;
              if (c + 32 <= jmax) {  // whole chunk valid: no per-element masking
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                  const float x = ex2f(fmaf(__uint_as_float(r[e]), sc, nm));
                  l_run += x;
                  r[e] = __float_as_uint(x);
                }
              } else {
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                  const float x = c + e < jmax ? ex2f(fmaf(__uint_as_float(r[e]), sc, nm)) : 0.f;
                  l_run += x;
                  r[e] = __float_as_uint(x);
                }
              }
              m_run = m_new;
            } else {
#pragma unroll
              for (int e = 0; e < 32; ++e) r[e] = 0u;
            }
            mch[j] = m_run;
            tmem_st32(t_row + c, r);
          }
        }
        tmem_wait_st();
        red_a[part * 128 + r_local] = m_run;
        red_b[part * 128 + r_local] = l_run;
        epi_bar();
        float m_row = red_a[r_local];
#pragma unroll
        for (int q = 1; q < 4; ++q) m_row = fmaxf(m_row, red_a[q * 128 + r_local]);
        float l_row = 0.f;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float mq = red_a[q * 128 + r_local];
          if (mq != -INFINITY) l_row += red_b[q * 128 + r_local] * ex2f(mq - m_row);
        }
        const float inv = l_row > 0.f ? 1.f / l_row : 0.f;
        // ---- pass 2: normalise (with the chunk's max correction), dropout,
        // stage, TMA store
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          const int c = (part + 4 * j) * 32;
          if (c >= p.S) {
            half_release(j);
            continue;
          }
          const float f = mch[j] != -INFINITY ? ex2f(mch[j] - m_row) * inv : 0.f;
          uint32_t rnd[4][4];
          if (p.store_pd) {
            uint64_t grp[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) grp[q] = ((uint64_t)grow * p.ld + c + 8 * q) >> 3;
            philox_n<4>(p.drop.seed, p.drop.stream, grp, rnd);
          }
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
          uint32_t r[32];
          tmem_ld32_nowait(t_row + c, r);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float pv[8], dv[8];
            uint32_t ph[4];  // P rounded once to bf16 pairs; pv = the same values widened
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              ph[e >> 1] = pack_bf16x2_(__uint_as_float(r[8 * q + e]) * f,
                                        __uint_as_float(r[8 * q + e + 1]) * f);
              pv[e] = __uint_as_float(ph[e >> 1] << 16);
              pv[e + 1] = __uint_as_float(ph[e >> 1] & 0xFFFF0000u);
            }
            const uint32_t addr = rbase + ((q ^ sw) << 4);
            st_shared_v4(addr, ph[0], ph[1], ph[2], ph[3]);
            if (p.store_pd) {
#pragma unroll
              for (int e = 0; e < 8; ++e)
                dv[e] = philox_keep_w(rnd[q], e, thr_hi) ? pv[e] * p.drop.scale : 0.f;
              st_shared_v4(addr + Cfg::kBufBytes, pack_bf16x2_(dv[0], dv[1]),
                           pack_bf16x2_(dv[2], dv[3]), pack_bf16x2_(dv[4], dv[5]),
                           pack_bf16x2_(dv[6], dv[7]));
            }
          }
          fence_async_shared();
          __syncwarp();
          if (lane == 0) {
            tma_store_4d(&tmO1, wbuf, c, m0 + quarter * 32, b1, b2);
            if (p.store_pd) tma_store_4d(&tmO2, wbuf + Cfg::kBufBytes, c, m0 + quarter * 32, b1, b2);
            bulk_commit();
          }
          half_release(j);
        }
      } else {
        // ---- backward: pass 1 dot = sum_j dP_j P_j (dP = dPd * keep * scale);
        // the keep decisions of each 32-column chunk stay in one register
        // (km) for pass 2, dP is re-read from TMEM
        const __nv_bfloat16* prow = p.P + grow * p.ld;
        uint32_t km[NCH];
        float dot = 0.f;
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          half_wait(j);
          const int c = (part + 4 * j) * 32;
          if (c < p.S) {
            uint64_t grp[4];
            uint32_t rnd[4][4];
#pragma unroll
            for (int q = 0; q < 4; ++q) grp[q] = ((uint64_t)grow * p.ld + c + 8 * q) >> 3;
            philox_n<4>(p.drop.seed, p.drop.stream, grp, rnd);
            km[j] = 0u;
            uint4 pr[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              pr[q] = (row_ok && c + 8 * q < p.S) ? *reinterpret_cast<const uint4*>(prow + c + 8 * q)
                                                  : make_uint4(0, 0, 0, 0);
            uint32_t r[32];
            tmem_ld32_nowait(t_row + c, r);
            tmem_wait_ld();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float pf[8];
              unpack_bf16x8(pr[q], pf);
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const bool keep = c + 8 * q + e < p.S && philox_keep_w(rnd[q], e, thr_hi);
                km[j] |= (keep ? 1u : 0u) << (8 * q + e);
                const float g = keep ? __uint_as_float(r[8 * q + e]) * p.drop.scale : 0.f;
                dot += g * pf[e];
              }
            }
          }
        }
        red_a[part * 128 + r_local] = dot;
        epi_bar();
        dot = (red_a[r_local] + red_a[128 + r_local]) + (red_a[256 + r_local] + red_a[384 + r_local]);
        // ---- pass 2: dS = P * (dP - dot) * scale -> stage -> TMA store
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          const int c = (part + 4 * j) * 32;
          if (c < p.S) {
            if (lane == 0) bulk_wait_read<0>();
            __syncwarp();
            uint4 pr[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              pr[q] = (row_ok && c + 8 * q < p.S) ? *reinterpret_cast<const uint4*>(prow + c + 8 * q)
                                                  : make_uint4(0, 0, 0, 0);
            uint32_t r[32];
            tmem_ld32_nowait(t_row + c, r);
            tmem_wait_ld();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float pf[8], ds[8];
              unpack_bf16x8(pr[q], pf);
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                // (columns >= S: g = 0 by the keep mask, and the TMA store
                // clips them, so no per-element bounds test is needed)
                const float g = ((km[j] >> (8 * q + e)) & 1u)
                                    ? __uint_as_float(r[8 * q + e]) * p.drop.scale
                                    : 0.f;
                ds[e] = pf[e] * (g - dot) * p.ds_scale;
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
          half_release(j);
        }
      }
      if constexpr (NC != 512) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
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
