// Flash attention backward, dK / dV kernel with TRANSPOSED scores (sm_100a).
//
// Work item = one 128-key block of one (sequence, head); inner loop over the
// 128-query blocks that see it. The scores are computed transposed, keys on
// the TMEM lanes:
//   S^T  = K Q_j^T      dP^T = V dO_j^T              (two 128 x 128 x 64 MMAs)
// so the score warps' outputs are already in the A-operand orientation of
//   dV  += Pd^T dO_j    dK  += dS^T Q_j              (M = keys, K = queries)
// and go straight back into tensor memory (tcgen05.st, bf16 pairs) where the
// accumulation MMAs read them as their A operand (tcgen05.mma A-from-TMEM):
// nothing is staged through shared memory and there is no per-block
// "staging buffer free" handshake (flash_bwd_kernel<0> wrote Pd / dS to
// shared memory and read them back as MN-major A operands - 64 KB of extra
// shared-memory traffic per block and a serialising barrier).
//
// Per-score algebra as flash_bwd_half (flash_sm100.cuh): with q the query
// (a TMEM column) and k the key (the lane),
//   P' = 2^(s sc - lse_s[q]),  f = keep(q, k) / (1 - p),
//   Pd = P' f / ds_scale,      dS = P' (dP f - D[q]),
// lse_s = lse - log2(ds_scale). lse / D of the block's 128 queries are staged
// in shared memory by the producer warp (padding queries get lse = +inf: P = 0).
// Dropout keep bits are stored query-major ([query][key / 32] words): each
// warp loads the 32 words of its 32 queries and transposes the 32 x 32 bit
// block across the warp (five shuffle rounds) into per-key words.
//
// Warps: 0 producer (TMA + lse / D staging), 1 MMA issuer, 2..17 score warps
// (TMEM lane quarter x 32-query slice). TMEM (512 columns): S^T double buffer
// [0, 256) - Pd^T / dS^T are written over the slice just read - dP^T [256,
// 384), dV [384, 448), dK [448, 512).
#pragma once

#include "flash_sm100.cuh"

namespace mimose_dev {

// 32 x 32 bit transpose across the warp: lane i holds row i on entry, column
// i on exit (bit r of lane i's result = bit i of row r).
__device__ __forceinline__ uint32_t warp_bit_transpose(uint32_t x, uint32_t lane) {
  constexpr uint32_t kMask[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    const int j = 16 >> t;
    const uint32_t m = kMask[t];
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
    x = (lane & j) ? ((x & ~m) | ((y >> j) & m)) : ((x & m) | ((y & m) << j));
  }
  return x;
}

// Ping-pong version: 64-query inner blocks alternate between two groups of
// eight score warps (block c -> group c & 1), and three 128-column TMEM
// regions (S^T | dP^T of one block each) rotate, so while one group turns
// block c's scores into Pd^T / dS^T the tensor pipe runs block c + 1's
// S^T / dP^T and block c - 1's accumulation: the tensor pipe, the MUFU pipe
// and the TMEM round trips of the two groups overlap instead of all sixteen
// warps stepping through one block at a time.
struct FlashBwdKv2Cfg {
  static constexpr int kThreads = 64 + 32 * 16;
  static constexpr int kKTile = 128 * 64 * 2;     // K or V of the item (128 keys)
  static constexpr int kQTile = 64 * 64 * 2;      // Q_j or dO_j (64 queries)
  static constexpr int kStages = 4;
  static constexpr int kStatBytes = 2 * 64 * 4;   // lse_s | D of the block's 64 queries
  static constexpr int kStageBytes = 2 * kQTile + 1024;  // + stats, 1024-aligned stride
  static constexpr int kSmemBytes = 2 * kKTile + kStages * kStageBytes + 1024 + 512;
};

template <bool DROP>
__global__ void __launch_bounds__(FlashBwdKv2Cfg::kThreads, 1)
    flash_bwd_kvt_kernel(const __grid_constant__ CUtensorMap tmQ,
                         const __grid_constant__ CUtensorMap tmK,
                         const __grid_constant__ CUtensorMap tmV,
                         const __grid_constant__ CUtensorMap tmO, const FlashParams p) {
  using Cfg = FlashBwdKv2Cfg;
  constexpr int NS = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sK = smem;
  uint8_t* sV = smem + Cfg::kKTile;
  uint8_t* sStage = smem + 2 * Cfg::kKTile;  // [NS] x (Q_j | dO_j | lse_s | D)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + NS * Cfg::kStageBytes);
  uint64_t* full = bars;             // [NS]
  uint64_t* empty = full + NS;       // [NS] (the block's accumulation MMAs done)
  uint64_t* fixfull = empty + NS;
  uint64_t* fixempty = fixfull + 1;
  uint64_t* sfull = fixempty + 1;    // [3] region r's S^T / dP^T landed
  uint64_t* rfree = sfull + 3;       // [3] region r's Pd^T / dS^T consumed
  uint64_t* pfull = rfree + 3;       // [2] group g wrote its block's Pd^T / dS^T
  uint64_t* accfull = pfull + 2;
  uint64_t* accempty = accfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 1);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const int nkb = (p.S + 127) / 128;  // 128-key items
  const int nqb = (p.S + 63) / 64;    // 64-query inner blocks
  const int num_items = nkb * p.nh * p.B;
  constexpr uint32_t kColDV = 384, kColDK = 448;
  auto decode = [&](int item, int& z, int& kb) {
    if (p.causal) {
      const int nz = p.nh * p.B;
      kb = item / nz;
      z = item % nz;
    } else {
      z = item / nkb;
      kb = item % nkb;
    }
  };
  auto lo_of = [&](int kb) { return p.causal ? 2 * kb : 0; };  // queries >= keys

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    tma_prefetch(&tmO);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(fixfull, 1);
    mbar_init(fixempty, 1);
    for (int r = 0; r < 3; ++r) {
      mbar_init(&sfull[r], 1);
      mbar_init(&rfree[r], 1);
    }
    mbar_init(&pfull[0], 8);
    mbar_init(&pfull[1], 8);
    mbar_init(accfull, 1);
    mbar_init(accempty, 16);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();
  const float kInf = __int_as_float(0x7f800000);

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    const float lse_shift = __log2f(p.ds_scale);
    int st = 0, ic = 0;
    for (int item = blockIdx.x; item < num_items; item += gridDim.x, ++ic) {
      int z, kb;
      decode(item, z, kb);
      const int h = z % p.nh, b = z / p.nh;
      if (lane == 0) {
        mbar_wait(fixempty, (ic & 1) ^ 1);
        mbar_arrive_expect_tx(fixfull, 2 * Cfg::kKTile);
        tma_load_4d(&tmK, fixfull, sK, 0, kb * 128, h, b);
        tma_load_4d(&tmV, fixfull, sV, 0, kb * 128, h, b);
      }
      for (int j = lo_of(kb); j < nqb; ++j, ++st) {
        const int s = st % NS;
        mbar_wait(&empty[s], ((st / NS) & 1) ^ 1);
        uint8_t* d = sStage + s * Cfg::kStageBytes;
        float* sl = reinterpret_cast<float*>(d + 2 * Cfg::kQTile);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int q = j * 64 + 2 * static_cast<int>(lane) + e;
          const bool ok = q < p.S;
          const int64_t g = (int64_t)z * p.S + (ok ? q : 0);
          sl[2 * lane + e] = ok ? p.lse[g] - lse_shift : kInf;
          sl[64 + 2 * lane + e] = ok ? p.dvec[g] : 0.f;
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_expect_tx(&full[s], 2 * Cfg::kQTile);
          tma_load_4d(&tmQ, &full[s], d, 0, j * 64, h, b);
          tma_load_4d(&tmO, &full[s], d + Cfg::kQTile, 0, j * 64, h, b);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc_s = idesc_bf16_f32(128, 64, false, false);
    const uint32_t idesc_acc = idesc_bf16_f32(128, 64, false, true);
    int st = 0, ic = 0, c = 0;  // c: global block counter (region c % 3, group c & 1)
    auto issue_acc = [&](int s, int cc, bool first) {
      const uint32_t dO = smem_u32(sStage + s * Cfg::kStageBytes + Cfg::kQTile);
      const uint32_t q = smem_u32(sStage + s * Cfg::kStageBytes);
      const uint32_t ta = tmem_base + (cc % 3) * 128;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {  // K = 64 queries, 16 per MMA
        const uint32_t col = 32 * (kk >> 1) + 8 * (kk & 1);
        umma_bf16_ts(tmem_base + kColDV, ta + col, smem_desc_sw128(dO + kk * 2048, 8192, 1024),
                     idesc_acc, (first && kk == 0) ? 0u : 1u);
        umma_bf16_ts(tmem_base + kColDK, ta + col + 16, smem_desc_sw128(q + kk * 2048, 8192, 1024),
                     idesc_acc, (first && kk == 0) ? 0u : 1u);
      }
      umma_commit(&rfree[cc % 3]);
      umma_commit(&empty[s]);
    };
    for (int item = blockIdx.x; item < num_items; item += gridDim.x, ++ic) {
      int z_, kb_;
      decode(item, z_, kb_);
      const int lo = lo_of(kb_);
      mbar_wait(fixfull, ic & 1);
      tc_fence_after();
      int prev_s = 0;
      for (int j = lo; j < nqb; ++j, ++st, ++c) {
        const int s = st % NS, r = c % 3;
        mbar_wait(&full[s], (st / NS) & 1);
        mbar_wait(&rfree[r], ((c / 3) & 1) ^ 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t k = smem_u32(sK), v = smem_u32(sV);
          const uint32_t q = smem_u32(sStage + s * Cfg::kStageBytes);
          const uint32_t dO = q + Cfg::kQTile;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // S^T = K Q_j^T (128 keys x 64 queries)
            umma_bf16(tmem_base + r * 128, smem_desc_sw128(k + kk * 32, 16, 1024),
                      smem_desc_sw128(q + kk * 32, 16, 1024), idesc_s, kk != 0 ? 1u : 0u);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // dP^T = V dO_j^T
            umma_bf16(tmem_base + r * 128 + 64, smem_desc_sw128(v + kk * 32, 16, 1024),
                      smem_desc_sw128(dO + kk * 32, 16, 1024), idesc_s, kk != 0 ? 1u : 0u);
          umma_commit(&sfull[r]);
          if (j == nqb - 1) umma_commit(fixempty);
        }
        __syncwarp();
        if (j > lo) {
          const int pc = c - 1;
          mbar_wait(&pfull[pc & 1], (pc >> 1) & 1);
          tc_fence_after();
          if (lane == 0) issue_acc(prev_s, pc, j - 1 == lo);
          __syncwarp();
        } else {
          mbar_wait(accempty, (ic & 1) ^ 1);
          tc_fence_after();
        }
        prev_s = s;
      }
      const int pc = c - 1;
      mbar_wait(&pfull[pc & 1], (pc >> 1) & 1);
      tc_fence_after();
      if (lane == 0) {
        issue_acc(prev_s, pc, nqb - 1 == lo);
        umma_commit(accfull);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ score warps
    const int ew = warp - 2;
    const int grp = ew >> 3;         // group: blocks c with (c & 1) == grp
    const int quarter = warp & 3;    // TMEM lane quarter: keys 32 quarter .. +31
    const int w = (ew >> 2) & 1;     // query slice: 32 w .. 32 w + 31 of the 64
    const uint32_t lane_base = tmem_base + ((uint32_t)(quarter * 32) << 16);
    const float fk = DROP ? p.drop.scale : 1.f, fkd = fk / p.ds_scale;
    const float2 sc2 = make_float2(p.sc, p.sc);
    int st = 0, ic = 0, c = 0;
    for (int item = blockIdx.x; item < num_items; item += gridDim.x, ++ic) {
      int z, kb;
      decode(item, z, kb);
      const int h = z % p.nh, b = z / p.nh;
      const int key = kb * 128 + quarter * 32 + static_cast<int>(lane);
      for (int j = lo_of(kb); j < nqb; ++j, ++st, ++c) {
        if ((c & 1) != grp) continue;
        const int s = st % NS, r = c % 3;
        const int q0 = j * 64 + 32 * w;
        uint32_t kw = 0xffffffffu;
        if (DROP) {
          const int qi = q0 + static_cast<int>(lane);
          const int chunk = kb * 4 + quarter;
          const uint32_t row = (qi < p.S && chunk < p.mw)
                                   ? p.mask[((int64_t)z * p.S + qi) * p.mw + chunk]
                                   : 0u;
          kw = warp_bit_transpose(row, lane);
        }
        int lim = 0;
        if (p.causal) lim = key - q0;
        const bool all_full = !p.causal || __all_sync(0xffffffffu, lim <= 0);
        const bool all_dead = p.causal && __all_sync(0xffffffffu, lim >= 32);
        mbar_wait(&full[s], (st / NS) & 1);
        const uint32_t sl = smem_u32(sStage + s * Cfg::kStageBytes + 2 * Cfg::kQTile) + 4 * 32 * w;
        mbar_wait(&sfull[r], (c / 3) & 1);
        tc_fence_after();
        uint32_t dr[16], sr[16];
        uint32_t pk_pd[16], pk_ds[16];
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          tmem_ld16u_nowait(lane_base + r * 128 + 64 + 32 * w + 16 * half, dr);
          tmem_ld16u_nowait(lane_base + r * 128 + 32 * w + 16 * half, sr);
          tmem_wait_ld();
          if (all_dead) {
#pragma unroll
            for (int e = 0; e < 8; ++e) pk_pd[8 * half + e] = pk_ds[8 * half + e] = 0u;
            continue;
          }
#pragma unroll
          for (int e4 = 16 * half; e4 < 16 * half + 16; e4 += 4) {
            const uint4 lsu = ld_shared_v4(sl + 4 * e4);
            const uint4 dvu = ld_shared_v4(sl + 4 * 64 + 4 * e4);
            const float lsv[4] = {__uint_as_float(lsu.x), __uint_as_float(lsu.y),
                                  __uint_as_float(lsu.z), __uint_as_float(lsu.w)};
            const float dvv[4] = {__uint_as_float(dvu.x), __uint_as_float(dvu.y),
                                  __uint_as_float(dvu.z), __uint_as_float(dvu.w)};
#pragma unroll
            for (int e2 = 0; e2 < 4; e2 += 2) {
              const int e = e4 + e2;
              const float2 x = make_float2(__uint_as_float(sr[e - 16 * half]),
                                           __uint_as_float(sr[e + 1 - 16 * half]));
              const float2 t = __ffma2_rn(x, sc2, make_float2(-lsv[e2], -lsv[e2 + 1]));
              float2 P = make_float2(fl_ex2(t.x), fl_ex2(t.y));
              if (!all_full) {
                if (e < lim) P.x = 0.f;
                if (e + 1 < lim) P.y = 0.f;
              }
              float2 f = make_float2(fk, fk), fd = make_float2(fkd, fkd);
              if (DROP) {
                if (!((kw >> e) & 1u)) f.x = fd.x = 0.f;
                if (!((kw >> (e + 1)) & 1u)) f.y = fd.y = 0.f;
              }
              const float2 dp = make_float2(__uint_as_float(dr[e - 16 * half]),
                                            __uint_as_float(dr[e + 1 - 16 * half]));
              const float2 dS =
                  __fmul2_rn(P, __ffma2_rn(dp, f, make_float2(-dvv[e2], -dvv[e2 + 1])));
              const float2 Pd = __fmul2_rn(P, fd);
              pk_pd[e >> 1] = fl_pack(Pd.x, Pd.y);
              pk_ds[e >> 1] = fl_pack(dS.x, dS.y);
            }
          }
        }
        // Pd^T over the first 16 columns of this warp's S^T slice, dS^T over the next 16
        tmem_st16u(lane_base + r * 128 + 32 * w, pk_pd);
        tmem_st16u(lane_base + r * 128 + 32 * w + 16, pk_ds);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[grp]);
      }
      // ---- item end: dV | dK rows (all sixteen warps: quarter x 32-column slice)
      mbar_wait(accfull, ic & 1);
      tc_fence_after();
      const int cs = (ew >> 2) & 3;  // 0, 1: dV halves; 2, 3: dK halves
      uint32_t o[32];
      tmem_ld32_nowait(lane_base + kColDV + 32 * cs, o);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(accempty);
      if (key < p.S) {
        const long long H = p.ctx_ld;
        __nv_bfloat16* dst = p.dqkv + ((long long)b * p.S + key) * 3 * H + (cs < 2 ? 2 * H : H) +
                             h * 64 + 32 * (cs & 1);
        uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          d4[q] = make_uint4(fl_pack(__uint_as_float(o[8 * q]), __uint_as_float(o[8 * q + 1])),
                             fl_pack(__uint_as_float(o[8 * q + 2]), __uint_as_float(o[8 * q + 3])),
                             fl_pack(__uint_as_float(o[8 * q + 4]), __uint_as_float(o[8 * q + 5])),
                             fl_pack(__uint_as_float(o[8 * q + 6]), __uint_as_float(o[8 * q + 7])));
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace mimose_dev
