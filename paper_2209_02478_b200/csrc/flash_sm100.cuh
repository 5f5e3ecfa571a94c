// Flash attention for sm_100a (head dim 64): the S x S scores never leave the
// SM. SURVEY §8(f)-4 ("a fused flash-style attention that removes the S^2
// term; a(x) becomes linear in x"): the block saves q | k | v, ctx and one
// fp32 log-sum-exp per row instead of the materialised P / Pd of the
// reference model's quadratic activation term (proj/models/bert12.model c2).
//
// Forward, one CTA per 128-query tile (persistent):
//   warp 0   TMA producer: Q tile once, then K_j / V_j (128 keys) per block
//   warp 1   MMA issuer:   S_j = Q K_j^T into one of two 128-column TMEM
//            buffers; O_w += P_j[:, slice w] V_j[slice w] for the four 32-key
//            slices, each into its own 64-column TMEM accumulator
//   warps 2+ 16 softmax warps: warp (lane quarter q, key slice w) owns rows
//            32q..32q+31 x keys 32w..32w+31 of every block and keeps its own
//            running max / sum for them -- no cross-warp exchange per block.
//            Lazy rescaling: O_w is corrected only when the slice max grows
//            by more than 2^8. Dropout (Philox, same element index as the
//            materialised path: row * ld + key) applies to the P operand of
//            the P V MMA, not to the row sum.
//   Tile end: the four slices of a row are combined once (max / sum through
//   shared memory), O = sum_w O_w 2^(m_w - M) / L * 1/(1-p) -> ctx, and
//   lse = M + log2 L (log2 units of the scaled scores) is stored for the
//   backward.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "ptx_sm100.cuh"

namespace mimose_dev {

struct FlashParams {
  int S, nh, B;
  int ld;               // dropout element index pitch (round8(S)), as the materialised path
  float sc;             // score scale * log2(e): scores live in log2 units
  DropoutCfg drop;
  int causal;           // keys j > query i masked
  __nv_bfloat16* ctx;   // fwd out: [B*S][ctx_ld], head h at columns 64h
  long long ctx_ld;
  float* lse;           // fwd out / bwd in: [B*nh][S]
  // backward
  const __nv_bfloat16* dctx;  // [B*S][ctx_ld]
  const float* dvec;          // [B*nh][S] rowsum(dO o O)
  __nv_bfloat16* dqkv;        // [B*S][3 * ctx_ld]
  float ds_scale;             // score scale folded into dS (1/sqrt(64))
};

struct FlashFwdCfg {
  static constexpr int kEW = 16;
  static constexpr int kThreads = 64 + 32 * kEW;
  static constexpr int kQBytes = 128 * 64 * 2;
  static constexpr int kKBytes = 128 * 64 * 2;
  static constexpr int kKVBytes = 2 * kKBytes;  // K block + V block
  static constexpr int kStages = 3;
  static constexpr int kPBytes = 128 * 128 * 2;  // two 64-key swizzled sub-tiles
  static constexpr int kXchBytes = 2 * 2 * 4 * 128 * 4;  // [tile parity][m|l][slice][row]
  static constexpr int kSmemBytes =
      kQBytes + kStages * kKVBytes + 2 * kPBytes + kXchBytes + 1024 + 512;
};

__device__ __forceinline__ float fl_ex2(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ uint32_t fl_pack(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void fl_epi_bar() { asm volatile("bar.sync 1, 512;" ::: "memory"); }

__global__ void __launch_bounds__(FlashFwdCfg::kThreads, 1)
    flash_fwd_kernel(const __grid_constant__ CUtensorMap tmQ,
                     const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const FlashParams p) {
  using Cfg = FlashFwdCfg;
  constexpr int NS = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + Cfg::kQBytes;
  uint8_t* sP = sKV + NS * Cfg::kKVBytes;
  float* xch = reinterpret_cast<float*>(sP + 2 * Cfg::kPBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(xch) + Cfg::kXchBytes);
  uint64_t* empty = full + NS;
  uint64_t* qfull = empty + NS;
  uint64_t* qempty = qfull + 1;
  uint64_t* sfull = qempty + 1;   // [2] S buffers
  uint64_t* sempty = sfull + 2;   // [2]
  uint64_t* pfull = sempty + 2;   // [2 P buffers][4 slices]
  uint64_t* pvdone = pfull + 8;   // [2][4]
  uint64_t* ofull = pvdone + 8;
  uint64_t* oempty = ofull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(oempty + 1);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const int tiles_m = (p.S + 127) / 128;
  const int num_tiles = tiles_m * p.nh * p.B;
  auto nkb_of = [&](int qt) { return p.causal ? (qt + 1 < tiles_m ? qt + 1 : tiles_m) : tiles_m; };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(qfull, 1);
    mbar_init(qempty, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sfull[b], 1);
      mbar_init(&sempty[b], Cfg::kEW);
    }
    for (int i = 0; i < 8; ++i) {
      mbar_init(&pfull[i], 4);  // the four lane-quarter warps of a slice
      mbar_init(&pvdone[i], 1);
    }
    mbar_init(ofull, 1);
    mbar_init(oempty, Cfg::kEW);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int kv = 0, tc = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tc) {
        const int z = tile / tiles_m, qt = tile % tiles_m;
        const int h = z % p.nh, b = z / p.nh;
        mbar_wait(qempty, (tc & 1) ^ 1);
        mbar_arrive_expect_tx(qfull, Cfg::kQBytes);
        tma_load_4d(&tmQ, qfull, sQ, 0, qt * 128, h, b);
        const int nkb = nkb_of(qt);
        for (int j = 0; j < nkb; ++j, ++kv) {
          const int s = kv % NS;
          mbar_wait(&empty[s], ((kv / NS) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], Cfg::kKVBytes);
          uint8_t* kd = sKV + s * Cfg::kKVBytes;
          tma_load_4d(&tmK, &full[s], kd, 0, j * 128, h, b);
          tma_load_4d(&tmV, &full[s], kd + Cfg::kKBytes, 0, j * 128, h, b);
          tma_load_4d(&tmV, &full[s], kd + Cfg::kKBytes + 8192, 0, j * 128 + 64, h, b);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc_s = idesc_bf16_f32(128, 128, false, false);
    const uint32_t idesc_pv = idesc_bf16_f32(128, 64, false, true);
    int kv = 0, jb = 0, tc = 0;
    // O_w += P_b[:, 32w..32w+31] V[32w..32w+31, :] for block b (j-th of its tile)
    auto issue_pv = [&](int b, int j, int stage) {
      if (j == 0) {
        mbar_wait(oempty, (tc & 1) ^ 1);  // the previous tile's O has been read
        tc_fence_after();
      }
#pragma unroll 1
      for (int w = 0; w < 4; ++w) {
        mbar_wait(&pfull[(b & 1) * 4 + w], (b >> 1) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t pa =
              smem_u32(sP + (b & 1) * Cfg::kPBytes + (w >> 1) * 16384) + (w & 1) * 64;
          const uint32_t va = smem_u32(sKV + stage * Cfg::kKVBytes + Cfg::kKBytes +
                                       (w >> 1) * 8192) + (w & 1) * 4096;
#pragma unroll
          for (int kk = 0; kk < 2; ++kk)
            umma_bf16(tmem_base + 256 + 64 * w, smem_desc_sw128(pa + kk * 32, 16, 1024),
                      smem_desc_sw128(va + kk * 2048, 8192, 1024), idesc_pv,
                      (j > 0 || kk > 0) ? 1u : 0u);
          umma_commit(&pvdone[(b & 1) * 4 + w]);
        }
        __syncwarp();
      }
      if (lane == 0) umma_commit(&empty[stage]);
      __syncwarp();
    };
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tc) {
      const int nkb = nkb_of(tile % tiles_m);
      mbar_wait(qfull, tc & 1);
      tc_fence_after();
      int prev_stage = 0;
      for (int j = 0; j < nkb; ++j, ++kv, ++jb) {
        const int s = kv % NS;
        mbar_wait(&full[s], (kv / NS) & 1);
        mbar_wait(&sempty[jb & 1], ((jb >> 1) & 1) ^ 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t qa = smem_u32(sQ), ka = smem_u32(sKV + s * Cfg::kKVBytes);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16(tmem_base + (jb & 1) * 128, smem_desc_sw128(qa + kk * 32, 16, 1024),
                      smem_desc_sw128(ka + kk * 32, 16, 1024), idesc_s, kk != 0 ? 1u : 0u);
          umma_commit(&sfull[jb & 1]);
          if (j == nkb - 1) umma_commit(qempty);
        }
        __syncwarp();
        // the previous block's P V goes after this block's S, so the softmax
        // warps have S_j in hand while P_{j-1} V_{j-1} runs
        if (j > 0) issue_pv(jb - 1, j - 1, prev_stage);
        prev_stage = s;
      }
      issue_pv(jb - 1, nkb - 1, prev_stage);
      if (lane == 0) umma_commit(ofull);
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    const int ew = warp - 2;
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int w = ew >> 2;         // key slice of every block
    const int r = quarter * 32 + static_cast<int>(lane);
    const uint32_t lane_base = tmem_base + ((uint32_t)(quarter * 32) << 16);
    const uint32_t thr_hi = p.drop.threshold << 16;
    const float kNegInf = -__int_as_float(0x7f800000);
    int jb = 0, tc = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tc) {
      const int z = tile / tiles_m, qt = tile % tiles_m;
      const int h = z % p.nh, b = z / p.nh;
      const int nkb = nkb_of(qt);
      const int i = qt * 128 + r;
      const bool row_ok = i < p.S;
      const int64_t grow = (int64_t)z * p.S + (row_ok ? i : 0);
      float m_used = kNegInf, l = 0.f;
      for (int j = 0; j < nkb; ++j, ++jb) {
        const int sb = jb & 1;
        mbar_wait(&sfull[sb], (jb >> 1) & 1);
        tc_fence_after();
        uint32_t raw[32];
        tmem_ld32_nowait(lane_base + sb * 128 + 32 * w, raw);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[sb]);
        const int c0 = j * 128 + 32 * w;
        int lim = p.S - c0;  // valid keys of the slice: c0 + e < S (and <= i if causal)
        if (p.causal && i - c0 + 1 < lim) lim = i - c0 + 1;
        float s[32];
        float mb = kNegInf;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          s[e] = e < lim ? __uint_as_float(raw[e]) * p.sc : kNegInf;
          mb = fmaxf(mb, s[e]);
        }
        if (j == 0) {
          m_used = mb;
        } else {
          const bool need = mb > m_used + 8.f;
          if (__any_sync(0xffffffffu, need)) {
            const float mn = fmaxf(m_used, mb);
            const float alpha = mn == kNegInf ? 1.f : fl_ex2(m_used - mn);
            // O_w holds P V of the blocks so far: wait for the last one to land
            const int pb = jb - 1;
            mbar_wait(&pvdone[(pb & 1) * 4 + w], (pb >> 1) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int part = 0; part < 4; ++part) {
              float o[16];
              const uint32_t ta = lane_base + 256 + 64 * w + 16 * part;
              tmem_ld16(ta, o);
#pragma unroll
              for (int e = 0; e < 16; ++e) o[e] *= alpha;
              tmem_st16(ta, o);
            }
            tmem_wait_st();
            l *= alpha;
            m_used = mn;
          }
        }
        // this P buffer is free once the P V of two blocks ago has run
        mbar_wait(&pvdone[sb * 4 + w], ((jb >> 1) & 1) ^ 1);
        const float m_eff = m_used == kNegInf ? 0.f : m_used;
        uint32_t rnd[4][4];
        if (thr_hi != 0) {
          uint64_t grp[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) grp[q] = ((uint64_t)grow * p.ld + c0 + 8 * q) >> 3;
          philox_n<4>(p.drop.seed, p.drop.stream, grp, rnd);
        }
        float psum = 0.f;
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          float a0 = fl_ex2(s[e] - m_eff), a1 = fl_ex2(s[e + 1] - m_eff);
          psum += a0 + a1;
          if (thr_hi != 0) {
            if (!philox_keep_w(rnd[e >> 3], e & 7, thr_hi)) a0 = 0.f;
            if (!philox_keep_w(rnd[e >> 3], (e & 7) + 1, thr_hi)) a1 = 0.f;
          }
          pk[e >> 1] = fl_pack(a0, a1);
        }
        l += psum;
        const uint32_t rowa = smem_u32(sP + sb * Cfg::kPBytes + (w >> 1) * 16384) + r * 128;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          st_shared_v4(rowa + ((((w & 1) * 4 + c) ^ (r & 7)) << 4), pk[4 * c], pk[4 * c + 1],
                       pk[4 * c + 2], pk[4 * c + 3]);
        fence_async_shared();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[sb * 4 + w]);
      }
      // ---- tile end: combine the four slices of each row
      mbar_wait(ofull, tc & 1);
      tc_fence_after();
      float* xm = xch + (tc & 1) * 1024;  // [4 slices][128 rows]
      float* xl = xm + 512;
      xm[w * 128 + r] = m_used;
      xl[w * 128 + r] = l;
      fl_epi_bar();
      float M = kNegInf;
#pragma unroll
      for (int t = 0; t < 4; ++t) M = fmaxf(M, xm[t * 128 + r]);
      float f[4], L = 0.f;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float mt = xm[t * 128 + r];
        f[t] = mt == kNegInf ? 0.f : fl_ex2(mt - M);
        L += f[t] * xl[t * 128 + r];
      }
      const float inv = p.drop.scale / L;
      float acc[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) acc[e] = 0.f;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        float o[16];
        tmem_ld16(lane_base + 256 + 64 * t + 16 * w, o);
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[e] = fmaf(o[e], f[t], acc[e]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(oempty);
      if (row_ok) {
        uint4* dst = reinterpret_cast<uint4*>(p.ctx + ((int64_t)b * p.S + i) * p.ctx_ld + h * 64 +
                                              16 * w);
        dst[0] = make_uint4(fl_pack(acc[0] * inv, acc[1] * inv), fl_pack(acc[2] * inv, acc[3] * inv),
                            fl_pack(acc[4] * inv, acc[5] * inv), fl_pack(acc[6] * inv, acc[7] * inv));
        dst[1] = make_uint4(fl_pack(acc[8] * inv, acc[9] * inv), fl_pack(acc[10] * inv, acc[11] * inv),
                            fl_pack(acc[12] * inv, acc[13] * inv),
                            fl_pack(acc[14] * inv, acc[15] * inv));
        if (w == 0) p.lse[grow] = M + __log2f(L);
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
