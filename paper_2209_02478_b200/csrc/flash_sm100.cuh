// Flash attention for sm_100a (head dim 64): the S x S scores never leave the
// SM. SURVEY §8(f)-4 ("a fused flash-style attention that removes the S^2
// term; a(x) becomes linear in x"): the block saves q | k | v, ctx and one
// fp32 log-sum-exp per row instead of the materialised P / Pd of the
// reference model's quadratic activation term (proj/models/bert12.model c2).
//
// Forward, one CTA per 128-query tile (persistent):
//   warp 0   TMA producer: Q tile once, then K_j / V_j (128 keys) per block
//   warp 1   MMA issuer:   S_j = Q K_j^T into the TMEM S buffer, issued as
//            soon as the softmax warps have loaded S_{j-1} into registers;
//            O_w += P_j[:, slice w] V_j[slice w] for the 32-key slices, each
//            into its own 64-column TMEM accumulator, P_j read from one of two
//            TMEM P buffers (so the next S never waits for a P V to finish)
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
//   backward -- deferred until after the next tile's first block, so the
//   wait for the tile's last P V MMA overlaps softmax work.
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
  uint32_t* mask;       // fwd / bwd in (dropout only): keep bits [B*nh*S][mw],
  int mw;               //   bit e of word (row, k) = key 32k + e kept
  // backward
  const __nv_bfloat16* dctx;  // [B*S][ctx_ld]
  float* dvec;                // [B*nh][S] rowsum(dO o O) (dQ kernel writes, dK/dV reads)
  __nv_bfloat16* dqkv;        // [B*S][3 * ctx_ld]
  float ds_scale;             // score scale folded into dS (1/sqrt(64))
};

// KB keys per block: 128 (one CTA per SM, 16 softmax warps = 4 lane quarters
// x 4 key slices, all 512 TMEM columns) or 64 (two CTAs per SM, 8 softmax
// warps each, 256 TMEM columns: two independent pipelines per SM hide each
// other's MMA / barrier latencies)
template <int KB>
struct FlashFwdCfg {
  static constexpr int kNSL = KB / 32;             // 32-key slices per block
  static constexpr int kEW = 4 * kNSL;             // softmax warps
  static constexpr int kThreads = 64 + 32 * kEW;
  static constexpr int kMinBlocks = KB == 64 ? 2 : 1;
  static constexpr int kQBytes = 128 * 64 * 2;
  static constexpr int kKBytes = KB * 64 * 2;
  static constexpr int kKVBytes = 2 * kKBytes;     // K block + V block
  static constexpr int kStages = 3;
  static constexpr int kXchBytes = 2 * 2 * kNSL * 128 * 4;  // [tile parity][m|l][slice][row]
  static constexpr int kTmemCols = 4 * KB;         // S (KB) + 2 P buffers (KB / 2) + kNSL O slices (64)
  static constexpr int kOCols = 64 / kNSL;         // output columns per warp in the combine
  // two Q buffers: the next tile's Q lands while this tile runs, so its first
  // Q K^T is issued before this tile's last P V (no tile-boundary bubble)
  static constexpr int kSmemBytes =
      2 * kQBytes + kStages * kKVBytes + kXchBytes + 1024 + 512;
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

// named barrier `id` (1..15) over N threads
template <int N>
__device__ __forceinline__ void fl_bar(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(N) : "memory");
}

// Store one 64-byte segment per lane (lane = a row; c = its four 16-byte
// chunks, dst = the row's segment, ok = the row exists) with coalesced warp
// stores: a 4x4 chunk transpose inside each group of four lanes (two
// shfl_xor rounds), after which store k has lane 4g + i write chunk i of row
// 4g + k - 8 whole 64-B segments per instruction instead of 32 scattered
// 16-B pieces (the row-per-lane form costs one L2 request per lane and
// stalled the attention epilogues for thousands of cycles).
__device__ __forceinline__ void fl_store_rows64(uint4 (&c)[4], void* dst, bool ok) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t m[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    m[j][0] = c[j].x; m[j][1] = c[j].y; m[j][2] = c[j].z; m[j][3] = c[j].w;
  }
  // round 1 (lanes i, i ^ 2): swap the off-diagonal 2x2 blocks
  const bool a = (lane >> 1) & 1;
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const uint32_t send = a ? m[k][w] : m[2 + k][w];
      const uint32_t got = __shfl_xor_sync(0xffffffffu, send, 2);
      if (a) m[k][w] = got;
      else m[2 + k][w] = got;
    }
  // round 2 (lanes i, i ^ 1): swap inside the 2x2 blocks
  const bool b = lane & 1;
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const uint32_t send = b ? m[2 * k][w] : m[2 * k + 1][w];
      const uint32_t got = __shfl_xor_sync(0xffffffffu, send, 1);
      if (b) m[2 * k][w] = got;
      else m[2 * k + 1][w] = got;
    }
  const uint64_t mine = reinterpret_cast<uint64_t>(dst);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int src = static_cast<int>(lane & ~3u) + k;
    const uint64_t row = __shfl_sync(0xffffffffu, mine, src);
    const bool rok = __shfl_sync(0xffffffffu, ok, src);
    if (rok)
      *reinterpret_cast<uint4*>(row + 16 * (lane & 3)) = make_uint4(m[k][0], m[k][1], m[k][2], m[k][3]);
  }
}

// Pipeline trace (build with -DMIMOSE_FLASH_TRACE): CTA 0 stamps SM clocks.
#ifdef MIMOSE_FLASH_TRACE
__device__ unsigned long long g_flash_trace[4096];
__device__ __forceinline__ unsigned long long fl_clk() {
  unsigned long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}
#define FT(i, v) if (blockIdx.x == 0 && (i) < 4096) g_flash_trace[i] = (v)
#define FT_CLK() fl_clk()
#else
#define FT(i, v)
#define FT_CLK() 0ull
#endif

// Dropout keep bits of the attention probabilities, one uint32 per (row, 32
// keys): bit e of word (row, k) keeps key 32k + e. Philox4x32-10 at the
// materialised path's element index row * ld + key (one call per 8 keys,
// 16-bit halves against the threshold: the same decisions as dropout_mask8).
// The bits depend only on (seed, stream, shape), so this runs at full
// occupancy ahead of the forward, which then tests one bit per score.
__global__ void flash_keep_mask_kernel(uint64_t seed, uint64_t stream, uint32_t threshold,
                                       uint32_t rows, int S, int ld, int mw, int causal,
                                       uint32_t* __restrict__ mask) {
  // 32-bit index math (the host guarantees rows * mw < 2^32): a 64-bit
  // division per word cost as many instructions as one of its Philox calls
  const uint32_t n = rows * (uint32_t)mw;
  const uint32_t thr_hi = threshold << 16;
  const uint32_t umw = (uint32_t)mw, uS = (uint32_t)S;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const uint32_t row = t / umw;
    const uint32_t k = t - row * umw;
    if (causal && 32 * k > row % uS) continue;  // all keys above the diagonal: never read
    // ld % 8 == 0: the word's four Philox groups are consecutive
    const uint64_t g0 = ((uint64_t)row * (uint32_t)ld + 32 * k) >> 3;
    uint64_t grp[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) grp[q] = g0 + q;
    uint32_t rnd[4][4];
    philox_n<4>(seed, stream, grp, rnd);
    uint32_t kw = 0;
#pragma unroll
    for (int e = 0; e < 32; ++e) kw |= (philox_keep_w(rnd[e >> 3], e & 7, thr_hi) ? 1u : 0u) << e;
    mask[t] = kw;
  }
}

// DROP: dropout on (keep bits read and applied); off = no per-score mask work
template <int KB, bool DROP>
__global__ void __launch_bounds__(FlashFwdCfg<KB>::kThreads, FlashFwdCfg<KB>::kMinBlocks)
    flash_fwd_kernel(const __grid_constant__ CUtensorMap tmQ,
                     const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const FlashParams p) {
  using Cfg = FlashFwdCfg<KB>;
  constexpr int NS = Cfg::kStages;
  constexpr int NSL = Cfg::kNSL;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;  // [2] Q buffers (tile parity)
  uint8_t* sKV = smem + 2 * Cfg::kQBytes;
  float* xch = reinterpret_cast<float*>(sKV + NS * Cfg::kKVBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(xch) + Cfg::kXchBytes);
  uint64_t* empty = full + NS;
  uint64_t* qfull = empty + NS;   // [2]
  uint64_t* qempty = qfull + 2;   // [2]
  // TMEM: one S buffer [0, KB) released as soon as the softmax warps have
  // loaded it (so S_{j+1} runs while they compute block j), two P buffers
  // [KB, 2 KB) (bf16 pairs, KB / 2 columns each) released by the P V commit,
  // the NSL per-slice O accumulators [2 KB, 2 KB + 64 NSL)
  uint64_t* sfull = qempty + 2;   // S landed
  uint64_t* sfree = sfull + 1;    // S loaded by every softmax warp
  uint64_t* pfull = sfree + 1;    // [2 P buffers][NSL slices]
  uint64_t* pempty = pfull + 2 * NSL;  // [2] P buffer read by its P V MMAs
  uint64_t* ofull = pempty + 2;
  uint64_t* oempty = ofull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(oempty + 1);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const int tiles_m = (p.S + 127) / 128;
  const int tiles_k = (p.S + KB - 1) / KB;
  const int num_tiles = tiles_m * p.nh * p.B;
  // key blocks of query tile qt (causal: up to the tile's last row)
  auto nkb_of = [&](int qt) {
    const int c = (qt + 1) * (128 / KB);
    return p.causal ? (c < tiles_k ? c : tiles_k) : tiles_k;
  };
  // tile -> (head z, query tile qt). Causal: longest tiles first, heads
  // fastest, so the static round-robin over CTAs stays balanced (with
  // z-major order and 148 % tiles_m == 0 a CTA would always get the same qt)
  auto decode = [&](int tile, int& z, int& qt) {
    if (p.causal) {
      const int nz = p.nh * p.B;
      qt = tiles_m - 1 - tile / nz;
      z = tile % nz;
    } else {
      z = tile / tiles_m;
      qt = tile % tiles_m;
    }
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&qfull[b], 1);
      mbar_init(&qempty[b], 1);
    }
    mbar_init(sfull, 1);
    mbar_init(sfree, Cfg::kEW);
    for (int i = 0; i < 2 * NSL; ++i) mbar_init(&pfull[i], 4);  // the slice's four lane-quarter warps
    for (int b = 0; b < 2; ++b) mbar_init(&pempty[b], 1);
    mbar_init(ofull, 1);
    mbar_init(oempty, Cfg::kEW);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::kTmemCols);
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
        int z, qt;
        decode(tile, z, qt);
        const int h = z % p.nh, b = z / p.nh;
        const int qb = tc & 1;
        mbar_wait(&qempty[qb], ((tc >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&qfull[qb], Cfg::kQBytes);
        tma_load_4d(&tmQ, &qfull[qb], sQ + qb * Cfg::kQBytes, 0, qt * 128, h, b);
        const int nkb = nkb_of(qt);
        for (int j = 0; j < nkb; ++j, ++kv) {
          const int s = kv % NS;
          mbar_wait(&empty[s], ((kv / NS) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], Cfg::kKVBytes);
          uint8_t* kd = sKV + s * Cfg::kKVBytes;
          tma_load_4d(&tmK, &full[s], kd, 0, j * KB, h, b);
#pragma unroll
          for (int v = 0; v < KB / 64; ++v)
            tma_load_4d(&tmV, &full[s], kd + Cfg::kKBytes + v * 8192, 0, j * KB + 64 * v, h, b);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc_s = idesc_bf16_f32(128, KB, false, false);
    const uint32_t idesc_pv = idesc_bf16_f32(128, 64, false, true);
    int kv = 0, jb = 0, tc = 0;
    // Warp-collective issue (umma_*_w: one lane elected inside the asm) with
    // descriptors as base + offset: the SWIZZLE_128B descriptor's start field
    // is addr >> 4, so a tile offset is added to it directly.
    const uint64_t qdesc = smem_desc_sw128(smem_u32(sQ), 16, 1024);
    const uint64_t kdesc = smem_desc_sw128(smem_u32(sKV), 16, 1024);                // K, stage 0
    const uint64_t vdesc = smem_desc_sw128(smem_u32(sKV + Cfg::kKBytes), 8192, 1024);  // V, stage 0
    // O_w += P_b[:, 32w..32w+31] V[32w..32w+31, :] for block b (j-th of tile
    // number btc)
    auto issue_pv = [&](int b, int j, int stage, int btc) {
      if (lane == 0 && b < 256) FT(b * 4 + 1, FT_CLK());
      if (j == 0) {
        mbar_wait(oempty, (btc & 1) ^ 1);  // the previous tile's O has been read
        tc_fence_after();
      }
#pragma unroll
      for (int w = 0; w < NSL; ++w) {
        mbar_wait(&pfull[(b & 1) * NSL + w], (b >> 1) & 1);
        tc_fence_after();
        // A = P_b[:, slice w] from TMEM (bf16 pairs, 16 columns of P buffer
        // b & 1), B = V rows of the slice (MN-major)
        const uint32_t pa = tmem_base + KB + (b & 1) * (KB / 2) + 16 * w;
        const uint64_t vd =
            vdesc + (uint64_t)((stage * Cfg::kKVBytes + (w >> 1) * 8192 + (w & 1) * 4096) >> 4);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk)
          umma_bf16_ts_w(tmem_base + 2 * KB + 64 * w, pa + 8 * kk, vd + (uint64_t)(kk * 2048 >> 4),
                         idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
      }
      umma_commit_w(&pempty[b & 1]);
      umma_commit_w(&empty[stage]);
      if (lane == 0 && b < 256) FT(b * 4 + 2, FT_CLK());
    };
    // One flat block sequence across tiles: block g's Q K^T goes in before
    // block g - 1's P V, also when g opens a new tile (its Q is already in the
    // other buffer), so the softmax warps find S ready at every tile boundary.
    bool have_prev = false, prev_last = false;
    int prev_b = 0, prev_j = 0, prev_stage = 0, prev_tc = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tc) {
      int z_, qt_;
      decode(tile, z_, qt_);
      const int nkb = nkb_of(qt_);
      const int qb = tc & 1;
      mbar_wait(&qfull[qb], (tc >> 1) & 1);
      tc_fence_after();
      const uint64_t qd = qdesc + (uint64_t)((qb * Cfg::kQBytes) >> 4);
      for (int j = 0; j < nkb; ++j, ++kv, ++jb) {
        const int s = kv % NS;
        mbar_wait(&full[s], (kv / NS) & 1);
        mbar_wait(sfree, (jb & 1) ^ 1);  // S_{jb-1} loaded by the softmax warps
        tc_fence_after();
        if (lane == 0 && jb < 256) FT(jb * 4 + 0, FT_CLK());
        const uint64_t kd = kdesc + (uint64_t)((s * Cfg::kKVBytes) >> 4);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16_w(tmem_base, qd + (uint64_t)(kk * 2), kd + (uint64_t)(kk * 2), idesc_s,
                      kk != 0 ? 1u : 0u);
        umma_commit_w(sfull);
        if (j == nkb - 1) umma_commit_w(&qempty[qb]);
        // the previous block's P V goes after this block's S, so the softmax
        // warps have S_j in hand while P_{j-1} V_{j-1} runs
        if (have_prev) {
          issue_pv(prev_b, prev_j, prev_stage, prev_tc);
          if (prev_last) umma_commit_w(ofull);
        }
        have_prev = true;
        prev_b = jb; prev_j = j; prev_stage = s; prev_tc = tc; prev_last = j == nkb - 1;
      }
    }
    if (have_prev) {
      issue_pv(prev_b, prev_j, prev_stage, prev_tc);
      umma_commit_w(ofull);
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    const int ew = warp - 2;
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int w = ew >> 2;         // key slice of every block
    const int r = quarter * 32 + static_cast<int>(lane);
    const uint32_t lane_base = tmem_base + ((uint32_t)(quarter * 32) << 16);
    const float kNegInf = -__int_as_float(0x7f800000);
    int jb = 0, tc = 0;
    // Tile end, software-pipelined: a tile's four slices are combined after
    // the NEXT tile's first block, so the wait for its last P V overlaps work
    bool pend = false, pend_ok = false;
    int pend_tc = 0;
    int64_t pend_ctx = 0, pend_grow = 0;
    auto finish = [&]() {
      mbar_wait(ofull, pend_tc & 1);
      tc_fence_after();
      // the quarter's NSL warps (the only writers of these rows' slice
      // statistics) have stored them: one named barrier per lane quarter
      fl_bar<32 * NSL>(1 + quarter);
      const float* xm = xch + (pend_tc & 1) * (2 * NSL * 128);
      const float* xl = xm + NSL * 128;
      float M = kNegInf;
#pragma unroll
      for (int t = 0; t < NSL; ++t) M = fmaxf(M, xm[t * 128 + r]);
      float f[NSL], L = 0.f;
#pragma unroll
      for (int t = 0; t < NSL; ++t) {
        const float mt = xm[t * 128 + r];
        f[t] = mt == kNegInf ? 0.f : fl_ex2(mt - M);
        L += f[t] * xl[t * 128 + r];
      }
      const float inv = p.drop.scale / L;
      constexpr int OC = Cfg::kOCols;  // this warp's output columns [OC w, OC w + OC)
      float acc[OC];
#pragma unroll
      for (int e = 0; e < OC; ++e) acc[e] = 0.f;
#pragma unroll
      for (int t = 0; t < NSL; ++t) {
#pragma unroll
        for (int q = 0; q < OC / 16; ++q) {
          uint32_t o[16];
          tmem_ld16u_nowait(lane_base + 2 * KB + 64 * t + OC * w + 16 * q, o);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) acc[16 * q + e] = fmaf(__uint_as_float(o[e]), f[t], acc[16 * q + e]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(oempty);
      if constexpr (OC == 32) {
        uint4 ch[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          ch[q] = make_uint4(fl_pack(acc[8 * q] * inv, acc[8 * q + 1] * inv),
                             fl_pack(acc[8 * q + 2] * inv, acc[8 * q + 3] * inv),
                             fl_pack(acc[8 * q + 4] * inv, acc[8 * q + 5] * inv),
                             fl_pack(acc[8 * q + 6] * inv, acc[8 * q + 7] * inv));
        fl_store_rows64(ch, p.ctx + pend_ctx, pend_ok);
      } else if (pend_ok) {
        uint4* dst = reinterpret_cast<uint4*>(p.ctx + pend_ctx);
#pragma unroll
        for (int q = 0; q < OC / 8; ++q)
          dst[q] = make_uint4(fl_pack(acc[8 * q] * inv, acc[8 * q + 1] * inv),
                              fl_pack(acc[8 * q + 2] * inv, acc[8 * q + 3] * inv),
                              fl_pack(acc[8 * q + 4] * inv, acc[8 * q + 5] * inv),
                              fl_pack(acc[8 * q + 6] * inv, acc[8 * q + 7] * inv));
      }
      if (pend_ok && w == 0) p.lse[pend_grow] = M + __log2f(L);
      pend = false;
    };
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tc) {
      int z, qt;
      decode(tile, z, qt);
      const int h = z % p.nh, b = z / p.nh;
      const int nkb = nkb_of(qt);
      const int i = qt * 128 + r;
      const bool row_ok = i < p.S;
      const int64_t grow = (int64_t)z * p.S + (row_ok ? i : 0);
      const bool warp_dead = qt * 128 + quarter * 32 >= p.S;  // all 32 rows past the end
      float m_used = kNegInf, l = 0.f;
      for (int j = 0; j < nkb; ++j, ++jb) {
        const int sb = jb & 1;
        const bool trw = lane == 0 && (ew == 0 || ew == Cfg::kEW - 1) && jb < 128;
        [[maybe_unused]] const int tro = 1024 + jb * 8 + (ew == Cfg::kEW - 1 ? 4 : 0);
        // keep bits first: the load overlaps the wait for S
        const int c0 = j * KB + 32 * w;
        int lim = p.S - c0;  // valid keys of the slice: c0 + e < S (and <= i if causal)
        if (p.causal && i - c0 + 1 < lim) lim = i - c0 + 1;
        if (warp_dead) lim = 0;
        const uint32_t kw = (DROP && lim > 0) ? p.mask[grow * p.mw + (c0 >> 5)] : 0u;
        if (trw) FT(tro + 0, FT_CLK());
        mbar_wait(sfull, jb & 1);
        tc_fence_after();
        uint32_t raw[32];
        tmem_ld32_nowait(lane_base + 32 * w, raw);
        tmem_wait_ld();
        // S is in registers: the buffer is free for the next block's Q K^T
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(sfree);
        if (trw) FT(tro + 1, FT_CLK());
        // warp-uniform paths: every key valid (no per-score test) / none valid
        // (past the sequence end or above the diagonal: P = 0, no Philox)
        const bool all_full = __all_sync(0xffffffffu, lim >= 32);
        const bool all_dead = __all_sync(0xffffffffu, lim <= 0);
        float x[32];
        // four independent max chains (a single 32-deep chain serialises on
        // the FMNMX latency)
        float mr[4] = {kNegInf, kNegInf, kNegInf, kNegInf};
        if (all_full) {
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            x[e] = __uint_as_float(raw[e]);
            mr[e & 3] = fmaxf(mr[e & 3], x[e]);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            x[e] = e < lim ? __uint_as_float(raw[e]) : kNegInf;
            mr[e & 3] = fmaxf(mr[e & 3], x[e]);
          }
        }
        const float mraw = fmaxf(fmaxf(mr[0], mr[1]), fmaxf(mr[2], mr[3]));
        const float mb = mraw * p.sc;
        if (j == 0) {
          m_used = mb;
        } else {
          const bool need = mb > m_used + 8.f;
          if (__any_sync(0xffffffffu, need)) {
            const float mn = fmaxf(m_used, mb);
            const float alpha = mn == kNegInf ? 1.f : fl_ex2(m_used - mn);
            // O_w holds P V of the blocks so far: wait for the last one to land
            const int pb = jb - 1;
            mbar_wait(&pempty[pb & 1], (pb >> 1) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int part = 0; part < 4; ++part) {
              float o[16];
              const uint32_t ta = lane_base + 2 * KB + 64 * w + 16 * part;
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
        const float m_eff = m_used == kNegInf ? 0.f : m_used;
        // row sums: two paired (f32x2) accumulators = four independent chains
        float2 ps2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        uint32_t pk[16];
        if (all_dead) {
#pragma unroll
          for (int e = 0; e < 16; ++e) pk[e] = 0u;
        } else {
          const float2 sc2 = make_float2(p.sc, p.sc), nm2 = make_float2(-m_eff, -m_eff);
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            // p = 2^(s * sc - m): one paired FFMA2 per two scores, then ex2 each
            const float2 t = __ffma2_rn(make_float2(x[e], x[e + 1]), sc2, nm2);
            float a0 = fl_ex2(t.x), a1 = fl_ex2(t.y);
            ps2[(e >> 1) & 1] = __fadd2_rn(ps2[(e >> 1) & 1], make_float2(a0, a1));
            if (DROP) {  // keep bits from flash_keep_mask_kernel
              if (!((kw >> e) & 1u)) a0 = 0.f;
              if (!((kw >> (e + 1)) & 1u)) a1 = 0.f;
            }
            pk[e >> 1] = fl_pack(a0, a1);
          }
        }
        l += (ps2[0].x + ps2[0].y) + (ps2[1].x + ps2[1].y);
        if (trw) FT(tro + 2, FT_CLK());
        // P (bf16 pairs) into P buffer sb, this warp's 16 columns: the P V
        // MMA's A operand, read from TMEM. The buffer's previous block (jb - 2)
        // must have been read by its P V MMAs.
        mbar_wait(&pempty[sb], ((jb >> 1) & 1) ^ 1);
        tc_fence_after();
        tmem_st16u(lane_base + KB + sb * (KB / 2) + 16 * w, pk);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[sb * NSL + w]);
        if (trw) FT(tro + 3, FT_CLK());
        if (j == 0 && pend) finish();  // the previous tile's combine
      }
      // this tile's row statistics for its (deferred) combine
      {
        float* xm = xch + (tc & 1) * (2 * NSL * 128);  // [m | l][slice][row]
        xm[w * 128 + r] = m_used;
        xm[NSL * 128 + w * 128 + r] = l;
      }
      pend = true;
      pend_tc = tc;
      pend_ok = row_ok;
      pend_ctx = ((int64_t)b * p.S + i) * p.ctx_ld + h * 64 + Cfg::kOCols * w;
      pend_grow = grow;
    }
    if (pend) finish();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
}

// ============================================================ backward
// Deterministic (no atomics), two kernels over the same per-score algebra,
// with the keep bits the forward stored (no Philox here):
//   P   = 2^(s sc - lse_i)                 (masked keys: 0)
//   Pd  = keep ? P / (1-p) : 0             dPd = dO_i . v_j  (TMEM)
//   dP  = keep ? dPd / (1-p) : 0           dS  = P (dP - D_i) * scale,
// D_i = dO_i . O_i (the dQ kernel, which runs first, computes it from its
// staged dO / O tiles and stores it for the dK / dV kernel). Both kernels compute S = Q K^T and
// dPd = dO V^T into TMEM with the query rows on the TMEM lanes (16 warps:
// lane quarter x 32-key slice, as the forward), then
//   flash_bwd_kv_kernel (one 128-key block per work item, loop over query
//   blocks): dV += Pd^T dO, dK += dS^T Q -- Pd / dS staged in smem as
//   [query][key] tiles and read by the MMA as MN-major A operands;
//   flash_bwd_q_kernel (one 128-query block per work item, loop over key
//   blocks): dQ += dS K with K read as an MN-major B operand.
// MODE 0 (dK / dV): 128-key items, 128-query inner blocks, 16 score warps,
// one CTA per SM. MODE 1 (dQ): 128-query items, KB-key inner blocks; KB = 64
// runs two CTAs per SM (8 score warps, 256 TMEM columns each).
template <int MODE, int KB>
struct FlashBwdCfg {
  static constexpr int kKB = MODE == 0 ? 128 : KB;  // keys per S tile
  static constexpr int kNSL = kKB / 32;              // 32-key slices
  static constexpr int kEW = 4 * kNSL;
  static constexpr int kThreads = 64 + 32 * kEW;
  static constexpr int kMinBlocks = (MODE == 1 && KB == 64) ? 2 : 1;
  static constexpr int kTile = 128 * 64 * 2;       // one 128-row x 64-dim bf16 tile
  static constexpr int kStrTile = (MODE == 0 ? 128 : KB) * 64 * 2;  // streamed tile
  // streamed (Q, dO) | (K, V) ring: a stage is released only when its block's
  // accumulation MMAs finish, so with two stages block j + 2's S / dPd MMAs
  // waited for block j's accumulation plus a TMA round trip (the measured
  // serialisation of the dK / dV kernel). The dQ kernel keeps dS in TMEM
  // (no staging tile), which leaves room for three stages in its two CTAs.
  // dK / dV smem split (A/B knob MIMOSE_FLASH_KV_CFG): 0 = two fixed K,V sets,
  // three ring stages, one staging buffer (default); 1 = one fixed set, two
  // stages, two staging buffers (no wait for the previous block's
  // accumulation before the Pd / dS stores); 2 = one fixed set, four stages
#ifndef MIMOSE_FLASH_KV_CFG
#define MIMOSE_FLASH_KV_CFG 0
#endif
  static constexpr int kKvCfg = MODE == 0 ? MIMOSE_FLASH_KV_CFG : 0;
  static constexpr int kStages = kKvCfg == 1 ? 2 : (kKvCfg == 2 ? 4 : 3);
  static constexpr int kSqBytes = 128 * kKB * 2;   // one [query][key] bf16 tile
  // staged score tiles per block: dK / dV stage Pd and dS in shared memory
  // ([query][key], read by the MMA as MN-major A operands); the dQ kernel
  // writes dS (bf16) into TMEM over the S slice it came from and the dQ MMA
  // reads its A operand from TMEM (no st.shared / proxy fence)
  static constexpr int kSqPer = MODE == 0 ? 2 : 0;
  static constexpr int kSqBufs = kKvCfg == 1 ? 2 : 1;
  static constexpr int kFix = MODE == 0 ? 2 : 3;   // K, V | Q, dO, O
  // dK / dV: the fixed K, V tiles are double-buffered, so the next item's
  // land while this one runs and its first S / dPd MMAs go in before this
  // item's last accumulation (no item-boundary bubble); the two-CTA dQ
  // kernel has no room for a second set
  static constexpr int kFixBufs = (MODE == 0 && kKvCfg == 0) ? 2 : 1;
  // S double buffer (2 kKB) + dPd (kKB) + accumulators (128 for dK / dV, 64 for dQ)
  static constexpr int kTmemCols = MODE == 0 ? 512 : (KB == 64 ? 256 : 512);
  static constexpr int kSmemBytes = kFixBufs * kFix * kTile + kStages * 2 * kStrTile +
                                    kSqBufs * kSqPer * kSqBytes + 1024 + 512;
};

// per-score backward algebra for 16 keys (columns e0..e0+15 of the thread's
// 32-key slice) of a query row; Pd (optional) and dS packed as bf16 pairs.
// The dS scale is folded into the exponent (lse_s = lse - log2(ds_scale):
// P' = P * ds_scale) and the keep bit into one factor f = keep / (1 - p):
//   dS = P' (dPd f - D),   Pd = P' f / ds_scale
// FULL: every key valid (no per-score test); DROP: dropout on.
template <bool FULL, bool WITH_PD, bool DROP>
__device__ __forceinline__ void flash_bwd_half(const uint32_t (&sraw)[16],
                                               const uint32_t (&dpraw)[16], int e0, int lim,
                                               float lse_s, float dvec, uint32_t kw, float fk,
                                               float fkd, float sc, uint32_t* pk_pd,
                                               uint32_t* pk_ds) {
  const float neg_inf = -__int_as_float(0x7f800000);
  // paired f32x2 math (FFMA2 / FMUL2): two scores per instruction
  const float2 sc2 = make_float2(sc, sc), nl2 = make_float2(-lse_s, -lse_s);
  const float2 nd2 = make_float2(-dvec, -dvec);
#pragma unroll
  for (int e = 0; e < 16; e += 2) {
    float2 x = make_float2(__uint_as_float(sraw[e]), __uint_as_float(sraw[e + 1]));
    if (!FULL) {
      if (e0 + e >= lim) x.x = neg_inf;
      if (e0 + e + 1 >= lim) x.y = neg_inf;
    }
    const float2 t = __ffma2_rn(x, sc2, nl2);
    const float2 P = make_float2(fl_ex2(t.x), fl_ex2(t.y));
    float2 f = make_float2(fk, fk), fd = make_float2(fkd, fkd);
    if (DROP) {
      if (!((kw >> (e0 + e)) & 1u)) f.x = fd.x = 0.f;
      if (!((kw >> (e0 + e + 1)) & 1u)) f.y = fd.y = 0.f;
    }
    const float2 dp = make_float2(__uint_as_float(dpraw[e]), __uint_as_float(dpraw[e + 1]));
    const float2 dS = __fmul2_rn(P, __ffma2_rn(dp, f, nd2));
    if constexpr (WITH_PD) {
      const float2 Pd = __fmul2_rn(P, fd);
      pk_pd[(e0 + e) >> 1] = fl_pack(Pd.x, Pd.y);
    }
    pk_ds[(e0 + e) >> 1] = fl_pack(dS.x, dS.y);
  }
}

// row r's 32-key slice w of a [query][key] tile (two 64-key SWIZZLE_128B sub-tiles)
__device__ __forceinline__ void flash_st_slice(uint8_t* tile, int r, int w,
                                               const uint32_t (&pk)[16]) {
  const uint32_t rowa = smem_u32(tile + (w >> 1) * 16384) + r * 128;
#pragma unroll
  for (int c = 0; c < 4; ++c)
    st_shared_v4(rowa + ((((w & 1) * 4 + c) ^ (r & 7)) << 4), pk[4 * c], pk[4 * c + 1],
                 pk[4 * c + 2], pk[4 * c + 3]);
}

// MODE 0: dK / dV kernel (work item = key block); MODE 1: dQ kernel (work item = query block)
template <int MODE, int KB>
__global__ void __launch_bounds__(FlashBwdCfg<MODE, KB>::kThreads,
                                  FlashBwdCfg<MODE, KB>::kMinBlocks)
    flash_bwd_kernel(const __grid_constant__ CUtensorMap tmQ,
                     const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV,
                     const __grid_constant__ CUtensorMap tmO,
                     const __grid_constant__ CUtensorMap tmC, const FlashParams p) {
  using Cfg = FlashBwdCfg<MODE, KB>;
  constexpr int NS = Cfg::kStages;
  constexpr int KBL = Cfg::kKB;  // keys per S tile
  constexpr bool KV = MODE == 0;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  // fixed tiles: KV ? (K, V) : (Q, dO, O); streamed pairs: KV ? (Q, dO) : (K, V)
  constexpr int kFix = Cfg::kFix;
  constexpr int NF = Cfg::kFixBufs;
  uint8_t* sFix = smem;  // [NF] fixed sets (item parity when NF = 2)
  uint8_t* sStr = smem + NF * kFix * Cfg::kTile;
  // staging buffer b: dS at sSq + b * kSqPer * kSqBytes, Pd (KV) right after
  uint8_t* sSq = sStr + NS * 2 * Cfg::kStrTile;
  constexpr int kSqBuf = Cfg::kSqPer * Cfg::kSqBytes;
  constexpr int NQ = Cfg::kSqBufs;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sSq + NQ * kSqBuf);
  uint64_t* full = bars;             // [NS]
  uint64_t* empty = full + NS;       // [NS]
  uint64_t* fixfull = empty + NS;     // [NF]
  uint64_t* fixempty = fixfull + NF;  // [NF]
  // S double-buffered in TMEM, dPd single: the score warps read dPd first and
  // release it, so the next block's S and dPd MMAs run while they compute
  uint64_t* sfull = fixempty + NF;  // [2] S[b] and dPd of a block landed
  uint64_t* sempty = sfull + 2;    // [2] S buffer b free (dK / dV: read; dQ: its dS consumed)
  uint64_t* dpempty = sempty + 2;  // dPd read
  // dK / dV: [NQ] staging buffer written by the score warps (the pdone wait
  // before each store keeps a fast warp from arriving for the next block
  // early); dQ: [2] by block parity -- with no staging wait a warp with dead
  // rows can run one block ahead, and one barrier would then complete a phase
  // on mixed arrivals (it cannot run two ahead: block j + 2's S needs block
  // j's accumulation, which needs pfull of block j)
  constexpr int NPF = KV ? NQ : 2;
  uint64_t* pfull = dpempty + 1;   // [NPF]
  uint64_t* pdone = pfull + NPF;   // [NQ] staging buffer read by the accumulation MMAs
  uint64_t* accfull = pdone + NQ;
  uint64_t* accempty = accfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 1);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const int nblk = (p.S + 127) / 128;       // 128-row item blocks
  const int nkb = (p.S + KBL - 1) / KBL;    // Q mode: KBL-key inner blocks
  const int num_items = nblk * p.nh * p.B;
  // inner blocks of work item `blk`: KV: query blocks [causal ? blk : 0, nblk);
  // Q: key blocks [0, causal ? blk + 1 : nblk)
  // item -> (head z, block). Causal: most inner blocks first, heads fastest
  auto decode = [&](int item, int& z, int& blk) {
    if (p.causal) {
      const int nz = p.nh * p.B;
      blk = KV ? item / nz : nblk - 1 - item / nz;
      z = item % nz;
    } else {
      z = item / nblk;
      blk = item % nblk;
    }
  };
  auto inner_range = [&](int blk, int& lo, int& hi) {
    if (KV) {
      lo = p.causal ? blk : 0;
      hi = nblk;
    } else {
      lo = 0;
      const int c = (blk + 1) * (128 / KBL);
      hi = p.causal ? (c < nkb ? c : nkb) : nkb;
    }
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    tma_prefetch(&tmO);
    if (!KV) tma_prefetch(&tmC);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int f = 0; f < NF; ++f) {
      mbar_init(&fixfull[f], 1);
      mbar_init(&fixempty[f], 1);
    }
    for (int b2 = 0; b2 < 2; ++b2) {
      mbar_init(&sfull[b2], 1);
      mbar_init(&sempty[b2], KV ? Cfg::kEW : 1);
    }
    mbar_init(dpempty, Cfg::kEW);
    for (int q = 0; q < NPF; ++q) mbar_init(&pfull[q], Cfg::kEW);
    for (int q = 0; q < NQ; ++q) mbar_init(&pdone[q], 1);
    mbar_init(accfull, 1);
    mbar_init(accempty, Cfg::kEW);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int st = 0, ic = 0;
      for (int item = blockIdx.x; item < num_items; item += gridDim.x, ++ic) {
        int z, blk;
        decode(item, z, blk);
        const int h = z % p.nh, b = z / p.nh;
        const int fb = ic % NF;
        const int fu = ic / NF;  // use count of set fb
        uint8_t* fx = sFix + fb * kFix * Cfg::kTile;
        mbar_wait(&fixempty[fb], (fu & 1) ^ 1);
        mbar_arrive_expect_tx(&fixfull[fb], kFix * Cfg::kTile);
        tma_load_4d(KV ? &tmK : &tmQ, &fixfull[fb], fx, 0, blk * 128, h, b);
        tma_load_4d(KV ? &tmV : &tmO, &fixfull[fb], fx + Cfg::kTile, 0, blk * 128, h, b);
        if (!KV) tma_load_4d(&tmC, &fixfull[fb], fx + 2 * Cfg::kTile, 0, blk * 128, h, b);
        int lo, hi;
        inner_range(blk, lo, hi);
        for (int j = lo; j < hi; ++j, ++st) {
          const int s = st % NS;
          mbar_wait(&empty[s], ((st / NS) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], 2 * Cfg::kStrTile);
          uint8_t* d = sStr + s * 2 * Cfg::kStrTile;
          const int rows = KV ? 128 : KBL;
          tma_load_4d(KV ? &tmQ : &tmK, &full[s], d, 0, j * rows, h, b);
          tma_load_4d(KV ? &tmO : &tmV, &full[s], d + Cfg::kStrTile, 0, j * rows, h, b);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc_s = idesc_bf16_f32(128, KBL, false, false);
    // KV: dV += Pd^T dO, dK += dS^T Q (A MN-major [query][key] tiles, B MN-major)
    // Q : dQ += dS K (A K-major [query][key] tile, B = K MN-major)
    const uint32_t idesc_acc = idesc_bf16_f32(128, 64, KV, true);
    int st = 0, ic = 0, blkc = 0;  // blkc: inner blocks processed (barrier phases)
    // warp-collective issue (umma_*_w), descriptors as base + (offset >> 4)
    const uint64_t d_str16 = smem_desc_sw128(smem_u32(sStr), 16, 1024);    // streamed, K-major
    const uint64_t d_fix16 = smem_desc_sw128(smem_u32(sFix), 16, 1024);    // fixed, K-major
    const uint64_t d_str8k = smem_desc_sw128(smem_u32(sStr), 8192, 1024);  // streamed, MN-major
    const uint64_t d_sq16k = smem_desc_sw128(smem_u32(sSq), 16384, 1024);  // staged, MN-major
    auto off = [](int bytes) { return (uint64_t)(bytes >> 4); };
    auto issue_sdp = [&](int s, int sb, int fb) {  // S = A0 B0^T, dPd = A1 B1^T (query rows)
      const uint64_t fx = d_fix16 + off(fb * kFix * Cfg::kTile);
      const uint64_t q = KV ? d_str16 + off(s * 2 * Cfg::kStrTile) : fx;
      const uint64_t k = KV ? fx : d_str16 + off(s * 2 * Cfg::kStrTile);
      constexpr int kQ2 = KV ? Cfg::kStrTile : Cfg::kTile;   // dO follows Q
      constexpr int kK2 = KV ? Cfg::kTile : Cfg::kStrTile;   // V follows K
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        umma_bf16_w(tmem_base + sb * KBL, q + off(kk * 32), k + off(kk * 32), idesc_s,
                    kk != 0 ? 1u : 0u);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        umma_bf16_w(tmem_base + 2 * KBL, q + off(kQ2 + kk * 32), k + off(kK2 + kk * 32), idesc_s,
                    kk != 0 ? 1u : 0u);
      umma_commit_w(&sfull[sb]);
    };
    auto issue_acc = [&](int s, int qb, int sb, bool first) {  // qb: staging buffer, sb: S buffer
      if (KV) {
        const uint64_t ds = d_sq16k + off(qb * kSqBuf), pd = ds + off(Cfg::kSqBytes);
        const uint64_t q = d_str8k + off(s * 2 * Cfg::kStrTile);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // K = 128 queries, 16 per MMA
          umma_bf16_w(tmem_base + 3 * KBL, pd + off(kk * 2048), q + off(Cfg::kStrTile + kk * 2048),
                      idesc_acc, (first && kk == 0) ? 0u : 1u);
          umma_bf16_w(tmem_base + 3 * KBL + 64, ds + off(kk * 2048), q + off(kk * 2048), idesc_acc,
                      (first && kk == 0) ? 0u : 1u);
        }
        umma_commit_w(&pdone[qb]);
      } else {
        // A = dS from TMEM: keys 32w..32w+31 of S buffer sb as bf16 pairs in
        // columns [32w, 32w + 16) of the buffer; 16 keys (8 columns) per MMA
        const uint32_t a0 = tmem_base + sb * KBL;
        const uint64_t k = d_str8k + off(s * 2 * Cfg::kStrTile);
#pragma unroll
        for (int kk = 0; kk < KBL / 16; ++kk)  // K = the block's keys
          umma_bf16_ts_w(tmem_base + 3 * KBL, a0 + (kk >> 1) * 32 + (kk & 1) * 8,
                         k + off(kk * 2048), idesc_acc, (first && kk == 0) ? 0u : 1u);
        umma_commit_w(&sempty[sb]);  // S buffer (and its dS) free for block + 2
      }
      umma_commit_w(&empty[s]);
    };
    // One flat block sequence across items: block g's S / dPd MMAs go in
    // before block g - 1's accumulation, also across an item boundary when the
    // next item's fixed tiles are in the other set (NF = 2).
    bool have_prev = false, prev_first = false, prev_last = false;
    int prev_s = 0, prev_pb = 0, prev_ic = 0;
    auto flush_prev = [&]() {
      if (prev_first) mbar_wait(accempty, (prev_ic & 1) ^ 1);  // previous item's drained
      mbar_wait(&pfull[prev_pb % NPF], (prev_pb / NPF) & 1);
      tc_fence_after();
      if (KV && lane == 0 && prev_pb < 256) FT(prev_pb * 4 + 1, FT_CLK());
      issue_acc(prev_s, prev_pb % NQ, prev_pb & 1, prev_first);
      if (KV && lane == 0 && prev_pb < 256) FT(prev_pb * 4 + 2, FT_CLK());
      if (prev_last) {
        umma_commit_w(accfull);
        // dQ: the score warps read the fixed dO / O tiles (D) and wait on
        // fixfull, so the set is released only after the item's last
        // accumulation -- an earlier release would let the producer
        // overwrite them, and lap fixfull, before the warps read
        if (!KV) umma_commit_w(&fixempty[prev_ic % NF]);
      }
      have_prev = false;
    };
    for (int item = blockIdx.x; item < num_items; item += gridDim.x, ++ic) {
      int lo, hi;
      int z_, blk_;
      decode(item, z_, blk_);
      inner_range(blk_, lo, hi);
      const int fb = ic % NF;
      // one fixed set: the previous item's last accumulation releases it
      if (NF == 1 && have_prev) flush_prev();
      mbar_wait(&fixfull[fb], (ic / NF) & 1);
      tc_fence_after();
      for (int j = lo; j < hi; ++j, ++st, ++blkc) {
        const int s = st % NS;
        mbar_wait(&full[s], (st / NS) & 1);
        mbar_wait(&sempty[blkc & 1], ((blkc >> 1) & 1) ^ 1);
        mbar_wait(dpempty, (blkc & 1) ^ 1);
        tc_fence_after();
        if (KV && lane == 0 && blkc < 256) FT(blkc * 4 + 0, FT_CLK());
        issue_sdp(s, blkc & 1, fb);
        // dK / dV: the fixed K, V tiles feed only the S / dPd MMAs (the
        // accumulation reads the staged tiles and the streamed pair), so the
        // set is released after the item's last S / dPd
        if (KV && j == hi - 1) umma_commit_w(&fixempty[fb]);
        if (have_prev) flush_prev();
        have_prev = true;
        prev_s = s; prev_pb = blkc; prev_ic = ic;
        prev_first = j == lo; prev_last = j == hi - 1;
      }
    }
    if (have_prev) flush_prev();
  } else {
    // ------------------------------------------------------------ score warps
    const int ew = warp - 2;
    const int quarter = warp & 3;
    const int w = ew >> 2;
    const int r = quarter * 32 + static_cast<int>(lane);
    const uint32_t lane_base = tmem_base + ((uint32_t)(quarter * 32) << 16);
    const bool dropout = p.drop.threshold != 0;
    int ic = 0, blkc = 0;
    // accumulators of item `dic` (TMEM lanes = its 128 key / query rows) -> dqkv
    auto drain = [&](int dic, int dblk, int dh, int db) {
        if (KV && ew == 0 && lane == 0 && dic < 256) FT(2048 + dic * 4 + 0, FT_CLK());
        mbar_wait(accfull, dic & 1);
        if (KV && ew == 0 && lane == 0 && dic < 256) FT(2048 + dic * 4 + 1, FT_CLK());
        tc_fence_after();
        const int row = dblk * 128 + r;  // key (KV) or query (Q) row of this lane
        if (KV) {
          uint32_t o[32];
          tmem_ld32_nowait(lane_base + 3 * KBL + 32 * w, o);  // w 0,1: dV halves; 2,3: dK halves
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(accempty);
          {
            const long long H = p.ctx_ld;
            const int rr = row < p.S ? row : 0;
            __nv_bfloat16* dst = p.dqkv + ((long long)db * p.S + rr) * 3 * H + (w < 2 ? 2 * H : H) +
                                 dh * 64 + 32 * (w & 1);
            uint4 ch[4];
  #pragma unroll
            for (int q = 0; q < 4; ++q)
              ch[q] = make_uint4(fl_pack(__uint_as_float(o[8 * q]), __uint_as_float(o[8 * q + 1])),
                                 fl_pack(__uint_as_float(o[8 * q + 2]), __uint_as_float(o[8 * q + 3])),
                                 fl_pack(__uint_as_float(o[8 * q + 4]), __uint_as_float(o[8 * q + 5])),
                                 fl_pack(__uint_as_float(o[8 * q + 6]), __uint_as_float(o[8 * q + 7])));
            fl_store_rows64(ch, dst, row < p.S);
          }
          if (ew == 0 && lane == 0 && dic < 256) FT(2048 + dic * 4 + 2, FT_CLK());
        } else {
          constexpr int OC = 64 / Cfg::kNSL;  // dQ columns of this warp
          float o[OC];
  #pragma unroll
          for (int q = 0; q < OC / 16; ++q) {
            uint32_t u[16];
            tmem_ld16u_nowait(lane_base + 3 * KBL + OC * w + 16 * q, u);
            tmem_wait_ld();
  #pragma unroll
            for (int e = 0; e < 16; ++e) o[16 * q + e] = __uint_as_float(u[e]);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(accempty);
          const long long H = p.ctx_ld;
          const int rr = row < p.S ? row : 0;
          __nv_bfloat16* dst = p.dqkv + ((long long)db * p.S + rr) * 3 * H + dh * 64 + OC * w;
          if constexpr (OC == 32) {
            uint4 ch[4];
  #pragma unroll
            for (int q = 0; q < 4; ++q)
              ch[q] = make_uint4(fl_pack(o[8 * q], o[8 * q + 1]), fl_pack(o[8 * q + 2], o[8 * q + 3]),
                                 fl_pack(o[8 * q + 4], o[8 * q + 5]),
                                 fl_pack(o[8 * q + 6], o[8 * q + 7]));
            fl_store_rows64(ch, dst, row < p.S);
          } else if (row < p.S) {
            uint4* d4 = reinterpret_cast<uint4*>(dst);
  #pragma unroll
            for (int q = 0; q < OC / 8; ++q)
              d4[q] = make_uint4(fl_pack(o[8 * q], o[8 * q + 1]), fl_pack(o[8 * q + 2], o[8 * q + 3]),
                                 fl_pack(o[8 * q + 4], o[8 * q + 5]),
                                 fl_pack(o[8 * q + 6], o[8 * q + 7]));
          }
        }
    };
    bool pend = false;
    int pend_ic = 0, pend_blk = 0, pend_h = 0, pend_b = 0;
    for (int item = blockIdx.x; item < num_items; item += gridDim.x, ++ic) {
      int z, blk;
      decode(item, z, blk);
      const int h = z % p.nh, b = z / p.nh;
      int lo, hi;
      inner_range(blk, lo, hi);
      // dQ kernel: D_i = dO_i . O_i of this lane's query row from the staged
      // dO / O tiles (this kernel runs first and stores D for the dK / dV one)
      float d_row = 0.f;
      if (!KV) {
        const uint8_t* fx = sFix + (ic % NF) * kFix * Cfg::kTile;
        mbar_wait(&fixfull[ic % NF], (ic / NF) & 1);
        const uint32_t ra = smem_u32(fx + Cfg::kTile) + r * 128;
        const uint32_t rc = smem_u32(fx + 2 * Cfg::kTile) + r * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint32_t off = (uint32_t)((c ^ (r & 7)) << 4);
          const uint4 x = ld_shared_v4(ra + off), y = ld_shared_v4(rc + off);
          const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&x);
          const __nv_bfloat162* y2 = reinterpret_cast<const __nv_bfloat162*>(&y);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 fx = __bfloat1622float2(x2[e]), fy = __bfloat1622float2(y2[e]);
            d_row = fmaf(fx.x, fy.x, d_row);
            d_row = fmaf(fx.y, fy.y, d_row);
          }
        }
        const int i = blk * 128 + r;
        if (w == 0 && i < p.S) p.dvec[(int64_t)z * p.S + i] = d_row;
      }
      if (KV && ew == 0 && lane == 0 && ic < 256) FT(2048 + ic * 4 + 3, FT_CLK());
      for (int j = lo; j < hi; ++j, ++blkc) {
        const int qb = KV ? j : blk, kb = KV ? blk : j;  // query / key block
        const int i = qb * 128 + r;
        const bool row_ok = i < p.S;
        const int64_t grow = (int64_t)z * p.S + (row_ok ? i : 0);
        // per-row scalars and keep bits first: their loads overlap the MMA
        const float lse = p.lse[grow], dv = KV ? p.dvec[grow] : d_row;
        const int c0 = kb * KBL + 32 * w;
        int lim = p.S - c0;
        if (p.causal && i - c0 + 1 < lim) lim = i - c0 + 1;
        if (!row_ok) lim = 0;
        const uint32_t kw = (dropout && lim > 0) ? p.mask[grow * p.mw + (c0 >> 5)] : 0u;
        const int sbuf = blkc & 1;
        const bool trw = KV && ew == 0 && lane == 0 && blkc < 256;
        if (trw) FT(1024 + blkc * 4 + 0, FT_CLK());
        mbar_wait(&sfull[sbuf], (blkc >> 1) & 1);
        if (trw) FT(1024 + blkc * 4 + 1, FT_CLK());
        tc_fence_after();
        const bool all_full = __all_sync(0xffffffffu, lim >= 32);
        const bool all_dead = __all_sync(0xffffffffu, lim <= 0);
        uint32_t pk_pd[16], pk_ds[16];
        // dPd first (whole slice, then its buffer is released), then S in two
        // 16-key halves; S buffer released once the second half is loaded
        uint32_t dpr[2][16];
        tmem_ld16u_nowait(lane_base + 2 * KBL + 32 * w, dpr[0]);
        tmem_ld16u_nowait(lane_base + 2 * KBL + 32 * w + 16, dpr[1]);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(dpempty);
        const float lse_s = lse - __log2f(p.ds_scale);
        const float fk = dropout ? p.drop.scale : 1.f, fkd = fk / p.ds_scale;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t sr[16];
          const uint32_t (&dr)[16] = dpr[half];
          tmem_ld16u_nowait(lane_base + sbuf * KBL + 32 * w + 16 * half, sr);
          tmem_wait_ld();
          if (KV && half == 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sempty[sbuf]);
          }
          if (all_dead) {
#pragma unroll
            for (int e = 0; e < 8; ++e) pk_pd[8 * half + e] = pk_ds[8 * half + e] = 0u;
          } else if (all_full) {
            if (dropout)
              flash_bwd_half<true, KV, true>(sr, dr, 16 * half, lim, lse_s, dv, kw, fk, fkd, p.sc,
                                             pk_pd, pk_ds);
            else
              flash_bwd_half<true, KV, false>(sr, dr, 16 * half, lim, lse_s, dv, kw, fk, fkd, p.sc,
                                              pk_pd, pk_ds);
          } else {
            if (dropout)
              flash_bwd_half<false, KV, true>(sr, dr, 16 * half, lim, lse_s, dv, kw, fk, fkd, p.sc,
                                              pk_pd, pk_ds);
            else
              flash_bwd_half<false, KV, false>(sr, dr, 16 * half, lim, lse_s, dv, kw, fk, fkd,
                                               p.sc, pk_pd, pk_ds);
          }
        }
        if (trw) FT(1024 + blkc * 4 + 2, FT_CLK());
        const int sq = blkc % NQ;
        if (KV) {
          // the accumulation MMAs of this staging buffer's previous block
          // (blkc - NQ) have read it
          mbar_wait(&pdone[sq], ((blkc / NQ) & 1) ^ 1);
          uint8_t* sDS = sSq + sq * kSqBuf;
          flash_st_slice(sDS + Cfg::kSqBytes, r, w, pk_pd);
          flash_st_slice(sDS, r, w, pk_ds);
          fence_async_shared();
        } else {
          // dS over the first half of this warp's own S slice (its S values
          // are already in registers; no other warp reads these columns)
          tmem_st16u(lane_base + sbuf * KBL + 32 * w, pk_ds);
          tmem_wait_st();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[blkc % NPF]);
        if (trw) FT(1024 + blkc * 4 + 3, FT_CLK());
        if (j == lo && pend) {  // the previous item's accumulators
          drain(pend_ic, pend_blk, pend_h, pend_b);
          pend = false;
        }
      }
      // item end: the accumulators are drained after the NEXT item's first
      // block (drain()), so the wait for this item's last accumulation and
      // the stores overlap that block's MMAs
      pend = true;
      pend_ic = ic; pend_blk = blk; pend_h = h; pend_b = b;
    }
    if (pend) drain(pend_ic, pend_blk, pend_h, pend_b);
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
}

}  // namespace mimose_dev
