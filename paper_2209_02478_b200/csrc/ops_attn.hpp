// Fused attention-score operators (attn.cu) and the tensor-map helpers they
// share with the GEMM (gemm.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "dropout_cfg.hpp"
#include "ops.hpp"

namespace mimose_ops {

// bf16 operand map over a 4-D view with a {64, box_rows} SWIZZLE_128B box
bool make_operand_map(CUtensorMap* map, const MatView& v, int nb1, int nb2, uint32_t box_rows);
// bf16 output map (rows x cols, pitch ld, batch strides) with a {box_cols, 32}
// box, SWIZZLE_128B (64 columns) or SWIZZLE_64B (32 columns)
bool make_output_map(CUtensorMap* map, void* ptr, int64_t rows, int64_t cols, int64_t ld,
                     int64_t bs1, int64_t bs2, int nb1, int nb2, uint32_t box_cols = 64,
                     bool sw64 = false);

bool attn_fused_supported(int S);
// P = softmax(alpha * Q K^T), Pd = dropout(P) (Pd may be null when p = 0)
// (causal: keys j > query i get P = 0)
cudaError_t attn_scores_fwd(const MatView& q, const MatView& k, void* P, void* Pd, int S, int ld,
                            int nh, int B, float alpha, const mimose_dev::DropoutCfg& drop,
                            cudaStream_t s, bool causal = false);
// dS = P * (dP - rowsum(dP * P)) * ds_scale with dP = dropout'(dO V^T)
cudaError_t attn_scores_bwd(const MatView& dout, const MatView& v, const void* P, void* dS, int S,
                            int ld, int nh, int B, float ds_scale,
                            const mimose_dev::DropoutCfg& drop, cudaStream_t s);

// Flash attention (flash_sm100.cuh, head dim 64): no S x S tensor in HBM.
// q / k / v: 4-D head views ([B][nh][S][64] over the packed qkv rows);
// ctx: [B*S][ctx_ld] (head h at columns 64h); lse: [B*nh][S] log2-sum-exp of
// the scaled scores. Dropout keep bits use the element index row * ld + key
// of the materialised path.
bool flash_supported(int S);
// Dropout keep bits [B*nh*S][ceil(S/32)] uint32 (bit e of word (row, k) =
// key 32k + e kept), Philox at the materialised path's element index; they
// depend only on (seed, stream, shape), so the trainer generates them on a
// side stream while the QKV projection runs. Read by flash_fwd / flash_bwd.
cudaError_t flash_keep_mask(uint32_t* mask, int S, int ld, int nh, int B,
                            const mimose_dev::DropoutCfg& drop, bool causal, cudaStream_t s);
// mask: required with dropout (flash_keep_mask output)
cudaError_t flash_fwd(const MatView& q, const MatView& k, const MatView& v, void* ctx,
                      int64_t ctx_ld, float* lse, uint32_t* mask, int S, int ld, int nh, int B,
                      float alpha, const mimose_dev::DropoutCfg& drop, bool causal,
                      cudaStream_t s);
// dqkv from dctx and the forward's ctx / lse / mask; dvec: [B*nh*S] fp32 workspace
cudaError_t flash_bwd(const MatView& q, const MatView& k, const MatView& v, const void* ctx,
                      const void* dctx, int64_t ctx_ld, const float* lse, const uint32_t* mask,
                      float* dvec, void* dqkv, int S, int ld, int nh, int B, float alpha,
                      const mimose_dev::DropoutCfg& drop, bool causal, cudaStream_t s);

}  // namespace mimose_ops
