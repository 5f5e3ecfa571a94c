// Launchers of the memory-bound kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "dropout_cfg.hpp"

namespace mimose_ops {

using mimose_dev::DropoutCfg;

// y = dropout_out(LN(z)), z = res + dropout_br(br)  (bf16 rows of H)
struct LnFwdArgs {
  int rows = 0;
  const void* res = nullptr;   // bf16 [rows][H] or null
  const void* br = nullptr;    // bf16 [rows][H]
  DropoutCfg br_drop;
  const float* gamma = nullptr;
  const float* beta = nullptr;
  float eps = 1e-12f;
  void* z = nullptr;           // bf16 saved LN input (null: not saved)
  void* stats = nullptr;       // float2 {mean, rstd} per row (null: not saved)
  void* y = nullptr;           // bf16 output
  DropoutCfg out_drop;
};

struct LnBwdArgs {
  int rows = 0;
  const void* dy = nullptr;    // bf16
  const void* dy2 = nullptr;   // bf16, added to dy (nullable)
  DropoutCfg in_drop;          // dropout that followed the LN (embedding)
  const void* z = nullptr;
  const void* stats = nullptr;
  const float* gamma = nullptr;
  void* dz = nullptr;          // bf16 grad of z (residual path)
  void* dbr = nullptr;         // bf16 grad of the dropped-out branch (nullable)
  DropoutCfg br_drop;
  float* partial = nullptr;    // [ln_bwd_blocks(rows)][3][H] scratch
};

struct AdamWArgs {
  float lr = 1e-4f, beta1 = 0.9f, beta2 = 0.999f, eps = 1e-8f, weight_decay = 0.01f;
  float bc1 = 1.f, bc2 = 1.f;  // bias corrections 1 - beta^t
  float max_grad_norm = 1.f;   // <= 0 disables clipping
  float grad_scale = 1.f;      // applied to raw grads (1/world after a sum-allreduce)
};

int ln_bwd_blocks(int rows);
int colsum_row_blocks(int rows);
int sumsq_blocks();

cudaError_t add_ln_fwd(const LnFwdArgs& a, int H, cudaStream_t s);
cudaError_t embed_ln_fwd(const LnFwdArgs& a, int H, const int32_t* tok, const int32_t* tt,
                         const void* word, const void* pos, const void* type, int S,
                         cudaStream_t s);
cudaError_t ln_bwd(const LnBwdArgs& a, int H, float* dgamma, float* dbeta, float* dbias,
                   cudaStream_t s);
// out[g][N] = sum over rows (with groups[r] == g) of x[r][:]; partial is
// [colsum_row_blocks(rows)][G][N] scratch
cudaError_t colsum(const void* x, int rows, int N, int64_t ld, const int32_t* groups, int G,
                   float* partial, float* out, cudaStream_t s);
cudaError_t softmax_fwd(const void* scores, void* P, void* Pd, int64_t rows, int S, int ld,
                        const DropoutCfg& d, cudaStream_t s);
cudaError_t softmax_bwd(const void* P, void* dPd, int64_t rows, int S, int ld,
                        const DropoutCfg& d, float scale, cudaStream_t s);
cudaError_t embed_word_grad(const void* de, int H, const int32_t* perm, const int32_t* seg,
                            const int32_t* uid, int n_unique, float* dword, cudaStream_t s);
cudaError_t embed_pos_grad(const void* de, int B, int S, int H, float* dpos, cudaStream_t s);
cudaError_t mc_head(const void* pre, int B, int H, int C, const float* wc, const float* bc,
                    const int32_t* labels, const DropoutCfg& d, float* loss, float* logits,
                    void* dpre, float* dwc, float* dbc, cudaStream_t s);
cudaError_t grad_norm2(const float* g, int64_t n, float* partial, float* out, cudaStream_t s);
cudaError_t adamw(float* p, float* m, float* v, const float* g, void* p16, int64_t n,
                  int64_t n_decay, const float* norm2, const AdamWArgs& a, cudaStream_t s);
cudaError_t f32_to_bf16(const float* in, void* out, int64_t n, cudaStream_t s);
cudaError_t init_normal(float* p, int64_t n, float mean, float std, uint64_t seed,
                        uint64_t stream, cudaStream_t s);

inline DropoutCfg make_dropout(float p, uint64_t seed, uint64_t stream) {
  DropoutCfg d;
  if (p <= 0.f) return d;
  d.seed = seed;
  d.stream = stream;
  const double t = static_cast<double>(p) * 65536.0 + 0.5;
  uint32_t thr = t >= 65535.0 ? 65535u : static_cast<uint32_t>(t);
  d.threshold = thr == 0 ? 1u : thr;
  d.scale = 1.f / (1.f - p);
  return d;
}

}  // namespace mimose_ops
