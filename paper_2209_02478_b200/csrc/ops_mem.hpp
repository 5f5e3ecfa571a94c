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
  bool skip_ln = false;        // y = dropout_out(z): plain (residual) sum, no LayerNorm
};

struct LnBwdArgs {
  int rows = 0;
  const void* dy = nullptr;    // bf16
  const void* dy2 = nullptr;   // bf16, added to dy (nullable)
  DropoutCfg in_drop;          // dropout that followed the LN (embedding)
  const void* z = nullptr;     // LN input z, or (beta != nullptr) the LN output y
  const void* stats = nullptr;
  const float* gamma = nullptr;
  // output-based x-hat: with beta set, `z` holds y = x-hat * gamma + beta (the
  // saved / retained LN output) and x-hat = (y - beta) / gamma; only rstd of
  // `stats` is read. Post-LN halves keep no LN input (lean saves).
  const float* beta = nullptr;
  void* dz = nullptr;          // bf16 grad of z (residual path)
  void* dbr = nullptr;         // bf16 grad of the dropped-out branch (nullable)
  DropoutCfg br_drop;
  const void* dres = nullptr;  // bf16 residual gradient added to dz AFTER the LN backward
                               // (pre-LN blocks: x + f(LN(x)))
  float* partial = nullptr;    // [ln_bwd_blocks(rows)][3][H] scratch
};

struct AdamWArgs {
  float lr = 1e-4f, beta1 = 0.9f, beta2 = 0.999f, eps = 1e-8f, weight_decay = 0.01f;
  float bc1 = 1.f, bc2 = 1.f;  // bias corrections 1 - beta^t
  float max_grad_norm = 1.f;   // <= 0 disables clipping
  float grad_scale = 1.f;      // applied to raw grads (1/world after a sum-allreduce)
};

int ln_bwd_blocks(int rows);
// row blocks of colsum over [rows][N]: one wave of the 256-thread partial
// kernel (ceil(N / 256) column groups x row blocks ~ the resident blocks);
// a function of (rows, N, SM count) only (deterministic partial layout)
int colsum_row_blocks(int rows, int N);
// scratch colsum needs for any (rows, N) and G <= 2
int64_t colsum_scratch_bytes();
int sumsq_blocks();

cudaError_t add_ln_fwd(const LnFwdArgs& a, int H, cudaStream_t s);
cudaError_t embed_ln_fwd(const LnFwdArgs& a, int H, const int32_t* tok, const int32_t* tt,
                         const void* word, const void* pos, const void* type, int S,
                         cudaStream_t s);
cudaError_t ln_bwd(const LnBwdArgs& a, int H, float* dgamma, float* dbeta, float* dbias,
                   cudaStream_t s);
// out[g][N] = sum over rows (with groups[r] == g) of x[r][:]; partial is
// [colsum_row_blocks(rows, N)][G][N] scratch (<= colsum_scratch_bytes())
cudaError_t colsum(const void* x, int rows, int N, int64_t ld, const int32_t* groups, int G,
                   float* partial, float* out, cudaStream_t s);
cudaError_t softmax_fwd(const void* scores, void* P, void* Pd, int64_t rows, int S, int ld,
                        const DropoutCfg& d, cudaStream_t s, bool causal = false);
cudaError_t softmax_bwd(const void* P, void* dPd, int64_t rows, int S, int ld,
                        const DropoutCfg& d, float scale, cudaStream_t s, bool causal = false);
cudaError_t embed_word_grad(const void* de, int H, const int32_t* perm, const int32_t* seg,
                            const int32_t* uid, int n_unique, float* dword, cudaStream_t s,
                            bool accumulate = false, int pad = -1);

// out = in * keep-mask * scale over n (multiple of 8) bf16 elements; element
// index = position in the buffer (the forward's dropout index)
cudaError_t dropout_apply(const void* in, void* out, int64_t n, const DropoutCfg& d,
                          cudaStream_t s);
// out = dg * gelu'(u)
cudaError_t dgelu_apply(const void* dg, const void* u, void* out, int64_t n, bool tanh_form,
                        cudaStream_t s);
// rows gather / scatter of bf16 [*, H]: dst[i] = src[idx[i]] ; dst[idx[i]] = src[i]
cudaError_t gather_rows(const void* src, const int32_t* idx, int n, int H, void* dst,
                        cudaStream_t s);
cudaError_t scatter_rows(const void* src, const int32_t* idx, int n, int H, void* dst,
                         cudaStream_t s);
// out = scale * sum(x[0..n)) in a fixed order (single CTA)
cudaError_t sum_f32(const float* x, int n, float scale, float* out, cudaStream_t s);

// extractive-QA head: logits[t] = (x[t] . w0 + b0, x[t] . w1 + b1); CE over the
// S positions of each sequence for start / end; dlogits [T][2] fp32 (scaled by
// 1 / (2 B)) and per-sequence loss partials (already / (2 B))
cudaError_t qa_head(const void* x, int B, int S, int H, const float* w, const float* b,
                    const int32_t* labels, float* logits, float* dlogits, float* loss_parts,
                    cudaStream_t s);
// dx[t] = dl[t][0] w0 + dl[t][1] w1 (bf16); partial sums for dW [2][H] and db [2]
cudaError_t qa_head_bwd(const void* x, const float* dlogits, int T, int H, const float* w,
                        void* dx, float* partial, float* dW, float* db, cudaStream_t s);
int qa_row_blocks(int T);
// row-wise softmax cross-entropy over V classes of bf16 logits [rows][ld]:
// loss_rows[r] = lse - logit[label] (0 for label < 0); logits are overwritten
// by dlogits = (softmax - onehot) * grad_scale (zero rows for ignored labels)
cudaError_t ce_rows(void* logits, int rows, int V, int ld, const int32_t* labels,
                    float grad_scale, float* loss_rows, cudaStream_t s);
cudaError_t embed_pos_grad(const void* de, int B, int S, int H, float* dpos, cudaStream_t s);
cudaError_t mc_head(const void* pre, int B, int H, int C, const float* wc, const float* bc,
                    const int32_t* labels, const DropoutCfg& d, float* loss, float* logits,
                    void* dpre, float* dwc, float* dbc, cudaStream_t s);
cudaError_t grad_norm2(const float* g, int64_t n, float* partial, float* out, cudaStream_t s);
cudaError_t adamw(float* p, float* m, float* v, const float* g, void* p16, int64_t n,
                  const uint8_t* decay_chunk, const float* norm2, const AdamWArgs& a,
                  cudaStream_t s);
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
