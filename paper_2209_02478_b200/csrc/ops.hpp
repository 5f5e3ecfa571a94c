// Internal (C++) interface of the device operators. The public boundary is the
// C ABI in include/mimose_cuda.h; this header is shared by the operator
// translation units and the training executor.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "dropout_cfg.hpp"

namespace mimose_ops {

// bf16 matrix view: logical [nb2][nb1][rows][cols], `cols` contiguous.
// Strides are in elements.
struct MatView {
  const void* ptr = nullptr;
  int64_t rows = 0, cols = 0, ld = 0, bs1 = 0, bs2 = 0;
};

enum Epi : int { kEpiBf16 = 0, kEpiBiasGelu = 1, kEpiDGelu = 2, kEpiF32 = 3 };

// D[z][m][n] = sum_k A[z][m][k] B[z][n][k]
//   A: a_mn == false -> view rows=M cols=K ; true -> view rows=K cols=M
//   B: b_mn == false -> view rows=N cols=K ; true -> view rows=K cols=N
struct GemmCall {
  int M = 0, N = 0, K = 0, nb1 = 1, nb2 = 1;
  MatView A;
  bool a_mn = false;
  MatView B;
  bool b_mn = false;
  int epi = kEpiBf16;
  void* out = nullptr;
  void* out2 = nullptr;
  const void* aux = nullptr;
  const float* bias = nullptr;
  int64_t ldo = 0, obs1 = 0, obs2 = 0;
  float alpha = 1.f, beta = 0.f;
  int force_bn = 0;  // 0 = heuristic; 64/128/256 for tests
  int force_ew = 0;  // 0 = heuristic; 8 / 16 epilogue warps for tests
  int force_cg = 0;  // 0 = heuristic; 1 / 2 (CTA pair) for tests
  bool direct_store = false;  // tests: force the per-thread store epilogue
  // deterministic split-K for fp32 (weight-gradient) outputs: partials go to
  // `workspace` ([splits][M][N] fp32) and are summed in a fixed order.
  // split_k: 0 = automatic when a workspace is given, 1 = off, >1 forced.
  int split_k = 0;
  void* workspace = nullptr;
  int64_t workspace_bytes = 0;
  int gelu_tanh = 0;              // GELU flavour for kEpiBiasGelu / kEpiDGelu
  int gelu_deriv = 0;             // kEpiBiasGelu: out = GELU'(u); kEpiDGelu: aux is GELU'(u)
  mimose_dev::DropoutCfg drop;    // kEpiBf16: dropout on the product before adding aux
  bool causal_tiles = false;      // skip tiles above the diagonal (causal S x S scores)
  int causal_k = 0;               // 1: only k <= row contributes, 2: only k >= row (causal)
  // kEpiF32 with MN-major A, unbatched, not causal: also write the sums of
  // A's rows over K to rowsum[M] (fp32, overwritten) -- the bias gradient
  // of a weight-gradient GEMM (A = dY), summed from the staged operand
  // tiles instead of a second pass over dY. Split-K partials take
  // splits * M floats of `workspace` after the [splits][M][N] block.
  float* rowsum = nullptr;
};

cudaError_t gemm(const GemmCall& c, cudaStream_t stream);
// programmatic dependent launch for the tcgen05 kernels (env MIMOSE_PDL=0 off)
bool pdl_enabled();
// split-K choice for an fp32 (weight-gradient) GEMM and the workspace it needs
int pick_split_k(int M, int N, int K, int bn, int cg = 1);
int64_t splitk_workspace_bytes(int M, int N, int K);
void gemm_profile_enable(bool on);
cudaError_t gemm_profile_read(double* flops, double* ms, int64_t* launches);
std::string gemm_profile_csv();

// Number of kernels launched by this module since process start (telemetry
// for the bench's gpu_launches count).
// g = GELU(u) elementwise, bit-identical to the bias+GELU epilogue's g
// (trainer: FFN halves that save u only regenerate g for the dW2 GEMM)
cudaError_t gelu_regen(const void* u, void* g, int64_t n, bool tanh_form, cudaStream_t s);

uint64_t launch_count();
void count_launch();

}  // namespace mimose_ops
