// C ABI implementation: context, allocator, operator entry points.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "allocator.hpp"
#include "capi_common.hpp"
#include "mimose_cuda.h"
#include "ops.hpp"
#include "ops_attn.hpp"
#include "ops_mem.hpp"
#include "prof.hpp"

using mimose_rt::ArenaBook;
using mimose_rt::DeviceArena;
using mimose_rt::MemStats;

namespace mimose_capi {
thread_local std::string g_last_error;
int fail(const std::string& msg) {
  g_last_error = msg;
  return 1;
}
int cuda_fail(cudaError_t e, const char* what) {
  return fail(std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace mimose_capi

using mimose_capi::cuda_fail;
using mimose_capi::fail;

struct mimose_book {
  ArenaBook book;
};

namespace {
void copy_stats(const MemStats& s, mimose_mem_stats* o) {
  o->budget = s.budget;
  o->reserved = s.reserved;
  o->peak_reserved = s.peak_reserved;
  o->requested = s.requested;
  o->peak_requested = s.peak_requested;
  o->largest_free = s.largest_free;
  o->n_live = s.n_live;
  o->n_allocs = s.n_allocs;
  o->n_failures = s.n_failures;
  for (int t = 0; t < MIMOSE_NUM_TAGS; ++t) {
    o->tag_requested[t] = s.tag_requested[t];
    o->tag_peak[t] = s.tag_peak[t];
  }
}
}  // namespace

extern "C" {

int mimose_abi_version(void) { return MIMOSE_ABI_VERSION; }
const char* mimose_last_error(void) { return mimose_capi::g_last_error.c_str(); }
uint64_t mimose_launch_count(void) { return mimose_ops::launch_count(); }

int mimose_ctx_create(int device, int64_t budget_bytes, mimose_ctx** out) {
  if (out == nullptr) return fail("mimose_ctx_create: null out");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  auto* ctx = new (std::nothrow) mimose_ctx();
  if (ctx == nullptr) return fail("out of host memory");
  ctx->device = device;
  std::string err = ctx->arena.init(budget_bytes);
  if (!err.empty()) {
    delete ctx;
    return fail("mimose_ctx_create: " + err);
  }
  *out = ctx;
  return 0;
}

int mimose_ctx_destroy(mimose_ctx* ctx) {
  delete ctx;
  return 0;
}

int mimose_alloc(mimose_ctx* ctx, int64_t bytes, int tag, void** out) {
  if (ctx == nullptr || out == nullptr) return fail("mimose_alloc: null argument");
  void* p = ctx->arena.alloc(bytes, tag);
  if (p == nullptr) {
    return fail("mimose_alloc: budget exceeded (request " + std::to_string(bytes) +
                " B, live " + std::to_string(ctx->arena.stats().reserved) + " B of " +
                std::to_string(ctx->arena.stats().budget) + " B)");
  }
  *out = p;
  return 0;
}

int mimose_free(mimose_ctx* ctx, void* ptr) {
  if (ctx == nullptr) return fail("mimose_free: null ctx");
  if (!ctx->arena.free(ptr)) return fail("mimose_free: pointer not owned by the arena");
  return 0;
}

int mimose_mem_stats_get(mimose_ctx* ctx, mimose_mem_stats* out) {
  if (ctx == nullptr || out == nullptr) return fail("mimose_mem_stats_get: null argument");
  copy_stats(ctx->arena.stats(), out);
  return 0;
}

int mimose_mem_reset_peak(mimose_ctx* ctx) {
  if (ctx == nullptr) return fail("mimose_mem_reset_peak: null ctx");
  ctx->arena.reset_peak();
  return 0;
}

int mimose_book_create(int64_t capacity, mimose_book** out) {
  if (out == nullptr || capacity <= 0) return fail("mimose_book_create: bad argument");
  *out = new mimose_book();
  (*out)->book.reset(capacity);
  return 0;
}
int mimose_book_destroy(mimose_book* b) {
  delete b;
  return 0;
}
int64_t mimose_book_alloc(mimose_book* b, int64_t bytes, int tag) {
  return b->book.allocate(bytes, tag);
}
int mimose_book_free(mimose_book* b, int64_t offset) {
  return b->book.release(offset) ? 0 : fail("mimose_book_free: unknown offset");
}
int mimose_book_stats(mimose_book* b, mimose_mem_stats* out) {
  copy_stats(b->book.stats(), out);
  return 0;
}

int mimose_gemm(const mimose_gemm_args* a, void* stream) {
  if (a == nullptr) return fail("mimose_gemm: null args");
  mimose_ops::GemmCall c;
  c.M = a->M; c.N = a->N; c.K = a->K; c.nb1 = a->nb1; c.nb2 = a->nb2;
  c.A = {a->a, a->a_rows, a->a_cols, a->lda, a->a_bs1, a->a_bs2};
  c.a_mn = a->a_mn != 0;
  c.B = {a->b, a->b_rows, a->b_cols, a->ldb, a->b_bs1, a->b_bs2};
  c.b_mn = a->b_mn != 0;
  c.epi = a->epi;
  c.out = a->out; c.out2 = a->out2; c.aux = a->aux; c.bias = a->bias;
  c.ldo = a->ldo; c.obs1 = a->obs1; c.obs2 = a->obs2;
  c.alpha = a->alpha; c.beta = a->beta;
  c.force_bn = a->force_bn;
  c.force_ew = a->force_ew;
  c.force_cg = a->force_cg;
  c.direct_store = a->direct_store != 0;
  c.split_k = a->split_k;
  c.workspace = a->workspace;
  c.workspace_bytes = a->workspace_bytes;
  c.rowsum = a->rowsum;
  cudaError_t e = mimose_ops::gemm(c, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "mimose_gemm");
  return 0;
}

namespace {
mimose_ops::MatView qkv_head_view(const void* qkv, int part, int S, int H) {
  mimose_ops::MatView v;
  v.ptr = static_cast<const uint16_t*>(qkv) + (int64_t)part * H;
  v.rows = S;
  v.cols = 64;
  v.ld = 3 * (int64_t)H;
  v.bs1 = 64;
  v.bs2 = (int64_t)S * 3 * H;
  return v;
}
}  // namespace

int mimose_flash_attn_fwd(const mimose_attn_args* a, void* stream) {
  if (a == nullptr || a->qkv == nullptr || a->ctx == nullptr || a->lse == nullptr)
    return fail("mimose_flash_attn_fwd: null argument");
  if (a->B <= 0 || a->S <= 0 || a->nh <= 0) return fail("mimose_flash_attn_fwd: bad shape");
  const int H = 64 * a->nh;
  const auto drop = mimose_ops::make_dropout(a->dropout_p, a->seed, a->stream_id);
  if (drop.threshold != 0 && a->keep_mask == nullptr)
    return fail("mimose_flash_attn_fwd: dropout needs keep_mask");
  cudaError_t e = mimose_ops::flash_keep_mask(a->keep_mask, a->S, (a->S + 7) / 8 * 8, a->nh, a->B,
                                              drop, a->causal != 0,
                                              static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "mimose_flash_attn_fwd");
  e = mimose_ops::flash_fwd(
      qkv_head_view(a->qkv, 0, a->S, H), qkv_head_view(a->qkv, 1, a->S, H),
      qkv_head_view(a->qkv, 2, a->S, H), a->ctx, H, a->lse, a->keep_mask, a->S,
      (a->S + 7) / 8 * 8, a->nh, a->B, a->scale, drop, a->causal != 0,
      static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "mimose_flash_attn_fwd");
  return 0;
}

int mimose_flash_attn_bwd(const mimose_attn_args* a, void* stream) {
  if (a == nullptr || a->qkv == nullptr || a->ctx == nullptr || a->lse == nullptr ||
      a->dctx == nullptr || a->dqkv == nullptr)
    return fail("mimose_flash_attn_bwd: null argument");
  if (a->B <= 0 || a->S <= 0 || a->nh <= 0) return fail("mimose_flash_attn_bwd: bad shape");
  if (a->dropout_p > 0.f && a->keep_mask == nullptr)
    return fail("mimose_flash_attn_bwd: dropout needs the forward's keep_mask");
  if (a->workspace == nullptr || a->workspace_bytes < (int64_t)4 * a->B * a->nh * a->S)
    return fail("mimose_flash_attn_bwd: workspace < 4 * B * nh * S bytes");
  const int H = 64 * a->nh;
  const auto drop = mimose_ops::make_dropout(a->dropout_p, a->seed, a->stream_id);
  cudaError_t e = mimose_ops::flash_bwd(
      qkv_head_view(a->qkv, 0, a->S, H), qkv_head_view(a->qkv, 1, a->S, H),
      qkv_head_view(a->qkv, 2, a->S, H), a->ctx, a->dctx, H, a->lse, a->keep_mask,
      static_cast<float*>(a->workspace), a->dqkv, a->S, (a->S + 7) / 8 * 8, a->nh, a->B, a->scale,
      drop, a->causal != 0, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "mimose_flash_attn_bwd");
  return 0;
}

int mimose_gemm_profile_enable(int enable) {
  mimose_ops::gemm_profile_enable(enable != 0);
  return 0;
}

int mimose_gemm_profile_csv(char** out) {
  const std::string s = mimose_ops::gemm_profile_csv();
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  *out = p;
  return 0;
}

int mimose_profile_enable(int enable) {
  mimose_ops::prof_enable(enable != 0);
  return 0;
}

int mimose_profile_read(const char* class_prefix, double* flops, double* bytes, double* ms,
                        int64_t* launches) {
  cudaError_t e = mimose_ops::prof_read(class_prefix != nullptr ? class_prefix : "", flops, bytes,
                                        ms, launches);
  if (e != cudaSuccess) return cuda_fail(e, "mimose_profile_read");
  return 0;
}

int mimose_profile_csv(char** out) { return mimose_gemm_profile_csv(out); }

int mimose_gemm_profile_read(double* flops, double* ms, int64_t* launches) {
  cudaError_t e = mimose_ops::gemm_profile_read(flops, ms, launches);
  if (e != cudaSuccess) return cuda_fail(e, "mimose_gemm_profile_read");
  return 0;
}

}  // extern "C"
