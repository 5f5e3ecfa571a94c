/* C ABI of the B200 execution side (libmimose_cuda.so).
 *
 * This is the device boundary SURVEY §8(b2) specifies: the reference keeps
 * the whole iteration on the host as byte/millisecond bookkeeping
 * (reference proj/include/mimose/simulator.hpp:104 `simulate_iteration`,
 * collector.hpp:115 `collect_iteration`); here those two calls become real
 * GPU iterations, driven through the entry points below.
 *
 * Conventions
 *   - every function returns int status, 0 = ok; on failure
 *     mimose_last_error() returns a thread-local message;
 *   - no C++ exceptions and no torch types cross this boundary: plain
 *     pointers, sizes and opaque handles only;
 *   - device work is stream-ordered (cudaStream_t passed as void*; NULL =
 *     legacy default stream);
 *   - one context per device, driven by one host thread. Every device byte
 *     the trainer uses comes from the context's budget arena.
 */
#ifndef MIMOSE_CUDA_H_
#define MIMOSE_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MIMOSE_ABI_VERSION 1

typedef struct mimose_ctx mimose_ctx;
typedef struct mimose_trainer mimose_trainer;

int mimose_abi_version(void);
const char* mimose_last_error(void);
/* Kernel launches issued by this library since load (telemetry). */
uint64_t mimose_launch_count(void);

/* ------------------------------------------------------------------ context
 * Replaces: the budget argument of reference scheduler.hpp:23
 * (SchedulerConfig::budget_bytes) becoming a hard device cap. */
int mimose_ctx_create(int device, int64_t budget_bytes, mimose_ctx** out);
int mimose_ctx_destroy(mimose_ctx* ctx);

/* ---------------------------------------------------------------- allocator
 * Replaces: the `resident` counter of reference simulator.hpp:113-155. */
#define MIMOSE_NUM_TAGS 8
typedef struct {
  int64_t budget;
  int64_t reserved;
  int64_t peak_reserved;
  int64_t requested;
  int64_t peak_requested;
  int64_t largest_free;
  int64_t n_live;
  int64_t n_allocs;
  int64_t n_failures;
  int64_t tag_requested[MIMOSE_NUM_TAGS];
  int64_t tag_peak[MIMOSE_NUM_TAGS];
} mimose_mem_stats;

int mimose_alloc(mimose_ctx* ctx, int64_t bytes, int tag, void** out);
int mimose_free(mimose_ctx* ctx, void* ptr);
int mimose_mem_stats_get(mimose_ctx* ctx, mimose_mem_stats* out);
int mimose_mem_reset_peak(mimose_ctx* ctx);

/* Host-only arena book-keeping (no device memory), for allocator tests. */
typedef struct mimose_book mimose_book;
int mimose_book_create(int64_t capacity, mimose_book** out);
int mimose_book_destroy(mimose_book* b);
int64_t mimose_book_alloc(mimose_book* b, int64_t bytes, int tag);
int mimose_book_free(mimose_book* b, int64_t offset);
int mimose_book_stats(mimose_book* b, mimose_mem_stats* out);

/* ------------------------------------------------------------ device ops
 * Stream-ordered operator entry points (device pointers). They are the
 * building blocks of the layer step and are exported for parity tests. */

/* D[z][m][n] = alpha * sum_k A[z][m][k] B[z][n][k] (+ epilogue)
 * A view: rows x cols with leading dim lda, batch strides (elements);
 * a_mn = 0 -> A view is [M][K]; a_mn = 1 -> A view is [K][M] (MN-major).
 * Same for B with N. epi: 0 bf16 (+bias), 1 bias+GELU (out=u, out2=gelu(u)),
 * 2 dGELU (out = acc * gelu'(aux)), 3 fp32 (out = alpha*acc + beta*out). */
typedef struct {
  int M, N, K, nb1, nb2;
  const void* a; int64_t a_rows, a_cols, lda, a_bs1, a_bs2; int a_mn;
  const void* b; int64_t b_rows, b_cols, ldb, b_bs1, b_bs2; int b_mn;
  int epi;
  void* out; void* out2; const void* aux; const float* bias;
  int64_t ldo, obs1, obs2;
  float alpha, beta;
  int force_bn;
} mimose_gemm_args;

int mimose_gemm(const mimose_gemm_args* args, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MIMOSE_CUDA_H_ */
