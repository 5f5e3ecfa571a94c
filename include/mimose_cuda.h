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

#define MIMOSE_ABI_VERSION 7

typedef struct mimose_ctx mimose_ctx;
typedef struct mimose_trainer mimose_trainer;
typedef struct mimose_dp mimose_dp;

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
  int force_bn;      /* 0 = heuristic tile width; 64 / 128 / 256 forces it */
  int direct_store;  /* 1 = per-thread stores instead of smem + TMA store (tests) */
  int split_k;       /* fp32 outputs: 0 auto (needs workspace), 1 off, >1 forced */
  void* workspace;   /* fp32 split-K partials, >= split_k * M * N * 4 bytes */
  int64_t workspace_bytes;
  int force_ew;      /* 0 = heuristic epilogue warps; 8 / 16 forces it */
  int force_cg;      /* 0 = heuristic; 1 = one SM per tile, 2 = CTA pair (cta_group::2) */
  float* rowsum;     /* epi 3 with a_mn = 1, unbatched: also rowsum[m] = sum_k A[m][k]
                        (fp32, overwritten: the bias gradient of a weight gradient);
                        split-K then needs split_k * M * (N + 1) * 4 workspace bytes */
} mimose_gemm_args;

int mimose_gemm(const mimose_gemm_args* args, void* stream);

/* Flash attention operator (head dim 64; the trainer's attn_fused = 3 path):
 * packed qkv [B*S][3H] bf16 (q | k | v thirds, head h at columns 64h of
 * each, H = 64 * nh). Forward writes ctx [B*S][H] bf16 and lse [B*nh][S] fp32
 * (log2-sum-exp of the scaled scores). Backward reads qkv, ctx, lse, dctx and
 * writes dqkv [B*S][3H]; workspace >= 4 * B * nh * S bytes. With dropout the
 * forward also writes one keep bit per score (keep_mask) for the backward. Dropout on the
 * probabilities uses the same Philox element index (row * round8(S) + key)
 * as the materialised path, so both paths drop the same entries. */
typedef struct mimose_attn_args {
  int B, S, nh, causal;
  float scale;        /* score scale (1/sqrt(64)) */
  float dropout_p;
  uint64_t seed, stream_id;
  const void* qkv;
  void* ctx;
  float* lse;
  uint32_t* keep_mask; /* dropout_p > 0: keep bits [B*nh*S][ceil(S/32)] (fwd out, bwd in) */
  const void* dctx;
  void* dqkv;
  void* workspace;
  int64_t workspace_bytes;
} mimose_attn_args;

int mimose_flash_attn_fwd(const mimose_attn_args* args, void* stream);
int mimose_flash_attn_bwd(const mimose_attn_args* args, void* stream);

/* GEMM profiling (roofline evidence): while enabled, every GEMM launch is
 * bracketed by CUDA events on its stream; read() synchronises and returns
 * the summed algorithmic flops (2*M*N*K*batch), summed kernel ms and the
 * number of launches since enable. */
int mimose_gemm_profile_enable(int enable);
int mimose_gemm_profile_read(double* flops, double* ms, int64_t* launches);
/* Per-launch CSV (class,desc,flops,bytes,ms); free with mimose_free_string. */
int mimose_gemm_profile_csv(char** out);

/* Kernel profiling across ALL instrumented launches (GEMMs and the
 * memory-bound stages). Each record carries its class ("gemm_dense",
 * "gemm_attn", "mem_softmax_fwd", "mem_ln_bwd", ...), algorithmic flops and
 * algorithmic HBM bytes. read() sums records whose class starts with
 * `class_prefix` ("" = all). The GEMM calls above are views of the same
 * recorder restricted to the "gemm" prefix. */
int mimose_profile_enable(int enable);
int mimose_profile_read(const char* class_prefix, double* flops, double* bytes, double* ms,
                        int64_t* launches);
int mimose_profile_csv(char** out);

/* ------------------------------------------------------------------ trainer
 * The training executor: BERT-style encoder blocks (post-LN, GELU FFN,
 * materialised attention) + multiple-choice head, trained with AdamW under
 * the context's byte budget. Replaces the reference's replayed iteration
 * (harness.hpp:139 run_experiment, Mimose branch harness.hpp:215-296) with a
 * real one; planning calls the host planner (include/mimose) in-process. */
enum { MIMOSE_ARCH_BERT = 0, MIMOSE_ARCH_GPT2 = 1 };
enum { MIMOSE_HEAD_MC = 0, MIMOSE_HEAD_QA = 1, MIMOSE_HEAD_LM = 2, MIMOSE_HEAD_MLM = 3 };

/* Label layouts per head (int32): MC [batch/num_choices] choice ids; QA
 * [2*batch] (start, end) positions; LM [batch*seq] next-token ids, -1 ignored;
 * MLM [batch*seq] original ids at masked positions, -1 elsewhere. LM and MLM
 * decoders are tied to the word embeddings. */
typedef struct {
  int layers, hidden, heads, ffn, vocab, max_pos, type_vocab; /* type_vocab 0: none */
  int num_choices;        /* multiple-choice group size C (batch % C == 0) */
  float hidden_dropout, attn_dropout, ln_eps, init_std;
  uint64_t seed;
  int arch;               /* MIMOSE_ARCH_BERT: post-LN block, embedding LayerNorm;
                             MIMOSE_ARCH_GPT2: pre-LN block, final LayerNorm */
  int head;               /* MIMOSE_HEAD_* */
  int causal;             /* causal self-attention mask */
  int gelu_tanh;          /* GELU tanh approximation (GPT-2 "gelu_new") instead of erf */
  int pad_token_id;       /* word-embedding row that receives no gradient (HF BERT
                             padding_idx = pad_token_id = 0); -1 = none (GPT-2) */
} mimose_model_cfg;

enum {
  MIMOSE_PLANNER_MIMOSE = 0, /* two-phase input-aware planner (the product) */
  MIMOSE_PLANNER_NONE = 1,   /* no checkpointing (throughput reference) */
  MIMOSE_PLANNER_ALL = 2,    /* checkpoint every block */
  MIMOSE_PLANNER_STATIC = 3, /* plan once for seq_max, reuse (baselines.hpp:20) */
  MIMOSE_PLANNER_DTR = 4     /* reactive eviction on the real arena (baselines.hpp:62) */
};

typedef struct {
  int planner;
  int batch;                   /* sequences per step B (x = B * S) */
  int seq_min, seq_max;        /* S range -> model input range [B*seq_min, B*seq_max] */
  int64_t reserve_bytes;       /* < 0: automatic (extras at seq_max + margin) */
  double bucket_tolerance;     /* scheduler.hpp:26 */
  double cache_tolerance;      /* scheduler.hpp:27 */
  int max_sheltered_iters;     /* collector.hpp:92 */
  int collect_new_sizes_always;/* collector.hpp:93 */
  int estimator_order;         /* harness.hpp:53 */
  float lr, beta1, beta2, adam_eps, weight_decay, max_grad_norm;
  int attn_fused;              /* 3: flash attention (default; no S x S tensor); 2: fused
                                  score + softmax kernels, whole key row in TMEM (S <= 512, else
                                  as 0); 0: QK^T GEMM + softmax kernels (materialised P / Pd) */
  int reserve_per_size;        /* automatic reserve: 1 = sized for this step's S and verified
                                  against the plan's own replay (simulate_iteration) - short
                                  inputs keep more units; 0 = worst case at seq_max */
  int ckpt_unit;               /* checkpoint unit the planner schedules: 0 = transformer block
                                  (the reference's layer granularity), 1 = block half (attention
                                  half, FFN half: 2 x layers units, finer-grained drops) */
  int ffn_regen_g;             /* 1: a kept FFN half saves the pre-activation u only and its
                                  backward regenerates g = GELU(u) (bit-identical) for the W2
                                  gradient: 8 H fewer bytes per token per kept block for one
                                  elementwise pass; 0: u and g both saved */
} mimose_train_cfg;

enum {
  MIMOSE_PHASE_PLANNED = 0,   /* responsive: cache hit or freshly generated plan */
  MIMOSE_PHASE_COLLECT = 1,   /* sheltered: measuring pass, all blocks dropped */
  MIMOSE_PHASE_SHELTERED = 2, /* sheltered: seen size, all blocks dropped */
  MIMOSE_PHASE_PLAIN = 3,     /* planner none / all / static / forced */
  MIMOSE_PHASE_FALLBACK = 4   /* post-window collection (too few sizes to fit) */
};

typedef struct {
  int64_t iter;
  int64_t x;
  int batch, seq;
  int phase;
  int cache_hit;
  int plan_size;
  int insufficient;
  int fit_order;               /* order of the fit performed this step, -1 none */
  float loss;                  /* filled by the host-input step (after D2H) */
  int64_t peak_requested;      /* arena peak during this step */
  int64_t peak_reserved;
  int64_t predicted_kept;      /* constant + predicted kept bytes (scheduler view) */
  int64_t budget;
  double plan_us;              /* lookup_or_plan wall time */
  double fit_us;               /* fit wall time */
  uint64_t dropped_mask_lo;    /* bit i = block i dropped (blocks 0..63) */
  double pred_err_mean;        /* |predict(l,x) - measured a_l(x)| / measured, kept blocks */
  double pred_err_max;
  int pred_layers;             /* kept blocks the error was measured on */
  double host_ms;              /* host wall time spent issuing this step's work */
  int64_t reserve_bytes;       /* scheduler reserve the plan was generated with */
} mimose_step_report;

typedef void (*mimose_grad_hook)(void* user, float* grads, int64_t n, void* stream);

int mimose_trainer_create(mimose_ctx* ctx, const mimose_model_cfg* m, const mimose_train_cfg* t,
                          mimose_trainer** out);
int mimose_trainer_destroy(mimose_trainer* tr);
/* Full step from HOST inputs (pinned for async copies): H2D, forward,
 * backward, grad hook, AdamW, loss D2H (synchronises the stream).
 * tokens/types: [batch*seq] int32, labels: [batch/num_choices] int32. */
int mimose_trainer_step(mimose_trainer* tr, const int32_t* tokens, const int32_t* types,
                        const int32_t* labels, int batch, int seq, void* stream,
                        mimose_step_report* rep);
/* Pipelined variant: same work, but the loss read-back is left in flight
 * (pinned ring of 4); fetch it with mimose_trainer_loss. Lets the host issue
 * step i+1 while step i runs. */
int mimose_trainer_step_async(mimose_trainer* tr, const int32_t* tokens, const int32_t* types,
                              const int32_t* labels, int batch, int seq, void* stream,
                              mimose_step_report* rep);
int mimose_trainer_loss(mimose_trainer* tr, int64_t iter, float* loss);
/* Same as mimose_trainer_step, without the optimizer (gradients left in the flat grad buffer). */
int mimose_trainer_forward_backward(mimose_trainer* tr, const int32_t* tokens,
                                    const int32_t* types, const int32_t* labels, int batch,
                                    int seq, void* stream, mimose_step_report* rep);
/* Step from DEVICE-resident inputs (no host sync; loss stays on device).
 * perm/seg/uid: token tables from mimose_build_token_tables. */
int mimose_trainer_step_device(mimose_trainer* tr, const int32_t* tokens, const int32_t* types,
                               const int32_t* labels, const int32_t* perm, const int32_t* seg,
                               const int32_t* uid, int n_unique, int batch, int seq,
                               int do_optimizer, void* stream, mimose_step_report* rep);
int mimose_trainer_optimizer_step(mimose_trainer* tr, float grad_scale, void* stream);
/* Force a plan (block ids) for subsequent steps (active=0 restores the planner). */
int mimose_trainer_force_plan(mimose_trainer* tr, const int* ids, int n, int active);
int mimose_trainer_set_grad_hook(mimose_trainer* tr, mimose_grad_hook fn, void* user);

/* Device buffers: fp32 master params, bf16 params, fp32 grads (flat). */
int mimose_trainer_buffers(mimose_trainer* tr, float** p32, void** p16, float** g32,
                           int64_t* n, float** d_loss, float** d_logits);
int mimose_trainer_param_count(mimose_trainer* tr);
int mimose_trainer_param_info(mimose_trainer* tr, int i, const char** name, int64_t* offset,
                              int64_t* numel);
/* Re-derive the bf16 copy after params_f32 was written externally. */
int mimose_trainer_sync_params(mimose_trainer* tr, void* stream);

/* Planner state as the reference's own text formats (caller frees with
 * mimose_free_string): collected samples (collector.hpp:198 CSV), fitted
 * estimator (estimator.hpp:182 dump), model document (model_spec.hpp:268). */
int mimose_trainer_samples_csv(mimose_trainer* tr, char** out);
int mimose_trainer_estimator_text(mimose_trainer* tr, char** out);
int mimose_trainer_model_text(mimose_trainer* tr, char** out);
/* The run so far through the reference's report writers (harness.hpp:339-379):
 * IterationRow CSV + key/value summary, with MEASURED peaks (arena) and
 * device milliseconds per iteration; recompute_ms from the fitted per-block
 * forward-time model; plain_* from that model (3 x sum f). */
int mimose_trainer_report(mimose_trainer* tr, char** summary, char** csv);
int mimose_trainer_info(mimose_trainer* tr, int64_t* constant_bytes, int64_t* reserve_bytes,
                        int64_t* budget, int* trained, int64_t* cache_hits,
                        int64_t* cache_misses);
void mimose_free_string(char* s);

/* Host helper: stable counting sort of token ids for the deterministic
 * word-embedding gradient. perm: [T], seg: [T+1], uid: [T]. */
int mimose_build_token_tables(const int32_t* tokens, int64_t T, int vocab, int32_t* perm,
                              int32_t* seg, int32_t* uid, int* n_unique);

/* ------------------------------------------------------- layer-level ABI
 * the per-unit operations of one training iteration, so a
 * caller can run the reference's training loop itself - the Mimose branch of
 * reference harness.hpp:215-296 with its simulate_iteration /
 * collect_iteration calls (harness.hpp:189,196,221,231,240,265,286) replaced
 * by these (tests/host/harness_gpu.cpp does exactly that, with the planner
 * from mimose_planner.h). Every buffer is a block of the trainer's budget
 * arena; buffers the library allocates are released with mimose_free.
 * A checkpoint unit is a transformer block (mimose_train_cfg.ckpt_unit 0) or
 * a block half (1: unit 2l = attention half of block l, 2l + 1 = FFN half). */
typedef struct mimose_saved mimose_saved;  /* saved set of one unit / the embeddings */
typedef struct {
  const int32_t* tokens;        /* device [batch*seq] */
  const int32_t* types;         /* device [batch*seq] (zeros when type_vocab == 0) */
  const int32_t* labels;        /* device, the head's layout (mimose_trainer_step) */
  const int32_t* perm;          /* device token tables (mimose_build_token_tables) */
  const int32_t* seg;
  const int32_t* uid;
  int n_unique;
  int batch, seq;
  int64_t step;                 /* iteration index: selects the dropout (Philox) streams */
} mimose_layer_io;

int mimose_trainer_units(mimose_trainer* tr, int* n_units);
/* *h0 = dropout(LN(word + pos + type)) (BERT) | dropout(word + pos) (GPT-2); *saved
 * receives the embedding's saved set. */
int mimose_embed_fwd(mimose_trainer* tr, const mimose_layer_io* io, void** h0,
                     mimose_saved** saved, void* stream);
/* Unit forward x_in -> x_out ([batch*seq][hidden] bf16, caller's arena block).
 * saved == NULL: no-save forward (the unit is dropped: only x_out stays);
 * else *saved receives the unit's saved set. Either way the unit's checkpoint
 * boundary is x_out plus (post-LN models) the output LayerNorm's statistics,
 * 8 B per token, which the trainer holds until the unit's backward (its LN
 * backward reads x-hat from the output). x_out must stay allocated until
 * mimose_layer_bwd of the unit. */
int mimose_layer_fwd(mimose_trainer* tr, int unit, const mimose_layer_io* io, const void* x_in,
                     void* x_out, mimose_saved** saved, void* stream);
/* Recompute of a dropped unit before its backward (reference: the
 * checkpointed layer's second forward, simulator.hpp:142-155): x_out is the
 * output this step's mimose_layer_fwd wrote (still held); only what the
 * backward reads is regenerated - same kernels and Philox streams, so the
 * saved set is bit-identical to a saving forward's - and the output
 * projection + LayerNorm that produced x_out are not rerun. *saved receives
 * the saved set. Fails when the unit's boundary is not held (e.g. a
 * both-halves-dropped block's attention half whose output was released: run
 * mimose_layer_fwd with saved != NULL for it instead). */
int mimose_layer_recompute(mimose_trainer* tr, int unit, const mimose_layer_io* io,
                           const void* x_in, void* x_out, mimose_saved** saved, void* stream);
/* Gives up a unit's boundary before its backward (the caller is about to free
 * x_out, e.g. the attention half of a block whose two halves are dropped):
 * releases the output statistics the trainer holds for it. */
int mimose_layer_release(mimose_trainer* tr, int unit);
/* Unit backward: consumes dy (arena block, grad of x_out) and saved; *dx =
 * grad of x_in (arena block). Units are differentiated last to first. */
int mimose_layer_bwd(mimose_trainer* tr, int unit, const mimose_layer_io* io, const void* x_in,
                     mimose_saved* saved, void* dy, void** dx, void* stream);
/* Final LayerNorm (GPT-2) + task head forward, loss (mimose_trainer_buffers
 * d_loss) and head backward; *dlast = grad of the last unit's output. */
int mimose_head_fwd_bwd(mimose_trainer* tr, const mimose_layer_io* io, const void* last,
                        void** dlast, void* stream);
/* Embedding backward: consumes dh0, h0 and the embedding's saved set. */
int mimose_embed_bwd(mimose_trainer* tr, const mimose_layer_io* io, mimose_saved* saved,
                     void* h0, void* dh0, void* stream);
int mimose_saved_free(mimose_trainer* tr, mimose_saved* saved);
/* Fused AdamW over the flat parameters (global-norm clipping; grad_scale on
 * the raw gradients). Same as mimose_trainer_optimizer_step. */
int mimose_adamw_step(mimose_trainer* tr, float grad_scale, void* stream);
/* Timing for the collector (cudaEvent wrappers; elapsed synchronises on end). */
int mimose_event_create(void** ev);
int mimose_event_record(void* ev, void* stream);
int mimose_event_elapsed(void* start, void* end, float* ms);
int mimose_event_destroy(void* ev);

/* ---- data parallelism (§8(b2) mimose_dp_*) --------------
 * One NCCL communicator per rank (NCCL resolved at run time). The unique id
 * (128 bytes) is made on rank 0 and broadcast by the caller (the reference
 * has no DP: SPEC.md:196 - this is new surface). */
int mimose_dp_unique_id(void* out128);
int mimose_dp_create(int device, const void* unique_id128, int rank, int world, mimose_dp** out);
/* Injectable transport: the same bucket schedule and comm-stream ordering,
 * but every reduction is handed to `fn` (buf: device pointer of n elements,
 * dtype 0 fp32 / 1 bf16, op 0 sum / 1 max, stream: the comm stream, already
 * ordered behind the backward work that produced the bucket). fn must leave
 * the cross-rank result in place (stream-ordered or synchronously) and
 * return 0. Used to run several ranks on one GPU (tests). */
typedef int (*mimose_dp_reduce_fn)(void* user, void* buf, int64_t n, int dtype, int op,
                                   void* stream);
int mimose_dp_create_custom(int device, int rank, int world, mimose_dp_reduce_fn fn, void* user,
                            mimose_dp** out);
/* Device bytes the NCCL communicator holds outside the budget arena (measured
 * around its init and first collective); 0 for custom transports. */
int mimose_dp_device_bytes(mimose_dp* dp, int64_t* out);
int mimose_dp_destroy(mimose_dp* dp);
/* in-place all-reduce of n elements; dtype 0 fp32 / 1 bf16, op 0 sum / 1 max */
int mimose_dp_allreduce(mimose_dp* dp, void* buf, int64_t n, int dtype, int op, void* stream);
/* Attach (dp != NULL) or detach: the trainer then sums its gradients across
 * ranks in buckets of >= bucket_bytes on the communicator's own stream as the
 * backward finishes each layer, and the optimizer waits for the last bucket
 * and scales by 1/world. */
int mimose_trainer_attach_dp(mimose_trainer* tr, mimose_dp* dp, int64_t bucket_bytes);
/* The bucket schedule in use: triples {after_unit, begin, end} (elements of
 * the flat gradient buffer; unit 0 = embeddings, 1..L = blocks, L+1 = head).
 * Returns the count in *n (at most cap triples written). */
int mimose_trainer_dp_buckets(mimose_trainer* tr, int64_t* triples, int cap, int* n);
/* Host-only: the same schedule for arbitrary unit offsets (n_units + 1 values). */
int mimose_dp_plan_buckets(const int64_t* unit_off, int n_units, int64_t bucket_elems,
                           int64_t* triples, int cap, int* n);

#ifdef __cplusplus
}
#endif

#endif /* MIMOSE_CUDA_H_ */
