/*
 * distattn_b200 — C ABI of the B200-native sequence-parallel causal attention
 * hot path (DistFlashAttn, arxiv 2310.03294).
 *
 * Every entry point replaces one function of the reference's C++ API in
 * /root/reference/proj/include/distattn (cited per declaration). Conventions:
 *   - device pointers owned by the caller, explicit CUDA stream (passed as
 *     void* so the header needs no CUDA include), no allocation on the hot
 *     path except the library's own small TMA-descriptor staging;
 *   - per-rank tensors are contiguous [heads, rows, d]: q/k/v/O bf16,
 *     accumulators o fp32 [H, rows, d], statistics m/l/lse/D fp32 [H, rows];
 *   - d = 128 (the Llama-shaped path the kernels are written for);
 *   - status codes mirror the reference exception taxonomy
 *     (errors.hpp:12-48); da_last_error() returns the thread-local message.
 *
 * Workers are 1-indexed as in the reference (schedule.hpp:7-8).
 */
#ifndef DISTATTN_B200_H
#define DISTATTN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define DA_ABI_VERSION 3

typedef enum da_status {
  DA_OK = 0,
  DA_ERR_SHAPE = 1,          /* ShapeError          errors.hpp:18-21 */
  DA_ERR_CONFIG = 2,         /* ConfigError         errors.hpp:24-27 */
  DA_ERR_SCHEDULE = 3,       /* ScheduleError       errors.hpp:30-33 */
  DA_ERR_STATE = 4,          /* StateError          errors.hpp:37-40 */
  DA_ERR_DEGENERATE_ROW = 5, /* DegenerateRowError  errors.hpp:45-48 */
  DA_ERR_CUDA = 6,           /* CUDA runtime / launch failure */
  DA_ERR_NCCL = 7,           /* NCCL failure (distributed runtime) */
  DA_ERR_UNSUPPORTED = 8     /* shape outside the sm_100a kernels (d != 128, ...) */
} da_status;

/* MaskMode, flashcore.hpp:30 */
typedef enum da_mask_mode { DA_MASK_DIAGONAL = 0, DA_MASK_FULL = 1, DA_MASK_EMPTY = 2 } da_mask_mode;

const char* da_last_error(void);
int da_abi_version(void);
/* 1 when the library was built for sm_100a and a device of that arch is present. */
int da_device_supported(void);

/* ------------------------------------------------------------------------
 * Per-chunk attention forward.
 *
 * Replaces block_attn_update (flashcore.hpp:135-197), fused with the
 * rescale merge of an incoming accumulator (flashcore.hpp:202-224) and,
 * when finalize != 0, with finalize (flashcore.hpp:227-240).
 *
 *   acc_in  = (o_in, m_in, l_in)  — NULL o_in means AttnAccumulator::fresh
 *   result  = rescale(acc_in, update(fresh, q, k, v, mask))
 *   finalize == 0: result -> (o_acc, m_acc, l_acc)  (may alias acc_in)
 *   finalize != 0: O = o / l -> o_out (bf16), lse = m + ln l -> lse_out;
 *                  rows with l <= 0 set *degenerate_flag (device int) to 1.
 *
 * m is kept in natural-log units of scale*q.k like the reference; the
 * kernel's lazy rescaling may leave m below the row maximum, which is a
 * valid accumulator representation (o/l and m + ln l are invariant).
 * GQA: q head h reads kv head h / (h_q / h_kv).
 * ------------------------------------------------------------------------ */
typedef struct da_fwd_args {
  const void* q; /* bf16 [h_q, rows_q, d]  */
  const void* k; /* bf16 [h_kv, rows_kv, d] */
  const void* v; /* bf16 [h_kv, rows_kv, d] */
  int64_t h_q, h_kv, rows_q, rows_kv, d;
  const float* o_in; /* fp32 [h_q, rows_q, d] or NULL */
  const float* m_in; /* fp32 [h_q, rows_q] */
  const float* l_in;
  float* o_acc; /* finalize == 0 */
  float* m_acc;
  float* l_acc;
  void* o_out;    /* bf16, finalize != 0 */
  float* lse_out; /* fp32 [h_q, rows_q] */
  int* degenerate_flag; /* optional device int */
  float scale;          /* <= 0 selects 1/sqrt(d) (runtime.cpp:150) */
  int mask;             /* da_mask_mode */
  int finalize;
} da_fwd_args;

da_status da_attn_fwd_chunk(const da_fwd_args* args, void* stream);

/* rescale (flashcore.hpp:202-224): (o,m,l)_out = a ⊕ b over [h, rows]. Out may alias a. */
da_status da_attn_merge(const float* o_a, const float* m_a, const float* l_a, const float* o_b,
                        const float* m_b, const float* l_b, float* o_out, float* m_out,
                        float* l_out, int64_t h, int64_t rows, int64_t d, void* stream);

/* finalize (flashcore.hpp:227-240): O = o/l (bf16), lse = m + ln l; degenerate rows flagged. */
da_status da_attn_finalize(const float* o, const float* m, const float* l, void* o_out,
                           float* lse_out, int* degenerate_flag, int64_t h, int64_t rows,
                           int64_t d, void* stream);

/* Reads back a device degenerate flag (synchronises the stream): DA_OK or
 * DA_ERR_DEGENERATE_ROW, the reference's DegenerateRowError. */
da_status da_check_degenerate(const int* degenerate_flag, void* stream);

/* ------------------------------------------------------------------------
 * Backward.
 *
 * da_attn_bwd_preprocess replaces backward_aux (flashcore.hpp:250-261):
 *   D = rowsum(dO ∘ O) computed once per query chunk (the reference
 *   recomputes it inside every block_attn_backward call, :294).
 *
 * da_attn_bwd_chunk replaces block_attn_backward (flashcore.hpp:269-337):
 *   P = exp(scale q kᵀ − lse), dv += Pᵀ dO, dS = P ∘ (dO vᵀ − D),
 *   dq += scale dS k, dk += scale dSᵀ q.
 *   dq_acc is fp32 [h_q, rows_q, d] and is always accumulated into
 *   (the reference's `s.dq += g.dq`, runtime.cpp:620,633).
 *   dk_acc / dv_acc are fp32 [h_kv, rows_kv, d]; accumulate_kv != 0 adds,
 *   otherwise overwrites (the reference returns the contribution, :290-291).
 *   lse is the GLOBAL logsumexp of the query rows (flashcore.hpp:263-266).
 * ------------------------------------------------------------------------ */
da_status da_attn_bwd_preprocess(const void* d_out, const void* out, float* d_vec, int64_t h,
                                 int64_t rows, int64_t d, void* stream);

typedef struct da_bwd_args {
  const void* q;     /* bf16 [h_q, rows_q, d] */
  const void* k;     /* bf16 [h_kv, rows_kv, d] */
  const void* v;     /* bf16 [h_kv, rows_kv, d] */
  const void* d_out; /* bf16 [h_q, rows_q, d] */
  const float* lse;  /* fp32 [h_q, rows_q] */
  const float* d_vec; /* fp32 [h_q, rows_q] from da_attn_bwd_preprocess */
  int64_t h_q, h_kv, rows_q, rows_kv, d;
  float* dq_acc; /* fp32 [h_q, rows_q, d], += */
  float* dk_acc; /* fp32 [h_kv, rows_kv, d] */
  float* dv_acc;
  int accumulate_kv;
  float scale;
  int mask;
  /* deterministic != 0: the fp32 dq partials of the kv tiles are added in a
   * fixed order (descending kv tile, enforced by per-(head, q tile)
   * semaphores), so dq_acc is bitwise reproducible run to run. Default 0 is
   * the faster unordered reduction (results agree to fp32 rounding). */
  int deterministic;
} da_bwd_args;

da_status da_attn_bwd_chunk(const da_bwd_args* args, void* stream);

/* fp32 -> bf16 conversion of gradient accumulators (dq/dk/dv outputs). */
da_status da_convert_f32_bf16(const float* src, void* dst, int64_t n, void* stream);

/* ------------------------------------------------------------------------
 * Host-buffer forms (fp64, row-major, ONE head: the reference's Mat<double>
 * per-head layout, numerics.hpp:26-32). What the signature-level drop-in
 * include/distattn/flashcore.hpp calls, so the reference's own call sites
 * (runtime.cpp:286-328, 605-716; ckptplan.cpp:146-155, 198-206) run on the
 * sm_100a kernels. Operands are rounded to the product precision on upload
 * (bf16 q/k/v/O/dO, fp32 accumulator and statistics); every call is
 * synchronous on a per-thread stream with per-thread staging buffers that
 * are grown once and reused (no allocation per call). d must be 128.
 * ------------------------------------------------------------------------ */
/* block_attn_update (flashcore.hpp:135-197): (o, m, l) updated in place; an
 * accumulator with every m = -inf and l = 0 is AttnAccumulator::fresh. */
da_status da_host_attn_update(const double* q, int64_t rows_q, const double* k, const double* v,
                              int64_t rows_kv, int64_t d, double* o, double* m, double* l,
                              int mask, double scale);
/* rescale (flashcore.hpp:202-224); the output may alias an input. */
da_status da_host_attn_merge(const double* o_a, const double* m_a, const double* l_a,
                             const double* o_b, const double* m_b, const double* l_b,
                             double* o_out, double* m_out, double* l_out, int64_t rows,
                             int64_t d);
/* finalize (flashcore.hpp:227-240): DA_ERR_DEGENERATE_ROW when a row has l <= 0. */
da_status da_host_attn_finalize(const double* o, const double* m, const double* l, int64_t rows,
                                int64_t d, double* out, double* lse);
/* backward_aux (flashcore.hpp:250-261). */
da_status da_host_backward_aux(const double* d_out, const double* out, int64_t rows, int64_t d,
                               double* d_vec);
/* block_attn_backward (flashcore.hpp:269-337): contributions dq [rows_q, d],
 * dk / dv [rows_kv, d] (overwritten); D = rowsum(dO o O) computed inside.
 * dq partials are added in a fixed order: bitwise reproducible. */
da_status da_host_attn_backward(const double* q, int64_t rows_q, const double* k,
                                const double* v, int64_t rows_kv, int64_t d, const double* out,
                                const double* lse, const double* d_out, int mask, double scale,
                                double* dq, double* dk, double* dv);
/* dense_oracle (flashcore.hpp:92-128) as one chunk launch: causal needs
 * rows_q == rows_kv (the Diagonal mask). */
da_status da_host_dense_attention(const double* q, int64_t rows_q, const double* k,
                                  const double* v, int64_t rows_kv, int64_t d, int causal,
                                  double scale, double* out, double* lse);

/* ------------------------------------------------------------------------
 * Host-buffer causal attention step with the PCIe copies overlapped per
 * head group (C++ host layer; the reference's runtime takes host matrices,
 * runtime.hpp:32-41, and prefetches the next operand during the current
 * compute, runtime.cpp:280-284). One step = forward (fused finalize) +
 * backward_aux + backward of a whole causal sequence on this GPU:
 *   in:  pinned host bf16 q [heads, rows, 128], k / v [heads_kv, rows, 128], dO
 *   out: pinned host bf16 dQ [heads, ...], dK / dV [heads_kv, ...]
 * The saved O / LSE stay on the device (da_pipeline_outputs). Consecutive
 * steps overlap (step i+1's copy-in of group g waits only for step i's
 * compute of group g). sync != 0 joins onto `stream` and checks degenerate
 * rows (DA_ERR_DEGENERATE_ROW); else call da_pipeline_join later.
 * ------------------------------------------------------------------------ */
typedef struct da_pipeline da_pipeline;
da_status da_pipeline_create(int64_t heads, int64_t heads_kv, int64_t rows, int64_t d,
                             int64_t heads_per_group, int compute_streams, da_pipeline** out);
void da_pipeline_destroy(da_pipeline* p);
da_status da_pipeline_step(da_pipeline* p, const void* hq, const void* hk, const void* hv,
                           const void* hdo, void* hdq, void* hdk, void* hdv, int sync,
                           void* stream);
/* `stream` waits for every step issued so far; check_degenerate != 0 also
 * reads the degenerate-row flag back (synchronises the stream). */
da_status da_pipeline_join(da_pipeline* p, void* stream, int check_degenerate);
/* Copies the last step's saved O (bf16 [heads, rows, 128]) and LSE (fp32
 * [heads, rows]) into caller device buffers (either may be NULL), in order
 * on `stream` after every step issued so far. */
da_status da_pipeline_outputs(da_pipeline* p, void* out, float* lse, void* stream);

/* ------------------------------------------------------------------------
 * Schedules (schedule.hpp:21-119, schedule.cpp:60-108).
 *
 * Flat, field-exact encoding of Schedule:
 *   tasks[i] = {step, kind, worker, query_owner, kv_owner, helper} (int32 x 6)
 *     kind: 0 LocalAttn, 1 RemoteAttn, 2 RescaleMerge, 3 Idle (TaskKind order)
 *     tasks appear step by step, P primaries ascending by worker then merges;
 *   messages[i] = {step, from, to, kind} (int32 x 4)
 *     kind: 0 KV, 1 Q, 2 PartialResult, 3 GradKV (PayloadKind order),
 *           4 KVHalf (half of a kv chunk's rows; DA_SCHEDULE_BALANCED_SPLIT).
 * Call once with NULL buffers to size them (counts are always written).
 * ------------------------------------------------------------------------ */
typedef enum da_schedule_kind {
  DA_SCHEDULE_RING = 0,         /* build_ring_schedule       schedule.cpp:60-77 */
  DA_SCHEDULE_BALANCED = 1,     /* build_balanced_schedule   schedule.cpp:79-108 */
  /* Backward schedules. The reference's backward is ring-only
   * (BackwardMode::Vanilla, runtime.hpp:110); RING_BWD makes its order explicit
   * (runtime.cpp:605-651), BALANCED_BWD is the load-balanced extension (SURVEY
   * §8(f)1): the forward task table with KV/GradKV for direct pairs,
   * Q = (q, dO, lse, D) bundle to the helper and Partial = dq contribution back. */
  DA_SCHEDULE_RING_BWD = 2,
  DA_SCHEDULE_BALANCED_BWD = 3,
  /* Forward extension (not in the reference): balanced with
   * the even-P last step split. At t = P/2 helper p computes the pair
   * (p + P/2, p) on the low half of its kv rows and the owner on the high
   * half, so no worker idles; the step costs half a chunk pair. For
   * RemoteAttn tasks the `helper` slot carries the kv row part:
   * 0 whole chunk, 1 rows [0, c/2), 2 rows [c/2, c). The owner's half arrives
   * as message kind 4 (KVHalf). Odd P: identical to DA_SCHEDULE_BALANCED. */
  DA_SCHEDULE_BALANCED_SPLIT = 4,
  /* Backward of the split schedule (extension): the DA_SCHEDULE_BALANCED_SPLIT
   * task table with the backward messages of BALANCED_BWD. At t = P/2 the
   * owner computes its pair on the high half of the kv rows (KVHalf in, the
   * half's GradKV back to the kv owner) and the helper on the low half (the
   * Q bundle in, the dq Partial back); the helper keeps its low half's dk/dv.
   * Odd P: identical to DA_SCHEDULE_BALANCED_BWD. */
  DA_SCHEDULE_BALANCED_SPLIT_BWD = 5
} da_schedule_kind;

da_status da_schedule_build(int workers, int kind, int32_t* steps_out, int32_t* tasks,
                            int64_t* n_tasks, int32_t* messages, int64_t* n_messages);

/* validate (schedule.cpp:121-258): returns the violation count; when nonzero
 * da_last_error() holds every violation message, newline-separated.
 * Negative on bad input. */
int64_t da_schedule_validate(int workers, int32_t steps, const int32_t* tasks, int64_t n_tasks,
                             const int32_t* messages, int64_t n_messages);

/* validate plus GradKV coverage for backward schedules (every direct pair
 * returns its dk/dv to the kv owner no earlier than its step). */
int64_t da_schedule_validate_backward(int workers, int32_t steps, const int32_t* tasks,
                                      int64_t n_tasks, const int32_t* messages,
                                      int64_t n_messages);

/* ------------------------------------------------------------------------
 * Peer-memory transport signals (replaces the message channel of the
 * reference's concurrent executor, runtime.cpp:413-487, for one process per
 * GPU): 32-bit monotonic counters in device memory, written and awaited by
 * stream memory operations, so ranks order their copy-engine pulls from each
 * other's HBM without host synchronisation or NCCL kernels.
 *   da_stream_write_u32:    *addr = value once prior work on `stream` is done
 *   da_stream_wait_u32_geq: `stream` waits until (int)(*addr - value) >= 0
 * addr may be local or a peer allocation mapped through CUDA IPC.
 * ------------------------------------------------------------------------ */
da_status da_stream_write_u32(void* stream, void* addr, uint32_t value);
da_status da_stream_wait_u32_geq(void* stream, const void* addr, uint32_t value);

/* ------------------------------------------------------------------------
 * Runtime (runtime.cpp:491-529, 720-750), P logical workers on ONE device —
 * the reference's stepper executor with device kernels: per step, every
 * worker's action runs in schedule order; "messages" are device buffers.
 * Shards are arrays of P device pointers, each [h, rows, d] (rows = N/P).
 * ------------------------------------------------------------------------ */
typedef struct da_shards {
  int32_t workers;
  int64_t h_q, h_kv, rows, d;
  const void* const* q; /* P pointers, bf16 */
  const void* const* k;
  const void* const* v;
  void* const* out;     /* bf16 O, written by forward  (SequenceShard.out) */
  float* const* lse;    /* fp32, written by forward    (SequenceShard.lse) */
  const void* const* d_out; /* bf16, read by backward (SequenceShard.d_out) */
  float* const* dq;     /* fp32, written by backward */
  float* const* dk;
  float* const* dv;
} da_shards;

typedef struct da_counters {
  /* CommCounters, runtime.hpp:49-63 (scalars per payload kind), plus bytes */
  int64_t kv_scalars, q_scalars, partial_scalars, grad_scalars;
  int64_t kv_messages, q_messages, partial_messages, grad_messages;
  int64_t attention_kernel_calls;
  int32_t max_remote_chunks_held;
} da_counters;

/* schedule_kind: da_schedule_kind. workspace is allocated internally on the
 * first call and cached per thread (not on the timed hot path). */
da_status da_run_forward(const da_shards* shards, int schedule_kind, da_counters* counters,
                         void* stream);
da_status da_run_backward(const da_shards* shards, da_counters* counters, void* stream);
/* run_backward with an explicit backward schedule (DA_SCHEDULE_RING_BWD is
 * identical to da_run_backward; DA_SCHEDULE_BALANCED_BWD balances the causal
 * pairs like the forward). */
da_status da_run_backward_sched(const da_shards* shards, int schedule_kind, da_counters* counters,
                                void* stream);
/* run_forward / run_backward over a caller-supplied schedule table in the
 * flat encoding of da_schedule_build (runtime.hpp:106-118 take `const
 * Schedule&`): any table that passes validate (schedule.cpp:121-258; the
 * backward one da_schedule_validate_backward) runs, else DA_ERR_SCHEDULE with
 * the first violation. */
da_status da_run_forward_table(const da_shards* shards, int32_t steps, const int32_t* tasks,
                               int64_t n_tasks, const int32_t* messages, int64_t n_messages,
                               da_counters* counters, void* stream);
da_status da_run_backward_table(const da_shards* shards, int32_t steps, const int32_t* tasks,
                                int64_t n_tasks, const int32_t* messages, int64_t n_messages,
                                da_counters* counters, void* stream);
/* Frees the cached runtime workspaces (one per stream; waits for each stream). */
void da_runtime_release(void);

/* ------------------------------------------------------------------------
 * Per-rank runtime: one process per GPU, each holding ONE contiguous chunk
 * of the sequence — the reference's worker (runtime.cpp:390-487 concurrent
 * executor, 653-716 backward). A pass is a fixed sequence of phases,
 * identical on every rank: operands(0), then per step t operands(t+1)
 * (prefetch depth 1, runtime.cpp:280-284) and results(t) (partials,
 * GradKV, dq partials), all on a high-priority side stream. Transports:
 *   DA_TRANSPORT_NCCL  one ncclGroupStart/Send/Recv/GroupEnd per phase
 *                      (NCCL is dlopen'ed: libnccl.so.2);
 *   DA_TRANSPORT_IPC   copy-engine pulls from the peer's HBM (CUDA IPC)
 *                      ordered by device counters (da_stream_write_u32 /
 *                      wait); ranks may share one GPU;
 *   DA_TRANSPORT_NONE  no transfer: receive slots are filled once from the
 *                      rank's own buffers — the same kernels on local data,
 *                      the no-communication timing arm (analyzer.cpp:60-64).
 * deterministic != 0 orders every dq reduction (bitwise reproducible
 * backward; the reference's executors are, runtime.hpp:7-9).
 *
 * Bootstrap (IPC handles, the NCCL unique id) and per-pass IPC publication
 * go through the caller's allgather (e.g. torch.distributed, MPI):
 * `fn(ctx, send, bytes, recv)` must gather `bytes` from every rank into
 * recv[world * bytes] in rank order and return 0. All da_rank_* calls are
 * collective over the ranks. Forward: q [h_q, rows, 128], k/v [h_kv, rows,
 * 128] bf16 of this rank; writes out (bf16) and lse (fp32) and keeps them (the
 * rematerialisation state) for da_rank_backward, which writes fp32 dq [h_q],
 * dk/dv [h_kv]. schedule_kind: DA_SCHEDULE_RING / BALANCED / BALANCED_SPLIT
 * (forward), DA_SCHEDULE_RING_BWD / BALANCED_BWD (backward).
 * ------------------------------------------------------------------------ */
typedef int (*da_allgather_fn)(void* ctx, const void* send, uint64_t bytes, void* recv);
typedef struct da_rank da_rank;

#define DA_TRANSPORT_IPC 0
#define DA_TRANSPORT_NCCL 1
#define DA_TRANSPORT_NONE 2

typedef struct da_rank_options {
  int transport;     /* DA_TRANSPORT_* */
  int deterministic; /* ordered dq reductions in every backward chunk */
  int nccl_max_ctas; /* > 0: cap the CTAs of NCCL's kernels (SMs left to attention) */
} da_rank_options;

/* da_rank_create = da_rank_create_ex with {DA_TRANSPORT_IPC, 0, 0}. */
da_status da_rank_create(int rank, int world, da_allgather_fn fn, void* ctx, da_rank** out);
da_status da_rank_create_ex(int rank, int world, da_allgather_fn fn, void* ctx,
                            const da_rank_options* opts, da_rank** out);
void da_rank_destroy(da_rank* r);
da_status da_rank_forward(da_rank* r, int schedule_kind, const void* q, const void* k,
                          const void* v, int64_t h_q, int64_t h_kv, int64_t rows, void* out,
                          float* lse, da_counters* counters, void* stream);
da_status da_rank_backward(da_rank* r, int schedule_kind, const void* d_out, float* dq, float* dk,
                           float* dv, da_counters* counters, void* stream);
/* The same passes over a caller-supplied validated schedule table (the flat
 * encoding of da_schedule_build; runtime.hpp:106-118 take `const Schedule&`).
 * Every rank must pass the same table. */
da_status da_rank_forward_table(da_rank* r, int32_t steps, const int32_t* tasks, int64_t n_tasks,
                                const int32_t* messages, int64_t n_messages, const void* q,
                                const void* k, const void* v, int64_t h_q, int64_t h_kv,
                                int64_t rows, void* out, float* lse, da_counters* counters,
                                void* stream);
da_status da_rank_backward_table(da_rank* r, int32_t steps, const int32_t* tasks, int64_t n_tasks,
                                 const int32_t* messages, int64_t n_messages, const void* d_out,
                                 float* dq, float* dk, float* dv, da_counters* counters,
                                 void* stream);
/* Re-installs a saved forward state (this rank's q, k, v, O, LSE of an
 * earlier pass) for the next da_rank_backward — the rematerialisation hook
 * of a checkpointed multi-layer model (ckptplan.cpp:198-206): each layer's
 * attention backward uses its own saved O / LSE, never a recompute. */
da_status da_rank_restore(da_rank* r, const void* q, const void* k, const void* v, void* out,
                          float* lse, int64_t h_q, int64_t h_kv, int64_t rows);
/* Wall-clock trace (the reference's ExecutionTrace,
 * runtime.hpp:66-89): with tracing on, every following pass records CUDA
 * events around each task kernel and each message phase. da_rank_trace
 * resolves the last pass of `pass` (0 forward, 1 backward) into records, times
 * in ms from the pass origin (synchronises on the events once):
 *   kind 0 task     code 1 local / 2 remote (direct) / 3 helper / 4 merge /
 *                   5 fold (GradKV or dq partial); peer = the other worker
 *   kind 1 send     code = buffer key, peer = destination rank, t0 = t1 = issue
 *   kind 2 receive  code = buffer key, peer = source rank, t1 = arrival
 * (step = schedule step, phase = 2t operands(t) / 2t+1 results(t); -1 for tasks). */
typedef struct da_trace_rec {
  int32_t kind, code, step, peer, phase, pad;
  float t0_ms, t1_ms;
} da_trace_rec;
void da_rank_set_trace(da_rank* r, int on);
da_status da_rank_trace(da_rank* r, int pass, da_trace_rec* out, int64_t cap, int64_t* n);
/* The message protocol of one rank without a device: 5 int32 per entry
 * {pass (0 forward, 1 backward), phase (2t = operands(t), 2t+1 = results(t)),
 * dir (0 send, 1 receive), peer rank, buffer key}; *n = entries (written up to
 * cap; out may be NULL to count). Every send must meet exactly one receive
 * of the same key in the same phase (checked by tests/test_rank_protocol.py). */
da_status da_rank_protocol(int world, int rank, int fwd_kind, int bwd_kind, int32_t* out,
                           int64_t cap, int64_t* n);


/* Device fill with the reference's splitmix64 stream (numerics.hpp:140-174):
 * out[i] = lo + (hi - lo) * unit(draw i of the stream whose CURRENT state is
 * `state`), stored as dtype 0 = fp32, 1 = bf16 (via fp32, round-to-nearest-
 * even), 2 = fp64. The caller advances its state by n * 0x9E3779B97F4A7C15.
 * Used by make_shards (runtime.cpp:24-46) to build parity inputs on device. */
da_status da_rng_uniform(uint64_t state, int64_t n, double lo, double hi, int dtype, void* out,
                         void* stream);

/* Debug: device buffer receiving, in DA_TRACE builds only, the backward
 * kernel's per-iteration clock64 timeline of CTA 0 (64 x 16 uint64) followed
 * by 8 uint64 per CTA (globaltimer / clock64 start and end, SM id, iteration
 * count, first / last MMA issue): size it 1024 + 8 * grid. NULL disables. */
void da_debug_set_bwd_trace(void* buf);
/* Debug: same layout for the forward kernel. */
void da_debug_set_fwd_trace(void* buf);

/* Debug: compute the raw score block S = q kᵀ (fp32, unscaled) of the first
 * 128x128 tile of head 0 through the forward kernel's MMA path. */
da_status da_debug_scores(const void* q, const void* k, int64_t rows, float* s_out, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* DISTATTN_B200_H */
