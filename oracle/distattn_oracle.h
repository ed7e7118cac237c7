/*
 * distattn_oracle — plain-C restatement of the reference's CPU algorithm
 * (/root/reference/proj) for this hot path. TEST INFRASTRUCTURE ONLY: it is
 * the checker for the sm_100a kernels (tests/, __graft_entry__.smoke(),
 * bench.py's cpu_baseline leg) and is never linked into or called by the
 * product library.
 *
 * Pinned against the reference itself: tests/test_oracle.py compares it with
 * outputs of the unmodified reference sources (oracle/_ref/ref_driver, built
 * by oracle/Makefile) and with the golden vectors in tests/golden/.
 *
 * Matrices are row-major float64 like the reference's Matd (numerics.hpp:26-32).
 * Return codes follow include/distattn_b200.h (0 ok, 1 shape, 2 config,
 * 3 schedule, 4 state, 5 degenerate row).
 */
#ifndef DISTATTN_ORACLE_H
#define DISTATTN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Rng: splitmix64, numerics.hpp:140-174 */
typedef struct dao_rng {
  uint64_t state;
} dao_rng;
uint64_t dao_rng_next_u64(dao_rng* r);
double dao_rng_next_unit(dao_rng* r);
void dao_rng_fork(dao_rng* r, dao_rng* child);
void dao_rng_matrix(dao_rng* r, int64_t rows, int64_t cols, double lo, double hi, double* out);
double dao_bf16_round(double x);

/* Parity inputs: per head h, head_rng = Rng(seed).fork() (h+1-th
 * fork); make_shards draws full q, k, v (runtime.cpp:24-46); then d_out. All
 * outputs [H][N][D]. bf16 != 0 rounds every value to bf16. */
int dao_make_inputs(uint64_t seed, int workers, int64_t n, int64_t d, int heads, int bf16,
                    double* q, double* k, double* v, double* d_out);

/* Schedules, schedule.cpp:60-108; flat encoding as include/distattn_b200.h */
int dao_schedule_build(int workers, int kind, int32_t* steps, int32_t* tasks, int64_t* n_tasks,
                       int32_t* messages, int64_t* n_messages);

/* flashcore.hpp:135-197 (mask 0 Diagonal, 1 Full, 2 Empty). In place on o/m/l. */
int dao_block_attn_update(const double* q, int64_t rq, const double* k, const double* v,
                          int64_t rk, int64_t d, double* o, double* m, double* l, int mask,
                          double scale, int64_t block_rows, int64_t block_cols);
/* flashcore.hpp:202-224 ; out may alias a */
void dao_rescale(const double* oa, const double* ma, const double* la, const double* ob,
                 const double* mb, const double* lb, int64_t rows, int64_t d, double* o,
                 double* m, double* l);
/* flashcore.hpp:227-240 */
int dao_finalize(const double* o, const double* m, const double* l, int64_t rows, int64_t d,
                 double* out, double* lse);
/* flashcore.hpp:250-261 */
void dao_backward_aux(const double* d_out, const double* out, int64_t rows, int64_t d, double* dv);
/* flashcore.hpp:269-337 ; writes contributions (zeroed first) */
int dao_block_attn_backward(const double* q, int64_t rq, const double* k, const double* v,
                            int64_t rk, int64_t d, const double* out, const double* lse,
                            const double* d_out, int mask, double scale, int64_t block_rows,
                            int64_t block_cols, double* dq, double* dk, double* dv);
/* flashcore.hpp:96-128 */
int dao_dense_oracle(const double* q, const double* k, const double* v, int64_t n, int64_t nk,
                     int64_t d, int causal, double scale, double* out, double* lse);
/* reference.hpp:21-74 */
int dao_dense_backward(const double* q, const double* k, const double* v, const double* d_out,
                       int64_t n, int64_t nk, int64_t d, int causal, double scale, double* dq,
                       double* dk, double* dv);

/* Stepper executors over P workers holding contiguous chunks of one head:
 * run_forward (runtime.cpp:266-330, 491-529) and run_backward
 * (runtime.cpp:605-651, 720-750). q/k/v/out/d_out/grads are [N][D] for the
 * whole sequence (worker p owns rows [(p-1)N/P, pN/P)). counters: 8 x int64
 * CommCounters (runtime.hpp:49-63) + kernel calls + max remote held. */
int dao_run_forward(int workers, int kind, int64_t n, int64_t d, const double* q, const double* k,
                    const double* v, double* out, double* lse, int64_t* counters10);
int dao_run_backward(int workers, int64_t n, int64_t d, const double* q, const double* k,
                     const double* v, const double* out, const double* lse, const double* d_out,
                     double* dq, double* dk, double* dv, int64_t* counters10);

/* block_attn_backward with a caller-supplied D (from dao_backward_aux). */
int dao_block_attn_backward_with_d(const double* q, int64_t rq, const double* k, const double* v,
                                   int64_t rk, int64_t d, const double* d_vec, const double* lse,
                                   const double* d_out, int mask, double scale, int64_t block_rows,
                                   int64_t block_cols, double* dq, double* dk, double* dv);

/* Backward over an explicit schedule table (kind 0 ring, 1 balanced, 4 the
 * balanced schedule with the even-P split; a split step's tasks use the kv row
 * window of their part, and a split direct pair's GradKV covers its half):
 * EXTENSION, the reference has only the ring order. Local/direct tasks follow
 * runtime.cpp:605-651 (dq += immediately, GradKV folded at the end of the step
 * in ascending receiver order); a helper h for owner o computes the pair
 * (o, h), adds dk/dv to its own chunk immediately and returns dq, which the
 * owner folds at the end of the step in merge order. Ring reproduces
 * dao_run_backward bit-exactly. */
int dao_run_backward_sched(int workers, int kind, int64_t n, int64_t d, const double* q,
                           const double* k, const double* v, const double* out,
                           const double* lse, const double* d_out, double* dq, double* dk,
                           double* dv, int64_t* counters10);

#ifdef __cplusplus
}
#endif
#endif
