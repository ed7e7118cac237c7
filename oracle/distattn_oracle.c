/*
 * Plain-C restatement of the reference CPU algorithm for the DistFlashAttn hot
 * path. TEST INFRASTRUCTURE ONLY (see distattn_oracle.h).
 *
 * Bit-exactness with the reference: every reduction below runs in the
 * reference's order (left to right, the same loop nests) and is compiled with
 * -ffp-contract=off like the reference build. The only liberty taken is
 * computing each exp(s - m) once and reusing it where the reference
 * recomputes the identical expression inside an inner loop
 * (flashcore.hpp:184-190): exp is a pure function, so the bits agree while the
 * oracle runs ~d times faster.
 */
#include "distattn_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define NEG_INF (-INFINITY)

/* std::max(a, b) of the reference: returns a unless a < b */
static inline double smax(double a, double b) { return (a < b) ? b : a; }

/* ---------------- numerics.hpp:140-174 ---------------- */
uint64_t dao_rng_next_u64(dao_rng* r) {
  r->state += 0x9E3779B97F4A7C15ULL;
  uint64_t z = r->state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

double dao_rng_next_unit(dao_rng* r) { return (double)(dao_rng_next_u64(r) >> 11) * 0x1.0p-53; }

void dao_rng_fork(dao_rng* r, dao_rng* child) { child->state = dao_rng_next_u64(r); }

void dao_rng_matrix(dao_rng* r, int64_t rows, int64_t cols, double lo, double hi, double* out) {
  for (int64_t i = 0; i < rows * cols; ++i) out[i] = lo + (hi - lo) * dao_rng_next_unit(r);
}

double dao_bf16_round(double x) {
  float f = (float)x;
  uint32_t u;
  memcpy(&u, &f, 4);
  u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
  memcpy(&f, &u, 4);
  return (double)f;
}

int dao_make_inputs(uint64_t seed, int workers, int64_t n, int64_t d, int heads, int bf16,
                    double* q, double* k, double* v, double* d_out) {
  if (workers < 1) return 2;
  if (n < 1 || d < 1) return 2;
  if (n % workers != 0) return 2;
  dao_rng root = {seed};
  const int64_t sz = n * d;
  for (int h = 0; h < heads; ++h) {
    dao_rng hr;
    dao_rng_fork(&root, &hr);
    /* make_shards draws the full q, then k, then v (runtime.cpp:36-38) */
    dao_rng_matrix(&hr, n, d, -1.0, 1.0, q + h * sz);
    dao_rng_matrix(&hr, n, d, -1.0, 1.0, k + h * sz);
    dao_rng_matrix(&hr, n, d, -1.0, 1.0, v + h * sz);
    if (d_out) dao_rng_matrix(&hr, n, d, -1.0, 1.0, d_out + h * sz);
    if (bf16) {
      for (int64_t i = 0; i < sz; ++i) {
        q[h * sz + i] = dao_bf16_round(q[h * sz + i]);
        k[h * sz + i] = dao_bf16_round(k[h * sz + i]);
        v[h * sz + i] = dao_bf16_round(v[h * sz + i]);
        if (d_out) d_out[h * sz + i] = dao_bf16_round(d_out[h * sz + i]);
      }
    }
  }
  return 0;
}

/* ---------------- schedule.cpp:60-108 ---------------- */
typedef struct {
  int32_t* t;
  int64_t n;
} ivec;

static void push6(int32_t* buf, int64_t* n, int32_t a, int32_t b, int32_t c, int32_t dd,
                  int32_t e, int32_t f) {
  if (buf) {
    int32_t* o = buf + 6 * (*n);
    o[0] = a; o[1] = b; o[2] = c; o[3] = dd; o[4] = e; o[5] = f;
  }
  ++(*n);
}

static void push4(int32_t* buf, int64_t* n, int32_t a, int32_t b, int32_t c, int32_t dd) {
  if (buf) {
    int32_t* o = buf + 4 * (*n);
    o[0] = a; o[1] = b; o[2] = c; o[3] = dd;
  }
  ++(*n);
}

int dao_schedule_build(int P, int kind, int32_t* steps, int32_t* tasks, int64_t* n_tasks,
                       int32_t* msgs, int64_t* n_msgs) {
  if (P < 1) return 2;
  int64_t nt = 0, nm = 0;
  if (kind == 0) { /* ring, schedule.cpp:60-77 */
    *steps = P;
    for (int p = 1; p <= P; ++p) push6(tasks, &nt, 0, 0, p, p, p, 0);
    for (int t = 1; t < P; ++t)
      for (int p = 1; p <= P; ++p) {
        if (p > t) {
          push6(tasks, &nt, t, 1, p, p, p - t, 0);
          push4(msgs, &nm, t, p - t, p, 0);
        } else {
          push6(tasks, &nt, t, 3, p, 0, 0, 0);
        }
      }
  } else { /* balanced, schedule.cpp:79-108; kind 4 = the even-P split extension
             * (SURVEY §8(f)2): at t = P/2 helper p takes pair (p + P/2, p) on the
             * low half of its kv rows (part 1, in the helper slot of the task),
             * the owner the high half (part 2) via a KVHalf (kind 4) message */
    const int split = (kind == 4) && (P % 2 == 0);
    const int half = P / 2;
    *steps = half + 1;
    for (int p = 1; p <= P; ++p) push6(tasks, &nt, 0, 0, p, p, p, 0);
    int32_t* merges = (int32_t*)malloc(sizeof(int32_t) * 6 * (size_t)(P + 1));
    for (int t = 1; t <= half; ++t) {
      int64_t nmg = 0;
      for (int p = 1; p <= P; ++p) {
        const int last_split = split && t == half;
        if (p > t) {
          push6(tasks, &nt, t, 1, p, p, p - t, last_split ? 2 : 0);
          push4(msgs, &nm, t, p - t, p, last_split ? 4 : 0);
        } else if (P % 2 == 0 && t == half && !split) {
          push6(tasks, &nt, t, 3, p, 0, 0, 0);
        } else {
          const int owner = p + P - t;
          push6(tasks, &nt, t, 1, p, owner, p, last_split ? 1 : 0);
          push4(msgs, &nm, t, owner, p, 1);
          push4(msgs, &nm, t, p, owner, 2);
          push6(merges, &nmg, t, 2, owner, 0, 0, p);
        }
      }
      for (int64_t i = 0; i < nmg; ++i) {
        const int32_t* m = merges + 6 * i;
        push6(tasks, &nt, m[0], m[1], m[2], m[3], m[4], m[5]);
      }
    }
    free(merges);
  }
  *n_tasks = nt;
  *n_msgs = nm;
  return 0;
}

/* ---------------- flashcore.hpp:135-197 ---------------- */
int dao_block_attn_update(const double* q, int64_t rq, const double* k, const double* v,
                          int64_t rk, int64_t d, double* o, double* m, double* l, int mask,
                          double scale, int64_t br0, int64_t bc0) {
  if (br0 <= 0 || bc0 <= 0) return 2;
  if (mask == 2) return 0; /* Empty: bit-identical accumulator */
  if (mask == 0 && rq != rk) return 1;
  double* s = (double*)malloc(sizeof(double) * (size_t)(br0 * bc0));
  double* e = (double*)malloc(sizeof(double) * (size_t)bc0);
  for (int64_t i0 = 0; i0 < rq; i0 += br0) {
    const int64_t br = br0 < rq - i0 ? br0 : rq - i0;
    for (int64_t j0 = 0; j0 < rk; j0 += bc0) {
      const int64_t bc = bc0 < rk - j0 ? bc0 : rk - j0;
      if (mask == 0 && j0 > i0 + br - 1) continue;
      for (int64_t r = 0; r < br; ++r)
        for (int64_t c = 0; c < bc; ++c) {
          if (mask == 0 && j0 + c > i0 + r) {
            s[r * bc + c] = NEG_INF;
            continue;
          }
          double dot = 0.0;
          for (int64_t x = 0; x < d; ++x) dot += q[(i0 + r) * d + x] * k[(j0 + c) * d + x];
          s[r * bc + c] = dot * scale;
        }
      for (int64_t r = 0; r < br; ++r) {
        double bm = s[r * bc];
        for (int64_t c = 1; c < bc; ++c) bm = smax(bm, s[r * bc + c]);
        const int64_t row = i0 + r;
        const double m_new = smax(m[row], bm);
        if (m_new == NEG_INF) continue;
        const double alpha = (m[row] == NEG_INF) ? 0.0 : exp(m[row] - m_new);
        double p_sum = 0.0;
        for (int64_t c = 0; c < bc; ++c) {
          e[c] = exp(s[r * bc + c] - m_new);
          p_sum += e[c];
        }
        l[row] = alpha * l[row] + p_sum;
        for (int64_t x = 0; x < d; ++x) {
          double contrib = 0.0;
          for (int64_t c = 0; c < bc; ++c) contrib += e[c] * v[(j0 + c) * d + x];
          o[row * d + x] = alpha * o[row * d + x] + contrib;
        }
        m[row] = m_new;
      }
    }
  }
  free(s);
  free(e);
  return 0;
}

/* ---------------- flashcore.hpp:202-224 ---------------- */
void dao_rescale(const double* oa, const double* ma, const double* la, const double* ob,
                 const double* mb, const double* lb, int64_t rows, int64_t d, double* o,
                 double* m, double* l) {
  for (int64_t r = 0; r < rows; ++r) {
    const double a_m = ma[r], b_m = mb[r], a_l = la[r], b_l = lb[r];
    const double m_new = smax(a_m, b_m);
    const double wa = (a_m == NEG_INF) ? 0.0 : exp(a_m - m_new);
    const double wb = (b_m == NEG_INF) ? 0.0 : exp(b_m - m_new);
    m[r] = m_new;
    l[r] = wa * a_l + wb * b_l;
    for (int64_t x = 0; x < d; ++x) o[r * d + x] = wa * oa[r * d + x] + wb * ob[r * d + x];
  }
}

/* ---------------- flashcore.hpp:227-240 ---------------- */
int dao_finalize(const double* o, const double* m, const double* l, int64_t rows, int64_t d,
                 double* out, double* lse) {
  for (int64_t r = 0; r < rows; ++r) {
    if (!(l[r] > 0.0)) return 5;
    for (int64_t x = 0; x < d; ++x) out[r * d + x] = o[r * d + x] / l[r];
    lse[r] = m[r] + log(l[r]);
  }
  return 0;
}

/* ---------------- flashcore.hpp:250-261 ---------------- */
void dao_backward_aux(const double* d_out, const double* out, int64_t rows, int64_t d, double* dv) {
  for (int64_t i = 0; i < rows; ++i) {
    double acc = 0.0;
    for (int64_t x = 0; x < d; ++x) acc += d_out[i * d + x] * out[i * d + x];
    dv[i] = acc;
  }
}

/* ---------------- flashcore.hpp:269-337 ---------------- */
int dao_block_attn_backward(const double* q, int64_t rq, const double* k, const double* v,
                            int64_t rk, int64_t d, const double* out, const double* lse,
                            const double* d_out, int mask, double scale, int64_t br0,
                            int64_t bc0, double* dq, double* dk, double* dv) {
  if (br0 <= 0 || bc0 <= 0) return 2;
  if (mask == 0 && rq != rk) return 1;
  memset(dq, 0, sizeof(double) * (size_t)(rq * d));
  memset(dk, 0, sizeof(double) * (size_t)(rk * d));
  memset(dv, 0, sizeof(double) * (size_t)(rk * d));
  if (mask == 2) return 0;
  double* big_d = (double*)malloc(sizeof(double) * (size_t)rq);
  dao_backward_aux(d_out, out, rq, d, big_d);
  double* p = (double*)malloc(sizeof(double) * (size_t)(br0 * bc0));
  for (int64_t j0 = 0; j0 < rk; j0 += bc0) {
    const int64_t bc = bc0 < rk - j0 ? bc0 : rk - j0;
    for (int64_t i0 = 0; i0 < rq; i0 += br0) {
      const int64_t br = br0 < rq - i0 ? br0 : rq - i0;
      if (mask == 0 && j0 > i0 + br - 1) continue;
      for (int64_t r = 0; r < br; ++r)
        for (int64_t c = 0; c < bc; ++c) {
          if (mask == 0 && j0 + c > i0 + r) {
            p[r * bc + c] = 0.0;
            continue;
          }
          double dot = 0.0;
          for (int64_t x = 0; x < d; ++x) dot += q[(i0 + r) * d + x] * k[(j0 + c) * d + x];
          p[r * bc + c] = exp(dot * scale - lse[i0 + r]);
        }
      for (int64_t r = 0; r < br; ++r)
        for (int64_t c = 0; c < bc; ++c) {
          const double pv = p[r * bc + c];
          for (int64_t x = 0; x < d; ++x) dv[(j0 + c) * d + x] += pv * d_out[(i0 + r) * d + x];
          double dp = 0.0;
          for (int64_t x = 0; x < d; ++x) dp += d_out[(i0 + r) * d + x] * v[(j0 + c) * d + x];
          p[r * bc + c] = pv * (dp - big_d[i0 + r]);
        }
      for (int64_t r = 0; r < br; ++r)
        for (int64_t c = 0; c < bc; ++c) {
          const double sp = scale * p[r * bc + c];
          for (int64_t x = 0; x < d; ++x) {
            dq[(i0 + r) * d + x] += sp * k[(j0 + c) * d + x];
            dk[(j0 + c) * d + x] += sp * q[(i0 + r) * d + x];
          }
        }
    }
  }
  free(p);
  free(big_d);
  return 0;
}

/* ---------------- flashcore.hpp:96-128 ---------------- */
int dao_dense_oracle(const double* q, const double* k, const double* v, int64_t n, int64_t nk,
                     int64_t d, int causal, double scale, double* out, double* lse) {
  double* s = (double*)malloc(sizeof(double) * (size_t)nk);
  int rc = 0;
  for (int64_t i = 0; i < n && rc == 0; ++i) {
    for (int64_t j = 0; j < nk; ++j) {
      double acc = 0.0;
      for (int64_t x = 0; x < d; ++x) acc += q[i * d + x] * k[j * d + x];
      s[j] = (causal && j > i) ? NEG_INF : acc * scale;
    }
    double m = s[0];
    for (int64_t j = 1; j < nk; ++j) m = smax(m, s[j]);
    if (m == NEG_INF) {
      rc = 5;
      break;
    }
    double l = 0.0;
    for (int64_t j = 0; j < nk; ++j) l += exp(s[j] - m);
    for (int64_t x = 0; x < d; ++x) {
      double acc = 0.0;
      for (int64_t j = 0; j < nk; ++j) acc += exp(s[j] - m) * v[j * d + x];
      out[i * d + x] = acc / l;
    }
    lse[i] = m + log(l);
  }
  free(s);
  return rc;
}

/* ---------------- reference.hpp:21-74 ---------------- */
int dao_dense_backward(const double* q, const double* k, const double* v, const double* d_out,
                       int64_t n, int64_t nk, int64_t d, int causal, double scale, double* dq,
                       double* dk, double* dv) {
  double* p = (double*)malloc(sizeof(double) * (size_t)(n * nk));
  double* ds = (double*)malloc(sizeof(double) * (size_t)(n * nk));
  for (int64_t i = 0; i < n; ++i) {
    double m = NEG_INF;
    for (int64_t j = 0; j < nk; ++j) {
      if (causal && j > i) {
        p[i * nk + j] = NEG_INF;
        continue;
      }
      double dot = 0.0;
      for (int64_t x = 0; x < d; ++x) dot += q[i * d + x] * k[j * d + x];
      p[i * nk + j] = dot * scale;
      m = smax(m, p[i * nk + j]);
    }
    double l = 0.0;
    for (int64_t j = 0; j < nk; ++j) {
      p[i * nk + j] = exp(p[i * nk + j] - m);
      l += p[i * nk + j];
    }
    for (int64_t j = 0; j < nk; ++j) p[i * nk + j] /= l;
  }
  for (int64_t i = 0; i < n; ++i) {
    double dsum = 0.0;
    for (int64_t j = 0; j < nk; ++j) {
      double dp = 0.0;
      for (int64_t x = 0; x < d; ++x) dp += d_out[i * d + x] * v[j * d + x];
      ds[i * nk + j] = dp;
      dsum += dp * p[i * nk + j];
    }
    for (int64_t j = 0; j < nk; ++j) ds[i * nk + j] = p[i * nk + j] * (ds[i * nk + j] - dsum);
  }
  /* dv = p^T d_out ; dq = (ds k) * scale ; dk = (ds^T q) * scale  (matmul order numerics.hpp:41-58) */
  for (int64_t j = 0; j < nk; ++j)
    for (int64_t x = 0; x < d; ++x) {
      double acc = 0.0;
      for (int64_t i = 0; i < n; ++i) acc += p[i * nk + j] * d_out[i * d + x];
      dv[j * d + x] = acc;
    }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t x = 0; x < d; ++x) {
      double acc = 0.0;
      for (int64_t j = 0; j < nk; ++j) acc += ds[i * nk + j] * k[j * d + x];
      dq[i * d + x] = acc * scale;
    }
  for (int64_t j = 0; j < nk; ++j)
    for (int64_t x = 0; x < d; ++x) {
      double acc = 0.0;
      for (int64_t i = 0; i < n; ++i) acc += ds[i * nk + j] * q[i * d + x];
      dk[j * d + x] = acc * scale;
    }
  free(p);
  free(ds);
  return 0;
}

/* ---------------- runtime.cpp:266-330, 491-529 (stepper forward) ---------------- */
static void count_msg(int64_t* c, int kind, int64_t rows, int64_t d) {
  /* runtime.cpp:50-83 */
  switch (kind) {
    case 0: c[0] += 2 * rows * d; ++c[4]; break;
    case 1: c[1] += rows * d; ++c[5]; break;
    case 2: c[2] += rows * (d + 2); ++c[6]; break;
    case 3: c[3] += 2 * rows * d; ++c[7]; break;
    case 4: c[0] += 2 * rows * d; ++c[4]; break; /* KVHalf: rows = the half */
  }
}

int dao_run_forward(int P, int kind, int64_t n, int64_t d, const double* q, const double* k,
                    const double* v, double* out, double* lse, int64_t* counters) {
  if (P < 1 || n % P != 0) return 2;
  const int64_t rows = n / P;
  const double scale = 1.0 / sqrt((double)d);
  int32_t steps = 0;
  int64_t nt = 0, nm = 0;
  dao_schedule_build(P, kind, &steps, NULL, &nt, NULL, &nm);
  int32_t* tasks = (int32_t*)malloc(sizeof(int32_t) * 6 * (size_t)nt);
  int32_t* msgs = (int32_t*)malloc(sizeof(int32_t) * 4 * (size_t)(nm + 1));
  dao_schedule_build(P, kind, &steps, tasks, &nt, msgs, &nm);
  const size_t osz = (size_t)(rows * d);
  double* o = (double*)calloc((size_t)P * osz, sizeof(double));
  double* m = (double*)malloc(sizeof(double) * (size_t)n);
  double* l = (double*)calloc((size_t)n, sizeof(double));
  double* po = (double*)malloc(sizeof(double) * (size_t)P * osz);
  double* pm = (double*)malloc(sizeof(double) * (size_t)n);
  double* pl = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) m[i] = NEG_INF;
  int64_t c[10] = {0};
  int held_any = 0;
  /* pending partial per (owner, helper) pair: one slot per helper suffices
   * because every partial is merged in the step that produced it */
  for (int t = 0; t < steps; ++t) {
    for (int64_t i = 0; i < nt; ++i) {
      const int32_t* tk = tasks + 6 * i;
      if (tk[0] != t || tk[1] == 3 || tk[1] == 2) continue;
      const int w = tk[2];
      ++c[8];
      double* ow = o + (size_t)(w - 1) * osz;
      if (tk[1] == 0) {
        dao_block_attn_update(q + (w - 1) * osz, rows, k + (w - 1) * osz, v + (w - 1) * osz, rows,
                              d, ow, m + (w - 1) * rows, l + (w - 1) * rows, 0, scale, 16, 16);
      } else if (tk[2] == tk[3]) {
        const int r = tk[4];
        /* kv row window: whole chunk, or the low/high half of the split step */
        const int64_t lo = rows / 2;
        const int64_t r0 = tk[5] == 2 ? lo : 0;
        const int64_t nr = tk[5] == 0 ? rows : (tk[5] == 1 ? lo : rows - lo);
        held_any = 1;
        count_msg(c, tk[5] == 0 ? 0 : 4, nr, d);
        dao_block_attn_update(q + (w - 1) * osz, rows, k + (r - 1) * osz + r0 * d,
                              v + (r - 1) * osz + r0 * d, nr, d, ow, m + (w - 1) * rows,
                              l + (w - 1) * rows, 1, scale, 16, 16);
      } else {
        const int owner = tk[3];
        const int64_t lo = rows / 2;
        const int64_t r0 = tk[5] == 2 ? lo : 0;
        const int64_t nr = tk[5] == 0 ? rows : (tk[5] == 1 ? lo : rows - lo);
        held_any = 1;
        count_msg(c, 1, rows, d);
        double* pw = po + (size_t)(w - 1) * osz;
        memset(pw, 0, sizeof(double) * osz);
        for (int64_t r = 0; r < rows; ++r) {
          pm[(w - 1) * rows + r] = NEG_INF;
          pl[(w - 1) * rows + r] = 0.0;
        }
        dao_block_attn_update(q + (owner - 1) * osz, rows, k + (w - 1) * osz + r0 * d,
                              v + (w - 1) * osz + r0 * d, nr, d, pw, pm + (w - 1) * rows,
                              pl + (w - 1) * rows, 1, scale, 16, 16);
      }
    }
    for (int64_t i = 0; i < nt; ++i) {
      const int32_t* tk = tasks + 6 * i;
      if (tk[0] != t || tk[1] != 2) continue;
      const int ow = tk[2], hw = tk[5];
      count_msg(c, 2, rows, d);
      double* oo = o + (size_t)(ow - 1) * osz;
      dao_rescale(oo, m + (ow - 1) * rows, l + (ow - 1) * rows, po + (size_t)(hw - 1) * osz,
                  pm + (hw - 1) * rows, pl + (hw - 1) * rows, rows, d, oo, m + (ow - 1) * rows,
                  l + (ow - 1) * rows);
    }
  }
  int rc = 0;
  for (int w = 0; w < P && rc == 0; ++w)
    rc = dao_finalize(o + (size_t)w * osz, m + w * rows, l + w * rows, rows, d, out + w * osz,
                      lse + w * rows);
  c[9] = held_any;
  if (counters) memcpy(counters, c, sizeof(c));
  free(tasks); free(msgs); free(o); free(m); free(l); free(po); free(pm); free(pl);
  return rc;
}

/* ---------------- runtime.cpp:605-651, 720-750 (stepper backward, ring) ---------------- */
int dao_run_backward(int P, int64_t n, int64_t d, const double* q, const double* k,
                     const double* v, const double* out, const double* lse, const double* d_out,
                     double* dq, double* dk, double* dv, int64_t* counters) {
  if (P < 1 || n % P != 0) return 2;
  const int64_t rows = n / P;
  const size_t osz = (size_t)(rows * d);
  const double scale = 1.0 / sqrt((double)d);
  memset(dq, 0, sizeof(double) * (size_t)(n * d));
  memset(dk, 0, sizeof(double) * (size_t)(n * d));
  memset(dv, 0, sizeof(double) * (size_t)(n * d));
  double* gq = (double*)malloc(sizeof(double) * osz);
  double* gk = (double*)malloc(sizeof(double) * osz);
  double* gv = (double*)malloc(sizeof(double) * osz);
  /* pending GradKV per (sender p, receiver p - t) for the current step */
  double* pk = (double*)malloc(sizeof(double) * osz * (size_t)P);
  double* pv = (double*)malloc(sizeof(double) * osz * (size_t)P);
  int64_t c[10] = {0};
  for (int t = 0; t < P; ++t) {
    for (int p = 1; p <= P; ++p) {
      const size_t po_ = (size_t)(p - 1) * osz;
      if (t == 0) {
        dao_block_attn_backward(q + po_, rows, k + po_, v + po_, rows, d, out + po_,
                                lse + (p - 1) * rows, d_out + po_, 0, scale, 16, 16, gq, gk, gv);
        ++c[8];
        for (size_t i = 0; i < osz; ++i) {
          dq[po_ + i] += gq[i];
          dk[po_ + i] += gk[i];
          dv[po_ + i] += gv[i];
        }
      } else if (t < p) {
        const int r = p - t;
        const size_t ro = (size_t)(r - 1) * osz;
        count_msg(c, 0, rows, d);
        c[9] = 1;
        dao_block_attn_backward(q + po_, rows, k + ro, v + ro, rows, d, out + po_,
                                lse + (p - 1) * rows, d_out + po_, 1, scale, 16, 16, gq,
                                pk + po_, pv + po_);
        ++c[8];
        for (size_t i = 0; i < osz; ++i) dq[po_ + i] += gq[i];
      }
    }
    if (t >= 1) {
      for (int r = 1; r <= P; ++r) {
        const int sender = r + t;
        if (sender > P) continue;
        count_msg(c, 3, rows, d);
        const size_t ro = (size_t)(r - 1) * osz, so = (size_t)(sender - 1) * osz;
        for (size_t i = 0; i < osz; ++i) {
          dk[ro + i] += pk[so + i];
          dv[ro + i] += pv[so + i];
        }
      }
    }
  }
  if (counters) memcpy(counters, c, sizeof(c));
  free(gq); free(gk); free(gv); free(pk); free(pv);
  return 0;
}

/* ---------------- backward over a schedule table (extension) ---------------- */
int dao_run_backward_sched(int P, int kind, int64_t n, int64_t d, const double* q,
                           const double* k, const double* v, const double* out,
                           const double* lse, const double* d_out, double* dq, double* dk,
                           double* dv, int64_t* counters) {
  if (P < 1 || n % P != 0) return 2;
  const int64_t rows = n / P;
  const size_t osz = (size_t)(rows * d);
  const double scale = 1.0 / sqrt((double)d);
  int32_t steps = 0;
  int64_t nt = 0, nm = 0;
  dao_schedule_build(P, kind, &steps, NULL, &nt, NULL, &nm);
  int32_t* tasks = (int32_t*)malloc(sizeof(int32_t) * 6 * (size_t)nt);
  int32_t* msgs = (int32_t*)malloc(sizeof(int32_t) * 4 * (size_t)(nm + 1));
  dao_schedule_build(P, kind, &steps, tasks, &nt, msgs, &nm);
  memset(dq, 0, sizeof(double) * (size_t)(n * d));
  memset(dk, 0, sizeof(double) * (size_t)(n * d));
  memset(dv, 0, sizeof(double) * (size_t)(n * d));
  double* gq = (double*)malloc(sizeof(double) * osz);
  double* gk = (double*)malloc(sizeof(double) * osz);
  double* gv = (double*)malloc(sizeof(double) * osz);
  /* pending GradKV indexed by sender, pending dq partial indexed by helper */
  double* pk = (double*)malloc(sizeof(double) * osz * (size_t)P);
  double* pv = (double*)malloc(sizeof(double) * osz * (size_t)P);
  double* pq = (double*)malloc(sizeof(double) * osz * (size_t)P);
  int* gk_to = (int*)malloc(sizeof(int) * (size_t)P); /* receiver of sender's GradKV, 0 = none */
  int64_t* gk_r0 = (int64_t*)malloc(sizeof(int64_t) * (size_t)P); /* its kv row window */
  int64_t* gk_nr = (int64_t*)malloc(sizeof(int64_t) * (size_t)P);
  int64_t c[10] = {0};
  for (int t = 0; t < steps; ++t) {
    for (int w = 0; w < P; ++w) gk_to[w] = 0;
    for (int64_t i = 0; i < nt; ++i) {
      const int32_t* tk = tasks + 6 * i;
      if (tk[0] != t || tk[1] == 3 || tk[1] == 2) continue;
      const int w = tk[2];
      const size_t wo = (size_t)(w - 1) * osz;
      ++c[8];
      if (tk[1] == 0) {
        dao_block_attn_backward(q + wo, rows, k + wo, v + wo, rows, d, out + wo,
                                lse + (w - 1) * rows, d_out + wo, 0, scale, 16, 16, gq, gk, gv);
        for (size_t x = 0; x < osz; ++x) {
          dq[wo + x] += gq[x];
          dk[wo + x] += gk[x];
          dv[wo + x] += gv[x];
        }
      } else if (tk[2] == tk[3]) { /* direct */
        const int r = tk[4];
        /* kv row window: whole chunk, or the low/high half of the split step */
        const int64_t lo = rows / 2;
        const int64_t r0 = tk[5] == 2 ? lo : 0;
        const int64_t nr = tk[5] == 0 ? rows : (tk[5] == 1 ? lo : rows - lo);
        const size_t ro = (size_t)(r - 1) * osz + (size_t)(r0 * d);
        count_msg(c, tk[5] == 0 ? 0 : 4, nr, d);
        c[9] = 1;
        dao_block_attn_backward(q + wo, rows, k + ro, v + ro, nr, d, out + wo,
                                lse + (w - 1) * rows, d_out + wo, 1, scale, 16, 16, gq, pk + wo,
                                pv + wo);
        gk_to[w - 1] = r;
        gk_r0[w - 1] = r0;
        gk_nr[w - 1] = nr;
        for (size_t x = 0; x < osz; ++x) dq[wo + x] += gq[x];
      } else { /* helper w for owner o on (a row window of) its own kv */
        const int o = tk[3];
        const size_t oo = (size_t)(o - 1) * osz;
        const int64_t lo = rows / 2;
        const int64_t r0 = tk[5] == 2 ? lo : 0;
        const int64_t nr = tk[5] == 0 ? rows : (tk[5] == 1 ? lo : rows - lo);
        const size_t wk = wo + (size_t)(r0 * d);
        c[1] += rows * (2 * d + 2);
        ++c[5];
        c[9] = 1;
        dao_block_attn_backward(q + oo, rows, k + wk, v + wk, nr, d, out + oo,
                                lse + (o - 1) * rows, d_out + oo, 1, scale, 16, 16, pq + wo, gk,
                                gv);
        for (size_t x = 0; x < (size_t)(nr * d); ++x) {
          dk[wk + x] += gk[x];
          dv[wk + x] += gv[x];
        }
      }
    }
    /* GradKV folds in ascending receiver order (runtime.cpp:636-649) */
    for (int r = 1; r <= P; ++r)
      for (int s = 1; s <= P; ++s)
        if (gk_to[s - 1] == r) {
          count_msg(c, 3, gk_nr[s - 1], d);
          const size_t ro = (size_t)(r - 1) * osz + (size_t)(gk_r0[s - 1] * d);
          const size_t so = (size_t)(s - 1) * osz;
          for (size_t x = 0; x < (size_t)(gk_nr[s - 1] * d); ++x) {
            dk[ro + x] += pk[so + x];
            dv[ro + x] += pv[so + x];
          }
        }
    /* dq partial folds in merge order */
    for (int64_t i = 0; i < nt; ++i) {
      const int32_t* tk = tasks + 6 * i;
      if (tk[0] != t || tk[1] != 2) continue;
      const int o = tk[2], h = tk[5];
      c[2] += rows * d;
      ++c[6];
      const size_t oo = (size_t)(o - 1) * osz, ho = (size_t)(h - 1) * osz;
      for (size_t x = 0; x < osz; ++x) dq[oo + x] += pq[ho + x];
    }
  }
  if (counters) memcpy(counters, c, sizeof(c));
  free(tasks); free(msgs); free(gq); free(gk); free(gv); free(pk); free(pv); free(pq); free(gk_to);
  free(gk_r0); free(gk_nr);
  return 0;
}

/* block_attn_backward with D = rowsum(dO * O) supplied by the caller (the
 * value backward_aux computes, flashcore.hpp:250-261): bit-identical to
 * dao_block_attn_backward when d_vec came from dao_backward_aux. */
int dao_block_attn_backward_with_d(const double* q, int64_t rq, const double* k, const double* v,
                                   int64_t rk, int64_t d, const double* d_vec, const double* lse,
                                   const double* d_out, int mask, double scale, int64_t br0,
                                   int64_t bc0, double* dq, double* dk, double* dv) {
  /* out is only used to form D: pass a fake O = d_vec spread so that
   * rowsum(dO * O) reproduces d_vec is not possible in general, so restate. */
  if (br0 <= 0 || bc0 <= 0) return 2;
  if (mask == 0 && rq != rk) return 1;
  memset(dq, 0, sizeof(double) * (size_t)(rq * d));
  memset(dk, 0, sizeof(double) * (size_t)(rk * d));
  memset(dv, 0, sizeof(double) * (size_t)(rk * d));
  if (mask == 2) return 0;
  double* p = (double*)malloc(sizeof(double) * (size_t)(br0 * bc0));
  for (int64_t j0 = 0; j0 < rk; j0 += bc0) {
    const int64_t bc = bc0 < rk - j0 ? bc0 : rk - j0;
    for (int64_t i0 = 0; i0 < rq; i0 += br0) {
      const int64_t br = br0 < rq - i0 ? br0 : rq - i0;
      if (mask == 0 && j0 > i0 + br - 1) continue;
      for (int64_t r = 0; r < br; ++r)
        for (int64_t c = 0; c < bc; ++c) {
          if (mask == 0 && j0 + c > i0 + r) {
            p[r * bc + c] = 0.0;
            continue;
          }
          double dot = 0.0;
          for (int64_t x = 0; x < d; ++x) dot += q[(i0 + r) * d + x] * k[(j0 + c) * d + x];
          p[r * bc + c] = exp(dot * scale - lse[i0 + r]);
        }
      for (int64_t r = 0; r < br; ++r)
        for (int64_t c = 0; c < bc; ++c) {
          const double pv = p[r * bc + c];
          for (int64_t x = 0; x < d; ++x) dv[(j0 + c) * d + x] += pv * d_out[(i0 + r) * d + x];
          double dp = 0.0;
          for (int64_t x = 0; x < d; ++x) dp += d_out[(i0 + r) * d + x] * v[(j0 + c) * d + x];
          p[r * bc + c] = pv * (dp - d_vec[i0 + r]);
        }
      for (int64_t r = 0; r < br; ++r)
        for (int64_t c = 0; c < bc; ++c) {
          const double sp = scale * p[r * bc + c];
          for (int64_t x = 0; x < d; ++x) {
            dq[(i0 + r) * d + x] += sp * k[(j0 + c) * d + x];
            dk[(j0 + c) * d + x] += sp * q[(i0 + r) * d + x];
          }
        }
    }
  }
  free(p);
  return 0;
}
