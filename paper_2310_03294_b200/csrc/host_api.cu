// Host-buffer (fp64, row-major, one head) entry points: the reference's
// flashcore API surface (flashcore.hpp:135-337) for callers that hold host
// matrices — what the signature-level drop-in include/distattn/flashcore.hpp
// calls, so the reference's own runtime.cpp / ckptplan.cpp run on the
// sm_100a kernels unmodified.
//
// Per calling thread: one non-blocking stream, one device arena and one
// pinned staging arena, grown on demand and reused (no allocation per call
// once the shapes are known). Each call converts its operands into the
// staging arena (bf16 for q/k/v/O/dO, fp32 for the accumulator and the
// statistics — the product layout of include/distattn_b200.h), does ONE
// host->device copy, launches the chunk kernels, ONE device->host copy, and
// synchronises its own stream only. Concurrent callers (the reference's
// thread-per-worker executor, runtime.cpp:351-388) therefore run their
// kernels concurrently on the device. The backward always orders its dq
// partials (deterministic): repeated calls are bitwise identical, as the
// reference's executors and checkpoint plans require (acceptance_main.cpp
// :316-412, ckptplan.cpp:235-305).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <initializer_list>
#include <limits>
#include <string>

#include "capi_internal.h"
#include "kernels.h"

namespace da {
namespace {

uint16_t to_bf16(double x) {
  const float f = static_cast<float>(x);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40);  // NaN
  u += 0x7fffu + ((u >> 16) & 1u);  // round to nearest even
  return static_cast<uint16_t>(u >> 16);
}

double from_bf16(uint16_t b) {
  const uint32_t u = static_cast<uint32_t>(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

struct HostCtx {
  cudaStream_t st = nullptr;
  char* dev = nullptr;
  size_t dev_bytes = 0;
  char* pin = nullptr;
  size_t pin_bytes = 0;
  ~HostCtx() {
    if (dev) cudaFree(dev);
    if (pin) cudaFreeHost(pin);
    if (st) cudaStreamDestroy(st);
  }
};
thread_local HostCtx g_ctx;

// Byte layout of one call's operands; the same offsets address the pinned
// staging arena and the device arena.
struct Layout {
  size_t bytes = 0;
  size_t add(size_t n) {
    const size_t off = bytes;
    bytes += (n + 255) & ~static_cast<size_t>(255);
    return off;
  }
};

da_status prepare(size_t bytes, HostCtx** out) {
  HostCtx& c = g_ctx;
  cudaError_t e = cudaSuccess;
  if (c.st == nullptr) e = cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking);
  if (e == cudaSuccess && bytes > c.dev_bytes) {
    if (c.dev) cudaFree(c.dev);
    c.dev = nullptr;
    c.dev_bytes = 0;
    e = cudaMalloc(&c.dev, bytes);
    if (e == cudaSuccess) c.dev_bytes = bytes;
  }
  if (e == cudaSuccess && bytes > c.pin_bytes) {
    if (c.pin) cudaFreeHost(c.pin);
    c.pin = nullptr;
    c.pin_bytes = 0;
    e = cudaMallocHost(&c.pin, bytes);
    if (e == cudaSuccess) c.pin_bytes = bytes;
  }
  if (e != cudaSuccess) return cuda_error(e, "host API workspace");
  *out = &c;
  return DA_OK;
}

void put_bf16(HostCtx* c, size_t off, const double* src, int64_t n) {
  uint16_t* d = reinterpret_cast<uint16_t*>(c->pin + off);
  for (int64_t i = 0; i < n; ++i) d[i] = to_bf16(src[i]);
}
void put_f32(HostCtx* c, size_t off, const double* src, int64_t n) {
  float* d = reinterpret_cast<float*>(c->pin + off);
  for (int64_t i = 0; i < n; ++i) d[i] = static_cast<float>(src[i]);
}
void get_f32(const HostCtx* c, size_t off, double* dst, int64_t n) {
  const float* s = reinterpret_cast<const float*>(c->pin + off);
  for (int64_t i = 0; i < n; ++i) dst[i] = s[i];
}
void get_bf16(const HostCtx* c, size_t off, double* dst, int64_t n) {
  const uint16_t* s = reinterpret_cast<const uint16_t*>(c->pin + off);
  for (int64_t i = 0; i < n; ++i) dst[i] = from_bf16(s[i]);
}

da_status upload(HostCtx* c, size_t bytes) {
  const cudaError_t e = cudaMemcpyAsync(c->dev, c->pin, bytes, cudaMemcpyHostToDevice, c->st);
  return e == cudaSuccess ? DA_OK : cuda_error(e, "host API upload");
}
da_status download(HostCtx* c, size_t off, size_t bytes) {
  cudaError_t e =
      cudaMemcpyAsync(c->pin + off, c->dev + off, bytes, cudaMemcpyDeviceToHost, c->st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->st);
  return e == cudaSuccess ? DA_OK : cuda_error(e, "host API download");
}

#define HOST_TRY(x)               \
  do {                            \
    const da_status s_ = (x);     \
    if (s_ != DA_OK) return s_;   \
  } while (0)

bool any_null(std::initializer_list<const void*> ps) {
  for (const void* p : ps)
    if (p == nullptr) return true;
  return false;
}

da_status check_dims(int64_t rows_q, int64_t rows_kv, int64_t d, const char* op) {
  if (d != 128) return set_error(DA_ERR_UNSUPPORTED, std::string(op) + ": d must be 128");
  if (rows_q < 0 || rows_kv < 0) return set_error(DA_ERR_SHAPE, std::string(op) + ": bad rows");
  return DA_OK;
}

bool all_fresh(const double* m, const double* l, int64_t rows) {
  for (int64_t i = 0; i < rows; ++i)
    if (!(std::isinf(m[i]) && m[i] < 0) || l[i] != 0.0) return false;
  return true;
}

}  // namespace
}  // namespace da

using namespace da;

extern "C" {

da_status da_host_attn_update(const double* q, int64_t rows_q, const double* k, const double* v,
                              int64_t rows_kv, int64_t d, double* o, double* m, double* l,
                              int mask, double scale) {
  if (any_null({q, k, v, o, m, l}))
    return set_error(DA_ERR_CONFIG, "block_attn_update: null host buffer");
  HOST_TRY(check_dims(rows_q, rows_kv, d, "block_attn_update"));
  if (mask == DA_MASK_EMPTY || rows_q == 0 || rows_kv == 0) return DA_OK;  // no-op (:148)
  if (mask == DA_MASK_DIAGONAL && rows_q != rows_kv)
    return set_error(DA_ERR_SHAPE, "block_attn_update: diagonal mask needs a square chunk");
  const int64_t nq = rows_q * d, nk = rows_kv * d;
  Layout L;
  const size_t oq = L.add(nq * 2), ok = L.add(nk * 2), ov = L.add(nk * 2);
  const size_t oo = L.add(nq * 4), om = L.add(rows_q * 4), ol = L.add(rows_q * 4);
  HostCtx* c = nullptr;
  HOST_TRY(prepare(L.bytes, &c));
  const bool fresh = all_fresh(m, l, rows_q);
  put_bf16(c, oq, q, nq);
  put_bf16(c, ok, k, nk);
  put_bf16(c, ov, v, nk);
  if (!fresh) {
    put_f32(c, oo, o, nq);
    put_f32(c, om, m, rows_q);
    put_f32(c, ol, l, rows_q);
  }
  HOST_TRY(upload(c, L.bytes));
  da_fwd_args a{};
  a.q = c->dev + oq;
  a.k = c->dev + ok;
  a.v = c->dev + ov;
  a.h_q = a.h_kv = 1;
  a.rows_q = rows_q;
  a.rows_kv = rows_kv;
  a.d = d;
  float* dev_o = reinterpret_cast<float*>(c->dev + oo);
  float* dev_m = reinterpret_cast<float*>(c->dev + om);
  float* dev_l = reinterpret_cast<float*>(c->dev + ol);
  if (!fresh) {
    a.o_in = dev_o;
    a.m_in = dev_m;
    a.l_in = dev_l;
  }
  a.o_acc = dev_o;
  a.m_acc = dev_m;
  a.l_acc = dev_l;
  a.scale = static_cast<float>(scale);
  a.mask = mask;
  HOST_TRY(da_attn_fwd_chunk(&a, c->st));
  HOST_TRY(download(c, oo, L.bytes - oo));
  get_f32(c, oo, o, nq);
  get_f32(c, om, m, rows_q);
  get_f32(c, ol, l, rows_q);
  return DA_OK;
}

da_status da_host_attn_merge(const double* o_a, const double* m_a, const double* l_a,
                             const double* o_b, const double* m_b, const double* l_b,
                             double* o_out, double* m_out, double* l_out, int64_t rows,
                             int64_t d) {
  if (any_null({o_a, m_a, l_a, o_b, m_b, l_b, o_out, m_out, l_out}))
    return set_error(DA_ERR_CONFIG, "rescale: null host buffer");
  HOST_TRY(check_dims(rows, rows, d, "rescale"));
  if (rows == 0) return DA_OK;
  const int64_t n = rows * d;
  Layout L;
  const size_t oa = L.add(n * 4), ma = L.add(rows * 4), la = L.add(rows * 4);
  const size_t ob = L.add(n * 4), mb = L.add(rows * 4), lb = L.add(rows * 4);
  HostCtx* c = nullptr;
  HOST_TRY(prepare(L.bytes, &c));
  put_f32(c, oa, o_a, n);
  put_f32(c, ma, m_a, rows);
  put_f32(c, la, l_a, rows);
  put_f32(c, ob, o_b, n);
  put_f32(c, mb, m_b, rows);
  put_f32(c, lb, l_b, rows);
  HOST_TRY(upload(c, L.bytes));
  auto F = [&](size_t off) { return reinterpret_cast<float*>(c->dev + off); };
  HOST_TRY(da_attn_merge(F(oa), F(ma), F(la), F(ob), F(mb), F(lb), F(oa), F(ma), F(la), 1, rows,
                         d, c->st));
  HOST_TRY(download(c, oa, ob - oa));
  get_f32(c, oa, o_out, n);
  get_f32(c, ma, m_out, rows);
  get_f32(c, la, l_out, rows);
  return DA_OK;
}

da_status da_host_attn_finalize(const double* o, const double* m, const double* l, int64_t rows,
                                int64_t d, double* out, double* lse) {
  if (any_null({o, m, l, out, lse}))
    return set_error(DA_ERR_CONFIG, "finalize: null host buffer");
  HOST_TRY(check_dims(rows, rows, d, "finalize"));
  if (rows == 0) return DA_OK;
  const int64_t n = rows * d;
  Layout L;
  const size_t oo = L.add(n * 4), om = L.add(rows * 4), ol = L.add(rows * 4);
  const size_t oout = L.add(n * 2), olse = L.add(rows * 4), oflag = L.add(4);
  HostCtx* c = nullptr;
  HOST_TRY(prepare(L.bytes, &c));
  put_f32(c, oo, o, n);
  put_f32(c, om, m, rows);
  put_f32(c, ol, l, rows);
  std::memset(c->pin + oflag, 0, 4);
  HOST_TRY(upload(c, L.bytes));
  auto F = [&](size_t off) { return reinterpret_cast<float*>(c->dev + off); };
  HOST_TRY(da_attn_finalize(F(oo), F(om), F(ol), c->dev + oout, F(olse),
                            reinterpret_cast<int*>(c->dev + oflag), 1, rows, d, c->st));
  HOST_TRY(download(c, oout, L.bytes - oout));
  int flag = 0;
  std::memcpy(&flag, c->pin + oflag, 4);
  if (flag != 0) return set_error(DA_ERR_DEGENERATE_ROW, "finalize: a row attended to no key");
  get_bf16(c, oout, out, n);
  get_f32(c, olse, lse, rows);
  return DA_OK;
}

da_status da_host_backward_aux(const double* d_out, const double* out, int64_t rows, int64_t d,
                               double* d_vec) {
  if (any_null({d_out, out, d_vec}))
    return set_error(DA_ERR_CONFIG, "backward_aux: null host buffer");
  HOST_TRY(check_dims(rows, rows, d, "backward_aux"));
  if (rows == 0) return DA_OK;
  const int64_t n = rows * d;
  Layout L;
  const size_t odo = L.add(n * 2), oo = L.add(n * 2), od = L.add(rows * 4);
  HostCtx* c = nullptr;
  HOST_TRY(prepare(L.bytes, &c));
  put_bf16(c, odo, d_out, n);
  put_bf16(c, oo, out, n);
  HOST_TRY(upload(c, od));
  HOST_TRY(da_attn_bwd_preprocess(c->dev + odo, c->dev + oo,
                                  reinterpret_cast<float*>(c->dev + od), 1, rows, d, c->st));
  HOST_TRY(download(c, od, rows * 4));
  get_f32(c, od, d_vec, rows);
  return DA_OK;
}

da_status da_host_attn_backward(const double* q, int64_t rows_q, const double* k,
                                const double* v, int64_t rows_kv, int64_t d, const double* out,
                                const double* lse, const double* d_out, int mask, double scale,
                                double* dq, double* dk, double* dv) {
  if (any_null({q, k, v, out, lse, d_out, dq, dk, dv}))
    return set_error(DA_ERR_CONFIG, "block_attn_backward: null host buffer");
  HOST_TRY(check_dims(rows_q, rows_kv, d, "block_attn_backward"));
  const int64_t nq = rows_q * d, nk = rows_kv * d;
  if (mask == DA_MASK_EMPTY || rows_q == 0 || rows_kv == 0) {  // zero contribution (:292)
    std::memset(dq, 0, sizeof(double) * nq);
    std::memset(dk, 0, sizeof(double) * nk);
    std::memset(dv, 0, sizeof(double) * nk);
    return DA_OK;
  }
  if (mask == DA_MASK_DIAGONAL && rows_q != rows_kv)
    return set_error(DA_ERR_SHAPE, "block_attn_backward: diagonal mask needs a square chunk");
  Layout L;
  const size_t oq = L.add(nq * 2), ok = L.add(nk * 2), ov = L.add(nk * 2);
  const size_t oo = L.add(nq * 2), odo = L.add(nq * 2), olse = L.add(rows_q * 4);
  const size_t odv = L.add(rows_q * 4);  // D (device only)
  const size_t gq = L.add(nq * 4), gk = L.add(nk * 4), gv = L.add(nk * 4);
  HostCtx* c = nullptr;
  HOST_TRY(prepare(L.bytes, &c));
  put_bf16(c, oq, q, nq);
  put_bf16(c, ok, k, nk);
  put_bf16(c, ov, v, nk);
  put_bf16(c, oo, out, nq);
  put_bf16(c, odo, d_out, nq);
  put_f32(c, olse, lse, rows_q);
  HOST_TRY(upload(c, odv));
  float* D = reinterpret_cast<float*>(c->dev + odv);
  const cudaError_t e = cudaMemsetAsync(c->dev + gq, 0, nq * 4, c->st);
  if (e != cudaSuccess) return cuda_error(e, "block_attn_backward dq zero");
  HOST_TRY(da_attn_bwd_preprocess(c->dev + odo, c->dev + oo, D, 1, rows_q, d, c->st));
  da_bwd_args a{};
  a.q = c->dev + oq;
  a.k = c->dev + ok;
  a.v = c->dev + ov;
  a.d_out = c->dev + odo;
  a.lse = reinterpret_cast<const float*>(c->dev + olse);
  a.d_vec = D;
  a.h_q = a.h_kv = 1;
  a.rows_q = rows_q;
  a.rows_kv = rows_kv;
  a.d = d;
  a.dq_acc = reinterpret_cast<float*>(c->dev + gq);
  a.dk_acc = reinterpret_cast<float*>(c->dev + gk);
  a.dv_acc = reinterpret_cast<float*>(c->dev + gv);
  a.accumulate_kv = 0;
  a.scale = static_cast<float>(scale);
  a.mask = mask;
  a.deterministic = 1;
  HOST_TRY(da_attn_bwd_chunk(&a, c->st));
  HOST_TRY(download(c, gq, L.bytes - gq));
  get_f32(c, gq, dq, nq);
  get_f32(c, gk, dk, nk);
  get_f32(c, gv, dv, nk);
  return DA_OK;
}

da_status da_host_dense_attention(const double* q, int64_t rows_q, const double* k,
                                  const double* v, int64_t rows_kv, int64_t d, int causal,
                                  double scale, double* out, double* lse) {
  if (any_null({q, k, v, out, lse}))
    return set_error(DA_ERR_CONFIG, "dense_oracle: null host buffer");
  HOST_TRY(check_dims(rows_q, rows_kv, d, "dense_oracle"));
  if (causal && rows_q != rows_kv)
    return set_error(DA_ERR_SHAPE, "dense_oracle: causal attention needs a square chunk");
  if (rows_q == 0) return DA_OK;
  if (rows_kv == 0) return set_error(DA_ERR_DEGENERATE_ROW, "dense_oracle: row attends to no key");
  const int64_t nq = rows_q * d, nk = rows_kv * d;
  Layout L;
  const size_t oq = L.add(nq * 2), ok = L.add(nk * 2), ov = L.add(nk * 2);
  const size_t oout = L.add(nq * 2), olse = L.add(rows_q * 4), oflag = L.add(4);
  HostCtx* c = nullptr;
  HOST_TRY(prepare(L.bytes, &c));
  put_bf16(c, oq, q, nq);
  put_bf16(c, ok, k, nk);
  put_bf16(c, ov, v, nk);
  std::memset(c->pin + oflag, 0, 4);
  HOST_TRY(upload(c, L.bytes));
  da_fwd_args a{};
  a.q = c->dev + oq;
  a.k = c->dev + ok;
  a.v = c->dev + ov;
  a.h_q = a.h_kv = 1;
  a.rows_q = rows_q;
  a.rows_kv = rows_kv;
  a.d = d;
  a.o_out = c->dev + oout;
  a.lse_out = reinterpret_cast<float*>(c->dev + olse);
  a.degenerate_flag = reinterpret_cast<int*>(c->dev + oflag);
  a.scale = static_cast<float>(scale);
  a.mask = causal ? DA_MASK_DIAGONAL : DA_MASK_FULL;
  a.finalize = 1;
  HOST_TRY(da_attn_fwd_chunk(&a, c->st));
  HOST_TRY(download(c, oout, L.bytes - oout));
  int flag = 0;
  std::memcpy(&flag, c->pin + oflag, 4);
  if (flag != 0) return set_error(DA_ERR_DEGENERATE_ROW, "dense_oracle: row attends to no key");
  get_bf16(c, oout, out, nq);
  get_f32(c, olse, lse, rows_q);
  return DA_OK;
}

}  // extern "C"
