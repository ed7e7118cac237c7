// extern "C" entry points of libdistattn_b200.so: argument checking with the
// reference's error taxonomy (errors.hpp:12-48), TMA descriptor encoding and
// kernel launches. No torch types cross this boundary.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "capi_internal.h"
#include "kernels.h"

namespace da {

namespace {
thread_local std::string g_last_error;

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}
}  // namespace

da_status set_error(da_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

da_status cuda_error(cudaError_t e, const char* where) {
  return set_error(DA_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

const char* last_error() { return g_last_error.c_str(); }

// bf16 [heads][rows][128] tensor -> 3D tensor map, box {64, box_rows, 1}, SWIZZLE_128B.
da_status make_tmap_3d(CUtensorMap* map, const void* base, int64_t heads, int64_t rows,
                       uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) return set_error(DA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {128, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(heads)};
  const cuuint64_t strides[2] = {128 * 2, static_cast<cuuint64_t>(rows) * 128 * 2};
  const cuuint32_t box[3] = {64, box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(DA_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return DA_OK;
}

da_status make_tmap_f32_acc(CUtensorMap* map, void* base, int64_t heads, int64_t rows,
                            bool swizzle128) {
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) return set_error(DA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {128, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(heads)};
  const cuuint64_t strides[2] = {128 * 4, static_cast<cuuint64_t>(rows) * 128 * 4};
  const cuuint32_t box[3] = {32, 32, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(DA_ERR_CUDA, "cuTensorMapEncodeTiled(f32) failed (" + std::to_string(r) + ")");
  return DA_OK;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

unsigned long long* g_bwd_trace = nullptr;

// Semaphores of the deterministic dQ order: one int per (query head, query
// tile), zeroed before every deterministic launch. One buffer PER STREAM
// (launches on one stream are serialised, so a reset can never overlap a
// kernel still spinning on the same counters; launches on different streams
// get different buffers). Growth is stream-ordered (cudaMallocAsync /
// cudaFreeAsync on that stream), so no in-flight launch loses its buffer.
struct SemBuffer {
  int* ptr = nullptr;
  size_t n = 0;
};
std::mutex g_sem_mu;
std::map<cudaStream_t, SemBuffer> g_dq_sem;

cudaError_t dq_semaphores(cudaStream_t st, size_t want, int** out) {
  std::lock_guard<std::mutex> lock(g_sem_mu);
  SemBuffer& b = g_dq_sem[st];
  if (want > b.n) {
    if (b.ptr) cudaFreeAsync(b.ptr, st);
    b.ptr = nullptr;
    b.n = 0;
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, want * sizeof(int), st);
    if (e != cudaSuccess) return e;
    b.ptr = static_cast<int*>(p);
    b.n = want;
  }
  *out = b.ptr;
  return cudaMemsetAsync(b.ptr, 0, want * sizeof(int), st);
}
unsigned long long* g_fwd_trace = nullptr;

}  // namespace da

using da::set_error;

extern "C" {

const char* da_last_error(void) { return da::last_error(); }
int da_abi_version(void) { return DA_ABI_VERSION; }

int da_device_supported(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return (major == 10 && minor == 0) ? 1 : 0;
}

da_status da_attn_fwd_chunk(const da_fwd_args* a, void* stream) {
  if (a == nullptr) return set_error(DA_ERR_CONFIG, "da_attn_fwd_chunk: null args");
  if (a->d != 128) return set_error(DA_ERR_UNSUPPORTED, "da_attn_fwd_chunk: d must be 128");
  if (a->h_q < 1 || a->h_kv < 1 || a->h_q % a->h_kv != 0)
    return set_error(DA_ERR_SHAPE, "block_attn_update: h_q must be a positive multiple of h_kv");
  if (a->rows_q < 0 || a->rows_kv < 0)
    return set_error(DA_ERR_SHAPE, "block_attn_update: negative row count");
  if (a->mask != DA_MASK_DIAGONAL && a->mask != DA_MASK_FULL && a->mask != DA_MASK_EMPTY)
    return set_error(DA_ERR_CONFIG, "block_attn_update: unknown mask mode");
  if (a->mask == DA_MASK_DIAGONAL && a->rows_q != a->rows_kv)
    return set_error(DA_ERR_SHAPE, "block_attn_update: diagonal mask needs a square chunk");
  if (a->o_in != nullptr && (a->m_in == nullptr || a->l_in == nullptr))
    return set_error(DA_ERR_CONFIG, "block_attn_update: partial input accumulator");
  if (a->finalize ? (a->o_out == nullptr || a->lse_out == nullptr)
                  : (a->o_acc == nullptr || a->m_acc == nullptr || a->l_acc == nullptr))
    return set_error(DA_ERR_CONFIG, "block_attn_update: missing output buffers");
  const int64_t rows_total = a->h_q * a->rows_q;
  if (rows_total > INT32_MAX / 128 || a->rows_kv * a->h_kv > INT32_MAX / 128)
    return set_error(DA_ERR_UNSUPPORTED, "block_attn_update: chunk too large for 32-bit rows");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (rows_total == 0) return DA_OK;

  const bool empty = a->mask == DA_MASK_EMPTY || a->rows_kv == 0;
  if (empty) {
    // Empty mask: the update is a no-op (flashcore.hpp:148); only the
    // accumulator plumbing (copy / finalize) remains.
    cudaError_t e = cudaSuccess;
    if (a->o_in == nullptr) {
      // fresh accumulator: o = 0, m = -inf, l = 0
      if (a->finalize) {
        // every row is degenerate (finalize would throw DegenerateRowError)
        e = cudaMemsetAsync(a->o_out, 0, rows_total * 128 * 2, st);
        if (e == cudaSuccess) e = da::launch_fill(a->lse_out, -INFINITY, rows_total, st);
        if (e == cudaSuccess && a->degenerate_flag)
          e = da::launch_fill(reinterpret_cast<float*>(a->degenerate_flag), 1.4e-45f, 1, st);
      } else {
        e = cudaMemsetAsync(a->o_acc, 0, rows_total * 128 * 4, st);
        if (e == cudaSuccess) e = cudaMemsetAsync(a->l_acc, 0, rows_total * 4, st);
        if (e == cudaSuccess) e = da::launch_fill(a->m_acc, -INFINITY, rows_total, st);
      }
    } else if (a->finalize) {
      e = da::launch_finalize(a->o_in, a->m_in, a->l_in, a->o_out, a->lse_out, a->degenerate_flag,
                              rows_total, st);
    } else if (a->o_in != a->o_acc) {
      e = da::launch_copy_acc(a->o_in, a->m_in, a->l_in, a->o_acc, a->m_acc, a->l_acc, rows_total,
                              st);
    }
    return e == cudaSuccess ? DA_OK : da::cuda_error(e, "block_attn_update(empty)");
  }

  if (!da::aligned16(a->q) || !da::aligned16(a->k) || !da::aligned16(a->v))
    return set_error(DA_ERR_CONFIG, "block_attn_update: q/k/v must be 16-byte aligned");
  CUtensorMap tq, tk, tv;
  da_status s;
  if ((s = da::make_tmap_3d(&tq, a->q, a->h_q, a->rows_q)) != DA_OK) return s;
  if ((s = da::make_tmap_3d(&tk, a->k, a->h_kv, a->rows_kv)) != DA_OK) return s;
  if ((s = da::make_tmap_3d(&tv, a->v, a->h_kv, a->rows_kv)) != DA_OK) return s;

  da::FwdParams p{};
  p.h_q = static_cast<int>(a->h_q);
  p.h_kv = static_cast<int>(a->h_kv);
  p.rows_q = static_cast<int>(a->rows_q);
  p.rows_kv = static_cast<int>(a->rows_kv);
  p.mask = a->mask;
  p.finalize = a->finalize ? 1 : 0;
  const float scale = a->scale > 0.f ? a->scale : 1.0f / std::sqrt(128.0f);
  p.scale_log2 = scale * 1.4426950408889634f;
  p.o_in = a->o_in;
  p.m_in = a->m_in;
  p.l_in = a->l_in;
  p.o_acc = a->o_acc;
  p.m_acc = a->m_acc;
  p.l_acc = a->l_acc;
  p.o_out = a->o_out;
  p.lse_out = a->lse_out;
  p.degenerate_flag = a->degenerate_flag;
  p.debug_s = nullptr;
  p.trace = da::g_fwd_trace;
  cudaError_t e;
  if (da::fwd_pair_enabled()) {
    CUtensorMap tk64;
    if ((s = da::make_tmap_3d(&tk64, a->k, a->h_kv, a->rows_kv, 64)) != DA_OK) return s;
    e = da::launch_attn_fwd_pair(tq, tk64, tv, p, st);
  } else {
    e = da::launch_attn_fwd(tq, tk, tv, p, st);
  }
  return e == cudaSuccess ? DA_OK : da::cuda_error(e, "da_attn_fwd_chunk launch");
}

da_status da_attn_merge(const float* o_a, const float* m_a, const float* l_a, const float* o_b,
                        const float* m_b, const float* l_b, float* o_out, float* m_out,
                        float* l_out, int64_t h, int64_t rows, int64_t d, void* stream) {
  if (d != 128) return set_error(DA_ERR_UNSUPPORTED, "rescale: d must be 128");
  if (h < 0 || rows < 0) return set_error(DA_ERR_SHAPE, "rescale: accumulator shapes disagree");
  cudaError_t e = da::launch_merge(o_a, m_a, l_a, o_b, m_b, l_b, o_out, m_out, l_out, h * rows,
                                   reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? DA_OK : da::cuda_error(e, "da_attn_merge");
}

da_status da_attn_finalize(const float* o, const float* m, const float* l, void* o_out,
                           float* lse_out, int* degenerate_flag, int64_t h, int64_t rows,
                           int64_t d, void* stream) {
  if (d != 128) return set_error(DA_ERR_UNSUPPORTED, "finalize: d must be 128");
  if (h < 0 || rows < 0) return set_error(DA_ERR_SHAPE, "finalize: bad shape");
  cudaError_t e = da::launch_finalize(o, m, l, o_out, lse_out, degenerate_flag, h * rows,
                                      reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? DA_OK : da::cuda_error(e, "da_attn_finalize");
}

da_status da_check_degenerate(const int* flag, void* stream) {
  if (flag == nullptr) return DA_OK;
  int host = 0;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(&host, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return da::cuda_error(e, "da_check_degenerate");
  if (host != 0) return set_error(DA_ERR_DEGENERATE_ROW, "finalize: a row attended to no key");
  return DA_OK;
}

da_status da_attn_bwd_preprocess(const void* d_out, const void* out, float* d_vec, int64_t h,
                                 int64_t rows, int64_t d, void* stream) {
  if (d != 128) return set_error(DA_ERR_UNSUPPORTED, "backward_aux: d must be 128");
  if (h < 0 || rows < 0) return set_error(DA_ERR_SHAPE, "backward_aux: shape mismatch");
  cudaError_t e = da::launch_bwd_preprocess(d_out, out, d_vec, h * rows,
                                            reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? DA_OK : da::cuda_error(e, "da_attn_bwd_preprocess");
}

da_status da_attn_bwd_chunk(const da_bwd_args* a, void* stream) {
  if (a == nullptr) return set_error(DA_ERR_CONFIG, "da_attn_bwd_chunk: null args");
  if (a->d != 128) return set_error(DA_ERR_UNSUPPORTED, "block_attn_backward: d must be 128");
  if (a->h_q < 1 || a->h_kv < 1 || a->h_q % a->h_kv != 0)
    return set_error(DA_ERR_SHAPE, "block_attn_backward: h_q must be a multiple of h_kv");
  if (a->rows_q < 0 || a->rows_kv < 0)
    return set_error(DA_ERR_SHAPE, "block_attn_backward: negative row count");
  if (a->mask != DA_MASK_DIAGONAL && a->mask != DA_MASK_FULL && a->mask != DA_MASK_EMPTY)
    return set_error(DA_ERR_CONFIG, "block_attn_backward: unknown mask mode");
  if (a->mask == DA_MASK_DIAGONAL && a->rows_q != a->rows_kv)
    return set_error(DA_ERR_SHAPE, "block_attn_backward: diagonal mask needs a square chunk");
  if (a->lse == nullptr || a->d_vec == nullptr)
    return set_error(DA_ERR_STATE, "block_attn_backward: requires logsumexp and D");
  if (a->h_q * a->rows_q > INT32_MAX / 128 || a->h_kv * a->rows_kv > INT32_MAX / 128)
    return set_error(DA_ERR_UNSUPPORTED, "block_attn_backward: chunk too large");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t kv_elems = a->h_kv * a->rows_kv * 128;
  if (a->mask == DA_MASK_EMPTY || a->rows_q == 0 || a->rows_kv == 0) {
    // Empty: zero contribution (flashcore.hpp:292)
    cudaError_t e = cudaSuccess;
    if (!a->accumulate_kv && kv_elems > 0) {
      e = cudaMemsetAsync(a->dk_acc, 0, kv_elems * 4, st);
      if (e == cudaSuccess) e = cudaMemsetAsync(a->dv_acc, 0, kv_elems * 4, st);
    }
    return e == cudaSuccess ? DA_OK : da::cuda_error(e, "block_attn_backward(empty)");
  }
  CUtensorMap tq, tk, tv, tdo, tdq;
  da_status s;
  if ((s = da::make_tmap_3d(&tq, a->q, a->h_q, a->rows_q)) != DA_OK) return s;
  if ((s = da::make_tmap_3d(&tk, a->k, a->h_kv, a->rows_kv)) != DA_OK) return s;
  if ((s = da::make_tmap_3d(&tv, a->v, a->h_kv, a->rows_kv)) != DA_OK) return s;
  if ((s = da::make_tmap_3d(&tdo, a->d_out, a->h_q, a->rows_q)) != DA_OK) return s;
  da::BwdParams p{};
  p.h_q = static_cast<int>(a->h_q);
  p.h_kv = static_cast<int>(a->h_kv);
  p.rows_q = static_cast<int>(a->rows_q);
  p.rows_kv = static_cast<int>(a->rows_kv);
  p.mask = a->mask;
  p.accumulate_kv = a->accumulate_kv ? 1 : 0;
  p.scale = a->scale > 0.f ? a->scale : 1.0f / std::sqrt(128.0f);
  p.scale_log2 = p.scale * 1.4426950408889634f;
  p.lse = a->lse;
  p.d_vec = a->d_vec;
  p.dq_acc = a->dq_acc;
  p.dk_acc = a->dk_acc;
  p.dv_acc = a->dv_acc;
  p.dq_sem = nullptr;
  if (a->deterministic) {
    const size_t n_sem = static_cast<size_t>(a->h_q) * ((a->rows_q + 127) / 128);
    int* sem = nullptr;
    cudaError_t e = da::dq_semaphores(st, n_sem, &sem);
    if (e != cudaSuccess) return da::cuda_error(e, "block_attn_backward deterministic workspace");
    p.dq_sem = sem;
  }
  p.trace = da::g_bwd_trace;
  cudaError_t e;
  if (p.dq_sem == nullptr && da::bwd_pair_enabled()) {
    // CTA-pair kernel (attn_bwd_pair_sm100.cu); the deterministic dQ order
    // lives in the single-CTA kernel
    CUtensorMap tq64, tdo64;
    if ((s = da::make_tmap_3d(&tq64, a->q, a->h_q, a->rows_q, 64)) != DA_OK) return s;
    if ((s = da::make_tmap_3d(&tdo64, a->d_out, a->h_q, a->rows_q, 64)) != DA_OK) return s;
    if ((s = da::make_tmap_f32_acc(&tdq, a->dq_acc, a->h_q, a->rows_q, true)) != DA_OK) return s;
    e = da::launch_attn_bwd_pair(tq, tq64, tk, tv, tdo, tdo64, tdq, p, st);
  } else {
    if ((s = da::make_tmap_f32_acc(&tdq, a->dq_acc, a->h_q, a->rows_q, false)) != DA_OK) return s;
    e = da::launch_attn_bwd(tq, tk, tv, tdo, tdq, p, st);
  }
  return e == cudaSuccess ? DA_OK : da::cuda_error(e, "da_attn_bwd_chunk launch");
}

da_status da_convert_f32_bf16(const float* src, void* dst, int64_t n, void* stream) {
  if (n % 4 != 0) return set_error(DA_ERR_SHAPE, "convert: n must be a multiple of 4");
  cudaError_t e = da::launch_convert(src, dst, n, reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? DA_OK : da::cuda_error(e, "da_convert_f32_bf16");
}

// Debug (DA_TRACE builds only record): device buffer of 64*16 uint64 per-iteration
// stamps of CTA 0 followed by 8 uint64 per CTA (timers, SM id, iterations).
void da_debug_set_bwd_trace(void* buf) { da::g_bwd_trace = static_cast<unsigned long long*>(buf); }
void da_debug_set_fwd_trace(void* buf) { da::g_fwd_trace = static_cast<unsigned long long*>(buf); }

da_status da_debug_scores(const void* q, const void* k, int64_t rows, float* s_out, void* stream) {
  CUtensorMap tq, tk;
  da_status s;
  if ((s = da::make_tmap_3d(&tq, q, 1, rows)) != DA_OK) return s;
  if ((s = da::make_tmap_3d(&tk, k, 1, rows)) != DA_OK) return s;
  // scratch outputs (discarded); the kernel dumps the raw first score tile
  float* scratch = nullptr;
  const size_t n = static_cast<size_t>(rows) * 128;
  cudaError_t e = cudaMalloc(&scratch, n * 4 * 2 + rows * 8);
  if (e != cudaSuccess) return da::cuda_error(e, "da_debug_scores alloc");
  da::FwdParams p{};
  p.h_q = 1;
  p.h_kv = 1;
  p.rows_q = static_cast<int>(rows);
  p.rows_kv = static_cast<int>(rows);
  p.mask = DA_MASK_FULL;
  p.finalize = 0;
  p.scale_log2 = 1.0f;
  p.o_acc = scratch;
  p.m_acc = scratch + n;
  p.l_acc = scratch + n + rows;
  p.debug_s = s_out;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  e = da::launch_attn_fwd(tq, tk, tq, p, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(scratch);
  return e == cudaSuccess ? DA_OK : da::cuda_error(e, "da_debug_scores");
}

}  // extern "C"
