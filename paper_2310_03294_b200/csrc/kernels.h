// Internal kernel parameter blocks and launchers (not part of the C ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>

#include "../../include/distattn_b200.h"

namespace da {

// One-time per-device setup (function attributes, cached device queries):
// runs `f` until it succeeds once on the current device. Thread-safe; two
// threads racing on the first call both run the (idempotent) setup.
template <class F>
inline cudaError_t once_per_device(std::atomic<uint64_t>& done, F&& f) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = f();
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

struct FwdParams {
  int h_q, h_kv, rows_q, rows_kv;
  int mask;        // da_mask_mode (DIAGONAL or FULL; EMPTY never launches)
  int finalize;
  float scale_log2;  // scale * log2(e)
  const float* o_in;
  const float* m_in;
  const float* l_in;
  float* o_acc;
  float* m_acc;
  float* l_acc;
  void* o_out;
  float* lse_out;
  int* degenerate_flag;
  float* debug_s;  // optional raw-score dump of tile (0,0) of head 0
  unsigned long long* trace;  // DA_TRACE builds: per-iteration clock64 stamps of CTA 0
};

struct BwdParams {
  int h_q, h_kv, rows_q, rows_kv;
  int mask;
  int accumulate_kv;
  float scale;       // softmax scale (dq/dk factor)
  float scale_log2;  // scale * log2(e)
  const float* lse;    // [h_q, rows_q] natural log
  const float* d_vec;  // [h_q, rows_q]
  float* dq_acc;
  float* dk_acc;
  float* dv_acc;
  int* dq_sem;  // deterministic mode: [h_q, q tiles] zeroed counters, else nullptr
  int head_group;  // kv heads whose CTAs are interleaved in the grid (bwd_head_group())
  unsigned long long* trace;  // DA_TRACE builds: per-iteration clock64 stamps of CTA 0
};

cudaError_t launch_attn_fwd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                            const FwdParams& p, cudaStream_t stream);

// CTA-pair forward (attn_fwd_pair_sm100.cu): tk64 is a 64-row-box map of k.
cudaError_t launch_attn_fwd_pair(const CUtensorMap& tq, const CUtensorMap& tk64,
                                 const CUtensorMap& tv, const FwdParams& p, cudaStream_t stream);
// whether the forward uses the CTA-pair kernel (DA_FWD_KERNEL=pair, read once per process)
bool fwd_pair_enabled();

cudaError_t launch_attn_bwd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                            const CUtensorMap& tdo, const CUtensorMap& tdq, const BwdParams& p,
                            cudaStream_t stream);

// CTA-pair backward (attn_bwd_pair_sm100.cu): q64/do64 are 64-row-box maps of
// q / d_out, tdq_sw the 128B-swizzled fp32 dq_acc map. Not deterministic.
cudaError_t launch_attn_bwd_pair(const CUtensorMap& tq, const CUtensorMap& tq64,
                                 const CUtensorMap& tk, const CUtensorMap& tv,
                                 const CUtensorMap& tdo, const CUtensorMap& tdo64,
                                 const CUtensorMap& tdq_sw, const BwdParams& p,
                                 cudaStream_t stream);
// whether the non-deterministic backward uses the CTA-pair kernel: only with
// DA_BWD_KERNEL=pair (read once per process). The pair kernel is correct but
// measured slower than the single-CTA kernel, so it is an
// opt-in experiment, not the product default.
bool bwd_pair_enabled();

cudaError_t launch_merge(const float* o_a, const float* m_a, const float* l_a, const float* o_b,
                         const float* m_b, const float* l_b, float* o_out, float* m_out,
                         float* l_out, int64_t rows_total, cudaStream_t stream);

cudaError_t launch_finalize(const float* o, const float* m, const float* l, void* o_out,
                            float* lse_out, int* flag, int64_t rows_total, cudaStream_t stream);

cudaError_t launch_bwd_preprocess(const void* d_out, const void* out, float* d_vec,
                                  int64_t rows_total, cudaStream_t stream);

cudaError_t launch_convert(const float* src, void* dst, int64_t n, cudaStream_t stream);

cudaError_t launch_add(float* dst, const float* src, int64_t n, cudaStream_t stream);

// dst[h][r0 + i][:] += src[h][i][:], i < n: fp32 [h, rows_dst, 128] += [h, n, 128]
cudaError_t launch_add_rows(float* dst, const float* src, int64_t h, int64_t rows_dst, int64_t r0,
                            int64_t n, cudaStream_t stream);

cudaError_t launch_copy_acc(const float* o, const float* m, const float* l, float* o_out,
                            float* m_out, float* l_out, int64_t rows_total, cudaStream_t stream);

}  // namespace da
