// Row-wise HBM-bound helpers around the chunk kernels (d = 128):
//   merge      — rescale (flashcore.hpp:202-224) of two partial accumulators
//   finalize   — finalize (flashcore.hpp:227-240)
//   preprocess — backward_aux D = rowsum(dO ∘ O) (flashcore.hpp:250-261)
//   convert    — fp32 gradient accumulators -> bf16
// One warp per row: lane i owns columns [4i, 4i+4) (one float4 / 8 bytes of
// bf16), so every warp-wide access is a single fully-coalesced 512 B / 256 B
// transaction. Grids are sized to a multiple of the SM count.
#include <cuda_bf16.h>

#include "kernels.h"
#include "sm100_ptx.cuh"

namespace da {
namespace {

constexpr int kD = 128;
constexpr int kWarpsPerBlock = 8;

__device__ __forceinline__ float2 bf16x2_to_f2(uint32_t u) {
  return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xFFFF0000u));
}

__global__ void merge_kernel(const float* __restrict__ o_a, const float* __restrict__ m_a,
                             const float* __restrict__ l_a, const float* __restrict__ o_b,
                             const float* __restrict__ m_b, const float* __restrict__ l_b,
                             float* o_out, float* m_out, float* l_out, int64_t rows) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * kWarpsPerBlock;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + threadIdx.x / 32; r < rows;
       r += warps) {
    const float ma = m_a[r], mb = m_b[r];
    const float mn = fmaxf(ma, mb);
    const float wa = (ma == -INFINITY) ? 0.f : __expf(ma - mn);
    const float wb = (mb == -INFINITY) ? 0.f : __expf(mb - mn);
    const float4 a = reinterpret_cast<const float4*>(o_a + r * kD)[lane];
    const float4 b = reinterpret_cast<const float4*>(o_b + r * kD)[lane];
    const float la = l_a[r], lb = l_b[r];
    __syncwarp();
    reinterpret_cast<float4*>(o_out + r * kD)[lane] =
        make_float4(wa * a.x + wb * b.x, wa * a.y + wb * b.y, wa * a.z + wb * b.z,
                    wa * a.w + wb * b.w);
    if (lane == 0) {
      m_out[r] = mn;
      l_out[r] = wa * la + wb * lb;
    }
  }
}

__global__ void finalize_kernel(const float* __restrict__ o, const float* __restrict__ m,
                                const float* __restrict__ l, __nv_bfloat16* __restrict__ o_out,
                                float* __restrict__ lse_out, int* flag, int64_t rows) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * kWarpsPerBlock;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + threadIdx.x / 32; r < rows;
       r += warps) {
    const float lr = l[r];
    const bool ok = lr > 0.f;
    if (!ok && lane == 0 && flag) atomicExch(flag, 1);
    const float inv = ok ? 1.f / lr : 0.f;
    const float4 x = reinterpret_cast<const float4*>(o + r * kD)[lane];
    uint2 w;
    w.x = pack_bf16x2(x.x * inv, x.y * inv);
    w.y = pack_bf16x2(x.z * inv, x.w * inv);
    reinterpret_cast<uint2*>(o_out + r * kD)[lane] = w;
    if (lane == 0) lse_out[r] = ok ? m[r] + __logf(lr) : -INFINITY;
  }
}

__global__ void preprocess_kernel(const __nv_bfloat16* __restrict__ d_out,
                                  const __nv_bfloat16* __restrict__ out, float* __restrict__ d_vec,
                                  int64_t rows) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * kWarpsPerBlock;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + threadIdx.x / 32; r < rows;
       r += warps) {
    const uint2 a = reinterpret_cast<const uint2*>(d_out + r * kD)[lane];
    const uint2 b = reinterpret_cast<const uint2*>(out + r * kD)[lane];
    const float2 a0 = bf16x2_to_f2(a.x), a1 = bf16x2_to_f2(a.y);
    const float2 b0 = bf16x2_to_f2(b.x), b1 = bf16x2_to_f2(b.y);
    float s = a0.x * b0.x + a0.y * b0.y + a1.x * b1.x + a1.y * b1.y;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) d_vec[r] = s;
  }
}

__global__ void convert_kernel(const float4* __restrict__ src, uint2* __restrict__ dst, int64_t n4) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += stride) {
    const float4 x = src[i];
    uint2 w;
    w.x = pack_bf16x2(x.x, x.y);
    w.y = pack_bf16x2(x.z, x.w);
    dst[i] = w;
  }
}

__global__ void copy_acc_kernel(const float* __restrict__ o, const float* __restrict__ m,
                                const float* __restrict__ l, float* o_out, float* m_out,
                                float* l_out, int64_t rows) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * kWarpsPerBlock;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + threadIdx.x / 32; r < rows;
       r += warps) {
    reinterpret_cast<float4*>(o_out + r * kD)[lane] =
        reinterpret_cast<const float4*>(o + r * kD)[lane];
    if (lane == 0) {
      m_out[r] = m[r];
      l_out[r] = l[r];
    }
  }
}

int sm_count() {
  static std::atomic<int> counts[64];  // per device, 0 = not queried yet
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  int n = counts[dev & 63].load(std::memory_order_relaxed);
  if (n == 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    counts[dev & 63].store(n, std::memory_order_relaxed);
  }
  return n;
}

unsigned row_grid(int64_t rows) {
  const int64_t need = (rows + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const int64_t cap = static_cast<int64_t>(sm_count()) * 8;  // 8 blocks (64 warps) per SM
  return static_cast<unsigned>(need < cap ? (need > 0 ? need : 1) : cap);
}

}  // namespace

cudaError_t launch_merge(const float* o_a, const float* m_a, const float* l_a, const float* o_b,
                         const float* m_b, const float* l_b, float* o_out, float* m_out,
                         float* l_out, int64_t rows, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  merge_kernel<<<row_grid(rows), kWarpsPerBlock * 32, 0, stream>>>(o_a, m_a, l_a, o_b, m_b, l_b,
                                                                    o_out, m_out, l_out, rows);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const float* o, const float* m, const float* l, void* o_out,
                            float* lse_out, int* flag, int64_t rows, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  finalize_kernel<<<row_grid(rows), kWarpsPerBlock * 32, 0, stream>>>(
      o, m, l, reinterpret_cast<__nv_bfloat16*>(o_out), lse_out, flag, rows);
  return cudaGetLastError();
}

cudaError_t launch_bwd_preprocess(const void* d_out, const void* out, float* d_vec, int64_t rows,
                                  cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  preprocess_kernel<<<row_grid(rows), kWarpsPerBlock * 32, 0, stream>>>(
      reinterpret_cast<const __nv_bfloat16*>(d_out), reinterpret_cast<const __nv_bfloat16*>(out),
      d_vec, rows);
  return cudaGetLastError();
}

__global__ void add_kernel(float4* __restrict__ dst, const float4* __restrict__ src, int64_t n4) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += stride) {
    float4 a = dst[i];
    const float4 b = src[i];
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
    dst[i] = a;
  }
}

// dst += src (fp32, n a multiple of 4): GradKV / dq-partial folds of the per-rank runtime
cudaError_t launch_add(float* dst, const float* src, int64_t n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int64_t n4 = n / 4;
  const int64_t blocks = (n4 + 255) / 256;
  const int64_t cap = static_cast<int64_t>(sm_count()) * 8;
  add_kernel<<<static_cast<unsigned>(blocks < cap ? blocks : cap), 256, 0, stream>>>(
      reinterpret_cast<float4*>(dst), reinterpret_cast<const float4*>(src), n4);
  return cudaGetLastError();
}

// dst[h][r0 + i][:] += src[h][i][:] for i < n (fp32 rows of 128): the fold of a
// kv row half (split schedules) into a [h, rows_dst, 128] accumulator
__global__ void add_rows_kernel(float4* __restrict__ dst, const float4* __restrict__ src,
                                int64_t rows_dst, int64_t r0, int64_t n, int64_t total4) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total4;
       i += stride) {
    const int64_t row = i / 32, c4 = i % 32;  // 32 float4 per 128-wide row
    const int64_t h = row / n, r = row % n;
    float4* d = dst + ((h * rows_dst + r0 + r) * 32 + c4);
    const float4 b = src[i];
    float4 a = *d;
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
    *d = a;
  }
}

cudaError_t launch_add_rows(float* dst, const float* src, int64_t h, int64_t rows_dst, int64_t r0,
                            int64_t n, cudaStream_t stream) {
  if (h <= 0 || n <= 0) return cudaSuccess;
  const int64_t total4 = h * n * 32;
  const int64_t blocks = (total4 + 255) / 256;
  const int64_t cap = static_cast<int64_t>(sm_count()) * 8;
  add_rows_kernel<<<static_cast<unsigned>(blocks < cap ? blocks : cap), 256, 0, stream>>>(
      reinterpret_cast<float4*>(dst), reinterpret_cast<const float4*>(src), rows_dst, r0, n,
      total4);
  return cudaGetLastError();
}

cudaError_t launch_convert(const float* src, void* dst, int64_t n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int64_t n4 = n / 4;
  const int64_t blocks = (n4 + 255) / 256;
  const int64_t cap = static_cast<int64_t>(sm_count()) * 8;
  convert_kernel<<<static_cast<unsigned>(blocks < cap ? blocks : cap), 256, 0, stream>>>(
      reinterpret_cast<const float4*>(src), reinterpret_cast<uint2*>(dst), n4);
  return cudaGetLastError();
}

cudaError_t launch_copy_acc(const float* o, const float* m, const float* l, float* o_out,
                            float* m_out, float* l_out, int64_t rows, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  copy_acc_kernel<<<row_grid(rows), kWarpsPerBlock * 32, 0, stream>>>(o, m, l, o_out, m_out,
                                                                      l_out, rows);
  return cudaGetLastError();
}

}  // namespace da

namespace da {
namespace {
__global__ void fill_kernel(float* dst, float v, int64_t n) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = v;
}
}  // namespace

cudaError_t launch_fill(float* dst, float value, int64_t n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = (n + 255) / 256;
  fill_kernel<<<static_cast<unsigned>(blocks < 1184 ? blocks : 1184), 256, 0, stream>>>(dst, value, n);
  return cudaGetLastError();
}
}  // namespace da
