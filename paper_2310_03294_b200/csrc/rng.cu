// Device-parallel splitmix64 stream: the reference's Rng (numerics.hpp:140-174)
// advances its state by a constant per draw, so draw i of a stream whose
// current state is s is mix(s + (i+1) * 0x9E3779B97F4A7C15) — independent of
// the other draws. Filling on the device reproduces make_shards'
// (runtime.cpp:24-46) values bit-exactly: double uniform in [lo, hi), then
// rounded to the storage dtype (double -> float -> bf16, round-to-nearest-even).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "capi_internal.h"
#include "kernels.h"

namespace da {
namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint16_t f32_to_bf16_rne(float f) {
  uint32_t u = __float_as_uint(f);
  u = u + 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

__global__ void rng_fill_kernel(uint64_t state, int64_t n, double lo, double hi, int dtype,
                                void* out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const uint64_t z = mix(state + static_cast<uint64_t>(i + 1) * kGolden);
    const double u = static_cast<double>(z >> 11) * 0x1.0p-53;
    const double x = lo + (hi - lo) * u;
    if (dtype == 0) {
      static_cast<float*>(out)[i] = static_cast<float>(x);
    } else if (dtype == 1) {
      static_cast<uint16_t*>(out)[i] = f32_to_bf16_rne(static_cast<float>(x));
    } else {
      static_cast<double*>(out)[i] = x;
    }
  }
}

}  // namespace
}  // namespace da

extern "C" da_status da_rng_uniform(uint64_t state, int64_t n, double lo, double hi, int dtype,
                                    void* out, void* stream) {
  if (n < 0 || dtype < 0 || dtype > 2) return da::set_error(DA_ERR_CONFIG, "rng: bad arguments");
  if (n == 0) return DA_OK;
  const int64_t blocks = (n + 255) / 256;
  da::rng_fill_kernel<<<static_cast<unsigned>(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0,
                        reinterpret_cast<cudaStream_t>(stream)>>>(state, n, lo, hi, dtype, out);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DA_OK : da::cuda_error(e, "da_rng_uniform");
}
