// Microbenchmark: TMEM read (tcgen05.ld 32x32b.x32, 4 KB per warp-instruction)
// and write (tcgen05.st) throughput per SM vs the number of warps (1..16).
#include <cstdio>
#include <cstdint>
#include "../../paper_2310_03294_b200/csrc/sm100_ptx.cuh"
using namespace da;

__global__ void __launch_bounds__(512, 1) kern(long long* out, int reps, int active_warps, int mode) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t lb = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  if (warp < active_warps) {
    uint32_t v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = i;
    for (int r = 0; r < reps; ++r) {
      if (mode == 0) {
        uint32_t w2[32];
        tmem_ld_32x32b_x32(lb, v);
        tmem_ld_32x32b_x32(lb + 32, w2);
        tmem_ld_wait();
        acc += v[3] + w2[17];
        tmem_ld_32x32b_x32(lb + 64, v);
        tmem_ld_32x32b_x32(lb + 96, w2);
        tmem_ld_wait();
        acc ^= v[30] ^ w2[9];
      } else {
        tmem_st_32x32b_x32(lb, v);
        tmem_st_32x32b_x32(lb + 32, v);
        tmem_st_32x32b_x32(lb + 64, v);
        tmem_st_32x32b_x32(lb + 96, v);
        tmem_st_wait();
      }
    }
  }
  __syncthreads();
  long long dt = clock64() - t0;
  if (threadIdx.x == 0) out[0] = dt;
  if (acc == 0xFFFFFFFF) out[1] = acc;
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
  long long* d; cudaMalloc(&d, 64);
  const int reps = 2000;
  for (int mode = 0; mode < 2; ++mode)
    for (int w : {1, 2, 4, 8, 12, 16}) {
      kern<<<1, 512>>>(d, reps, w, mode);
      cudaError_t e = cudaDeviceSynchronize();
      long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      const double bytes = static_cast<double>(w) * reps * 4 * 4096;
      printf("%s warps %2d: %.1f B/clk per SM (%s)\n", mode ? "st" : "ld", w, bytes / h,
             cudaGetErrorString(e));
    }
  return 0;
}
