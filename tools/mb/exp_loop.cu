// Microbenchmark: the forward softmax's exponential loop on one SM.
// 4 warps (one per SMSP) or 8 warps; each thread exponentiates 128 values per
// "tile" like attn_fwd_sm100.cu: x = s*scale - m (FFMA2), p = ex2(x) (2 MUFU),
// row sum (FADD2), bf16 pack (F2FP or integer). Reports clk per tile per warp.
#include <cstdio>
#include <cstdint>
#include "../../paper_2310_03294_b200/csrc/sm100_ptx.cuh"
using namespace da;

template <int kMode>
__global__ void __launch_bounds__(256, 1) kern(long long* out, float* sink, int reps, int nwarps) {
  const int warp = threadIdx.x / 32;
  float v[128];
#pragma unroll
  for (int i = 0; i < 128; ++i) v[i] = -0.001f * (i + threadIdx.x);
  const float2 sl = make_float2(0.12f, 0.12f), nm = make_float2(-0.5f, -0.5f);
  float2 acc[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) acc[u] = make_float2(0.f, 0.f);
  uint32_t pk[64];
  __syncthreads();
  long long t0 = clock64();
  if (warp < nwarps) {
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int i = 0; i < 128; i += 2) {
        float2 x = make_float2(v[i], v[i + 1]);
        if (kMode >= 1) x = ffma2(x, sl, nm);
        float2 p;
        if (kMode >= 5 && ((i / 2) % (kMode - 3)) == kMode - 4)
          p = ex2_emu2(x);
        else
          p = make_float2(ex2_approx(x.x), ex2_approx(x.y));
        if (kMode >= 2) acc[(i / 2) & 7] = fadd2(acc[(i / 2) & 7], p);
        if (kMode == 3) pk[i / 2] = pack_bf16x2(p.x, p.y);
        if (kMode == 4 || kMode >= 5) pk[i / 2] = pack_bf16x2_int(p.x, p.y);
        if (kMode < 3) pk[i / 2] = __float_as_uint(p.x) ^ __float_as_uint(p.y);
      }
#pragma unroll
      for (int i = 0; i < 128; i += 2) v[i] += __uint_as_float(pk[i / 2] & 0x3u);  // keep live
    }
  }
  __syncthreads();
  long long dt = clock64() - t0;
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += acc[u].x + acc[u].y;
#pragma unroll
  for (int i = 0; i < 128; ++i) s += v[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) out[0] = dt / reps;
}

int main() {
  long long* d; cudaMalloc(&d, 64);
  float* sink; cudaMalloc(&sink, 1 << 20);
  const char* names[8] = {"MUFU only", "+FFMA2", "+FADD2", "+F2FP pack", "+int pack (no F2FP)",
                          "int pack, emu 1/2", "int pack, emu 1/3", "int pack, emu 1/4"};
  for (int nw : {4, 8}) {
    for (int m = 0; m < 8; ++m) {
      auto f = m == 0 ? kern<0> : m == 1 ? kern<1> : m == 2 ? kern<2> : m == 3 ? kern<3>
             : m == 4 ? kern<4> : m == 5 ? kern<5> : m == 6 ? kern<6> : kern<7>;
      f<<<1, 256>>>(d, sink, 200, nw);
      cudaError_t e = cudaDeviceSynchronize();
      long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("warps %d  %-20s %lld clk per 128-value tile (MUFU bound %d) %s\n", nw, names[m], h,
             nw <= 4 ? 1024 : 2048, cudaGetErrorString(e));
    }
  }
  return 0;
}
