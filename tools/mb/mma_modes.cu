// Microbenchmark: tcgen05 bf16 MMA throughput on one SM (one issuing thread).
// A "GEMM" is 8 K=16 steps of M=128, N=128 (128^3). Modes:
//   0 SS, one accumulator (each step depends on the previous)
//   1 SS, two accumulators interleaved step by step
//   2 TS (A in TMEM), one accumulator
//   3 TS, two accumulators interleaved
//   4 SS, N=256, one accumulator (counted as two 128^3 GEMMs)
//   5 SS, four accumulators interleaved
//   6 SS, N=64 x 2 interleaved (half-width tiles)
//   7 SS, two accumulators issued one whole chain after the other
//   8 SS, two accumulators interleaved two steps at a time
//   9 TS chain then SS chain (independent accumulators, issued sequentially)
// Reports the best of 3 runs, clk per 128^3 GEMM (ideal 512 at 4096 MAC/clk).
#include <cstdio>
#include <cstdint>
#include "../../paper_2310_03294_b200/csrc/sm100_ptx.cuh"
using namespace da;

constexpr int kModes = 11;
__global__ void __launch_bounds__(128, 1) kern(long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* smem = raw + smem_align_pad(raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tbase;
  // deterministic operands: small bf16 values everywhere (smem) and in the TMEM A region
  for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) {
    const uint32_t x = static_cast<uint32_t>(i * 2654435761u);
    const uint16_t lo = 0x3C00 | ((x >> 8) & 0x7F), hi = 0xBC00 | ((x >> 16) & 0x7F);  // ~+-0.008
    reinterpret_cast<uint32_t*>(smem)[i] = (static_cast<uint32_t>(hi) << 16) | lo;
  }
  {
    uint32_t v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = 0x3C00BC00u;
    const uint32_t lb = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    tmem_st_32x32b_x32(lb + 384, v);
    tmem_st_32x32b_x32(lb + 416, v);
    tmem_st_wait();
  }
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    const uint32_t kBox = 32768;  // room for 256-row boxes
    int phase = 0;
    for (int round = 0; round < 3; ++round)
      for (int mode = 0; mode < kModes; ++mode) {
        const uint32_t nn = mode == 4 ? 256 : (mode == 6 ? 64 : 128);
        const uint32_t idesc = make_idesc_bf16(128, nn, false, false);
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * kBox + (kk & 3) * 32;
            const uint64_t da = make_sdesc_sw128(a + off, 16, 1024);
            const uint64_t db = make_sdesc_sw128(b + off, 16, 1024);
            const uint32_t acc = kk > 0 ? 1u : 0u;
            if (mode == 0 || mode == 4) {
              mma_ss(tmem, da, db, idesc, acc);
            } else if (mode == 1) {
              mma_ss(tmem, da, db, idesc, acc);
              mma_ss(tmem + 128, da, db, idesc, acc);
            } else if (mode == 5) {
              mma_ss(tmem, da, db, idesc, acc);
              mma_ss(tmem + 128, da, db, idesc, acc);
              mma_ss(tmem + 256, da, db, idesc, acc);
              mma_ss(tmem + 384, da, db, idesc, acc);
            } else if (mode == 6) {
              mma_ss(tmem, da, db, idesc, acc);
              mma_ss(tmem + 64, da, db, idesc, acc);
            } else if (mode == 7 || mode == 9) {
              // handled below (sequential chains)
            } else if (mode == 8) {
              if ((kk & 1) == 0) {
                const uint32_t off1 = ((kk + 1) >> 2) * kBox + ((kk + 1) & 3) * 32;
                const uint64_t da1 = make_sdesc_sw128(a + off1, 16, 1024);
                const uint64_t db1 = make_sdesc_sw128(b + off1, 16, 1024);
                mma_ss(tmem, da, db, idesc, acc);
                mma_ss(tmem, da1, db1, idesc, 1u);
                mma_ss(tmem + 128, da, db, idesc, acc);
                mma_ss(tmem + 128, da1, db1, idesc, 1u);
              }
            } else if (mode == 2) {
              mma_ts(tmem, tmem + 384 + kk * 8, db, idesc, acc);
            } else if (mode == 3) {
              mma_ts(tmem, tmem + 384 + kk * 8, db, idesc, acc);
              mma_ts(tmem + 128, tmem + 384 + kk * 8, db, idesc, acc);
            }
          }
          if (mode == 10) {  // the backward's five-GEMM mix: SS, SS, TS, TS, SS chains
            for (int g = 0; g < 5; ++g)
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) {
                const uint32_t off = (kk >> 2) * kBox + (kk & 3) * 32;
                const uint64_t da = make_sdesc_sw128(a + off, 16, 1024);
                const uint64_t db = make_sdesc_sw128(b + off, 16, 1024);
                const uint32_t acc = kk > 0 ? 1u : 0u;
                if (g == 2 || g == 3)
                  mma_ts(tmem + 256 + (g - 2) * 64, tmem + 384 + (g - 2) * 64 + kk * 8, db, idesc,
                         acc);
                else
                  mma_ss(tmem + (g == 4 ? 0u : static_cast<uint32_t>(g % 2) * 128u), da, db, idesc,
                         acc);
              }
          }
          if (mode == 7 || mode == 9) {
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) {
                const uint32_t off = (kk >> 2) * kBox + (kk & 3) * 32;
                const uint64_t da = make_sdesc_sw128(a + off, 16, 1024);
                const uint64_t db = make_sdesc_sw128(b + off, 16, 1024);
                const uint32_t acc = kk > 0 ? 1u : 0u;
                if (mode == 9 && c == 0) mma_ts(tmem, tmem + 384 + kk * 8, db, idesc, acc);
                else mma_ss(tmem + 128 * c, da, db, idesc, acc);
              }
          }
        }
        mma_commit(&bar);
        mbar_wait(&bar, phase & 1);
        ++phase;
        const long long dt = clock64() - t0;
        const double gemms = mode == 10 ? 5.0 * reps : mode == 5 ? 4.0 * reps
                             : (mode == 1 || mode == 3 || mode == 4 || mode >= 7) ? 2.0 * reps : 1.0 * reps;
        const long long per = static_cast<long long>(dt / gemms);
        if (round == 0 || per < out[mode]) out[mode] = per;
      }
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
  long long* d; cudaMalloc(&d, 256);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  const char* names[kModes] = {"SS 1 accumulator", "SS 2 interleaved", "TS 1 accumulator",
                               "TS 2 interleaved", "SS N=256", "SS 4 interleaved", "SS N=64 x2",
                               "SS 2 sequential", "SS 2 by pairs", "TS then SS",
                               "bwd 5-GEMM mix"};
  for (int grid : {1, 148}) {
    kern<<<grid, 128, 200000>>>(d, 4000);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[kModes]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    for (int m = 0; m < kModes; ++m)
      printf("grid %3d  %-18s %lld clk per 128^3 GEMM (%s)\n", grid, names[m], h[m],
             cudaGetErrorString(e));
  }
  return 0;
}
