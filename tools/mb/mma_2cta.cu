// Microbenchmark: tcgen05 cta_group::2 (CTA pair, M=256) bf16 MMA throughput,
// per SM, in clk per 128^3 GEMM-equivalent (compare tools/mb/mma_modes.cu).
// Modes: 0 M=256 N=128 one accumulator; 1 two accumulators interleaved;
//        2 M=256 N=256 one accumulator; 3 TS (A from TMEM) M=256 N=128 one acc;
//        4 TS M=256 N=128 two accumulators interleaved (the backward's dV/dK pattern);
//        5 SS M=128 (cta_group::2: 64 rows per CTA) N=128 one accumulator;
//        6 the backward's five-GEMM mix per iteration: SS, SS, TS, TS, SS into
//          four accumulators (S, dP, dV, dK, dQ-like), K = 128 each.
#include <cstdio>
#include <cstdint>
#include "../../paper_2310_03294_b200/csrc/sm100_ptx.cuh"
using namespace da;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
               "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
               ::"r"(smem_u32(bar)), "h"(mask) : "memory");
}

constexpr int kModes = 7;
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) kern(long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* smem = raw + smem_align_pad(raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  const uint32_t rank = cta_rank();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tbase)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) {
    const uint32_t x = static_cast<uint32_t>(i * 2654435761u);
    const uint16_t lo = 0x3C00 | ((x >> 8) & 0x7F), hi = 0xBC00 | ((x >> 16) & 0x7F);
    reinterpret_cast<uint32_t*>(smem)[i] = (static_cast<uint32_t>(hi) << 16) | lo;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tbase;
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
  tc_fence_before(); __syncthreads(); cluster_sync_all(); tc_fence_after();
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    const uint32_t kBox = 32768;
    int phase = 0;
    for (int round = 0; round < 3; ++round)
      for (int mode = 0; mode < kModes; ++mode) {
        const uint32_t nn = mode == 2 ? 256 : 128;
        const uint32_t idesc = make_idesc_bf16(256, nn, false, false);
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * kBox + (kk & 3) * 32;
            const uint64_t da = make_sdesc_sw128(a + off, 16, 1024);
            const uint64_t db = make_sdesc_sw128(b + off, 16, 1024);
            const uint32_t acc = kk > 0 ? 1u : 0u;
            if (mode == 0 || mode == 2) {
              mma2_ss(tmem, da, db, idesc, acc);
            } else if (mode == 1) {
              mma2_ss(tmem, da, db, idesc, acc);
              mma2_ss(tmem + 128, da, db, idesc, acc);
            } else if (mode == 3) {
              mma2_ts(tmem, tmem + 384 + kk * 8, db, idesc, acc);
            } else if (mode == 4) {
              mma2_ts(tmem, tmem + 384 + kk * 8, db, idesc, acc);
              mma2_ts(tmem + 128, tmem + 448 + kk * 8, db, idesc, acc);
            } else if (mode == 5) {
              mma2_ss(tmem, da, db, make_idesc_bf16(128, 128, false, false), acc);
            }
          }
          if (mode == 6) {  // five GEMMs, each a full K = 128 chain
            for (int g = 0; g < 5; ++g)
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) {
                const uint32_t off = (kk >> 2) * kBox + (kk & 3) * 32;
                const uint64_t da = make_sdesc_sw128(a + off, 16, 1024);
                const uint64_t db = make_sdesc_sw128(b + off, 16, 1024);
                const uint32_t acc = kk > 0 ? 1u : 0u;
                const uint32_t d = tmem + (g == 4 ? 0u : static_cast<uint32_t>(g % 2) * 128u);
                if (g == 2 || g == 3)
                  mma2_ts(tmem + 256 + (g - 2) * 64, tmem + 384 + (g - 2) * 64 + kk * 8, db, idesc,
                          acc);
                else
                  mma2_ss(d, da, db, idesc, acc);
              }
          }
        }
        commit2(&bar, 1);
        mbar_wait(&bar, phase & 1);
        ++phase;
        const long long dt = clock64() - t0;
        // per SM: M=256 N=128 is one 128^3 per SM per 8 steps
        const double gemms = (mode == 1 || mode == 2 || mode == 4) ? 2.0 * reps
                             : mode == 5                           ? 0.5 * reps
                             : mode == 6                           ? 5.0 * reps
                                                                   : 1.0 * reps;
        const long long per = static_cast<long long>(dt / gemms);
        if (round == 0 || per < out[mode]) out[mode] = per;
      }
  }
  tc_fence_before(); __syncthreads(); cluster_sync_all();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
  }
}

int main() {
  long long* d; cudaMalloc(&d, 256);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  const char* names[kModes] = {"2CTA M256 N128 1 acc", "2CTA M256 N128 2 intl", "2CTA M256 N256 1 acc",
                               "2CTA TS M256 N128", "2CTA TS M256 N128 2 intl",
                               "2CTA M128 N128 1 acc", "2CTA bwd 5-GEMM mix"};
  for (int grid : {2, 148}) {
    kern<<<grid, 128, 200000>>>(d, 4000);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[kModes]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    for (int m = 0; m < kModes; ++m)
      printf("grid %3d  %-22s %lld clk per 128^3 per SM (%s)\n", grid, names[m], h[m],
             cudaGetErrorString(e));
  }
  return 0;
}
