// Chunk-attention backward for sm_100a, warp-specialised: the probability
// pass (P) and the gradient-of-scores pass (dS) run on different warps, so
// P of the next query tile is computed while dS of the current one is.
//
// Reference semantics: block_attn_backward (flashcore.hpp:269-337)
//   P = exp(scale q k^T - lse); dV += P^T dO; dS = P o (dO v^T - D);
//   dQ += scale dS k;  dK += scale dS^T q;   D = rowsum(dO o O) precomputed.
//
// Per CTA = one kv head x one 128-row kv tile; loops over every (query head of
// the GQA group, query tile) that sees the kv tile. 512 threads:
//   warps 0-3   P warps:  P = exp2(S^T*scale*log2e - lse2) -> TMEM (bf16, packed)
//   warps 4-7   dS warps: read P, release the S region, dS = P o (dP - D)
//                         -> TMEM (A of dK) and smem (B of dQ^T)
//   warps 8-11  dQ drain: tcgen05.ld of dQ^T, TMA reduce-add into dq_acc
//   warp 12     MMA issuer, warp 13 loader (TMA), warps 14-15 idle
// TMEM (512 cols): dV [0,128) dK [128,256) S|P [256,384) dP|dS|dQ^T [384,512)
//   S^T  = K Q^T   (SS)            -> S region
//   dP^T = V dO^T  (SS)            -> dP region
//   dV  += P^T dO  (TS, A = P^T packed in the S region, B = dO MN-major)
//   dK  += dS^T Q  (TS, A = dS^T packed in the dP region, B = Q MN-major)
//   dQ^T = K^T dS^T (SS, both MN-major) -> dP region: head dim on TMEM lanes
// Per-iteration MMA order: dV(i), S(i+1) [after the dS warps read P(i)],
// dK(i), dQ^T(i) [after dS(i)], dP(i+1) [after dQ^T(i) is drained]. The P
// warps therefore compute P(i+1) while the dS warps compute dS(i).
//
// Bound (measured): besides the five 128^3 GEMMs per (kv tile, q tile), each
// pair reduce-adds a 64 KB fp32 dQ partial into L2 via TMA; at 32K x 32 heads
// that is 69 GB of L2 reductions per launch, and removing it (experiment
// build) takes the kernel from 21.1 to 17.4 ms, half of it to 19.9 ms. Plain
// TMA stores of the same bytes cost about as much (20.9 ms), LSU red.global
// from registers far more (29.5 ms): the cost is the partial's path through
// shared memory (64 KB STS + 64 KB TMA read per pair) competing with the MMA
// operand traffic (256 KB per pair), not the L2 reduction itself.
#include <cuda.h>
#include <cuda_bf16.h>

#include "kernels.h"
#include "sm100_ptx.cuh"

namespace da {
namespace bwdws {

#ifdef DA_TRACE
#define BWS_TRACE(cond, it, slot)                                             \
  do {                                                                        \
    if ((cond) && p.trace != nullptr && blockIdx.x == 0 && (it) < 64)         \
      p.trace[(it) * 16 + (slot)] = clock64();                                \
  } while (0)
// per-CTA record after the 64x16 iteration stamps: globaltimer start/end,
// clock64 start/end, smid, iterations, first MMA issue, last MMA commit
#define BWS_CTA_TRACE(slot, val)                                              \
  do {                                                                        \
    if (p.trace != nullptr)                                                   \
      p.trace[1024 + static_cast<size_t>(blockIdx.x) * 8 + (slot)] = (val);   \
  } while (0)
__device__ __forceinline__ unsigned long long bws_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long bws_smid() {
  uint32_t s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}
#else
#define BWS_TRACE(cond, it, slot) \
  do {                            \
  } while (0)
#define BWS_CTA_TRACE(slot, val) \
  do {                           \
  } while (0)
#endif

// Grid order: the CTAs of `head_group` kv heads are interleaved, so the
// co-resident CTAs share those heads' Q / dO tiles and dQ reduction targets
// in L2. Chosen per launch by the host (launch_attn_bwd): 2 while two heads'
// working set (dQ fp32 + Q + dO, ~1 KB per query row) fits the 126 MB L2,
// else 1 — e.g. the 64K x 64K Full chunk pair of cfg4 runs 1032 vs 907
// TFLOP/s with 1 (profiles/ab_r2_bwd_head_group.txt). DA_BWD_HEAD_GROUP
// forces a value (experiments).
#ifndef DA_BWD_HEAD_GROUP
#define DA_BWD_HEAD_GROUP 0
#endif
constexpr int kHeadGroupForced = DA_BWD_HEAD_GROUP;
constexpr int kBM = 128;  // query rows per iteration
constexpr int kBN = 128;  // kv rows per CTA
constexpr int kHD = 128;
constexpr uint32_t kTileBytes = 128 * 128 * 2;
constexpr uint32_t kHalfTile = kTileBytes / 2;
constexpr int kThreads = 512;
constexpr int kLaunchRegs = 128;  // the setmaxnreg budget below assumes exactly this
constexpr uint32_t kColDV = 0;
constexpr uint32_t kColDK = 128;
constexpr uint32_t kColS = 256;
constexpr uint32_t kColDP = 384;

struct SmemLayout {
  static constexpr uint32_t k = 0;
  static constexpr uint32_t v = k + kTileBytes;
  static constexpr uint32_t q = v + kTileBytes;         // 2 stages
  static constexpr uint32_t dout = q + 2 * kTileBytes;  // 1 stage
  static constexpr uint32_t ds = dout + kTileBytes;     // dS^T [kv][q] bf16, SW128
  static constexpr uint32_t vecs = ds + kTileBytes;     // 2 stages x (-lse2[128], -D[128])
  static constexpr uint32_t bars = vecs + 2 * 2 * 128 * 4;
  // 4 drain warps x 2 boxes of [32 q][32 d] fp32: two TMA reductions in flight
  // per warp (the drain throughput is bounded by bytes in flight / latency)
  static constexpr uint32_t dq_stage = bars + 256;
  static constexpr uint32_t total = dq_stage + 4 * 2 * 32 * 32 * 4;
};
// The dynamic window starts 1024-aligned on sm_100 (after the 1 KB reserved
// per CTA), so no alignment slack is reserved; the kernel traps if it is not.
constexpr size_t kSmemBytes = SmemLayout::total;
static_assert(kSmemBytes <= 232448, "dynamic shared memory per CTA");

struct Bars {
  uint64_t kv_full;
  uint64_t q_full[2];
  uint64_t q_empty[2];
  uint64_t vec_full[2];
  uint64_t vec_empty[2];  // P + dS warps (one arrive per warp) -> loader
  uint64_t do_full;
  uint64_t do_empty;
  uint64_t s_full;
  uint64_t dp_full;
  uint64_t p_full;   // P warps -> MMA: P(i) packed in the S region
  uint64_t p_read;   // dS warps -> MMA: P(i) is in registers, S region reusable
  uint64_t ds_full;  // dS warps -> MMA: dS(i) in TMEM and smem
  uint64_t dq_full;
  uint64_t dq_drained;
  uint64_t acc_full;
  uint32_t tmem_base;
};
static_assert(sizeof(Bars) <= 256, "barrier block");

// dK/dV epilogue: each thread stores its accumulator row (TMEM lane) from
// registers. (Staging the rows in the free smem tiles and writing them with TMA
// stores measured ~5% slower overall: the bulk stores delay the next CTA's
// loads on the same SM.)
__device__ __forceinline__ void store_acc_rows_lsu(float* dst, bool valid, uint32_t tmem_cols,
                                                   float f, bool accumulate) {
#pragma unroll 1
  for (int c = 0; c < 4; ++c) {
    uint32_t a[32];
    tmem_ld_32x32b_x32(tmem_cols + c * 32, a);
    tmem_ld_wait();
    if (!valid) continue;
    float4* d4 = reinterpret_cast<float4*>(dst + c * 32);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float4 x = make_float4(f * __uint_as_float(a[4 * i]), f * __uint_as_float(a[4 * i + 1]),
                             f * __uint_as_float(a[4 * i + 2]), f * __uint_as_float(a[4 * i + 3]));
      if (accumulate) {
        const float4 o = d4[i];
        x.x += o.x; x.y += o.y; x.z += o.z; x.w += o.w;
      }
      d4[i] = x;
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    attn_bwd_ws_kernel(const __grid_constant__ CUtensorMap tmap_q,
                       const __grid_constant__ CUtensorMap tmap_k,
                       const __grid_constant__ CUtensorMap tmap_v,
                       const __grid_constant__ CUtensorMap tmap_do,
                       const __grid_constant__ CUtensorMap tmap_dq, const BwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // SW128 tiles need 1024-byte alignment: checked, not padded (see kSmemBytes)
  if (smem_align_pad(smem_raw) != 0) __trap();  // see kSmemBytes
  uint8_t* smem = smem_raw;
  Bars* bars = reinterpret_cast<Bars*>(smem + SmemLayout::bars);
  float* vecs = reinterpret_cast<float*>(smem + SmemLayout::vecs);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;

  // ---- work: head-major, within a head the kv tiles with most query tiles first
  const int n_q_tiles = (p.rows_q + kBM - 1) / kBM;
  const int n_kv_tiles = (p.rows_kv + kBN - 1) / kBN;
  // kv heads in groups of head_group, interleaved within a group (L2 holds the
  // group's Q/dO; the last wave mixes heads instead of one head's tiles)
  const int b = static_cast<int>(blockIdx.x);
  const int head_group = p.head_group;
  const int g0 = (b / (head_group * n_kv_tiles)) * head_group;
  const int g_heads = min(head_group, p.h_kv - g0);
  const int r_in = b - g0 * n_kv_tiles;
  const int kv_head = g0 + r_in % g_heads;
  const int slot = r_in / g_heads;
  // deterministic mode launches each head's kv tiles lightest-first: a CTA
  // only ever waits for a higher kv tile, which was launched before it
  const int jt = p.dq_sem != nullptr ? n_kv_tiles - 1 - slot : slot;
  const int group = p.h_q / p.h_kv;
  const int i0 = (p.mask == DA_MASK_DIAGONAL) ? jt : 0;
  const int n_i = n_q_tiles - i0;
  const int n_it = n_i > 0 ? group * n_i : 0;
  if (threadIdx.x == 0) {
    BWS_CTA_TRACE(0, bws_gtimer());
    BWS_CTA_TRACE(2, clock64());
  }

  if (warp == 0) {
    if (lane == 0) {
      mbar_init(&bars->kv_full, 1);
      for (int s = 0; s < 2; ++s) {
        mbar_init(&bars->q_full[s], 1);
        mbar_init(&bars->q_empty[s], 1);
        mbar_init(&bars->vec_full[s], 1);
        mbar_init(&bars->vec_empty[s], 8);
      }
      mbar_init(&bars->do_full, 1);
      mbar_init(&bars->do_empty, 1);
      mbar_init(&bars->s_full, 1);
      mbar_init(&bars->dp_full, 1);
      mbar_init(&bars->p_full, 128);
      mbar_init(&bars->p_read, 128);
      mbar_init(&bars->ds_full, 128);
      mbar_init(&bars->dq_full, 1);
      mbar_init(&bars->dq_drained, 128);
      mbar_init(&bars->acc_full, 1);
      fence_barrier_init();
    }
  } else if (warp == 13) {
    if (lane == 0) {
      tma_prefetch_desc(&tmap_q);
      tma_prefetch_desc(&tmap_k);
      tma_prefetch_desc(&tmap_v);
      tma_prefetch_desc(&tmap_do);
    }
  } else if (warp == 8) {
    if (lane == 0) tma_prefetch_desc(&tmap_dq);
  } else if (warp == 12) {
    tmem_alloc<512>(&bars->tmem_base);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  // Register budget (setmaxnreg is warpgroup-granular; launch = 512 x 128):
  // the MMA/loader and P warpgroups (-> 96) give 2 x 32 x 128 registers to the
  // dS and drain warpgroups (-> 160).
  if (warp >= 12 || warp < 4) setmaxnreg_dec<96>();

  // iteration it -> (query head, query tile), stepped without division
  struct ItCursor {
    int hq, qt, i0, q_end;
    __device__ __forceinline__ void next() {
      if (++qt == q_end) {
        qt = i0;
        ++hq;
      }
    }
  };
  const ItCursor cur0{kv_head * group, i0, i0, n_q_tiles};

  if (warp == 13) {
    // ===================== loader =====================
    constexpr float kLog2e = 1.4426950408889634f;
    if (lane == 0) {
      mbar_arrive_expect_tx(&bars->kv_full, 2 * kTileBytes);
      tma_load_3d(smem + SmemLayout::k, &tmap_k, &bars->kv_full, 0, jt * kBN, kv_head);
      tma_load_3d(smem + SmemLayout::k + kHalfTile, &tmap_k, &bars->kv_full, 64, jt * kBN, kv_head);
      tma_load_3d(smem + SmemLayout::v, &tmap_v, &bars->kv_full, 0, jt * kBN, kv_head);
      tma_load_3d(smem + SmemLayout::v + kHalfTile, &tmap_v, &bars->kv_full, 64, jt * kBN, kv_head);
    }
    ItCursor cur = cur0;
    for (int it = 0; it < n_it; ++it, cur.next()) {
      const int st = it & 1;
      const uint32_t ph = (it >> 1) & 1;
      const int hq = cur.hq;
      const int row0 = cur.qt * kBM;
      mbar_wait(&bars->q_empty[st], ph ^ 1);
      if (lane == 0) {
#ifdef DA_BWD_EXPERIMENT_NO_RELOAD  // (cost probe only: reuses stale Q/dO tiles)
        if (it >= 2) {
          mbar_arrive(&bars->q_full[st]);
        } else
#endif
        {
        mbar_arrive_expect_tx(&bars->q_full[st], kTileBytes);
        uint8_t* qs = smem + SmemLayout::q + st * kTileBytes;
        tma_load_3d(qs, &tmap_q, &bars->q_full[st], 0, row0, hq);
        tma_load_3d(qs + kHalfTile, &tmap_q, &bars->q_full[st], 64, row0, hq);
        }
      }
      // -lse (log2 units) and -D for the 128 query rows; padding rows get
      // -lse2 = -inf so their probabilities are exactly zero
      float l2[4], dd[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int row = row0 + lane * 4 + k;
        l2[k] = -INFINITY;
        dd[k] = 0.f;
        if (row < p.rows_q) {
          const size_t idx = static_cast<size_t>(hq) * p.rows_q + row;
          l2[k] = -p.lse[idx] * kLog2e;
          dd[k] = -p.d_vec[idx] * p.scale;  // the softmax scale rides on dS
        }
      }
      if (lane == 0) {
        mbar_wait(&bars->do_empty, (it & 1) ^ 1);
#ifdef DA_BWD_EXPERIMENT_NO_RELOAD
        if (it >= 1) {
          mbar_arrive(&bars->do_full);
        } else
#endif
        {
        mbar_arrive_expect_tx(&bars->do_full, kTileBytes);
        tma_load_3d(smem + SmemLayout::dout, &tmap_do, &bars->do_full, 0, row0, hq);
        tma_load_3d(smem + SmemLayout::dout + kHalfTile, &tmap_do, &bars->do_full, 64, row0, hq);
        }
      }
      float* lse2 = vecs + st * 256;
      float* dvec = lse2 + 128;
      mbar_wait(&bars->vec_empty[st], ph ^ 1);  // iteration it-2 done reading this stage
      *reinterpret_cast<float4*>(lse2 + lane * 4) = make_float4(l2[0], l2[1], l2[2], l2[3]);
      *reinterpret_cast<float4*>(dvec + lane * 4) = make_float4(dd[0], dd[1], dd[2], dd[3]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->vec_full[st]);
    }
  } else if (warp == 12) {
    // ===================== MMA issuer =====================
    if (lane == 0 && n_it > 0) {
      constexpr uint32_t idesc_kk = make_idesc_bf16(128, 128, false, false);  // S, dP
      constexpr uint32_t idesc_kmn = make_idesc_bf16(128, 128, false, true);  // dV, dK
      constexpr uint32_t idesc_mnmn = make_idesc_bf16(128, 128, true, true);  // dQ^T
      const uint32_t k_addr = smem_u32(smem + SmemLayout::k);
      const uint32_t v_addr = smem_u32(smem + SmemLayout::v);
      const uint32_t q_addr = smem_u32(smem + SmemLayout::q);
      const uint32_t do_addr = smem_u32(smem + SmemLayout::dout);
      const uint32_t ds_addr = smem_u32(smem + SmemLayout::ds);

      // D = A B^T with both operands K-major [128][128] SW128 tiles
      auto gemm_kk = [&](uint32_t d_tmem, uint32_t a, uint32_t b) {
#pragma unroll
        for (int kk = 0; kk < kHD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kHalfTile + (kk & 3) * 32;
          mma_ss(d_tmem, make_sdesc_sw128(a + off, 16, 1024), make_sdesc_sw128(b + off, 16, 1024),
                 idesc_kk, kk > 0 ? 1u : 0u);
        }
      };
      // D (+)= A[tmem, packed bf16 pairs, K = 128 query columns] * B (MN-major [q][d])
      auto gemm_ts = [&](uint32_t d_tmem, uint32_t a_tmem, uint32_t b, bool acc) {
#pragma unroll
        for (int kk = 0; kk < kBM / 16; ++kk)
          mma_ts(d_tmem, a_tmem + kk * 8, make_sdesc_sw128(b + kk * 2048, kHalfTile, 1024),
                 idesc_kmn, (acc || kk > 0) ? 1u : 0u);
      };

      mbar_wait(&bars->kv_full, 0);
      mbar_wait(&bars->q_full[0], 0);
      BWS_CTA_TRACE(6, clock64());
      tc_fence_after();
      gemm_kk(tmem + kColS, k_addr, q_addr);
      mma_commit(&bars->s_full);
      mbar_wait(&bars->do_full, 0);
      tc_fence_after();
      gemm_kk(tmem + kColDP, v_addr, do_addr);
      mma_commit(&bars->dp_full);

      for (int it = 0; it < n_it; ++it) {
        const int st = it & 1;
        const bool has_next = it + 1 < n_it;
        // dV += P^T dO
        mbar_wait(&bars->p_full, it & 1);
        BWS_TRACE(true, it, 0);
        tc_fence_after();
        gemm_ts(tmem + kColDV, tmem + kColS, do_addr, it > 0);
        mma_commit(&bars->do_empty);
        // next S^T once the dS warps hold P(it) in registers (dV precedes it in
        // the in-order pipe, so it has consumed P by the time S is written)
        if (has_next) {
          const int st1 = (it + 1) & 1;
          mbar_wait(&bars->p_read, it & 1);
          mbar_wait(&bars->q_full[st1], ((it + 1) >> 1) & 1);
          tc_fence_after();
          gemm_kk(tmem + kColS, k_addr, q_addr + st1 * kTileBytes);
          mma_commit(&bars->s_full);
        }
        // dK += dS^T Q, then dQ^T = K^T dS^T over the same region (in order)
        mbar_wait(&bars->ds_full, it & 1);
        BWS_TRACE(true, it, 1);
        tc_fence_after();
        gemm_ts(tmem + kColDK, tmem + kColDP, q_addr + st * kTileBytes, it > 0);
        mma_commit(&bars->q_empty[st]);
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk) {
          mma_ss(tmem + kColDP, make_sdesc_sw128(k_addr + kk * 2048, kHalfTile, 1024),
                 make_sdesc_sw128(ds_addr + kk * 2048, kHalfTile, 1024), idesc_mnmn,
                 kk > 0 ? 1u : 0u);
        }
        mma_commit(&bars->dq_full);
        // next dP^T once dQ^T has left TMEM
        if (has_next) {
          mbar_wait(&bars->dq_drained, it & 1);
          BWS_TRACE(true, it, 2);
          mbar_wait(&bars->do_full, (it + 1) & 1);
          tc_fence_after();
          gemm_kk(tmem + kColDP, v_addr, do_addr);
          mma_commit(&bars->dp_full);
        }
      }
      mma_commit(&bars->acc_full);
      BWS_CTA_TRACE(7, clock64());
    }
  } else if (warp >= 14) {
    // idle warps of the MMA/loader warpgroup
  } else if (warp >= 8) {
    // ===================== dQ drain =====================
    setmaxnreg_inc<160>();
    const uint32_t dw = warp - 8;
    const uint32_t lane_base = tmem + (dw * 32u << 16);
    ItCursor cur = cur0;
    for (int it = 0; it < n_it; ++it, cur.next()) {
      const int hq = cur.hq;
      const int row0 = cur.qt * kBM;
      mbar_wait(&bars->dq_full, it & 1);
#ifdef DA_BWD_EXPERIMENT_MMA_ONLY  // (cost probe only: no dQ, P or dS math)
      tc_fence_before();
      mbar_arrive(&bars->dq_drained);
      continue;
#endif
      BWS_TRACE(dw == 0 && lane == 0, it, 8);
      tc_fence_after();
      uint32_t r[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(lane_base + kColDP + c * 32, r[c]);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&bars->dq_drained);
      BWS_TRACE(dw == 0 && lane == 0, it, 9);
      // deterministic order: the partials of query tile (hq, qt) are added by
      // descending kv tile; wait until every higher contributor has landed
      int* sem = nullptr;
      if (p.dq_sem != nullptr) {
        sem = p.dq_sem + static_cast<size_t>(hq) * n_q_tiles + cur.qt;
        const int turn = (p.mask == DA_MASK_DIAGONAL ? cur.qt : n_kv_tiles - 1) - jt;
        if (dw == 0 && lane == 0) {
          while (ld_acquire_gpu(sem) != turn) __nanosleep(64);
        }
        named_bar_sync(1, 128);
        fence_proxy_async_global();
      }
      // stage [32 q][32 d] boxes (this warp's 32 head-dim columns) and let TMA
      // reduce them into dq_acc: no LSU atomics; OOB query rows are clipped
      float* box2 = reinterpret_cast<float*>(smem + SmemLayout::dq_stage) + dw * 2 * 32 * 32;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float* box = box2 + (c & 1) * 32 * 32;
        // the reduction that last read this box was committed two groups ago
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 32; ++k) box[k * 32 + lane] = __uint_as_float(r[c][k]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
#if defined(DA_BWD_EXPERIMENT_DQ_STORE)  // (cost probe only: overwrites dQ)
          tma_store_3d(&tmap_dq, box, dw * 32, row0 + c * 32, hq);
#elif !defined(DA_BWD_EXPERIMENT_NO_DQ_REDUCE)  // (cost probe only: drops dQ)
          tma_reduce_add_3d(&tmap_dq, box, dw * 32, row0 + c * 32, hq);
#endif
          bulk_commit();
        }
      }
      BWS_TRACE(dw == 0 && lane == 0, it, 10);
      if (sem != nullptr) {
        // this CTA's partial is complete in global memory: pass the turn on
        if (lane == 0) bulk_wait<0>();
        __syncwarp();
        fence_proxy_async_global();
        named_bar_sync(1, 128);
        if (dw == 0 && lane == 0) {
          __threadfence();
          red_release_gpu_add(sem, 1);
        }
      }
    }
    // the staging boxes must outlive the TMA reads; the global adds complete
    // on their own before the grid is considered done
    if (lane == 0) bulk_wait_read<0>();
  } else if (warp < 4) {
    // ===================== P warps =====================
    const int quarter = warp;
    const int r = quarter * 32 + lane;  // kv row within the tile = TMEM lane
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const uint32_t s_tmem = lane_base + kColS;
    const float sl2 = p.scale_log2;
    ItCursor cur = cur0;
    for (int it = 0; it < n_it; ++it, cur.next()) {
      const int st = it & 1;
      const bool diag = (p.mask == DA_MASK_DIAGONAL) && (cur.qt == jt);
      const float* lse2 = vecs + st * 256;  // -lse * log2(e)
      mbar_wait(&bars->vec_full[st], (it >> 1) & 1);
      mbar_wait(&bars->s_full, it & 1);
#ifdef DA_BWD_EXPERIMENT_MMA_ONLY
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->vec_empty[st]);
      tc_fence_before();
      mbar_arrive(&bars->p_full);
      continue;
#endif
      BWS_TRACE(quarter == 0 && lane == 0, it, 3);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) {  // query columns [32 c, 32 c + 32)
        uint32_t sr[32];
        tmem_ld_32x32b_x32(s_tmem + c * 32, sr);
        tmem_ld_wait();
        if (diag) {
          // query column q is visible from kv row r iff q >= r: masked scores
          // become -inf (exact zeros) so the exp loop stays branch-free
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c * 32 + i < r) sr[i] = __float_as_uint(-INFINITY);
        }
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
#ifdef DA_BWD_VECS_FROM_GLOBAL
          // sanitizer-evidence build only: -lse2 straight from global memory,
          // bypassing the mbarrier-ordered smem ring (see profiles/sanitizer_r2.txt)
          float lv[4];
          for (int u = 0; u < 4; ++u) {
            const int row = cur.qt * kBM + c * 32 + i + u;
            lv[u] = row < p.rows_q
                        ? -p.lse[static_cast<size_t>(cur.hq) * p.rows_q + row] * 1.4426950408889634f
                        : -INFINITY;
          }
          const float4 l4 = make_float4(lv[0], lv[1], lv[2], lv[3]);
#else
          const float4 l4 = *reinterpret_cast<const float4*>(lse2 + c * 32 + i);
#endif
          const float2 x01 = ffma2(make_float2(__uint_as_float(sr[i]), __uint_as_float(sr[i + 1])),
                                   make_float2(sl2, sl2), make_float2(l4.x, l4.y));
          const float2 x23 =
              ffma2(make_float2(__uint_as_float(sr[i + 2]), __uint_as_float(sr[i + 3])),
                    make_float2(sl2, sl2), make_float2(l4.z, l4.w));
          pk[i / 2] = pack_bf16x2(ex2_approx(x01.x), ex2_approx(x01.y));
          pk[i / 2 + 1] = pack_bf16x2(ex2_approx(x23.x), ex2_approx(x23.y));
        }
        // packed pairs: column j of the S region holds P[r][2j], P[r][2j+1]
        // (columns [16 c, 16 c + 16): already read)
        tmem_st_32x32b_x16(s_tmem + c * 16, pk);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->vec_empty[st]);  // lse2[st] no longer read
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&bars->p_full);
      BWS_TRACE(quarter == 0 && lane == 0, it, 4);
    }
    // ---- epilogue: dV rows
    if (n_it > 0) {
      mbar_wait(&bars->acc_full, 0);
      tc_fence_after();
      store_acc_rows_lsu(p.dv_acc + (static_cast<size_t>(kv_head) * p.rows_kv + jt * kBN + r) * kHD,
                         jt * kBN + r < p.rows_kv, lane_base + kColDV, 1.f, p.accumulate_kv != 0);
    } else if (p.mask != DA_MASK_EMPTY && !p.accumulate_kv) {
      // no query tile sees this kv tile: the contribution is zero
      const int row = jt * kBN + r;
      if (row < p.rows_kv) {
        float4* d4 = reinterpret_cast<float4*>(
            p.dv_acc + (static_cast<size_t>(kv_head) * p.rows_kv + row) * kHD);
        for (int i = 0; i < 32; ++i) d4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  } else {
    // ===================== dS warps (4-7) =====================
    setmaxnreg_inc<160>();
    const int quarter = warp - 4;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const uint32_t s_tmem = lane_base + kColS;
    const uint32_t dp_tmem = lane_base + kColDP;
    uint8_t* ds_row = smem + SmemLayout::ds + r * 128;
    const float2 sc2 = make_float2(p.scale, p.scale);
    ItCursor cur = cur0;
    for (int it = 0; it < n_it; ++it, cur.next()) {
      const int st = it & 1;
      const float* dvec = vecs + st * 256 + 128;  // -D
      mbar_wait(&bars->vec_full[st], (it >> 1) & 1);
      mbar_wait(&bars->p_full, it & 1);  // P(it) written (P warps)
      mbar_wait(&bars->dp_full, it & 1);
#ifdef DA_BWD_EXPERIMENT_MMA_ONLY
      tc_fence_before();
      mbar_arrive(&bars->p_read);
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->vec_empty[st]);
      fence_proxy_async_smem();
      mbar_arrive(&bars->ds_full);
      continue;
#endif
      BWS_TRACE(quarter == 0 && lane == 0, it, 5);
      tc_fence_after();
      // P(it) (64 packed columns) into registers, then release the S region
      uint32_t pk[2][32];
      tmem_ld_32x32b_x32(s_tmem, pk[0]);
      tmem_ld_32x32b_x32(s_tmem + 32, pk[1]);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&bars->p_read);
      BWS_TRACE(quarter == 0 && lane == 0, it, 6);
#pragma unroll
      for (int c = 0; c < 4; ++c) {  // query columns [32 c, 32 c + 32)
        uint32_t dr[32];
        tmem_ld_32x32b_x32(dp_tmem + c * 32, dr);
        tmem_ld_wait();
        uint32_t dsk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const int qc = c * 32 + i;
#ifdef DA_BWD_VECS_FROM_GLOBAL  // sanitizer-evidence build only (see above)
          float dv4[4];
          for (int u = 0; u < 4; ++u) {
            const int row = cur.qt * kBM + qc + u;
            dv4[u] = row < p.rows_q ? -p.d_vec[static_cast<size_t>(cur.hq) * p.rows_q + row] * p.scale : 0.f;
          }
          const float4 d4 = make_float4(dv4[0], dv4[1], dv4[2], dv4[3]);
#else
          const float4 d4 = *reinterpret_cast<const float4*>(dvec + qc);
#endif
          const uint32_t a = pk[qc >> 6][(qc & 63) / 2], b = pk[qc >> 6][(qc & 63) / 2 + 1];
          // t = scale (dP - D) = scale dP + (-scale D): dS, hence dQ and dK, come
          // out scaled, so neither the dQ drain nor the dK epilogue multiplies
          const float2 t01 = ffma2(make_float2(__uint_as_float(dr[i]), __uint_as_float(dr[i + 1])),
                                   sc2, make_float2(d4.x, d4.y));
          const float2 t23 =
              ffma2(make_float2(__uint_as_float(dr[i + 2]), __uint_as_float(dr[i + 3])), sc2,
                    make_float2(d4.z, d4.w));
          // dS = P o bf16(dP - D) as one packed bf16 multiply per column pair:
          // the subtraction stays fp32 (no cancellation loss); dS is a bf16 MMA
          // operand either way. Against unpacking P and an fp32 multiply this
          // drops 3 of 5 instructions per pair on the dS warps (the cycle's
          // critical phase): backward -2.5% time, max rel. error of dq/dk
          // ~1.3x higher (e.g. dk 4.3e-3 -> 5.5e-3 at 4 x 4K; bar 2e-2),
          // profiles/ab_r2_bwd_ds_bf16mul.txt
          dsk[i / 2] = mul_bf16x2(a, pack_bf16x2(t01.x, t01.y));
          dsk[i / 2 + 1] = mul_bf16x2(b, pack_bf16x2(t23.x, t23.y));
        }
        // dS^T packed into the (already read) low columns of the dP region ...
        tmem_st_32x32b_x16(dp_tmem + c * 16, dsk);
        // ... and into smem (SW128, 64-column boxes): 4 x 16-byte chunks
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          const int chunk = (c & 1) * 4 + ch;
          const int phys = chunk ^ (r & 7);
          *reinterpret_cast<uint4*>(ds_row + (c >> 1) * kHalfTile + phys * 16) =
              make_uint4(dsk[4 * ch + 0], dsk[4 * ch + 1], dsk[4 * ch + 2], dsk[4 * ch + 3]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->vec_empty[st]);  // dvec[st] no longer read
      fence_proxy_async_smem();
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&bars->ds_full);
      BWS_TRACE(quarter == 0 && lane == 0, it, 7);
    }
    // ---- epilogue: dK rows (scaled)
    if (n_it > 0) {
      mbar_wait(&bars->acc_full, 0);
      tc_fence_after();
      store_acc_rows_lsu(p.dk_acc + (static_cast<size_t>(kv_head) * p.rows_kv + jt * kBN + r) * kHD,
                         jt * kBN + r < p.rows_kv, lane_base + kColDK, 1.f, p.accumulate_kv != 0);
    } else if (p.mask != DA_MASK_EMPTY && !p.accumulate_kv) {
      const int row = jt * kBN + r;
      if (row < p.rows_kv) {
        float4* d4 = reinterpret_cast<float4*>(
            p.dk_acc + (static_cast<size_t>(kv_head) * p.rows_kv + row) * kHD);
        for (int i = 0; i < 32; ++i) d4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 12) tmem_dealloc<512>(tmem);
  if (threadIdx.x == 0) {
    BWS_CTA_TRACE(1, bws_gtimer());
    BWS_CTA_TRACE(3, clock64());
    BWS_CTA_TRACE(4, bws_smid());
    BWS_CTA_TRACE(5, static_cast<unsigned long long>(n_it));
  }
}

}  // namespace bwdws

cudaError_t launch_attn_bwd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                            const CUtensorMap& tdo, const CUtensorMap& tdq, const BwdParams& p,
                            cudaStream_t stream) {
  static std::atomic<uint64_t> configured{0};
  cudaError_t e = once_per_device(configured, [] {
    cudaError_t r = cudaFuncSetAttribute(bwdws::attn_bwd_ws_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(bwdws::kSmemBytes));
    if (r != cudaSuccess) return r;
    cudaFuncAttributes attr{};
    r = cudaFuncGetAttributes(&attr, bwdws::attn_bwd_ws_kernel);
    if (r != cudaSuccess) return r;
    // setmaxnreg redistributes a fixed CTA budget; any other launch register
    // count would make the drain warps' increase wait forever.
    return attr.numRegs == bwdws::kLaunchRegs ? cudaSuccess : cudaErrorInvalidConfiguration;
  });
  if (e != cudaSuccess) return e;
  const int n_kv_tiles = (p.rows_kv + bwdws::kBN - 1) / bwdws::kBN;
  dim3 grid(n_kv_tiles * p.h_kv);
  BwdParams pp = p;
  if (bwdws::kHeadGroupForced > 0) {
    pp.head_group = bwdws::kHeadGroupForced;
  } else {
    constexpr double kL2Budget = 80.0 * (1 << 20);  // of the 126 MB L2
    pp.head_group = 2.0 * static_cast<double>(p.rows_q) * 1024.0 <= kL2Budget ? 2 : 1;
  }
  bwdws::attn_bwd_ws_kernel<<<grid, bwdws::kThreads, bwdws::kSmemBytes, stream>>>(tq, tk, tv, tdo,
                                                                                  tdq, pp);
  return cudaGetLastError();
}

}  // namespace da

