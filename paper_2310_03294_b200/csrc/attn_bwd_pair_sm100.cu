// Chunk-attention backward for sm_100a on CTA pairs (tcgen05 cta_group::2).
//
// Reference semantics: block_attn_backward (flashcore.hpp:269-337)
//   P = exp(scale q k^T - lse); dV += P^T dO; dS = P o (dO v^T - D);
//   dQ += scale dS k;  dK += scale dS^T q;   D = rowsum(dO o O) precomputed.
//
// Why pairs. The single-CTA kernel (attn_bwd_ws_sm100.cu) is bound by the
// SM's shared-memory bandwidth: 512 KB per (kv tile, q tile) of 128 x 128,
// of which 256 KB are MMA operand reads and 128 KB the dQ partial's staging.
// In a CTA pair every GEMM is M = 256: each CTA supplies its own 128 rows of
// A and HALF of B, and the tensor cores exchange the B halves, so B reads per
// SM halve. The pair owns two adjacent kv tiles (CTA r: kv tile 2*jp + r) and
// walks the same query tiles:
//   S^T  = K Q^T       (SS, M = 256 kv rows, N = 128 q)   -> S region
//   dP^T = V dO^T      (SS)                               -> dP region
//   dV  += P^T dO      (TS, A = P^T packed in TMEM, N = head dim)
//   dK  += dS^T Q      (TS, A = dS^T packed in TMEM)
//   dQ   = dS K        (SS, M = 256 = two query tiles, K = 256 kv rows)
// dQ needs M = 256 query rows, so it runs once per TWO query tiles: tile t is
// owned by CTA (t & 1); both CTAs write their dS^T(t) (their kv rows) into the
// owner's shared memory (the partner's half over DSMEM), and one GEMM gives
// each CTA the complete dQ of its tile over the pair's 256 kv rows. The dQ
// partial leaving the SM is therefore per (kv PAIR, q tile): half the L2
// reductions and half the staging of the single-CTA kernel.
//
// Shared memory per (kv tile, q tile) and SM: 176 KB MMA operands (S^T 48,
// dP^T 48, dV 16, dK 16, dQ 48), 64 KB Q/dO TMA writes, 32 KB dS stores,
// 64 KB dQ staging, 32 KB -lse/-D broadcasts: 368 KB vs 512 KB.
//
// Capacity (227 KB per CTA) is met by single-buffering every streamed operand
// as two pieces with separate lifetimes (the S^T/dP^T B half "XZ" = 64 query
// rows x 128, the dV/dK B half "Y" = 128 query rows x 64 head-dim columns,
// each refilled one MMA period ahead), and by time-sharing the dQ GEMM's
// K pieces with the dQ staging buffer (the K pieces are re-read after each
// drain, 16 KB per iteration).
//
// Warps (512 threads per CTA): 0-3 P, 4-7 dS, 8-11 dQ drain, 12 MMA (the
// leader CTA's lane 0 issues for the pair), 13 TMA loader, 14 -lse/-D loader.
//
// Measured (round 2, profiles/bwd_pair_r2.txt): correct (the backward parity
// suites pass with DA_BWD_KERNEL=pair) but SLOWER than the single-CTA kernel,
// 33 ms vs 21 ms at 32 heads x 32K. The per-iteration timeline
// (tools/trace_bwd2.py, DA_TRACE build) shows why:
//   * the DSMEM exchange of the partner's dS half (32 KB per query tile,
//     st.shared::cluster + fence.proxy.async.shared::cluster) costs ~2 us per
//     tile on the non-owner's dS warps;
//   * with the exchange removed (cost probe DA_BWD2_PROBE_NO_XCTA, wrong dQ)
//     an iteration still takes ~2.6 us at 16K, the single-CTA kernel's period:
//     the bound is the MMA dependency chain, not shared-memory bandwidth. Each
//     GEMM is one 8-instruction accumulator chain (~90-120 clk per M=256
//     instruction), S(i+1) must queue behind dV(i) (P(i) aliases the S
//     columns), and the dQ GEMM shares TMEM with dP, so every other iteration
//     serialises dK -> dQ -> drain -> dP.
// Cluster-scope release/acquire (mbarrier .release.cluster / .acquire.cluster)
// compile to MEMBAR.ALL.GPU / CCTL.IVALL and cost ~1 us per hand-off; the
// kernel therefore uses default-semantics arrives and waits (as CUTLASS does).
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdlib>
#include <cstring>

#include "kernels.h"
#include "sm100_ptx.cuh"

namespace da {
namespace bwd2 {

#ifndef DA_BWD_HEAD_GROUP
#define DA_BWD_HEAD_GROUP 0
#endif
constexpr int kHeadGroupForced = DA_BWD_HEAD_GROUP;
constexpr int kBM = 128;  // query rows per iteration
constexpr int kBN = 128;  // kv rows per CTA
constexpr int kHD = 128;
constexpr uint32_t kTile = 32768;    // 128 x 128 bf16
constexpr uint32_t kHalf = 16384;    // 128 x 64 bf16 (one SW128 box)
constexpr uint32_t kQuarter = 8192;  // 64 x 64 bf16
constexpr int kThreads = 512;
constexpr int kLaunchRegs = 128;
constexpr uint32_t kColDV = 0;
constexpr uint32_t kColDK = 128;
constexpr uint32_t kColS = 256;
constexpr uint32_t kColDP = 384;

#ifdef DA_TRACE
// per-iteration globaltimer stamps of pair 0 (CTA 0 and CTA 1: comparable
// across the two SMs), 32 iterations x 32 slots
#define B2_TRACE(cond, it, slot)                                                    \
  do {                                                                            \
    if ((cond) && p.trace != nullptr && blockIdx.x < 2 && (it) < 32)              \
      p.trace[(it) * 32 + (slot)] = globaltimer_ns();                             \
  } while (0)
#else
#define B2_TRACE(cond, it, slot) \
  do {                           \
  } while (0)
#endif

struct SmemLayout {
  static constexpr uint32_t k = 0;                // own K tile [dh0 | dh1], K-major A of S^T
  static constexpr uint32_t v = k + kTile;        // own V tile, A of dP^T
  static constexpr uint32_t kdq = v + kTile;      // K[tile 2jp][dh r] | K[tile 2jp+1][dh r]; dQ staging
  static constexpr uint32_t qxz = kdq + kTile;    // Q rows [64r, 64r+64): [dh0 | dh1]
  static constexpr uint32_t qy = qxz + kHalf;     // Q rows [0,128) x dh r
  static constexpr uint32_t doxz = qy + kHalf;
  static constexpr uint32_t doy = doxz + kHalf;
  static constexpr uint32_t ds = doy + kHalf;     // slot s = kv tile 2jp+s: dS^T [kv][q] as [qh0 | qh1]
  static constexpr uint32_t vecs = ds + 2 * kTile;  // 2 stages x (-lse2[128], -D[128])
  static constexpr uint32_t bars = vecs + 2 * 2 * 128 * 4;
  static constexpr uint32_t total = bars + 256;
};
constexpr size_t kSmemBytes = SmemLayout::total;
static_assert(kSmemBytes <= 232448, "dynamic shared memory per CTA");

struct Bars {
  // leader (rank 0) barriers: TMA completions of both CTAs, arrivals of both CTAs' warps
  uint64_t kv_full;
  uint64_t kdq_full;
  uint64_t qxz_full, qy_full, doxz_full, doy_full;
  uint64_t p_full;      // P(i) packed in TMEM, 4 warps x 2 CTAs
  uint64_t p_read;      // dS warps hold P(i) in registers: S region reusable
  uint64_t ds_full;     // dS(i) in TMEM and in the owner's smem
  uint64_t dq_drained;  // dQ left TMEM (both CTAs)
  // local barriers (pair MMA commits arrive in both CTAs)
  uint64_t qxz_empty, qy_empty, doxz_empty, doy_empty;
  uint64_t s_full, dp_full, dq_full, acc_full;
  uint64_t vec_full[2], vec_empty[2];
  uint64_t p_local;  // this CTA's P warps -> its dS warps
  uint32_t tmem_base;
};
static_assert(sizeof(Bars) <= 256, "barrier block");

__device__ __forceinline__ void store_acc_rows(float* dst, bool valid, uint32_t tmem_cols, float f,
                                               bool accumulate) {
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

// iteration -> (query head, query tile), stepped without division
struct ItCursor {
  int hq, qt, i0, q_end;
  __device__ __forceinline__ void next() {
    if (++qt == q_end) {
      qt = i0;
      ++hq;
    }
  }
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    attn_bwd_pair_kernel(const __grid_constant__ CUtensorMap tmap_q,
                         const __grid_constant__ CUtensorMap tmap_q64,
                         const __grid_constant__ CUtensorMap tmap_k,
                         const __grid_constant__ CUtensorMap tmap_v,
                         const __grid_constant__ CUtensorMap tmap_do,
                         const __grid_constant__ CUtensorMap tmap_do64,
                         const __grid_constant__ CUtensorMap tmap_dq, const BwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (smem_align_pad(smem_raw) != 0) __trap();
  uint8_t* smem = smem_raw;
  Bars* bars = reinterpret_cast<Bars*>(smem + SmemLayout::bars);
  float* vecs = reinterpret_cast<float*>(smem + SmemLayout::vecs);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  auto lead = [](uint64_t* b) { return mapa_shared(smem_u32(b), 0); };

  // ---- work: the pair's kv tiles (2 jp, 2 jp + 1) of one kv head
  const int n_q_tiles = (p.rows_q + kBM - 1) / kBM;
  const int n_kv_tiles = (p.rows_kv + kBN - 1) / kBN;
  const int n_pairs = (n_kv_tiles + 1) / 2;
  const int pb = static_cast<int>(blockIdx.x >> 1);
  const int head_group = p.head_group;
  const int g0 = (pb / (head_group * n_pairs)) * head_group;
  const int g_heads = min(head_group, p.h_kv - g0);
  const int r_in = pb - g0 * n_pairs;
  const int kv_head = g0 + r_in % g_heads;
  const int jp = r_in / g_heads;
  const int jt = 2 * jp + static_cast<int>(rank);
  const int group = p.h_q / p.h_kv;
  const int i0 = (p.mask == DA_MASK_DIAGONAL) ? 2 * jp : 0;
  const int n_i = n_q_tiles - i0;
  const int n_it = n_i > 0 ? group * n_i : 0;
  const int n_dq = (n_it + 1) / 2;

  if (warp == 0) {
    if (lane == 0) {
      mbar_init(&bars->kv_full, 1);
      mbar_init(&bars->kdq_full, 1);
      mbar_init(&bars->qxz_full, 1);
      mbar_init(&bars->qy_full, 1);
      mbar_init(&bars->doxz_full, 1);
      mbar_init(&bars->doy_full, 1);
      mbar_init(&bars->p_full, 8);
      mbar_init(&bars->p_read, 8);
      mbar_init(&bars->ds_full, 8);
      mbar_init(&bars->dq_drained, 8);
      mbar_init(&bars->qxz_empty, 1);
      mbar_init(&bars->qy_empty, 1);
      mbar_init(&bars->doxz_empty, 1);
      mbar_init(&bars->doy_empty, 1);
      mbar_init(&bars->s_full, 1);
      mbar_init(&bars->dp_full, 1);
      mbar_init(&bars->dq_full, 1);
      mbar_init(&bars->acc_full, 1);
      for (int s = 0; s < 2; ++s) {
        mbar_init(&bars->vec_full[s], 1);
        mbar_init(&bars->vec_empty[s], 8);
      }
      mbar_init(&bars->p_local, 4);
      fence_barrier_init();
    }
  } else if (warp == 13) {
    if (lane == 0) {
      tma_prefetch_desc(&tmap_q);
      tma_prefetch_desc(&tmap_q64);
      tma_prefetch_desc(&tmap_k);
      tma_prefetch_desc(&tmap_v);
      tma_prefetch_desc(&tmap_do);
      tma_prefetch_desc(&tmap_do64);
    }
  } else if (warp == 8) {
    if (lane == 0) tma_prefetch_desc(&tmap_dq);
  } else if (warp == 12) {
    tmem_alloc_pair<512>(&bars->tmem_base);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // peer barriers initialised before any remote arrive / TMA signal
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp >= 12 || warp < 4) setmaxnreg_dec<96>();

  const ItCursor cur0{kv_head * group, i0, i0, n_q_tiles};

  if (warp == 13) {
    // ===================== TMA loader (both CTAs, own smem, leader's barriers) =====
    if (lane == 0 && n_it > 0) {
      const int r64 = static_cast<int>(rank) * 64;
      if (rank == 0) mbar_arrive_expect_tx(&bars->kv_full, 2 * 2 * kTile);
      tma_load_3d_pair(smem + SmemLayout::k, &tmap_k, lead(&bars->kv_full), 0, jt * kBN, kv_head);
      tma_load_3d_pair(smem + SmemLayout::k + kHalf, &tmap_k, lead(&bars->kv_full), 64, jt * kBN,
                       kv_head);
      tma_load_3d_pair(smem + SmemLayout::v, &tmap_v, lead(&bars->kv_full), 0, jt * kBN, kv_head);
      tma_load_3d_pair(smem + SmemLayout::v + kHalf, &tmap_v, lead(&bars->kv_full), 64, jt * kBN,
                       kv_head);
      if (rank == 0) mbar_arrive_expect_tx(&bars->kdq_full, 2 * kTile);
      tma_load_3d_pair(smem + SmemLayout::kdq, &tmap_k, lead(&bars->kdq_full), r64,
                       (2 * jp) * kBN, kv_head);
      tma_load_3d_pair(smem + SmemLayout::kdq + kHalf, &tmap_k, lead(&bars->kdq_full), r64,
                       (2 * jp + 1) * kBN, kv_head);
      ItCursor cur = cur0;
      for (int j = 0; j < n_it; ++j, cur.next()) {
        const int hq = cur.hq;
        const int row0 = cur.qt * kBM;
        const uint32_t pe = (j - 1) & 1;
        // S^T(j)'s B half: query rows [64 r, 64 r + 64), both head-dim halves
        if (j > 0) mbar_wait(&bars->qxz_empty, pe);
        B2_TRACE(rank == 0, j, 27);
        if (rank == 0) mbar_arrive_expect_tx(&bars->qxz_full, 2 * kHalf);
        tma_load_3d_pair(smem + SmemLayout::qxz, &tmap_q64, lead(&bars->qxz_full), 0, row0 + r64, hq);
        tma_load_3d_pair(smem + SmemLayout::qxz + kQuarter, &tmap_q64, lead(&bars->qxz_full), 64,
                         row0 + r64, hq);
        // dP^T(j)'s B half
        if (j > 0) mbar_wait(&bars->doxz_empty, pe);
        B2_TRACE(rank == 0, j, 28);
        if (rank == 0) mbar_arrive_expect_tx(&bars->doxz_full, 2 * kHalf);
        tma_load_3d_pair(smem + SmemLayout::doxz, &tmap_do64, lead(&bars->doxz_full), 0, row0 + r64,
                         hq);
        tma_load_3d_pair(smem + SmemLayout::doxz + kQuarter, &tmap_do64, lead(&bars->doxz_full), 64,
                         row0 + r64, hq);
        // dV(j)'s B half: all 128 query rows, head-dim half r
        if (j > 0) mbar_wait(&bars->doy_empty, pe);
        B2_TRACE(rank == 0, j, 29);
        if (rank == 0) mbar_arrive_expect_tx(&bars->doy_full, 2 * kHalf);
        tma_load_3d_pair(smem + SmemLayout::doy, &tmap_do, lead(&bars->doy_full), r64, row0, hq);
        // dK(j)'s B half
        if (j > 0) mbar_wait(&bars->qy_empty, pe);
        B2_TRACE(rank == 0, j, 30);
        if (rank == 0) mbar_arrive_expect_tx(&bars->qy_full, 2 * kHalf);
        tma_load_3d_pair(smem + SmemLayout::qy, &tmap_q, lead(&bars->qy_full), r64, row0, hq);
      }
    }
  } else if (warp == 14) {
    // ===================== -lse (log2 units) / -D loader =====================
    constexpr float kLog2e = 1.4426950408889634f;
    ItCursor cur = cur0;
    for (int j = 0; j < n_it; ++j, cur.next()) {
      const int st = j & 1;
      const int row0 = cur.qt * kBM;
      float l2[4], dd[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int row = row0 + lane * 4 + k;
        l2[k] = -INFINITY;  // padding rows: probabilities exactly zero
        dd[k] = 0.f;
        if (row < p.rows_q) {
          const size_t idx = static_cast<size_t>(cur.hq) * p.rows_q + row;
          l2[k] = -p.lse[idx] * kLog2e;
          dd[k] = -p.d_vec[idx];
        }
      }
      float* lse2 = vecs + st * 256;
      float* dvec = lse2 + 128;
      mbar_wait(&bars->vec_empty[st], ((j >> 1) & 1) ^ 1);
      *reinterpret_cast<float4*>(lse2 + lane * 4) = make_float4(l2[0], l2[1], l2[2], l2[3]);
      *reinterpret_cast<float4*>(dvec + lane * 4) = make_float4(dd[0], dd[1], dd[2], dd[3]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->vec_full[st]);
    }
  } else if (warp == 12) {
    // ===================== MMA issuer (leader CTA only) =====================
    if (rank == 0 && lane == 0 && n_it > 0) {
      constexpr uint32_t idesc_ss = make_idesc_bf16(256, 128, false, false);  // S^T, dP^T
      constexpr uint32_t idesc_ts = make_idesc_bf16(256, 128, false, true);   // dV, dK
      constexpr uint32_t idesc_dq = make_idesc_bf16(256, 128, true, true);    // dQ
      const uint32_t k_addr = smem_u32(smem + SmemLayout::k);
      const uint32_t v_addr = smem_u32(smem + SmemLayout::v);
      const uint32_t kdq_addr = smem_u32(smem + SmemLayout::kdq);
      const uint32_t qxz_addr = smem_u32(smem + SmemLayout::qxz);
      const uint32_t qy_addr = smem_u32(smem + SmemLayout::qy);
      const uint32_t doxz_addr = smem_u32(smem + SmemLayout::doxz);
      const uint32_t doy_addr = smem_u32(smem + SmemLayout::doy);
      const uint32_t ds_addr = smem_u32(smem + SmemLayout::ds);
      // D = A B^T: A = own [128 kv][128 d] K-major, B = [64 q][128 d] K-major (per CTA)
      auto gemm_kk = [&](uint32_t d_tmem, uint32_t a, uint32_t b) {
#pragma unroll
        for (int kk = 0; kk < kHD / 16; ++kk) {
          const uint32_t ao = (kk >> 2) * kHalf + (kk & 3) * 32;
          const uint32_t bo = (kk >> 2) * kQuarter + (kk & 3) * 32;
          mma2_ss(d_tmem, make_sdesc_sw128(a + ao, 16, 1024), make_sdesc_sw128(b + bo, 16, 1024),
                  idesc_ss, kk > 0 ? 1u : 0u);
        }
      };
      // D (+)= A[tmem, packed bf16 pairs over 128 query columns] * B ([128 q][64 d] MN-major)
      auto gemm_ts = [&](uint32_t d_tmem, uint32_t a_tmem, uint32_t b, bool acc) {
#pragma unroll
        for (int kk = 0; kk < kBM / 16; ++kk)
          mma2_ts(d_tmem, a_tmem + kk * 8, make_sdesc_sw128(b + kk * 2048, kHalf, 1024), idesc_ts,
                  (acc || kk > 0) ? 1u : 0u);
      };

      mbar_wait(&bars->kv_full, 0);
      mbar_wait(&bars->qxz_full, 0);
      tc_fence_after();
      gemm_kk(tmem + kColS, k_addr, qxz_addr);
      mma2_commit_both(&bars->s_full);
      mma2_commit_both(&bars->qxz_empty);
      mbar_wait(&bars->doxz_full, 0);
      tc_fence_after();
      gemm_kk(tmem + kColDP, v_addr, doxz_addr);
      mma2_commit_both(&bars->dp_full);
      mma2_commit_both(&bars->doxz_empty);

      for (int it = 0; it < n_it; ++it) {
        const uint32_t ph = it & 1;
        const uint32_t ph1 = (it + 1) & 1;
        const bool has_next = it + 1 < n_it;
        // dV += P^T dO
        mbar_wait(&bars->p_full, ph);
        B2_TRACE(true, it, 0);
        mbar_wait(&bars->doy_full, ph);
        tc_fence_after();
        gemm_ts(tmem + kColDV, tmem + kColS, doy_addr, it > 0);
        mma2_commit_both(&bars->doy_empty);
        B2_TRACE(true, it, 25);
        // next S^T once both CTAs' dS warps hold P(it) in registers
        if (has_next) {
          mbar_wait(&bars->p_read, ph);
          B2_TRACE(true, it, 1);
          mbar_wait(&bars->qxz_full, ph1);
          tc_fence_after();
          gemm_kk(tmem + kColS, k_addr, qxz_addr);
          mma2_commit_both(&bars->s_full);
          mma2_commit_both(&bars->qxz_empty);
          B2_TRACE(true, it, 26);
        }
        // dK += dS^T Q
        mbar_wait(&bars->ds_full, ph);
        B2_TRACE(true, it, 2);
        mbar_wait(&bars->qy_full, ph);
        tc_fence_after();
        gemm_ts(tmem + kColDK, tmem + kColDP, qy_addr, it > 0);
        mma2_commit_both(&bars->qy_empty);
        // dQ of query tiles (it - 1, it) [or (it, -) at an odd end] over the pair's kv rows
        const bool do_dq = (it & 1) || !has_next;
        const int g = it >> 1;
        if (do_dq) {
          mbar_wait(&bars->kdq_full, g & 1);
          B2_TRACE(true, it, 3);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 2 * kBN / 16; ++kk) {
            const uint32_t ao = (kk >> 3) * kTile + (kk & 7) * 2048;
            const uint32_t bo = (kk >> 3) * kHalf + (kk & 7) * 2048;
            mma2_ss(tmem + kColDP, make_sdesc_sw128(ds_addr + ao, kHalf, 1024),
                    make_sdesc_sw128(kdq_addr + bo, kHalf, 1024), idesc_dq, kk > 0 ? 1u : 0u);
          }
          mma2_commit_both(&bars->dq_full);
        }
        // next dP^T (after dQ has left TMEM)
        if (has_next) {
          if (do_dq) mbar_wait(&bars->dq_drained, g & 1);
          B2_TRACE(true, it, 4);
          mbar_wait(&bars->doxz_full, ph1);
          B2_TRACE(true, it, 5);
          tc_fence_after();
          gemm_kk(tmem + kColDP, v_addr, doxz_addr);
          mma2_commit_both(&bars->dp_full);
          mma2_commit_both(&bars->doxz_empty);
        }
      }
      mma2_commit_both(&bars->acc_full);
    }
  } else if (warp == 15) {
    // idle
  } else if (warp >= 8) {
    // ===================== dQ drain =====================
    setmaxnreg_inc<160>();
    const uint32_t dw = warp - 8;
    const uint32_t lane_base = tmem + (dw * 32u << 16);
    ItCursor cur = cur0;
    if (rank == 1) cur.next();
    float* stage2 = reinterpret_cast<float*>(smem + SmemLayout::kdq) + dw * 2 * 32 * 32;
    const uint32_t kdq_bar = lead(&bars->kdq_full);
    for (int g = 0; g < n_dq; ++g) {
      const bool valid = 2 * g + static_cast<int>(rank) < n_it;
      mbar_wait(&bars->dq_full, g & 1);
      B2_TRACE(rank == 0 && dw == 0 && lane == 0, 2 * g + 1, 22);
      tc_fence_after();
      uint32_t r[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(lane_base + kColDP + c * 32, r[c]);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(lead(&bars->dq_drained));
      B2_TRACE(rank == 0 && dw == 0 && lane == 0, 2 * g + 1, 23);
      if (valid) {
        // thread = query row (TMEM lane); [32 q][32 d] fp32 boxes, 128B-swizzled
        const int row0 = cur.qt * kBM + static_cast<int>(dw) * 32;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          float* box = stage2 + (b & 1) * 32 * 32;
          if (b >= 2) {
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
          }
          uint8_t* row_base = reinterpret_cast<uint8_t*>(box) + lane * 128;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            const float4 x = make_float4(
                p.scale * __uint_as_float(r[b][4 * ch]), p.scale * __uint_as_float(r[b][4 * ch + 1]),
                p.scale * __uint_as_float(r[b][4 * ch + 2]), p.scale * __uint_as_float(r[b][4 * ch + 3]));
            *reinterpret_cast<float4*>(row_base + ((ch ^ (lane & 7)) << 4)) = x;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_reduce_add_3d(&tmap_dq, box, b * 32, row0, cur.hq);
            bulk_commit();
          }
        }
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
      }
      B2_TRACE(rank == 0 && dw == 0 && lane == 0, 2 * g + 1, 24);
      cur.next();
      cur.next();
      // staging read back: the region holds the K pieces of the next dQ GEMM again
      named_bar_sync(1, 128);
      if (g + 1 < n_dq && dw == 0 && lane == 0) {
        if (rank == 0) mbar_arrive_expect_tx(&bars->kdq_full, 2 * kTile);
        tma_load_3d_pair(smem + SmemLayout::kdq, &tmap_k, kdq_bar, static_cast<int>(rank) * 64,
                         (2 * jp) * kBN, kv_head);
        tma_load_3d_pair(smem + SmemLayout::kdq + kHalf, &tmap_k, kdq_bar,
                         static_cast<int>(rank) * 64, (2 * jp + 1) * kBN, kv_head);
      }
    }
  } else if (warp < 4) {
    // ===================== P warps =====================
    const int quarter = warp;
    const int r = quarter * 32 + lane;  // kv row within the tile = TMEM lane
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const uint32_t s_tmem = lane_base + kColS;
    const float sl2 = p.scale_log2;
    const uint32_t p_full_bar = lead(&bars->p_full);
    ItCursor cur = cur0;
    for (int it = 0; it < n_it; ++it, cur.next()) {
      const int st = it & 1;
      // query column q is visible from kv row r iff qt*128 + q >= jt*128 + r
      const bool masked = (p.mask == DA_MASK_DIAGONAL) && (cur.qt <= jt);
      const int mlim = r + (jt - cur.qt) * kBM;
      const float* lse2 = vecs + st * 256;
      mbar_wait(&bars->vec_full[st], (it >> 1) & 1);
      mbar_wait(&bars->s_full, it & 1);
      B2_TRACE(quarter == 0 && lane == 0, it, rank ? 8 : 6);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t sr[32];
        tmem_ld_32x32b_x32(s_tmem + c * 32, sr);
        tmem_ld_wait();
        if (masked) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c * 32 + i < mlim) sr[i] = __float_as_uint(-INFINITY);
        }
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 l4 = *reinterpret_cast<const float4*>(lse2 + c * 32 + i);
          const float2 x01 = ffma2(make_float2(__uint_as_float(sr[i]), __uint_as_float(sr[i + 1])),
                                   make_float2(sl2, sl2), make_float2(l4.x, l4.y));
          const float2 x23 =
              ffma2(make_float2(__uint_as_float(sr[i + 2]), __uint_as_float(sr[i + 3])),
                    make_float2(sl2, sl2), make_float2(l4.z, l4.w));
          pk[i / 2] = pack_bf16x2(ex2_approx(x01.x), ex2_approx(x01.y));
          pk[i / 2 + 1] = pack_bf16x2(ex2_approx(x23.x), ex2_approx(x23.y));
        }
        tmem_st_32x32b_x16(s_tmem + c * 16, pk);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->vec_empty[st]);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&bars->p_local);
        mbar_arrive_cluster(p_full_bar);
      }
      B2_TRACE(quarter == 0 && lane == 0, it, rank ? 9 : 7);
    }
    // ---- epilogue: dV rows
    if (n_it > 0) {
      mbar_wait(&bars->acc_full, 0);
      tc_fence_after();
      store_acc_rows(p.dv_acc + (static_cast<size_t>(kv_head) * p.rows_kv + jt * kBN + r) * kHD,
                     jt * kBN + r < p.rows_kv, lane_base + kColDV, 1.f, p.accumulate_kv != 0);
    } else if (p.mask != DA_MASK_EMPTY && !p.accumulate_kv) {
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
    // this CTA's kv rows land in slot `rank` of the owner's dS buffer
    const uint32_t ds_row = smem_u32(smem + SmemLayout::ds + rank * kTile + r * 128);
    const uint32_t ds_row_peer = mapa_shared(ds_row, rank ^ 1u);
    const uint32_t p_read_bar = lead(&bars->p_read);
    const uint32_t ds_full_bar = lead(&bars->ds_full);
    for (int it = 0; it < n_it; ++it) {
      const int st = it & 1;
      const bool local = static_cast<uint32_t>(it & 1) == rank;  // tile it is owned by CTA it & 1
      const float* dvec = vecs + st * 256 + 128;
      mbar_wait(&bars->vec_full[st], (it >> 1) & 1);
      mbar_wait(&bars->p_local, it & 1);
      mbar_wait(&bars->dp_full, it & 1);
      B2_TRACE(quarter == 0 && lane == 0, it, rank ? 16 : 10);
      tc_fence_after();
      uint32_t pk[2][32];
      tmem_ld_32x32b_x32(s_tmem, pk[0]);
      tmem_ld_32x32b_x32(s_tmem + 32, pk[1]);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(p_read_bar);
      B2_TRACE(quarter == 0 && lane == 0, it, rank ? 17 : 11);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c == 2) B2_TRACE(quarter == 0 && lane == 0, it, rank ? 18 : 12);
        uint32_t dr[32];
        tmem_ld_32x32b_x32(dp_tmem + c * 32, dr);
        tmem_ld_wait();
        uint32_t dsk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const int qc = c * 32 + i;
          const float4 d4 = *reinterpret_cast<const float4*>(dvec + qc);
          const uint32_t a = pk[qc >> 6][(qc & 63) / 2], b = pk[qc >> 6][(qc & 63) / 2 + 1];
          const float2 t01 = fadd2(make_float2(__uint_as_float(dr[i]), __uint_as_float(dr[i + 1])),
                                   make_float2(d4.x, d4.y));
          const float2 t23 =
              fadd2(make_float2(__uint_as_float(dr[i + 2]), __uint_as_float(dr[i + 3])),
                    make_float2(d4.z, d4.w));
          const float2 s01 =
              fmul2(make_float2(__uint_as_float(a << 16), __uint_as_float(a & 0xFFFF0000u)), t01);
          const float2 s23 =
              fmul2(make_float2(__uint_as_float(b << 16), __uint_as_float(b & 0xFFFF0000u)), t23);
          dsk[i / 2] = pack_bf16x2(s01.x, s01.y);
          dsk[i / 2 + 1] = pack_bf16x2(s23.x, s23.y);
        }
        // dS^T packed into the (already read) low columns of the dP region ...
        tmem_st_32x32b_x16(dp_tmem + c * 16, dsk);
        // ... and into the owner's dS buffer (SW128 [kv][64 q] boxes, MN-major A of dQ)
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          const int chunk = (c & 1) * 4 + ch;
          const uint32_t off = (c >> 1) * kHalf + ((chunk ^ (r & 7)) << 4);
          const uint4 v4 = make_uint4(dsk[4 * ch + 0], dsk[4 * ch + 1], dsk[4 * ch + 2], dsk[4 * ch + 3]);
#ifdef DA_BWD2_PROBE_NO_XCTA  // cost probe only: the partner half is not exchanged
          if (!local) continue;
#endif
          if (local) {
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(ds_row + off), "r"(v4.x),
                         "r"(v4.y), "r"(v4.z), "r"(v4.w)
                         : "memory");
          } else {
            st_cluster_v4(ds_row_peer + off, v4);
          }
        }
      }
      B2_TRACE(quarter == 0 && lane == 0, it, rank ? 19 : 13);
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->vec_empty[st]);
      if (local)
        fence_proxy_async_smem();
#ifndef DA_BWD2_PROBE_NO_XCTA
      else
        fence_proxy_async_smem_cluster();
#endif
      tmem_st_wait();
      B2_TRACE(quarter == 0 && lane == 0, it, rank ? 20 : 14);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(ds_full_bar);
      B2_TRACE(quarter == 0 && lane == 0, it, rank ? 21 : 15);
    }
    // ---- epilogue: dK rows (scaled)
    if (n_it > 0) {
      mbar_wait(&bars->acc_full, 0);
      tc_fence_after();
      store_acc_rows(p.dk_acc + (static_cast<size_t>(kv_head) * p.rows_kv + jt * kBN + r) * kHD,
                     jt * kBN + r < p.rows_kv, lane_base + kColDK, p.scale, p.accumulate_kv != 0);
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
  cluster_sync();  // the peer's MMAs, DSMEM stores and TMA signals into this CTA are done
  if (warp == 12) tmem_dealloc_pair<512>(tmem);
}

}  // namespace bwd2

cudaError_t launch_attn_bwd_pair(const CUtensorMap& tq, const CUtensorMap& tq64,
                                 const CUtensorMap& tk, const CUtensorMap& tv,
                                 const CUtensorMap& tdo, const CUtensorMap& tdo64,
                                 const CUtensorMap& tdq_sw, const BwdParams& p,
                                 cudaStream_t stream) {
  static std::atomic<uint64_t> configured{0};
  cudaError_t e = once_per_device(configured, [] {
    cudaError_t r = cudaFuncSetAttribute(bwd2::attn_bwd_pair_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(bwd2::kSmemBytes));
    if (r != cudaSuccess) return r;
    cudaFuncAttributes attr{};
    r = cudaFuncGetAttributes(&attr, bwd2::attn_bwd_pair_kernel);
    if (r != cudaSuccess) return r;
    return attr.numRegs == bwd2::kLaunchRegs ? cudaSuccess : cudaErrorInvalidConfiguration;
  });
  if (e != cudaSuccess) return e;
  const int n_kv_tiles = (p.rows_kv + bwd2::kBN - 1) / bwd2::kBN;
  const int n_pairs = (n_kv_tiles + 1) / 2;
  dim3 grid(2 * n_pairs * p.h_kv);
  BwdParams pp = p;
  if (bwd2::kHeadGroupForced > 0) {
    pp.head_group = bwd2::kHeadGroupForced;
  } else {
    constexpr double kL2Budget = 80.0 * (1 << 20);  // of the 126 MB L2
    pp.head_group = 2.0 * static_cast<double>(p.rows_q) * 1024.0 <= kL2Budget ? 2 : 1;
  }
  bwd2::attn_bwd_pair_kernel<<<grid, bwd2::kThreads, bwd2::kSmemBytes, stream>>>(
      tq, tq64, tk, tv, tdo, tdo64, tdq_sw, pp);
  return cudaGetLastError();
}

}  // namespace da

namespace da {
bool bwd_pair_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DA_BWD_KERNEL");
    return e != nullptr && std::strcmp(e, "pair") == 0;
  }();
  return on;
}
}  // namespace da
