// Chunk-attention forward for sm_100a on CTA pairs (tcgen05 cta_group::2).
//
// Reference semantics: block_attn_update (flashcore.hpp:135-197) followed by
// rescale (flashcore.hpp:202-224) with the caller's accumulator and, on the
// last step, finalize (flashcore.hpp:227-240) -- the same contract as the
// single-CTA kernel (attn_fwd_sm100.cu), whose softmax it keeps.
//
// Why pairs. The single-CTA forward is bound by the SM's shared-memory
// bandwidth: 192 KB per (query tile, kv tile) pair of 128 x 128 (S reads
// Q 32 + K 32, PV reads P 32 + V 32, K/V TMA writes 32, P stores 32) against
// 128 B/clk. In a CTA pair every GEMM is M = 256: each CTA supplies its own
// 128 query rows of A and HALF of B, so per tile pair an SM reads
// S: Q 32 + K/2 16, PV: P 32 + V/2 16, writes K/V halves 16 and P 32:
// 144 KB (-25%), and the kv stream an SM loads halves.
//
// Cluster of 2 CTAs = one head x a quad of query tiles 4u .. 4u+3. Slot t of
// CTA r holds query tile 4u + 2t + r; slot t's MMAs are M = 256 over both
// CTAs' tiles of that slot and walk the kv tiles of the later one (causal:
// the earlier CTA's last kv tile is fully masked, ~0.4% extra MMA work).
//   warp 0-3  softmax of slot 0 (thread = query row = TMEM lane)
//   warp 4-7  softmax of slot 1
//   warp 8    MMA issuer (lane 0 of the leader CTA, rank 0, issues for both)
//   warp 9    TMA producer (each CTA loads its own Q tiles and B halves; the
//             completions are counted on the leader's barriers)
// TMEM (512 cols, both CTAs): S_0 [0,128) S_1 [128,256) O_0 [256,384)
// O_1 [384,512). P_t goes to shared memory (K-major SW128) as in the
// single-CTA kernel, so S_t(j+1) is computed while softmax t still works on
// S_t(j); the two slots' exponential loops ping-pong on the MUFU.
// Hand-offs to the leader (s_free, p_full) are one arrive per warp of either
// CTA (count 8), default semantics (a cluster-scope release costs ~1 us,
// attn_bwd_pair_sm100.cu); MMA completions are multicast to both CTAs.
//
// Measured (round 2, profiles/ab_r2_fwd_pair.txt): correct (the forward
// parity suites pass with DA_FWD_KERNEL=pair) but not faster: 8.55 vs 8.19 ms
// in the sustained 32K step. With the softmax removed (cost probe
// DA_FWD2_EXPERIMENT_MMA_ONLY) both kernels take ~5.8 ms: the MMA stream is
// issue/latency bound at ~750 clk per 128^3, not shared-memory bound, so the
// saved bytes do not turn into speed, and the pair runs at the pace of the
// slower CTA's softmax. Opt-in only.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "kernels.h"
#include "sm100_ptx.cuh"

namespace da {
namespace fwd2 {

#ifndef DA_FWD2_HEAD_GROUP
#define DA_FWD2_HEAD_GROUP 2
#endif
constexpr int kHeadGroup = DA_FWD2_HEAD_GROUP;
constexpr int kBM = 128;
constexpr int kBN = 128;
constexpr int kHD = 128;
constexpr uint32_t kTile = 32768;    // 128 x 128 bf16
constexpr uint32_t kHalf = 16384;    // 128 x 64 bf16 (one SW128 box) = a B half
constexpr uint32_t kQuarter = 8192;  // 64 x 64 bf16
constexpr int kThreads = 320;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
#ifndef DA_FWD2_K_STAGES
#define DA_FWD2_K_STAGES 3
#endif
#ifndef DA_FWD2_V_STAGES
#define DA_FWD2_V_STAGES 3
#endif
#ifndef DA_FWD2_EX2_EMU_MOD
#define DA_FWD2_EX2_EMU_MOD 0
#endif
constexpr int kEx2EmuMod = DA_FWD2_EX2_EMU_MOD;
constexpr int kKStages = DA_FWD2_K_STAGES;
constexpr int kVStages = DA_FWD2_V_STAGES;

struct SmemLayout {
  // all tiles 1024B aligned (SW128)
  static constexpr uint32_t q0 = 0;                               // own query tile, slot 0
  static constexpr uint32_t q1 = q0 + kTile;                      // slot 1
  static constexpr uint32_t k = q1 + kTile;                       // K halves [64 kv][dh0 | dh1]
  static constexpr uint32_t v = k + kKStages * kHalf;             // V halves [128 kv][64 d]
  static constexpr uint32_t pbuf = v + kVStages * kHalf;          // P_0, P_1
  static constexpr uint32_t bars = pbuf + 2 * kTile;
  static constexpr uint32_t total = bars + 256;
};
constexpr size_t kSmemBytes = SmemLayout::total;
static_assert(kSmemBytes <= 232448, "dynamic shared memory per CTA");

struct Bars {
  // leader (rank 0): TMA completions of both CTAs, arrivals of both CTAs' warps
  uint64_t q_full;
  uint64_t k_full[kKStages];
  uint64_t v_full[kVStages];
  uint64_t p_full[2];  // P_t(j) in both CTAs' shared memory: 4 warps x 2 CTAs
  uint64_t s_free[2];  // softmax t of both CTAs holds S_t(j) in registers
  // local (pair MMA commits arrive in both CTAs)
  uint64_t k_empty[kKStages];
  uint64_t v_empty[kVStages];
  uint64_t s_full[2];
  uint64_t o_done[2];
  uint32_t tmem_base;
};
static_assert(sizeof(Bars) <= 256, "barrier block");

__device__ __forceinline__ int tiles_for(int mask, int qt, int n_kv_tiles) {
  // Diagonal: query tile qt sees kv tiles 0..qt. Full: every kv tile.
  return mask == DA_MASK_DIAGONAL ? min(qt + 1, n_kv_tiles) : n_kv_tiles;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    attn_fwd_pair_kernel(const __grid_constant__ CUtensorMap tmap_q,
                         const __grid_constant__ CUtensorMap tmap_k64,
                         const __grid_constant__ CUtensorMap tmap_v, const FwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (smem_align_pad(smem_raw) != 0) __trap();
  uint8_t* smem = smem_raw;
  Bars* bars = reinterpret_cast<Bars*>(smem + SmemLayout::bars);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  auto lead = [](uint64_t* b) { return mapa_shared(smem_u32(b), 0); };

  // ---- work: heads in groups of kHeadGroup, heaviest (latest) quads first
  const int n_q_tiles = (p.rows_q + kBM - 1) / kBM;
  const int n_kv_tiles = (p.rows_kv + kBN - 1) / kBN;
  const int n_quads = (n_q_tiles + 3) / 4;
  const int cl = static_cast<int>(blockIdx.x >> 1);
  const int g0 = (cl / (kHeadGroup * n_quads)) * kHeadGroup;
  const int g_heads = min(kHeadGroup, p.h_q - g0);
  const int r_in = cl - g0 * n_quads;
  const int head = g0 + r_in % g_heads;
  const int quad = n_quads - 1 - r_in / g_heads;
  const int kv_head = head / (p.h_q / p.h_kv);
  // slot t: pair-level kv tile count (the later of the two CTAs' tiles)
  auto slot_tiles = [&](int a) {
    return (a + 1 < n_q_tiles) ? tiles_for(p.mask, a + 1, n_kv_tiles)
           : (a < n_q_tiles)   ? tiles_for(p.mask, a, n_kv_tiles)
                               : 0;
  };
  const int n0 = slot_tiles(4 * quad), n1 = slot_tiles(4 * quad + 2);
  const int nmax = max(n0, n1);

  if (warp == 0) {
    if (lane == 0) {
      mbar_init(&bars->q_full, 1);
      for (int s = 0; s < kKStages; ++s) {
        mbar_init(&bars->k_full[s], 1);
        mbar_init(&bars->k_empty[s], 1);
      }
      for (int s = 0; s < kVStages; ++s) {
        mbar_init(&bars->v_full[s], 1);
        mbar_init(&bars->v_empty[s], 1);
      }
      for (int t = 0; t < 2; ++t) {
        mbar_init(&bars->s_full[t], 1);
        mbar_init(&bars->p_full[t], 8);
        mbar_init(&bars->o_done[t], 1);
        mbar_init(&bars->s_free[t], 8);
      }
      fence_barrier_init();
    }
  } else if (warp == 9) {
    if (lane == 0) {
      tma_prefetch_desc(&tmap_q);
      tma_prefetch_desc(&tmap_k64);
      tma_prefetch_desc(&tmap_v);
    }
  } else if (warp == 8) {
    tmem_alloc_pair<512>(&bars->tmem_base);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // peer barriers initialised before any remote arrive / TMA signal
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 9) {
    // ===================== TMA producer (own smem, leader's barriers) =====================
    if (lane == 0 && nmax > 0) {
      const int n_slots = (n0 > 0 ? 1 : 0) + (n1 > 0 ? 1 : 0);
      if (rank == 0) mbar_arrive_expect_tx(&bars->q_full, static_cast<uint32_t>(n_slots) * 2 * kTile);
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if ((t == 0 ? n0 : n1) == 0) continue;
        // a CTA whose own tile is past the end loads a real tile (rows not stored)
        const int qt = min(4 * quad + 2 * t + static_cast<int>(rank), n_q_tiles - 1);
        uint8_t* dst = smem + (t == 0 ? SmemLayout::q0 : SmemLayout::q1);
        tma_load_3d_pair(dst, &tmap_q, lead(&bars->q_full), 0, qt * kBM, head);
        tma_load_3d_pair(dst + kHalf, &tmap_q, lead(&bars->q_full), 64, qt * kBM, head);
      }
      for (int j = 0; j < nmax; ++j) {
        {  // K(j): kv rows [64 r, 64 r + 64) of the tile, both head-dim halves
          const int s = j % kKStages;
          uint8_t* ks = smem + SmemLayout::k + s * kHalf;
          mbar_wait(&bars->k_empty[s], ((j / kKStages) & 1) ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&bars->k_full[s], 2 * kHalf);
          int r0 = j * kBN + 64 * static_cast<int>(rank);
          if (r0 >= p.rows_kv) r0 = 0;  // fully past the end: masked columns, any real rows
          tma_load_3d_pair(ks, &tmap_k64, lead(&bars->k_full[s]), 0, r0, kv_head);
          tma_load_3d_pair(ks + kQuarter, &tmap_k64, lead(&bars->k_full[s]), 64, r0, kv_head);
        }
        {  // V(j): all 128 kv rows, head-dim columns [64 r, 64 r + 64)
          const int s = j % kVStages;
          uint8_t* vs = smem + SmemLayout::v + s * kHalf;
          mbar_wait(&bars->v_empty[s], ((j / kVStages) & 1) ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&bars->v_full[s], 2 * kHalf);
          tma_load_3d_pair(vs, &tmap_v, lead(&bars->v_full[s]), 64 * static_cast<int>(rank),
                           j * kBN, kv_head);
        }
      }
    }
  } else if (warp == 8) {
    // ===================== MMA issuer (leader CTA) =====================
    if (rank == 0 && lane == 0 && nmax > 0) {
      constexpr uint32_t idesc_qk = make_idesc_bf16(256, 128, false, false);
      constexpr uint32_t idesc_pv = make_idesc_bf16(256, 128, false, true);
      const uint32_t q_addr = smem_u32(smem + SmemLayout::q0);  // q1 = q0 + kTile
      const uint32_t k_addr = smem_u32(smem + SmemLayout::k);
      const uint32_t v_addr = smem_u32(smem + SmemLayout::v);
      const uint32_t p_base = smem_u32(smem + SmemLayout::pbuf);

      // S_t = Q_t K^T: A = own [128 q][128 d], B = [64 kv][128 d] per CTA (K-major)
      auto issue_s = [&](int t, int stage) {
        const uint32_t kb = k_addr + stage * kHalf;
#pragma unroll
        for (int kk = 0; kk < kHD / 16; ++kk) {
          const uint64_t a =
              make_sdesc_sw128(q_addr + t * kTile + (kk >> 2) * kHalf + (kk & 3) * 32, 16, 1024);
          const uint64_t b = make_sdesc_sw128(kb + (kk >> 2) * kQuarter + (kk & 3) * 32, 16, 1024);
          mma2_ss(tmem + t * 128, a, b, idesc_qk, kk > 0 ? 1u : 0u);
        }
      };
      // O_t += P_t V: A = own P [128 q][128 kv] (K-major), B = [128 kv][64 d] per CTA (MN-major)
      auto issue_pv = [&](int t, int stage, bool acc) {
        const uint32_t vb = v_addr + stage * kHalf;
        const uint32_t pa = p_base + t * kTile;
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk) {
          const uint64_t a = make_sdesc_sw128(pa + (kk >> 2) * kHalf + (kk & 3) * 32, 16, 1024);
          const uint64_t b = make_sdesc_sw128(vb + kk * 2048, kHalf, 1024);
          mma2_ss(tmem + 256 + t * 128, a, b, idesc_pv, (acc || kk > 0) ? 1u : 0u);
        }
      };

      mbar_wait(&bars->q_full, 0);
      mbar_wait(&bars->k_full[0], 0);
      tc_fence_after();
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if ((t == 0 ? n0 : n1) > 0) {
          issue_s(t, 0);
          mma2_commit_both(&bars->s_full[t]);
        }
      }
      mma2_commit_both(&bars->k_empty[0]);
      for (int j = 0; j < nmax; ++j) {
        if (j + 1 < nmax) {
          // S_t(j+1) once softmax t of both CTAs holds S_t(j) in registers
          const int s1 = (j + 1) % kKStages;
          mbar_wait(&bars->k_full[s1], ((j + 1) / kKStages) & 1);
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            if (j + 1 < (t == 0 ? n0 : n1)) {
              mbar_wait(&bars->s_free[t], j & 1);
              tc_fence_after();
              issue_s(t, s1);
              mma2_commit_both(&bars->s_full[t]);
            }
          }
          mma2_commit_both(&bars->k_empty[s1]);
        }
        // PV_t(j) once P_t(j) is in both CTAs' shared buffers
        const int sv = j % kVStages;
        mbar_wait(&bars->v_full[sv], (j / kVStages) & 1);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          if (j < (t == 0 ? n0 : n1)) {
            mbar_wait(&bars->p_full[t], j & 1);
            tc_fence_after();
            issue_pv(t, sv, j > 0);
            mma2_commit_both(&bars->o_done[t]);
          }
        }
        mma2_commit_both(&bars->v_empty[sv]);
      }
    }
  } else {
    // ===================== softmax / epilogue (warps 0-7) =====================
    const int t = warp / 4;
    const int quarter = warp % 4;
    const int row_in_tile = quarter * 32 + lane;
    const int qt = 4 * quad + 2 * t + static_cast<int>(rank);
    const int n_tiles = t == 0 ? n0 : n1;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const uint32_t s_tmem = lane_base + t * 128;
    const uint32_t o_tmem = lane_base + 256 + t * 128;
    const uint32_t s_free_bar = lead(&bars->s_free[t]);
    const uint32_t p_full_bar = lead(&bars->p_full[t]);
    const float sl2 = p.scale_log2;
    const float neg_inf = -INFINITY;

    float m_run = neg_inf;  // running max, log2 units of scale*q.k
    float l_run = 0.f;

    for (int j = 0; j < n_tiles; ++j) {
      mbar_wait(&bars->s_full[t], j & 1);
      tc_fence_after();
#ifdef DA_FWD2_EXPERIMENT_MMA_ONLY  // (cost probe only: no softmax, garbage output)
      if (j > 0) mbar_wait(&bars->o_done[t], (j - 1) & 1);
      tc_fence_before();
      __syncwarp();
      if (lane == 0 && j + 1 < n_tiles) mbar_arrive_cluster(s_free_bar);
      if (lane == 0) mbar_arrive_cluster(p_full_bar);
      l_run = 1.f;
      continue;
#endif
      uint32_t sr[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(s_tmem + c * 32, sr[c]);
      tmem_ld_wait();
      if (j + 1 < n_tiles) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(s_free_bar);  // S_t(j+1) may overwrite the S columns
      }

      // masking: causal inside the diagonal tile (kv tiles past it: this
      // CTA's tile is the earlier one of the slot, every column masked),
      // ragged kv tail
      const bool diag = (p.mask == DA_MASK_DIAGONAL) && (j >= qt);
      const int kv_valid = p.rows_kv - j * kBN;  // columns >= kv_valid are padding
      const bool masked_tile = diag || kv_valid < kBN;
      if (masked_tile) {
        const int lim = !diag ? kv_valid : (j > qt ? 0 : min(row_in_tile + 1, kv_valid));
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c * 32 + i >= lim) sr[c][i] = __float_as_uint(neg_inf);
      }
      // row max as a tree of 8 independent chains
      float mx;
      {
        float mc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) mc[u] = __uint_as_float(sr[u >> 1][(u & 1) * 16]);
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int u = c * 2 + i / 16;
            if ((i & 15) != 0) mc[u] = fmaxf(mc[u], __uint_as_float(sr[c][i]));
          }
        mx = fmaxf(fmaxf(fmaxf(mc[0], mc[1]), fmaxf(mc[2], mc[3])),
                   fmaxf(fmaxf(mc[4], mc[5]), fmaxf(mc[6], mc[7])));
      }
      mx *= sl2;

      float alpha = 1.f;
      const float m_new = fmaxf(m_run, mx);
      const bool need = m_new > m_run + kRescaleThreshold;
      if (need) {
        alpha = (m_run == neg_inf) ? 0.f : ex2_approx(m_run - m_new);
        m_run = m_new;
      }
      const float neg_m = (m_run == neg_inf) ? 0.f : -m_run;

      // P = 2^(s*scale*log2e - m): packed FFMA2 arguments, 8 packed FADD2 row-sum chains
      float2 rs2[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) rs2[u] = make_float2(0.f, 0.f);
      uint32_t pk[2][32];
      const float2 sl2x2 = make_float2(sl2, sl2);
      const float2 nm2 = make_float2(neg_m, neg_m);
      // MUFU ping-pong of the two slots (named barriers 1/2, 256 threads)
      if (t == 0 ? (j > 0 && j <= n1) : (j < n0)) named_bar_sync(1 + t, 256);
      // on unmasked tiles every kEx2EmuMod-th column pair is exponentiated on
      // the FMA pipe (offloads the MUFU; masked entries need the exact zeros
      // of the MUFU path)
      auto exp_tile = [&](auto emulate) {
        constexpr bool kEmu = decltype(emulate)::value;
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float2 x = ffma2(
                make_float2(__uint_as_float(sr[c][i]), __uint_as_float(sr[c][i + 1])), sl2x2, nm2);
            const int pr = c * 16 + i / 2;
            float2 pv;
            if (kEmu && (pr % kEx2EmuMod) == kEx2EmuMod - 1) {
              pv = ex2_emu2(x);
            } else {
              pv = make_float2(ex2_approx(x.x), ex2_approx(x.y));
            }
            rs2[pr & 7] = fadd2(rs2[pr & 7], pv);
            pk[c >> 1][(c & 1) * 16 + i / 2] = pack_bf16x2_int(pv.x, pv.y);
          }
      };
      if (kEx2EmuMod == 0 || masked_tile) {
        exp_tile(std::false_type{});
      } else {
        exp_tile(std::integral_constant<bool, (kEx2EmuMod > 0)>{});
      }
      if (t == 0 ? (j < n1) : (j + 1 < n0)) named_bar_arrive(2 - t, 256);
#pragma unroll
      for (int u = 0; u < 4; ++u) rs2[u] = fadd2(rs2[u], rs2[u + 4]);
      rs2[0] = fadd2(rs2[0], rs2[2]);
      rs2[1] = fadd2(rs2[1], rs2[3]);
      rs2[0] = fadd2(rs2[0], rs2[1]);
      const float rs = rs2[0].x + rs2[0].y;
      l_run = l_run * alpha + rs;

      // PV(j-1) complete: O may be corrected and P_t(j-1)'s buffer is free
      if (j > 0) mbar_wait(&bars->o_done[t], (j - 1) & 1);
      if (j > 0 && __any_sync(0xffffffffu, need)) {
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t orr[32];
          tmem_ld_32x32b_x32(o_tmem + c * 32, orr);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) orr[i] = __float_as_uint(__uint_as_float(orr[i]) * alpha);
          tmem_st_32x32b_x32(o_tmem + c * 32, orr);
        }
      }
      {
        // K-major SW128 tile [128 q][128 kv] bf16 as two 64-column boxes
        uint8_t* prow = smem + SmemLayout::pbuf + t * kTile + row_in_tile * 128;
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int ch = 0; ch < 8; ++ch)
            *reinterpret_cast<uint4*>(prow + b * kHalf + ((ch ^ (row_in_tile & 7)) * 16)) =
                make_uint4(pk[b][4 * ch], pk[b][4 * ch + 1], pk[b][4 * ch + 2], pk[b][4 * ch + 3]);
        fence_proxy_async_smem();
        tmem_st_wait();  // the O correction, if any
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(p_full_bar);
    }

    // ===================== epilogue =====================
    if (n_tiles > 0) {
      mbar_wait(&bars->o_done[t], (n_tiles - 1) & 1);
      tc_fence_after();
      const int row = qt * kBM + row_in_tile;
      const bool valid = row < p.rows_q;
      const size_t srow = static_cast<size_t>(head) * p.rows_q + (valid ? row : 0);
      constexpr float kLn2 = 0.69314718055994530942f;
      const float m_k = m_run * kLn2;  // natural-log units
      float wa = 0.f, wb = 1.f, m_out = m_k, l_out = l_run;
      if (valid && p.o_in != nullptr) {
        const float m_i = p.m_in[srow];
        const float l_i = p.l_in[srow];
        m_out = fmaxf(m_i, m_k);
        wa = (m_i == neg_inf) ? 0.f : __expf(m_i - m_out);
        wb = (m_k == neg_inf) ? 0.f : __expf(m_k - m_out);
        l_out = wa * l_i + wb * l_run;
      }
      float inv_l = 0.f;
      if (p.finalize && valid) {
        if (!(l_out > 0.f)) {
          if (p.degenerate_flag) atomicExch(p.degenerate_flag, 1);
        } else {
          inv_l = 1.f / l_out;
        }
      }
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t orr[32];
        tmem_ld_32x32b_x32(o_tmem + c * 32, orr);
        tmem_ld_wait();
        if (!valid) continue;
        float o[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] = __uint_as_float(orr[i]) * wb;
        if (p.o_in != nullptr) {
          const float4* src = reinterpret_cast<const float4*>(p.o_in + srow * kHD + c * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 x = src[i];
            o[4 * i + 0] = fmaf(wa, x.x, o[4 * i + 0]);
            o[4 * i + 1] = fmaf(wa, x.y, o[4 * i + 1]);
            o[4 * i + 2] = fmaf(wa, x.z, o[4 * i + 2]);
            o[4 * i + 3] = fmaf(wa, x.w, o[4 * i + 3]);
          }
        }
        if (p.finalize) {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.o_out) +
                                                srow * kHD + c * 32);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            uint4 w;
            w.x = pack_bf16x2(o[8 * i + 0] * inv_l, o[8 * i + 1] * inv_l);
            w.y = pack_bf16x2(o[8 * i + 2] * inv_l, o[8 * i + 3] * inv_l);
            w.z = pack_bf16x2(o[8 * i + 4] * inv_l, o[8 * i + 5] * inv_l);
            w.w = pack_bf16x2(o[8 * i + 6] * inv_l, o[8 * i + 7] * inv_l);
            dst[i] = w;
          }
        } else {
          float4* dst = reinterpret_cast<float4*>(p.o_acc + srow * kHD + c * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            dst[i] = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
        }
      }
      if (valid) {
        if (p.finalize) {
          p.lse_out[srow] = (l_out > 0.f) ? m_out + __logf(l_out) : neg_inf;
        } else {
          p.m_acc[srow] = m_out;
          p.l_acc[srow] = l_out;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the leader's MMAs into this CTA's TMEM and all remote arrives are done
  if (warp == 8) tmem_dealloc_pair<512>(tmem);
}

}  // namespace fwd2

cudaError_t launch_attn_fwd_pair(const CUtensorMap& tq, const CUtensorMap& tk64,
                                 const CUtensorMap& tv, const FwdParams& p, cudaStream_t stream) {
  static std::atomic<uint64_t> configured{0};
  cudaError_t e = once_per_device(configured, [] {
    return cudaFuncSetAttribute(fwd2::attn_fwd_pair_kernel,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(fwd2::kSmemBytes));
  });
  if (e != cudaSuccess) return e;
  const int n_q_tiles = (p.rows_q + fwd2::kBM - 1) / fwd2::kBM;
  const int n_quads = (n_q_tiles + 3) / 4;
  dim3 grid(2 * n_quads * p.h_q);
  fwd2::attn_fwd_pair_kernel<<<grid, fwd2::kThreads, fwd2::kSmemBytes, stream>>>(tq, tk64, tv, p);
  return cudaGetLastError();
}

bool fwd_pair_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DA_FWD_KERNEL");
    return e != nullptr && std::strcmp(e, "pair") == 0;
  }();
  return on;
}

}  // namespace da
