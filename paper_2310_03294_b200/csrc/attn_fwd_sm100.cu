// Chunk-attention forward for sm_100a: one (query chunk, kv chunk) online-
// softmax update with the incoming-accumulator merge and finalize fused into
// the epilogue.
//
// Reference semantics: block_attn_update (flashcore.hpp:135-197) followed by
// rescale (flashcore.hpp:202-224) with the caller's accumulator and, on the
// last step, finalize (flashcore.hpp:227-240).
//
// Design (per CTA = one head x two 128-row query tiles "pair"):
//   warp 0-3  softmax for query tile 0  (thread = query row = TMEM lane)
//   warp 4-7  softmax for query tile 1
//   warp 8    MMA issuer (one thread): S_t = Q_t K_j^T (SS), O_t += P_t V_j (SS)
//   warp 9    TMA producer: Q once, K_j single-stage, V_j through a 2-stage ring
// TMEM (512 cols): S_0 [0,128) S_1 [128,256) O_0 [256,384) O_1 [384,512);
// P_t (bf16) is written to its own smem tile, so S_t(j+1) is computed while
// softmax t still works on S_t(j) (it holds S_t(j) in registers). The two
// query tiles' exponential loops ping-pong on the MUFU.
// O is rescaled lazily (only when the running max grows by > 2^8).
#include <cuda.h>
#include <cuda_bf16.h>

#include <type_traits>

#include "kernels.h"
#include "sm100_ptx.cuh"

namespace da {
namespace fwd {

#ifdef DA_TRACE
#define FWD_TRACE(cond, j, slot)                                                \
  do {                                                                          \
    if ((cond) && p.trace != nullptr && blockIdx.x == 0 && (j) < 64)            \
      p.trace[(j) * 16 + (slot)] = clock64();                                   \
  } while (0)
// per-CTA record after the 64x16 stamps (same layout as the backward's):
// globaltimer start/end, clock64 start/end, smid, kv tiles
#define FWD_CTA_TRACE(slot, val)                                                \
  do {                                                                          \
    if (p.trace != nullptr)                                                     \
      p.trace[1024 + static_cast<size_t>(blockIdx.x) * 8 + (slot)] = (val);     \
  } while (0)
__device__ __forceinline__ unsigned long long fwd_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long fwd_smid() {
  uint32_t s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}
#else
#define FWD_TRACE(cond, j, slot) \
  do {                           \
  } while (0)
#define FWD_CTA_TRACE(slot, val) \
  do {                           \
  } while (0)
#endif

#ifndef DA_FWD_HEAD_GROUP
#define DA_FWD_HEAD_GROUP 2
#endif
constexpr int kHeadGroup = DA_FWD_HEAD_GROUP;
constexpr int kBM = 128;
constexpr int kBN = 128;
constexpr int kHD = 128;
constexpr int kStages = 2;
constexpr uint32_t kTileBytes = kBM * kHD * 2;  // 32 KB, one 128x128 bf16 tile
constexpr uint32_t kHalfTile = kTileBytes / 2;  // one 64-column SW128 box
constexpr int kThreads = 320;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
#ifndef DA_FWD_EX2_EMU_MOD
#define DA_FWD_EX2_EMU_MOD 0
#endif
// every kEx2EmuMod-th pair of columns is exponentiated on the FMA pipe (0: none)
constexpr int kEx2EmuMod = DA_FWD_EX2_EMU_MOD;
#ifndef DA_FWD_NO_PINGPONG
constexpr bool kMufuPingPong = true;
#else
constexpr bool kMufuPingPong = false;
#endif
// P through shared memory (one 32 KB buffer per tile) and PV as an SS MMA:
// S(j+1) no longer has to wait for PV(j) to consume P(j) in the S columns, so
// a tile's next softmax follows its current one directly. The smem for the
// two P tiles comes from a single-stage V ring.
#ifndef DA_FWD_P_SMEM
#define DA_FWD_P_SMEM 1
#endif
constexpr bool kPSmem = DA_FWD_P_SMEM != 0;
// With P in smem one K or V stage has to go: K single-stage (refilled once
// both tiles' S(j) are done) and V double-stage measured marginally ahead of
// the opposite split (7.85 vs 7.88 ms in the sustained step).
#ifndef DA_FWD_K_STAGES
#define DA_FWD_K_STAGES 1
#endif
constexpr int kKStages = kPSmem ? DA_FWD_K_STAGES : 2;
constexpr int kVStages = kPSmem ? 3 - kKStages : 2;

struct SmemLayout {
  // all tiles 1024B aligned (SW128)
  static constexpr uint32_t q0 = 0;
  static constexpr uint32_t q1 = q0 + kTileBytes;
  static constexpr uint32_t k = q1 + kTileBytes;                 // kStages tiles
  static constexpr uint32_t v = k + kKStages * kTileBytes;       // kVStages tiles
  static constexpr uint32_t pbuf = v + kVStages * kTileBytes;    // P_0, P_1 (kPSmem)
  static constexpr uint32_t bars = pbuf + (kPSmem ? 2 * kTileBytes : 0);  // barriers
  static constexpr uint32_t total = bars + 256;
};
constexpr size_t kSmemBytes = SmemLayout::total + (kPSmem ? 0 : 1024);  // + alignment slack
static_assert(kSmemBytes <= 232448, "dynamic shared memory per CTA");

struct Bars {
  uint64_t q_full;
  uint64_t k_full[kStages];
  uint64_t k_empty[kStages];
  uint64_t v_full[kStages];
  uint64_t v_empty[kStages];
  uint64_t s_full[2];
  uint64_t p_full[2];
  uint64_t o_done[2];
  uint64_t s_free[2];     // kPSmem: softmax t holds S_t(j) in registers
  uint32_t tmem_base;
};
static_assert(sizeof(Bars) <= 256, "barrier block");

__device__ __forceinline__ int tiles_for(int mask, int qt, int n_kv_tiles) {
  // Diagonal: query tile qt sees kv tiles 0..qt. Full: every kv tile.
  return mask == DA_MASK_DIAGONAL ? min(qt + 1, n_kv_tiles) : n_kv_tiles;
}

__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmap_q,
                    const __grid_constant__ CUtensorMap tmap_k,
                    const __grid_constant__ CUtensorMap tmap_v, const FwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment (SW128) by offsetting the __shared__ symbol itself, so
  // the compiler keeps the shared address space (STS/LDS, not generic ST/LD)
  // (kPSmem: no slack left, so the 1024-aligned window is checked instead)
  if (kPSmem && smem_align_pad(smem_raw) != 0) __trap();
  uint8_t* smem = smem_raw + smem_align_pad(smem_raw);
  Bars* bars = reinterpret_cast<Bars*>(smem + SmemLayout::bars);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;

  // ---- work assignment: heavy (late) query pairs first under causal masks
  const int n_q_tiles = (p.rows_q + kBM - 1) / kBM;
  const int n_kv_tiles = (p.rows_kv + kBN - 1) / kBN;
  const int n_pairs = (n_q_tiles + 1) / 2;
  // heads in groups of kHeadGroup: the co-resident CTAs share a group's K/V in
  // L2; within a group the heaviest (latest) query pairs launch first, the
  // group's heads interleaved, so the last wave is short light pairs rather
  // than one head's long ones (head-major left a ~2% tail)
  const int b = static_cast<int>(blockIdx.x);
  const int g0 = (b / (kHeadGroup * n_pairs)) * kHeadGroup;
  const int g_heads = min(kHeadGroup, p.h_q - g0);
  const int r_in = b - g0 * n_pairs;
  const int head = g0 + r_in % g_heads;
  const int pair = n_pairs - 1 - r_in / g_heads;
  const int kv_head = head / (p.h_q / p.h_kv);
  const int qt0 = 2 * pair;
  const bool has_t1 = (qt0 + 1) < n_q_tiles;
  const int n0 = tiles_for(p.mask, qt0, n_kv_tiles);
  const int n1 = has_t1 ? tiles_for(p.mask, qt0 + 1, n_kv_tiles) : 0;
  const int nmax = max(n0, n1);
  if (threadIdx.x == 0) {
    FWD_CTA_TRACE(0, fwd_gtimer());
    FWD_CTA_TRACE(2, clock64());
  }

  if (warp == 0) {
    if (lane == 0) {
      mbar_init(&bars->q_full, 1);
      for (int s = 0; s < kStages; ++s) {
        mbar_init(&bars->k_full[s], 1);
        mbar_init(&bars->k_empty[s], 1);
        mbar_init(&bars->v_full[s], 1);
        mbar_init(&bars->v_empty[s], 1);
      }
      for (int t = 0; t < 2; ++t) {
        mbar_init(&bars->s_full[t], 1);
        mbar_init(&bars->p_full[t], 128);
        mbar_init(&bars->o_done[t], 1);
        mbar_init(&bars->s_free[t], 128);
      }
      fence_barrier_init();
    }
  } else if (warp == 9) {
    if (lane == 0) {
      tma_prefetch_desc(&tmap_q);
      tma_prefetch_desc(&tmap_k);
      tma_prefetch_desc(&tmap_v);
    }
  } else if (warp == 8) {
    tmem_alloc<512>(&bars->tmem_base);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 9) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      const int row0 = qt0 * kBM;
      mbar_arrive_expect_tx(&bars->q_full, (has_t1 ? 2u : 1u) * kTileBytes);
      tma_load_3d(smem + SmemLayout::q0, &tmap_q, &bars->q_full, 0, row0, head);
      tma_load_3d(smem + SmemLayout::q0 + kHalfTile, &tmap_q, &bars->q_full, 64, row0, head);
      if (has_t1) {
        tma_load_3d(smem + SmemLayout::q1, &tmap_q, &bars->q_full, 0, row0 + kBM, head);
        tma_load_3d(smem + SmemLayout::q1 + kHalfTile, &tmap_q, &bars->q_full, 64, row0 + kBM,
                    head);
      }
      auto load_k = [&](int j) {
        const int s = j % kKStages;
        uint8_t* ks = smem + SmemLayout::k + s * kTileBytes;
        mbar_wait(&bars->k_empty[s], ((j / kKStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&bars->k_full[s], kTileBytes);
        tma_load_3d(ks, &tmap_k, &bars->k_full[s], 0, j * kBN, kv_head);
        tma_load_3d(ks + kHalfTile, &tmap_k, &bars->k_full[s], 64, j * kBN, kv_head);
      };
      auto load_v = [&](int j) {
        const int s = j % kVStages;
        uint8_t* vs = smem + SmemLayout::v + s * kTileBytes;
        mbar_wait(&bars->v_empty[s], ((j / kVStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&bars->v_full[s], kTileBytes);
        tma_load_3d(vs, &tmap_v, &bars->v_full[s], 0, j * kBN, kv_head);
        tma_load_3d(vs + kHalfTile, &tmap_v, &bars->v_full[s], 64, j * kBN, kv_head);
      };
      for (int j = 0; j < nmax; ++j) {
        if (kPSmem && kKStages == 1) {
          // V(j) first (its stage frees early), then K(j+1) once S(j) is done
          if (j == 0) load_k(0);
          load_v(j);
          if (j + 1 < nmax) load_k(j + 1);
        } else if (kPSmem) {
          // K runs a tile ahead of V (the single V stage frees only after both PVs)
          if (j == 0) load_k(0);
          if (j + 1 < nmax) load_k(j + 1);
          load_v(j);
        } else {
          load_k(j);
          load_v(j);
        }
      }
    }
  } else if (warp == 8) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      constexpr uint32_t idesc_qk = make_idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_pv = make_idesc_bf16(128, 128, false, true);
      const uint32_t q_addr[2] = {smem_u32(smem + SmemLayout::q0), smem_u32(smem + SmemLayout::q1)};
      const uint32_t k_addr = smem_u32(smem + SmemLayout::k);
      const uint32_t v_addr = smem_u32(smem + SmemLayout::v);
      const int n_t[2] = {n0, n1};

      auto issue_s = [&](int t, int stage) {
        const uint32_t kb = k_addr + stage * kTileBytes;
        const uint32_t d_tmem = tmem + t * 128;
#pragma unroll
        for (int kk = 0; kk < kHD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kHalfTile + (kk & 3) * 32;
          const uint64_t a = make_sdesc_sw128(q_addr[t] + off, 16, 1024);
          const uint64_t b = make_sdesc_sw128(kb + off, 16, 1024);
          mma_ss(d_tmem, a, b, idesc_qk, kk > 0 ? 1u : 0u);
        }
      };
      auto issue_pv = [&](int t, int stage, bool acc) {
        const uint32_t vb = v_addr + stage * kTileBytes;
        const uint32_t d_tmem = tmem + 256 + t * 128;
        const uint32_t p_tmem = tmem + t * 128 + 64;
        const uint32_t p_addr = smem_u32(smem + SmemLayout::pbuf) + t * kTileBytes;
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk) {
          const uint64_t b = make_sdesc_sw128(vb + kk * 2048, kHalfTile, 1024);
          if (kPSmem) {
            const uint32_t off = (kk >> 2) * kHalfTile + (kk & 3) * 32;
            mma_ss(d_tmem, make_sdesc_sw128(p_addr + off, 16, 1024), b, idesc_pv,
                   (acc || kk > 0) ? 1u : 0u);
          } else {
            mma_ts(d_tmem, p_tmem + kk * 8, b, idesc_pv, (acc || kk > 0) ? 1u : 0u);
          }
        }
      };

      mbar_wait(&bars->q_full, 0);
      if (nmax > 0) {
        mbar_wait(&bars->k_full[0], 0);
        tc_fence_after();
        for (int t = 0; t < 2; ++t) {
          if (n_t[t] > 0) {
            issue_s(t, 0);
            mma_commit(&bars->s_full[t]);
          }
        }
        mma_commit(&bars->k_empty[0]);
      }
      for (int j = 0; kPSmem && j < nmax; ++j) {
        const bool has_next = j + 1 < nmax;
        const int s1 = (j + 1) % kKStages;
        const uint32_t ph1 = ((j + 1) / kKStages) & 1;
        FWD_TRACE(true, j, 0);
        // S_t(j+1) as soon as softmax t holds S_t(j) in registers
        if (has_next) {
          mbar_wait(&bars->k_full[s1], ph1);
          for (int t = 0; t < 2; ++t) {
            if (j + 1 < n_t[t]) {
              mbar_wait(&bars->s_free[t], j & 1);
              tc_fence_after();
              issue_s(t, s1);
              mma_commit(&bars->s_full[t]);
            }
          }
          mma_commit(&bars->k_empty[s1]);
        }
        // PV_t(j) once P_t(j) is in its shared buffer
        const int sv = j % kVStages;
        mbar_wait(&bars->v_full[sv], (j / kVStages) & 1);
        for (int t = 0; t < 2; ++t) {
          if (j < n_t[t]) {
            mbar_wait(&bars->p_full[t], j & 1);
            FWD_TRACE(true, j, 1 + t);
            tc_fence_after();
            issue_pv(t, sv, j > 0);
            mma_commit(&bars->o_done[t]);
          }
        }
        mma_commit(&bars->v_empty[sv]);
      }
      for (int j = 0; !kPSmem && j < nmax; ++j) {
        const int s = j % kStages;
        const uint32_t ph = (j / kStages) & 1;
        const bool has_next = j + 1 < nmax;
        const int s1 = (j + 1) % kStages;
        const uint32_t ph1 = ((j + 1) / kStages) & 1;
        FWD_TRACE(true, j, 0);
        mbar_wait(&bars->v_full[s], ph);

        if (has_next) mbar_wait(&bars->k_full[s1], ph1);

        tc_fence_after();
        for (int t = 0; t < 2; ++t) {
          if (j < n_t[t]) {
            mbar_wait(&bars->p_full[t], j & 1);
            FWD_TRACE(true, j, 1 + t);
            tc_fence_after();
            issue_pv(t, s, j > 0);
            mma_commit(&bars->o_done[t]);
            if (j + 1 < n_t[t]) {
              issue_s(t, s1);
              mma_commit(&bars->s_full[t]);
            }
          }
        }
        mma_commit(&bars->v_empty[s]);
        if (has_next) mma_commit(&bars->k_empty[s1]);
      }
    }
  } else {
    // ===================== softmax / epilogue (warps 0-7) =====================
    const int t = warp / 4;
    const int quarter = warp % 4;
    const int row_in_tile = quarter * 32 + lane;
    const int qt = qt0 + t;
    const int n_tiles = t == 0 ? n0 : n1;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const uint32_t s_tmem = lane_base + t * 128;
    const uint32_t p_tmem = s_tmem + 64;
    const uint32_t o_tmem = lane_base + 256 + t * 128;
    const float sl2 = p.scale_log2;
    const float neg_inf = -INFINITY;

    float m_run = neg_inf;  // running max, log2 units of scale*q.k
    float l_run = 0.f;

    for (int j = 0; j < n_tiles; ++j) {
      mbar_wait(&bars->s_full[t], j & 1);
      FWD_TRACE(quarter == 0 && lane == 0, j, 3 + 6 * t);
      tc_fence_after();
#ifdef DA_FWD_EXPERIMENT_MMA_ONLY  // (cost probe only: no softmax, garbage output)
      if (j > 0) mbar_wait(&bars->o_done[t], (j - 1) & 1);
      tc_fence_before();
      if (kPSmem && j + 1 < n_tiles) mbar_arrive(&bars->s_free[t]);
      mbar_arrive(&bars->p_full[t]);
      l_run = 1.f;
      continue;
#endif
      uint32_t sr[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(s_tmem + c * 32, sr[c]);
      tmem_ld_wait();
      if (kPSmem && j + 1 < n_tiles) {
        tc_fence_before();
        mbar_arrive(&bars->s_free[t]);  // S_t(j+1) may overwrite the S columns
      }
      FWD_TRACE(quarter == 0 && lane == 0, j, 4 + 6 * t);

      if (p.debug_s != nullptr && j == 0 && t == 0 && blockIdx.x == 0) {
        // raw (unscaled, unmasked) scores of the first tile, for layout tests
        float* dst = p.debug_s + static_cast<size_t>(row_in_tile) * kBN;
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i) dst[c * 32 + i] = __uint_as_float(sr[c][i]);
      }

      // masking: causal inside the diagonal tile, ragged kv tail
      const bool diag = (p.mask == DA_MASK_DIAGONAL) && (j == qt);
      const int kv_valid = p.rows_kv - j * kBN;  // columns >= kv_valid are padding
      const bool masked_tile = diag || kv_valid < kBN;
      if (masked_tile) {
        const int lim = diag ? min(row_in_tile + 1, kv_valid) : kv_valid;
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c * 32 + i >= lim) sr[c][i] = __float_as_uint(neg_inf);
      }
      // row max as a tree of 8 independent chains (latency, not a 128-long chain)
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
      FWD_TRACE(quarter == 0 && lane == 0, j, 5 + 6 * t);

      float alpha = 1.f;
      const float m_new = fmaxf(m_run, mx);
      const bool need = m_new > m_run + kRescaleThreshold;
      if (need) {
        alpha = (m_run == neg_inf) ? 0.f : ex2_approx(m_run - m_new);
        m_run = m_new;
      }
      const float neg_m = (m_run == neg_inf) ? 0.f : -m_run;

      // P = 2^(s*scale*log2e - m): packed FFMA2 for the argument, packed FADD2
      // row sums (4 independent accumulators); on unmasked tiles every
      // kEx2EmuMod-th column pair is exponentiated on the FMA pipe
      // 8 independent packed accumulators: no FADD2 dependency stalls
      float2 rs2[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) rs2[u] = make_float2(0.f, 0.f);
      uint32_t pk[2][32];
      const float2 sl2x2 = make_float2(sl2, sl2);
      const float2 nm2 = make_float2(neg_m, neg_m);
      auto exp_tile = [&](auto emulate) {
        constexpr bool kEmu = decltype(emulate)::value;
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float2 x = ffma2(
                make_float2(__uint_as_float(sr[c][i]), __uint_as_float(sr[c][i + 1])), sl2x2, nm2);
            const int pair = c * 16 + i / 2;
            float2 pv;
            if (kEmu && (pair % kEx2EmuMod) == kEx2EmuMod - 1) {
              pv = ex2_emu2(x);
            } else {
              pv = make_float2(ex2_approx(x.x), ex2_approx(x.y));
            }
            rs2[pair & 7] = fadd2(rs2[pair & 7], pv);
            // integer-pipe rounding (P in [0, 1]): keeps F2FP off the
            // exponential loop (+1% forward, sustained bench A/B)
            pk[c >> 1][(c & 1) * 16 + i / 2] = pack_bf16x2_int(pv.x, pv.y);
          }
      };
      // MUFU ping-pong: the two tiles' exponential loops take turns (named
      // barriers 1/2, 256 threads = both softmax warpgroups), so each runs at
      // the full ex2 rate while the tensor core works on the other tile.
      // Turn order per j: tile 0, then tile 1 (counts match for n0 <= n1).
      if (kMufuPingPong) {
        if (t == 0 ? (j > 0 && j <= n1) : (j < n0)) named_bar_sync(1 + t, 256);
      }
      FWD_TRACE(quarter == 0 && lane == 0, j, 6 + 6 * t);
      // masked entries must give exact zeros: the MUFU path only
      if (kEx2EmuMod == 0 || masked_tile) {
        exp_tile(std::false_type{});
      } else {
        exp_tile(std::integral_constant<bool, (kEx2EmuMod > 0)>{});
      }
      if (kMufuPingPong) {
        if (t == 0 ? (j < n1) : (j + 1 < n0)) named_bar_arrive(2 - t, 256);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) rs2[u] = fadd2(rs2[u], rs2[u + 4]);
      rs2[0] = fadd2(rs2[0], rs2[2]);
      rs2[1] = fadd2(rs2[1], rs2[3]);
      rs2[0] = fadd2(rs2[0], rs2[1]);
      const float rs = rs2[0].x + rs2[0].y;
      FWD_TRACE(quarter == 0 && lane == 0, j, 7 + 6 * t);
      l_run = l_run * alpha + rs;

      // PV(j-1) complete: O may be corrected and (kPSmem) P_t(j-1)'s buffer is
      // free. Without kPSmem it never blocks (S(j) was committed after it).
      // Waited every iteration, which keeps the protocol checkable (synccheck).
      if (j > 0) mbar_wait(&bars->o_done[t], (j - 1) & 1);
      // lazy O correction: only warps with a row whose max jumped
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

      if (kPSmem) {
        // P_t(j-1) was consumed: PV_t(j-1) completed (o_done waited above).
        // K-major SW128 tile [128 q][128 kv] bf16 as two 64-column boxes
        uint8_t* prow = smem + SmemLayout::pbuf + t * kTileBytes + row_in_tile * 128;
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int ch = 0; ch < 8; ++ch)
            *reinterpret_cast<uint4*>(prow + b * kHalfTile + ((ch ^ (row_in_tile & 7)) * 16)) =
                make_uint4(pk[b][4 * ch], pk[b][4 * ch + 1], pk[b][4 * ch + 2], pk[b][4 * ch + 3]);
        fence_proxy_async_smem();
        tmem_st_wait();  // the O correction, if any
      } else {
        tmem_st_32x32b_x32(p_tmem, pk[0]);
        tmem_st_32x32b_x32(p_tmem + 32, pk[1]);
        tmem_st_wait();
      }

      tc_fence_before();
      mbar_arrive(&bars->p_full[t]);
      FWD_TRACE(quarter == 0 && lane == 0, j, 8 + 6 * t);
    }

    // ===================== epilogue =====================
    if (n_tiles > 0) {
      mbar_wait(&bars->o_done[t], (n_tiles - 1) & 1);
      tc_fence_after();
      const int row = qt * kBM + row_in_tile;
      const bool valid = row < p.rows_q;
      const size_t srow = static_cast<size_t>(head) * p.rows_q + row;
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
  if (warp == 8) tmem_dealloc<512>(tmem);
  if (threadIdx.x == 0) {
    FWD_CTA_TRACE(1, fwd_gtimer());
    FWD_CTA_TRACE(3, clock64());
    FWD_CTA_TRACE(4, fwd_smid());
    FWD_CTA_TRACE(5, static_cast<unsigned long long>(nmax));
    FWD_CTA_TRACE(6, 0ull);
    FWD_CTA_TRACE(7, 0ull);
  }
}

}  // namespace fwd

cudaError_t launch_attn_fwd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                            const FwdParams& p, cudaStream_t stream) {
  static std::atomic<uint64_t> configured{0};
  cudaError_t e = once_per_device(configured, [] {
    return cudaFuncSetAttribute(fwd::attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(fwd::kSmemBytes));
  });
  if (e != cudaSuccess) return e;
  const int n_q_tiles = (p.rows_q + fwd::kBM - 1) / fwd::kBM;
  const int n_pairs = (n_q_tiles + 1) / 2;
  dim3 grid(n_pairs * p.h_q);
  fwd::attn_fwd_kernel<<<grid, fwd::kThreads, fwd::kSmemBytes, stream>>>(tq, tk, tv, p);
  return cudaGetLastError();
}

}  // namespace da
