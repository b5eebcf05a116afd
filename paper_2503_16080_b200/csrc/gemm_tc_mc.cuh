// gemm_tc_mc.cuh — the single-CTA limb GEMM of gemm_tc.cuh in 2-CTA clusters that SHARE the X
// limb tiles by TMA multicast (SURVEY.md §8(a) a4 + a5).
//
// Same MMA (tcgen05.mma.cta_group::1.kind::i8, M = 128 U^T columns × N = 256 = 4 limbs × 64 rows,
// accumulator in each CTA's own TMEM) and the same epilogue; the difference is where the
// operands come from.  The two CTAs of a cluster work on the SAME 64 rows of X and on adjacent
// 128-column blocks of U (j-tiles 2t and 2t+1): CTA c loads its own U^T tile (16 KB per K-block)
// and limbs {2c, 2c+1} of the shared X tile (16 KB), the latter MULTICAST into both CTAs' shared
// memory, so every SM pulls 32 KB instead of 48 KB per K-block from L2 (−33 % L2→SM traffic) —
// a lever on the power-capped GEMM (energy, not issue rate, is the limit).
//
// Synchronisation (stage s, identical smem offsets in both CTAs):
//   full[s]   local, 1 arrival (own arrive.expect_tx of 48 KB) + the bytes of own U load, own
//             X half and the peer's X half (both multicasts complete_tx on each CTA's full[s]).
//   empty[s]  local, 2 arrivals: own MMA commit and the peer's (each MMA thread commits with
//             .multicast::cluster to both CTAs) — a stage is refilled only after BOTH CTAs' MMAs
//             read it, because the refill writes into both.
//   tfull / tempty: local, as in gemm_tc.cuh.
#pragma once
#include <cstdint>

#include "gemm_tc.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace ctpt {

constexpr int MC_X_HALF = 2 * TC_BLOCK_R * TC_BLOCK_K;  // 2 limbs × 64 rows × 128 B = 16 KB

// 5-D TMA load multicast to the CTAs in `mask` (same smem / mbarrier offsets in each).
__device__ __forceinline__ void tma_load_5d_mc(uint32_t dst, const CUtensorMap* m, uint32_t bar, int32_t c0,
                                               int32_t c1, int32_t c2, int32_t c3, int32_t c4, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar), "h"(mask)
      : "memory");
}
// tcgen05.commit of this CTA's MMAs, arriving on the barrier at `bar` in every CTA of `mask`.
__device__ __forceinline__ void mma_commit_mc(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"(mask)
      : "memory");
}

// cluster tile t (a pair of j-tiles × one 64-row tile) → (j-tile pair, r-tile), raster groups of
// group_j PAIRS so a group's U panels stay in L2 while the X panels stream
__device__ __forceinline__ void mc_tile_coords(int32_t tile, const TcParams& P, int32_t tiles_jp, int32_t& tjp,
                                               int32_t& tr) {
  const int32_t per_group = P.group_j * P.tiles_r;
  const int32_t g = tile / per_group;
  const int32_t rem = tile - g * per_group;
  const int32_t gj = min(P.group_j, tiles_jp - g * P.group_j);
  tjp = g * P.group_j + rem % gj;
  tr = rem / gj;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS, 1)
    k_gemm_tc_mc(const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmX,
                 const __grid_constant__ TcParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_base = sbase + TC_STAGES * TC_STAGE_BYTES;
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto empty_bar = [&](int s) { return bar_base + 8u * (TC_STAGES + s); };
  auto tfull_bar = [&](int b) { return bar_base + 8u * (2 * TC_STAGES + b); };
  auto tempty_bar = [&](int b) { return bar_base + 8u * (2 * TC_STAGES + 2 + b); };
  const uint32_t tmem_slot = bar_base + 8u * (2 * TC_STAGES + 4);
  uint32_t* tmem_slot_ptr = reinterpret_cast<uint32_t*>(smem + TC_STAGES * TC_STAGE_BYTES + 8 * (2 * TC_STAGES + 4));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int32_t cl = static_cast<int32_t>(blockIdx.x >> 1);
  const int32_t ncl = static_cast<int32_t>(gridDim.x >> 1);
  const int32_t tiles_jp = (P.tiles_j + 1) / 2;
  const int32_t ntiles = tiles_jp * P.tiles_r;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmU);
    tma_prefetch(&tmX);
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 2);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull_bar(b), 1);
      mbar_init(tempty_bar(b), 128);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();  // both CTAs' barriers initialised before any multicast lands
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int32_t tile = cl; tile < ntiles; tile += ncl) {
        int32_t tjp, tr;
        mc_tile_coords(tile, P, tiles_jp, tjp, tr);
        const int32_t jrow = P.j_off + (2 * tjp + static_cast<int32_t>(rank)) * TC_BLOCK_J;
        for (int32_t kb = 0; kb < P.num_kb; ++kb) {
          mbar_wait(empty_bar(stage), phase ^ 1);  // both CTAs' MMAs have read this stage
          const uint32_t su = sbase + stage * TC_STAGE_BYTES;
          mbar_arrive_expect_tx(full_bar(stage), TC_STAGE_BYTES);
          tma_load_3d(su, &tmU, full_bar(stage), kb * TC_BLOCK_K, jrow, P.plane);
          tma_load_5d_mc(su + TC_U_BYTES + rank * MC_X_HALF, &tmX, full_bar(stage), 0, 0, 2 * static_cast<int32_t>(rank), kb,
                         tr, 0x3);
          if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_i8(TC_BLOCK_J, TC_ACC_COLS, /*a_signed=*/!P.u_unsigned, /*b_signed=*/false);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int32_t tile = cl; tile < ntiles; tile += ncl) {
        mbar_wait(tempty_bar(acc), acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * TC_ACC_COLS;
        for (int32_t kb = 0; kb < P.num_kb; ++kb) {
          mbar_wait(full_bar(stage), phase);
          tc_fence_after();
          const uint32_t su = sbase + stage * TC_STAGE_BYTES;
#pragma unroll
          for (int kk = 0; kk < TC_BLOCK_K / TC_MMA_K; ++kk)
            mma_i8(d_tmem, umma_desc_sw128(su + kk * TC_MMA_K), umma_desc_sw128(su + TC_U_BYTES + kk * TC_MMA_K), idesc,
                   (kb | kk) != 0);
          mma_commit_mc(empty_bar(stage), 0x3);  // frees the stage in BOTH CTAs' accounting
          if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(tfull_bar(acc));
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue (128 threads)
    const int quad = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int32_t tile = cl; tile < ntiles; tile += ncl) {
      int32_t tjp, tr;
      mc_tile_coords(tile, P, tiles_jp, tjp, tr);
      mbar_wait(tfull_bar(acc), acc_phase);
      tc_fence_after();
      const int64_t j = static_cast<int64_t>(2 * tjp + static_cast<int32_t>(rank)) * TC_BLOCK_J + quad * 32 + lane;
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * TC_ACC_COLS;
#pragma unroll 1
      for (int c = 0; c < TC_BLOCK_R / 16; ++c) {
        uint32_t v0[16], v1[16], v2[16], v3[16];
        tmem_ld16(t_row + 0 * TC_BLOCK_R + c * 16, v0);
        tmem_ld16(t_row + 1 * TC_BLOCK_R + c * 16, v1);
        tmem_ld16(t_row + 2 * TC_BLOCK_R + c * 16, v2);
        tmem_ld16(t_row + 3 * TC_BLOCK_R + c * 16, v3);
        tmem_ld_wait();
        if (j < P.o.d3_loc) {
          uint32_t res[16];
#pragma unroll
          for (int i = 0; i < 16; ++i)
            res[i] = recombine_mod(static_cast<int32_t>(v0[i]), static_cast<int32_t>(v1[i]),
                                   static_cast<int32_t>(v2[i]), static_cast<int32_t>(v3[i]), P.m);
          store16(P.o, P.m, j, static_cast<int64_t>(tr) * TC_BLOCK_R + c * 16, res);
        }
      }
      tc_fence_before();
      mbar_arrive(tempty_bar(acc));
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp == 2 || warp == 3) {
    // ---------------------------------------------------------------- next prime's limb split
    if (P.sj.x) side_split_rows(P.sj, 2 * static_cast<int64_t>(blockIdx.x) + (warp - 2), 2 * static_cast<int64_t>(gridDim.x), lane);
  }

  tc_fence_before();
  cluster_sync();  // every multicast into / commit onto the peer has landed before either exits
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

}  // namespace ctpt
