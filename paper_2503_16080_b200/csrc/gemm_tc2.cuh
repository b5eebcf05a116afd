// gemm_tc2.cuh — the limb GEMM on a CTA PAIR (tcgen05 cta_group::2), SURVEY.md §8(a) a4 + a5.
//
// Same mathematics and epilogue as gemm_tc.cuh; the difference is the operand delivery:
// one MMA of M = 256 (U^T columns j) × N = 256 (4 limbs × 64 rows of X) × K = 32 is issued by
// the leader CTA of a 2-CTA cluster and executed on both SMs:
//   CTA c holds U^T rows [j0 + 128c, j0 + 128c + 128) (its half of M)
//           and byte limbs {2c, 2c+1} of the 64 X rows (its half of N),
//   D in CTA c's TMEM = its 128 j-lanes × all 256 (ℓ, r) columns → the epilogue is unchanged.
// Per SM and per K byte this moves 128 (U) + 128 (X) bytes for 128×256 MACs (128 MAC/B)
// instead of 128 + 256 bytes (85 MAC/B) for the single-CTA tile, and each SM's shared memory
// feeds half of B: less L2→SMEM traffic and less SMEM read bandwidth per MAC.
//
// Synchronisation (all mbarriers at identical offsets in both CTAs):
//   full[s]   leader only, 1 arrival: the leader's arrive.expect_tx of both CTAs' 64 KB;
//             both CTAs' TMAs complete_tx on it (cp.async.bulk.tensor … .cta_group::2).
//             (A remote arrive.release.cluster from the peer here compiled to a MEMBAR that
//             waited for the peer's in-flight TMA and halved the pipeline: measured.)
//   empty[s]  both CTAs, 1 arrival: the leader's tcgen05.commit multicast to {0,1}.
//   tfull[b]  both CTAs, 1 arrival: leader's commit multicast when accumulator b is final.
//   tempty[b] leader only, 8 arrivals: one per epilogue warp of both CTAs.
#pragma once
#include <cstdint>

#include "kernels.cuh"
#include "ptx.cuh"

namespace ctpt {

constexpr int T2_BLOCK_J = 256;                                // MMA M over the pair
constexpr int T2_BLOCK_R = 64;                                 // X rows per tile (× 4 limbs = N)
constexpr int T2_BLOCK_K = 128;
constexpr int T2_STAGES = 6;
constexpr int T2_MMA_K = 32;
constexpr int T2_U_BYTES = 128 * T2_BLOCK_K;                   // this CTA's half of U^T: 16 KB
constexpr int T2_X_BYTES = 2 * T2_BLOCK_R * T2_BLOCK_K;        // this CTA's 2 limbs: 16 KB
constexpr int T2_STAGE_BYTES = T2_U_BYTES + T2_X_BYTES;        // 32 KB
constexpr int T2_ACC_COLS = 4 * T2_BLOCK_R;                    // 256
constexpr int T2_THREADS = 256;
constexpr int T2_SMEM_BYTES = T2_STAGES * T2_STAGE_BYTES + 256 + 1024;
constexpr int T2_GROUP_J_DEFAULT = 8;                          // pair-tiles (256 columns) per raster group

__device__ __forceinline__ void t2_tile_coords(int32_t tile, const TcParams& P, int32_t& tj, int32_t& tr) {
  const int32_t per_group = P.group_j * P.tiles_r;
  const int32_t g = tile / per_group;
  const int32_t rem = tile - g * per_group;
  const int32_t gj = min(P.group_j, P.tiles_j - g * P.group_j);
  tj = g * P.group_j + rem % gj;
  tr = rem / gj;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(T2_THREADS, 1)
    k_gemm_tc2(const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmX,
               const __grid_constant__ TcParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_base = sbase + T2_STAGES * T2_STAGE_BYTES;
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto empty_bar = [&](int s) { return bar_base + 8u * (T2_STAGES + s); };
  auto tfull_bar = [&](int b) { return bar_base + 8u * (2 * T2_STAGES + b); };
  auto tempty_bar = [&](int b) { return bar_base + 8u * (2 * T2_STAGES + 2 + b); };
  const uint32_t tmem_slot = bar_base + 8u * (2 * T2_STAGES + 4);
  uint32_t* tmem_slot_ptr = reinterpret_cast<uint32_t*>(smem + T2_STAGES * T2_STAGE_BYTES + 8 * (2 * T2_STAGES + 4));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();  // 0 = leader
  const int32_t pair = static_cast<int32_t>(blockIdx.x >> 1);
  const int32_t npairs = static_cast<int32_t>(gridDim.x >> 1);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmU);
    tma_prefetch(&tmX);
    for (int s = 0; s < T2_STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull_bar(b), 1);
      mbar_init(tempty_bar(b), 8);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();  // peer barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int32_t tile = pair; tile < P.num_tiles; tile += npairs) {
        int32_t tj, tr;
        t2_tile_coords(tile, P, tj, tr);
        const int32_t jrow = P.j_off + tj * T2_BLOCK_J + static_cast<int32_t>(rank) * 128;
        for (int32_t kb = 0; kb < P.num_kb; ++kb) {
          mbar_wait(empty_bar(stage), phase ^ 1);
          const uint32_t su = sbase + stage * T2_STAGE_BYTES;
          const uint32_t lbar = mapa_shared(full_bar(stage), 0);
          // Only the leader arms its barrier, for the bytes of BOTH CTAs; the peer's TMA
          // completes its bytes on it directly (no remote arrive, no cluster-scope fence).
          if (rank == 0) mbar_arrive_expect_tx(full_bar(stage), 2 * T2_STAGE_BYTES);
          tma_load_3d_pair(su, &tmU, lbar, kb * T2_BLOCK_K, jrow, P.plane);
          tma_load_5d_pair(su + T2_U_BYTES, &tmX, lbar, 0, 0, 2 * static_cast<int32_t>(rank), kb, tr);
          if (++stage == T2_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (leader only)
    if (rank == 0 && lane == 0) {
      const uint32_t idesc = idesc_i8(T2_BLOCK_J, T2_ACC_COLS, /*a_signed=*/!P.u_unsigned, /*b_signed=*/false);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int32_t tile = pair; tile < P.num_tiles; tile += npairs) {
        mbar_wait(tempty_bar(acc), acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * T2_ACC_COLS;
        for (int32_t kb = 0; kb < P.num_kb; ++kb) {
          mbar_wait(full_bar(stage), phase);
          tc_fence_after();
          const uint32_t su = sbase + stage * T2_STAGE_BYTES;
#pragma unroll
          for (int kk = 0; kk < T2_BLOCK_K / T2_MMA_K; ++kk) {
            const uint64_t ad = umma_desc_sw128(su + kk * T2_MMA_K);
            const uint64_t bd = umma_desc_sw128(su + T2_U_BYTES + kk * T2_MMA_K);
            mma_i8_pair(d_tmem, ad, bd, idesc, (kb | kk) != 0);
          }
          mma_commit_pair_mc(empty_bar(stage), 0x3);  // frees this stage in both CTAs
          if (++stage == T2_STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit_pair_mc(tfull_bar(acc), 0x3);  // accumulator final in both CTAs
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue (both CTAs)
    const int quad = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int32_t tile = pair; tile < P.num_tiles; tile += npairs) {
      int32_t tj, tr;
      t2_tile_coords(tile, P, tj, tr);
      mbar_wait(tfull_bar(acc), acc_phase);
      tc_fence_after();
      const int64_t j = static_cast<int64_t>(tj) * T2_BLOCK_J + rank * 128 + quad * 32 + lane;
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * T2_ACC_COLS;
#pragma unroll 1
      for (int c = 0; c < T2_BLOCK_R / 16; ++c) {
        uint32_t v0[16], v1[16], v2[16], v3[16];
        tmem_ld16(t_row + 0 * T2_BLOCK_R + c * 16, v0);
        tmem_ld16(t_row + 1 * T2_BLOCK_R + c * 16, v1);
        tmem_ld16(t_row + 2 * T2_BLOCK_R + c * 16, v2);
        tmem_ld16(t_row + 3 * T2_BLOCK_R + c * 16, v3);
        tmem_ld_wait();
        uint32_t res[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          res[i] = recombine_mod(static_cast<int32_t>(v0[i]), static_cast<int32_t>(v1[i]),
                                 static_cast<int32_t>(v2[i]), static_cast<int32_t>(v3[i]), P.m);
        if (j < P.o.d3_loc) {
          const int64_t r0 = static_cast<int64_t>(tr) * T2_BLOCK_R + c * 16;
          store16(P.o, P.m, j, r0, res);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(tempty_bar(acc), 0));
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  tc_fence_before();
  cluster_sync();  // neither CTA leaves while the pair still uses its SMEM / TMEM
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem_base);
  }
}

}  // namespace ctpt
