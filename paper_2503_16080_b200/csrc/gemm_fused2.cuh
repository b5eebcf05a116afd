// gemm_fused2.cuh — the skinny-U fused split + limb GEMM on a CTA PAIR (tcgen05 cta_group::2)
// for 128 < d3_loc ≤ 256 (Table 4's skinny shapes).
//
// Same contraction, split and epilogue as gemm_fused.cuh (C_ℓ = X_ℓ·U over Z,
// out = Σ 2^{8ℓ} C_ℓ mod p; X read from HBM exactly once), but the two U^T groups
// of the single-CTA kernel (NG = 2: two M = 128 MMAs reading the SAME 64-row limb tile) become
// ONE M = 256 MMA over a 2-CTA cluster:
//   CTA c holds U^T rows [j_off + 128c, +128)            (its half of M = 256)
//          and the four limbs of X rows [64t + 32c, +32) (its half of N = 256:
//          N index c·128 + ℓ·32 + r, ℓ = limb, r = row within the half)
//   D in CTA c's TMEM = its 128 j-lanes × all 256 (half, ℓ, r) columns — each output's four limb
//   sums still sit in one lane, so the epilogue needs no exchange.
// Each CTA converts only ITS 32 rows (raw int32 TMA ring → LDS.128 → PRMT byte transpose →
// SWIZZLE_128B STS), so per 32 rows of X an SM moves ≈ 96 KB through shared memory instead of
// ≈ 112 KB (the limb tile is no longer read by two MMA groups), and TMEM holds two accumulator
// buffers of 256 columns (the NG = 2 single-CTA kernel had to drain its only one between tiles).
//
// Synchronisation (all mbarriers at identical offsets in both CTAs):
//   full[s]    LEADER only: 1 arrive.expect_tx (both CTAs' U halves, 2 × 16 KB, completed by
//              their cta_group::2 TMAs) + 8 local converter-warp arrivals + 8 REMOTE arrivals
//              from the peer's converter warps (fence.proxy.async, then a remote arrive).
//   empty[s]   both CTAs, 1 arrival: the leader's tcgen05.commit multicast to {0, 1}.
//   tfull[b]   both CTAs, 1 arrival: the leader's commit multicast when accumulator b is final.
//   tempty[b]  leader only, 8 arrivals: one per epilogue warp of both CTAs.
//   raw_full / raw_empty: local to each CTA (its own raw X ring), as in gemm_fused.cuh.
// Status: opt-in (CTPT_FUSED2=pair).  Bit-exact in every test, but not faster than the
// single-CTA NG = 2 kernel on c4's ciphertexts (2.05–2.22 vs 2.02–2.14 ms per launch for
// d3 = 129..256; profiles/r01/fused2_pair/): its time does not follow d3, i.e. the MMA is not the
// bound — the converters' per-K-block latency chain and the pair's lock-step stages are.  (One
// early run ended in a launch failure: an mbarrier parity alias with two converter groups on an
// odd-length raw ring, fixed below.)
// Warp roles (512 threads per CTA): w0 U^T TMA, w1 MMA issuer (leader), w2 TMEM allocator,
// w3 raw X TMA, w4–7 epilogue, w8–15 converters (4 rows each).
#pragma once
#include <cstdint>

#include "gemm_fused.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace ctpt {

constexpr int F2_ROWS = 32;                                  // X rows per CTA per tile (pair: 64)
constexpr int F2_BLOCK_K = 128;
constexpr int F2_U_BYTES = 128 * F2_BLOCK_K;                 // this CTA's half of U^T: 16 KB
constexpr int F2_X_BYTES = 4 * F2_ROWS * F2_BLOCK_K;         // this CTA's 4 limbs × 32 rows: 16 KB
constexpr int F2_STAGE_BYTES = F2_U_BYTES + F2_X_BYTES;      // 32 KB
constexpr int F2_STAGES = 4;
constexpr int F2_RAW_BYTES = F2_ROWS * F2_BLOCK_K * 4;       // 16 KB raw int32 tile
constexpr int F2_RAW_STAGES = 6;                             // 96 KB of X in flight per SM
// Both rings' lengths must be multiples of the converter-group count CG (≤ 2): group g then
// always meets the same stages, so its previous use of a stage is its own and an mbarrier parity
// wait can never match a phase two behind.  (With 5 raw stages the groups alternated over a
// stage: a group could pass raw_full(s) while the OTHER group's earlier fill of s was still in
// flight — a TMA landing out of order — and read a stale tile: the one unexplained launch
// failure of the first measurements.)
constexpr int F2_ACC_COLS = 256;
constexpr int F2_THREADS = 512;
constexpr int F2_CONV_WARPS = 8;
constexpr int F2_ROWS_PER_WARP = F2_ROWS / F2_CONV_WARPS;   // 4
constexpr int F2_SMEM_BYTES = F2_STAGES * F2_STAGE_BYTES + F2_RAW_STAGES * F2_RAW_BYTES + 256 + 1024;

// Remote arrive on the leader's barrier after the converters' limb stores were fenced into the
// async proxy (fence.proxy.async.shared::cta).  Default semantics (release at CTA scope): the
// .release.cluster form compiles to MEMBAR.ALL.GPU + CCTL.IVALL per arrival and halved the
// kernel (measured: 3.93 vs 1.99 ms per launch on c4's ciphertexts).
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

template <int CG>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(F2_THREADS, 1)
    k_gemm_fused2(const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmX,
                  const __grid_constant__ FusedParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t raw_base = sbase + F2_STAGES * F2_STAGE_BYTES;
  const uint32_t bar_base = raw_base + F2_RAW_STAGES * F2_RAW_BYTES;
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto empty_bar = [&](int s) { return bar_base + 8u * (F2_STAGES + s); };
  auto tfull_bar = [&](int b) { return bar_base + 8u * (2 * F2_STAGES + b); };
  auto tempty_bar = [&](int b) { return bar_base + 8u * (2 * F2_STAGES + 2 + b); };
  const uint32_t tmem_slot = bar_base + 8u * (2 * F2_STAGES + 4);
  uint32_t* tmem_slot_ptr = reinterpret_cast<uint32_t*>(smem + F2_STAGES * F2_STAGE_BYTES +
                                                        F2_RAW_STAGES * F2_RAW_BYTES + 8 * (2 * F2_STAGES + 4));
  auto raw_full = [&](int s) { return bar_base + 8u * (2 * F2_STAGES + 5 + s); };
  auto raw_empty = [&](int s) { return bar_base + 8u * (2 * F2_STAGES + 5 + F2_RAW_STAGES + s); };

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();  // 0 = leader
  const int32_t pair = static_cast<int32_t>(blockIdx.x >> 1);
  const int32_t npairs = static_cast<int32_t>(gridDim.x >> 1);
  const int32_t my_tiles = (P.num_tiles > pair) ? (P.num_tiles - 1 - pair) / npairs + 1 : 0;
  const int64_t n_it = static_cast<int64_t>(my_tiles) * P.num_kb;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmU);
    tma_prefetch(&tmX);
    for (int s = 0; s < F2_STAGES; ++s) {
      mbar_init(full_bar(s), 1 + 2 * (F2_CONV_WARPS / CG));  // U tx + both CTAs' converter warps
      mbar_init(empty_bar(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull_bar(b), 1);
      mbar_init(tempty_bar(b), 8);
    }
    for (int s = 0; s < F2_RAW_STAGES; ++s) {
      mbar_init(raw_full(s), 1);
      mbar_init(raw_empty(s), F2_CONV_WARPS / CG);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;

  if (warp == 0) {
    // ---------------------------------------------------------------- U^T TMA (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const int32_t jrow = P.j_off + static_cast<int32_t>(rank) * 128;
      for (int64_t it = 0; it < n_it; ++it) {
        const int32_t kb = static_cast<int32_t>(it % P.num_kb);
        mbar_wait(empty_bar(stage), phase ^ 1);
        const uint32_t su = sbase + stage * F2_STAGE_BYTES;
        if (rank == 0) mbar_arrive_expect_tx(full_bar(stage), 2 * F2_U_BYTES);
        tma_load_3d_pair(su, &tmU, mapa_shared(full_bar(stage), 0), kb * F2_BLOCK_K, jrow, P.plane);
        if (++stage == F2_STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (leader only)
    if (rank == 0 && lane == 0) {
      const uint32_t idesc = idesc_i8(256, F2_ACC_COLS, /*a_signed=*/!P.u_unsigned, /*b_signed=*/false);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int32_t t = 0; t < my_tiles; ++t) {
        mbar_wait(tempty_bar(acc), acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * F2_ACC_COLS;
        for (int32_t kb = 0; kb < P.num_kb; ++kb) {
          mbar_wait(full_bar(stage), phase);
          tc_fence_after();
          const uint32_t su = sbase + stage * F2_STAGE_BYTES;
#pragma unroll
          for (int kk = 0; kk < F2_BLOCK_K / FU_MMA_K; ++kk)
            mma_i8_pair(d_tmem, umma_desc_sw128(su + kk * FU_MMA_K), umma_desc_sw128(su + F2_U_BYTES + kk * FU_MMA_K),
                        idesc, (kb | kk) != 0);
          mma_commit_pair_mc(empty_bar(stage), 0x3);
          if (++stage == F2_STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit_pair_mc(tfull_bar(acc), 0x3);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp == 3) {
    // ---------------------------------------------------------------- raw X TMA (both CTAs)
    if (lane == 0) {
      int rs = 0;
      uint32_t rphase = 0;
      for (int64_t it = 0; it < n_it; ++it) {
        const int32_t tr = pair + static_cast<int32_t>(it / P.num_kb) * npairs;
        const int32_t kb = static_cast<int32_t>(it % P.num_kb);
        mbar_wait(raw_empty(rs), rphase ^ 1);
        mbar_arrive_expect_tx(raw_full(rs), F2_RAW_BYTES);
        tma_load_2d(raw_base + rs * F2_RAW_BYTES, &tmX, raw_full(rs), kb * F2_BLOCK_K,
                    tr * 64 + static_cast<int32_t>(rank) * F2_ROWS);
        if (++rs == F2_RAW_STAGES) { rs = 0; rphase ^= 1; }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------------------------------------------------------- epilogue (both CTAs)
    const int quad = warp & 3;
    const int64_t j = static_cast<int64_t>(rank) * 128 + quad * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int32_t t = 0; t < my_tiles; ++t) {
      const int32_t tr = pair + t * npairs;
      mbar_wait(tfull_bar(acc), acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * F2_ACC_COLS;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {  // rows 16c .. 16c+15 of the 64-row tile
        const uint32_t col = (c >> 1) * 128 + (c & 1) * 16;
        uint32_t v0[16], v1[16], v2[16], v3[16];
        tmem_ld16(t_row + col + 0 * 32, v0);
        tmem_ld16(t_row + col + 1 * 32, v1);
        tmem_ld16(t_row + col + 2 * 32, v2);
        tmem_ld16(t_row + col + 3 * 32, v3);
        tmem_ld_wait();
        if (j < P.o.d3_loc) {
          uint32_t res[16];
#pragma unroll
          for (int i = 0; i < 16; ++i)
            res[i] = recombine_mod(static_cast<int32_t>(v0[i]), static_cast<int32_t>(v1[i]),
                                   static_cast<int32_t>(v2[i]), static_cast<int32_t>(v3[i]), P.m);
          store16(P.o, P.m, j, static_cast<int64_t>(tr) * 64 + c * 16, res);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(tempty_bar(acc), 0));
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp >= 8) {
    // ---------------------------------------------------------------- converters (both CTAs)
    // CG groups of 8/CG warps; group g converts the K-blocks it ≡ g (mod CG), so CG K-blocks are
    // in flight at once and each warp amortises its per-iteration latency chain (barrier waits,
    // two proxy fences) over 4·CG rows.  Warp w of a group owns rows w + (8/CG)·i of this CTA's
    // 32-row half; lane owns residues 4·lane .. 4·lane+3 (one 512-B row segment per instruction).
    static_assert(F2_RAW_STAGES % CG == 0 && F2_STAGES % CG == 0, "ring lengths must be multiples of CG");
  constexpr int WPG = F2_CONV_WARPS / CG;       // warps per group
    constexpr int RPW = F2_ROWS / WPG;            // rows per warp
    const int cw = warp - 8;
    const int grp = cw / WPG, w = cw % WPG;
    for (int64_t it = grp; it < n_it; it += CG) {
      const int rs = static_cast<int>(it % F2_RAW_STAGES);
      const uint32_t rphase = static_cast<uint32_t>((it / F2_RAW_STAGES) & 1);
      const int stage = static_cast<int>(it % F2_STAGES);
      const uint32_t phase = static_cast<uint32_t>((it / F2_STAGES) & 1);
      mbar_wait(raw_full(rs), rphase);
      const uint32_t sraw = raw_base + rs * F2_RAW_BYTES;
      uint32_t lw[RPW][4];
#pragma unroll
      for (int i = 0; i < RPW; ++i) {
        const uint4 v = lds128(sraw + (w + WPG * i) * 512 + lane * 16);
        byte_transpose4(v.x, v.y, v.z, v.w, lw[i][0], lw[i][1], lw[i][2], lw[i][3]);
      }
      // hand the raw tile back once its values are consumed, behind a proxy fence (the next
      // TMA into it is an async-proxy write after these generic reads; gemm_fused.cuh)
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(raw_empty(rs));

      mbar_wait(empty_bar(stage), phase ^ 1);
      const uint32_t sx = sbase + stage * F2_STAGE_BYTES + F2_U_BYTES;
#pragma unroll
      for (int i = 0; i < RPW; ++i) {
        const int row = w + WPG * i;
        const uint32_t off =
            static_cast<uint32_t>(row) * 128u + ((((lane >> 2) ^ (row & 7)) << 4) | ((lane & 3) << 2));
#pragma unroll
        for (int l = 0; l < 4; ++l) sts32(sx + l * F2_ROWS * 128 + off, lw[i][l]);
      }
      fence_proxy_async_smem();  // the limb stores are read by the tensor cores (async proxy)
      __syncwarp();
      if (lane == 0) {
        if (rank == 0)
          mbar_arrive(full_bar(stage));
        else
          mbar_arrive_remote(mapa_shared(full_bar(stage), 0));
      }
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
