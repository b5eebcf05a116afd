// gemm_fused.cuh — the skinny-U limb GEMM with the limb split fused into its load path
// (d3 ≤ 256, including CP-Mv at d3 = 1; Table 4's d3 ∈ {1, 2^6, 2^7},
// P:1575–1582; CP-Mv).
//
// Same contraction and epilogue as gemm_tc.cuh (C_ℓ = X_ℓ·U over Z, out = Σ 2^{8ℓ} C_ℓ mod p,
// P:1380–1388), but for d3 ≤ 256 the step is HBM-bound (≈ d3 limb MACs per byte of X, below the
// ridge), so the schedule is built around reading X exactly once:
//   * one tile = 64 rows of X × ALL of U's d3_loc columns (NG = ⌈d3_loc/128⌉ ≤ 2 MMA groups of
//     M = 128 U^T rows) × the full K loop — X is never re-read;
//   * the residues are read as int32 straight from the stacked K-major X of ctpt_layout (TMA
//     into a raw shared-memory ring, then LDS.128 by eight converter warps), split
//     into their four base-2^8 digits with a PRMT byte transpose in registers and stored into the
//     SWIZZLE_128B K-major shared-memory image the UMMA descriptor expects — no limb workspace,
//     8 B/residue of HBM traffic saved against split + GEMM (4 B read instead of 4 + 4 + 4);
//   * U^T tiles (≤ 256 × 128 B per K-block, L2-resident) arrive by TMA on the same stage barrier.
// Warp roles (512 threads): w0 U TMA, w1 MMA issuer, w2 TMEM allocator, w3 raw X TMA, w4–7 epilogue,
// w8–15 converters.  Stage barrier `full` completes on 1 TMA arrival (+ tx bytes) and 8 converter
// warp arrivals; converters fence their generic-proxy stores (fence.proxy.async) first.
#pragma once
#include <cstdint>

#include "kernels.cuh"
#include "ptx.cuh"

namespace ctpt {

constexpr int FU_BLOCK_R = 64;     // rows of X per tile (× 4 limbs = MMA N = 256)
constexpr int FU_BLOCK_K = 128;    // K bytes (= int32 residues) per stage
constexpr int FU_MMA_K = 32;
constexpr int FU_U_BYTES = 128 * FU_BLOCK_K;                 // one U^T group tile: 16 KB
constexpr int FU_X_BYTES = 4 * FU_BLOCK_R * FU_BLOCK_K;      // 4 limb tiles: 32 KB
constexpr int FU_ACC_COLS = 4 * FU_BLOCK_R;                  // 256 TMEM columns per group
constexpr int FU_THREADS = 512;
constexpr int FU_CONV_WARP0 = 8;
constexpr int FU_CONV_WARPS = 8;
constexpr int FU_ROWS_PER_WARP = FU_BLOCK_R / FU_CONV_WARPS; // 8
// X reaches the converters through a ring of RAW shared-memory stages filled by TMA (warp 3):
// raw int32 tiles of 64 rows × 128 residues (32 KB), 96–128 KB in flight per SM without any
// register cost; converters read them with LDS.128.  (Measured against register loads two
// K-blocks ahead, a half-TMA / half-register hybrid and two converter groups: the TMA ring was
// best or tied, profiles/r01/skinny_sweep_*.jsonl, fused_tma2/; those variants were removed.)
constexpr int FU_RAW_BYTES = FU_BLOCK_R * FU_BLOCK_K * 4;   // 32 KB
constexpr int FU_STAGES = 2;                                 // limb stages
__host__ __device__ constexpr int fu_raw_stages(int ng) { return ((ng == 1 ? 128 : 96) * 1024) / FU_RAW_BYTES; }
__host__ __device__ constexpr int fu_stage_bytes(int ng) { return ng * FU_U_BYTES + FU_X_BYTES; }
__host__ __device__ constexpr int fu_smem_bytes(int ng) {
  return FU_STAGES * fu_stage_bytes(ng) + fu_raw_stages(ng) * FU_RAW_BYTES + 256 + 1024;
}

struct FusedParams {
  const uint32_t* x;   // stacked K-major X of this prime (or chunk): [R][d2p] int32 residues
  int64_t R, d2p;
  int32_t j_off;       // first U column (col_begin)
  int32_t plane;       // U digit plane (3rd TMA coordinate)
  int32_t num_kb;      // ceil(d2p / 128)
  int32_t num_tiles;   // ceil(R / 64)
  int32_t u_unsigned;  // U plane is u8 (U + u_offset) instead of balanced s8 digits
  ModP m;
  OutParams o;         // d3_loc ≤ 128·NG
};

template <int NG>
__global__ void __launch_bounds__(FU_THREADS, 1)
    k_gemm_fused(const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmX,
                 const __grid_constant__ FusedParams P) {
  constexpr int STAGES = FU_STAGES;
  constexpr int RAW = fu_raw_stages(NG);
  constexpr int RAW_BYTES = FU_RAW_BYTES;
  constexpr int STAGE_BYTES = fu_stage_bytes(NG);
  constexpr int NBUF = (NG == 1) ? 2 : 1;  // accumulator buffers (NBUF·NG·256 ≤ 512 columns)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t raw_base = sbase + STAGES * STAGE_BYTES;
  const uint32_t bar_base = raw_base + RAW * RAW_BYTES;
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto empty_bar = [&](int s) { return bar_base + 8u * (STAGES + s); };
  auto tfull_bar = [&](int b) { return bar_base + 8u * (2 * STAGES + b); };
  auto tempty_bar = [&](int b) { return bar_base + 8u * (2 * STAGES + 2 + b); };
  const uint32_t tmem_slot = bar_base + 8u * (2 * STAGES + 4);
  uint32_t* tmem_slot_ptr =
      reinterpret_cast<uint32_t*>(smem + STAGES * STAGE_BYTES + RAW * RAW_BYTES + 8 * (2 * STAGES + 4));
  auto raw_full = [&](int s) { return bar_base + 8u * (2 * STAGES + 5 + s); };
  auto raw_empty = [&](int s) { return bar_base + 8u * (2 * STAGES + 5 + RAW + s); };

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // this CTA's (tile, kb) iterations, flattened: tile = blockIdx.x + (it / num_kb)·gridDim.x
  const int32_t my_tiles =
      (P.num_tiles > static_cast<int32_t>(blockIdx.x)) ? (P.num_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t n_it = static_cast<int64_t>(my_tiles) * P.num_kb;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmU);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1 + FU_CONV_WARPS);
      mbar_init(empty_bar(s), 1);
    }
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(tfull_bar(b), 1);
      mbar_init(tempty_bar(b), 128);
    }
    for (int s = 0; s < RAW; ++s) {
      mbar_init(raw_full(s), 1);
      mbar_init(raw_empty(s), FU_CONV_WARPS);
    }
    tma_prefetch(&tmX);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;

  if (warp == 0) {
    // ---------------------------------------------------------------- U^T TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t it = 0; it < n_it; ++it) {
        const int32_t kb = static_cast<int32_t>(it % P.num_kb);
        mbar_wait(empty_bar(stage), phase ^ 1);
        const uint32_t su = sbase + stage * STAGE_BYTES;
        mbar_arrive_expect_tx(full_bar(stage), NG * FU_U_BYTES);
#pragma unroll
        for (int g = 0; g < NG; ++g)
          tma_load_3d(su + g * FU_U_BYTES, &tmU, full_bar(stage), kb * FU_BLOCK_K, P.j_off + g * 128, P.plane);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_i8(128, FU_ACC_COLS, /*a_signed=*/!P.u_unsigned, /*b_signed=*/false);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int32_t t = 0; t < my_tiles; ++t) {
        mbar_wait(tempty_bar(acc), acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * NG * FU_ACC_COLS;
        for (int32_t kb = 0; kb < P.num_kb; ++kb) {
          mbar_wait(full_bar(stage), phase);
          tc_fence_after();
          const uint32_t su = sbase + stage * STAGE_BYTES;
#pragma unroll
          for (int kk = 0; kk < FU_BLOCK_K / FU_MMA_K; ++kk) {
            const uint64_t bd = umma_desc_sw128(su + NG * FU_U_BYTES + kk * FU_MMA_K);
#pragma unroll
            for (int g = 0; g < NG; ++g)
              mma_i8(d_tmem + g * FU_ACC_COLS, umma_desc_sw128(su + g * FU_U_BYTES + kk * FU_MMA_K), bd, idesc,
                     (kb | kk) != 0);
          }
          mma_commit(empty_bar(stage));
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(tfull_bar(acc));
        if (++acc == NBUF) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp == 3) {
    // ---------------------------------------------------------------- raw X TMA producer
    if (lane == 0) {
      int rs = 0;
      uint32_t rphase = 0;
      for (int64_t it = 0; it < n_it; ++it) {
        const int32_t tr = static_cast<int32_t>(blockIdx.x) + static_cast<int32_t>(it / P.num_kb) * gridDim.x;
        const int32_t kb = static_cast<int32_t>(it % P.num_kb);
        mbar_wait(raw_empty(rs), rphase ^ 1);
        mbar_arrive_expect_tx(raw_full(rs), RAW_BYTES);
        tma_load_2d(raw_base + rs * RAW_BYTES, &tmX, raw_full(rs), kb * FU_BLOCK_K, tr * FU_BLOCK_R);
        if (++rs == RAW) { rs = 0; rphase ^= 1; }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------------------------------------------------------- epilogue (128 threads)
    const int quad = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int32_t t = 0; t < my_tiles; ++t) {
      const int32_t tr = static_cast<int32_t>(blockIdx.x) + t * static_cast<int32_t>(gridDim.x);
      mbar_wait(tfull_bar(acc), acc_phase);
      tc_fence_after();
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        const int64_t j = g * 128 + quad * 32 + lane;
        const uint32_t t_row =
            tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + (acc * NG + g) * FU_ACC_COLS;
#pragma unroll 1
        for (int c = 0; c < FU_BLOCK_R / 16; ++c) {
          uint32_t v0[16], v1[16], v2[16], v3[16];
          tmem_ld16(t_row + 0 * FU_BLOCK_R + c * 16, v0);
          tmem_ld16(t_row + 1 * FU_BLOCK_R + c * 16, v1);
          tmem_ld16(t_row + 2 * FU_BLOCK_R + c * 16, v2);
          tmem_ld16(t_row + 3 * FU_BLOCK_R + c * 16, v3);
          tmem_ld_wait();
          if (j < P.o.d3_loc) {
            uint32_t res[16];
#pragma unroll
            for (int i = 0; i < 16; ++i)
              res[i] = recombine_mod(static_cast<int32_t>(v0[i]), static_cast<int32_t>(v1[i]),
                                     static_cast<int32_t>(v2[i]), static_cast<int32_t>(v3[i]), P.m);
            const int64_t r0 = static_cast<int64_t>(tr) * FU_BLOCK_R + c * 16;
            store16(P.o, P.m, j, r0, res);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(tempty_bar(acc));
      if (++acc == NBUF) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp >= FU_CONV_WARP0) {
    // ---------------------------------------------------------------- converters (256 threads)
    // Warp cw owns rows cw + 8·i (i < 8) of every 64-row tile; lane owns residues 4·lane..4·lane+3
    // of the K-block (LDS.128 of the raw tile's 512-B rows).
    const int cw = warp - FU_CONV_WARP0;
    int stage = 0;
    uint32_t phase = 0;
    int rs = 0;
    uint32_t rphase = 0;
    for (int64_t it = 0; it < n_it; ++it) {
      mbar_wait(raw_full(rs), rphase);
      const uint32_t sraw = raw_base + rs * RAW_BYTES;
      uint32_t lw[FU_ROWS_PER_WARP][4];
#pragma unroll
      for (int i = 0; i < FU_ROWS_PER_WARP; ++i) {
        CTPT_CHECK(sraw + (cw + FU_CONV_WARPS * i) * 512 + lane * 16 + 16 <= raw_base + RAW * RAW_BYTES);
        const uint4 v = lds128(sraw + (cw + FU_CONV_WARPS * i) * 512 + lane * 16);
        byte_transpose4(v.x, v.y, v.z, v.w, lw[i][0], lw[i][1], lw[i][2], lw[i][3]);
      }
      // Hand the raw tile back to the TMA producer as soon as its values are CONSUMED (the
      // byte transposes above depend on every LDS), behind a proxy fence (a generic read
      // followed by an async-proxy write of the same bytes), and before waiting for a free limb
      // stage — so the raw ring keeps streaming while the MMAs drain.  Releasing it right after
      // merely issuing the LDS corrupted whole output rows intermittently (K ≥ 32 blocks).
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(raw_empty(rs));
      if (++rs == RAW) { rs = 0; rphase ^= 1; }
      // store the limb words of this warp's 8 rows into the next limb stage (SWIZZLE_128B
      // K-major: 16-B chunk c of row r at chunk position c ^ (r & 7)) and arrive on its barrier
      mbar_wait(empty_bar(stage), phase ^ 1);
      const uint32_t sx = sbase + stage * STAGE_BYTES + NG * FU_U_BYTES;
#pragma unroll
      for (int i = 0; i < FU_ROWS_PER_WARP; ++i) {
        const int row = cw + FU_CONV_WARPS * i;
        const uint32_t off =
            static_cast<uint32_t>(row) * 128u + ((((lane >> 2) ^ (row & 7)) << 4) | ((lane & 3) << 2));
        sts32(sx + 0 * FU_BLOCK_R * 128 + off, lw[i][0]);
        sts32(sx + 1 * FU_BLOCK_R * 128 + off, lw[i][1]);
        sts32(sx + 2 * FU_BLOCK_R * 128 + off, lw[i][2]);
        sts32(sx + 3 * FU_BLOCK_R * 128 + off, lw[i][3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(full_bar(stage));
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

}  // namespace ctpt
