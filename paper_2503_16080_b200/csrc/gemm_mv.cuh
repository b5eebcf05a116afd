// gemm_mv.cuh — the very-skinny regime (d3_loc ≤ 32, including CP-Mv at d3 = 1):
// the residues' bytes go to the tensor cores AS LOADED, with no limb split at all.
//
// Read the stacked int32 X as a byte matrix: row r, byte column k' = 4k + ℓ is byte ℓ of x[r][k].
// With the EXPANDED plaintext U_exp ∈ Z^{(4·d3p)×(4·d2p)},
//     U_exp[ℓ·d3p + j][4k + ℓ'] = U[k][j] if ℓ' = ℓ, else 0,
// one byte-level contraction gives every limb product at once:
//     D[r][ℓ·d3p + j] = Σ_k' byte(X)[r][k'] · U_exp[ℓ·d3p + j][k'] = Σ_k x_ℓ[r][k]·U[k][j] = C_ℓ[r][j].
// So the MMA's A operand is the raw X tile itself (TMA, SWIZZLE_128B, no converter warps, no
// workspace round trip), B = U_exp (N = 4·d3p ≤ 128 rows), D in TMEM: lane = row r of X, columns
// (ℓ, j) — every limb sum of output (r, j) lands in the thread that owns row r, so recombination
// is local and the output column stores are coalesced across the 128 threads.
// The MMA does 4·d3p/d3-fold padded work (3 of 4 bytes of every U_exp row are 0), which is free
// here: at d3 ≤ 32 the tensor pipe is < 40 % busy when HBM is saturated.  Shared-memory traffic
// per X byte: TMA write 1 + MMA read 1 + U_exp (N·128 B per 16 KB of X) — about half the
// converter kernel's.
//
// Load balance: a tile is 128 rows × all K; with few tiles (R/128) the K loop is split into S
// parts; each (tile, split) unit writes its exact int32 partial C_ℓ to the workspace, and the
// last arriving unit of a tile (atomic ticket, threadfence pattern — no waiting) adds them up and
// runs the epilogue.  Partial sums are exact: |C_ℓ| ≤ d2·255·128 < 2^31 for the full K already.
// Warp roles (256 threads): w0 TMA, w1 MMA, w2 TMEM, w4–7 epilogue (row r = TMEM lane).
#pragma once
#include <cstdint>

#include "kernels.cuh"
#include "ptx.cuh"

namespace ctpt {

constexpr int MV_BLOCK_R = 128;                 // MMA M: rows of X per tile
constexpr int MV_BLOCK_K = 128;                 // bytes of the byte-view K per stage (32 residues)
constexpr int MV_MAX_N = 128;                   // 4 limbs × d3p ≤ 128  →  d3 ≤ 32 (TMEM buffer stride)
constexpr int MV_A_BYTES = MV_BLOCK_R * MV_BLOCK_K;  // 16 KB
constexpr int MV_B_BYTES = MV_MAX_N * MV_BLOCK_K;    // ≤ 16 KB
constexpr int MV_STAGE_BYTES = MV_A_BYTES + MV_B_BYTES;
constexpr int MV_STAGES = 6;
constexpr int MV_THREADS = 256;
constexpr int MV_SMEM_BYTES = MV_STAGES * MV_STAGE_BYTES + 256 + 1024;

struct MvParams {
  int32_t num_kb;      // (4·d2p) / 128 byte-blocks of K
  int32_t num_tiles;   // ceil(R / 128)
  int32_t splits;      // K splits per tile (S)
  int32_t u_unsigned;
  int32_t* partial;    // [num_tiles·S][NC][128] int32 (S > 1)
  uint32_t* tickets;   // [num_tiles], zero on entry; left zero on exit
  ModP m;
  OutParams o;
};

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// NC = N = 4·d3p columns of D (d3p = U columns per limb group, padded to a multiple of 4)
template <int NC>
__global__ void __launch_bounds__(MV_THREADS, 1)
    k_gemm_mv(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmUe,
              const __grid_constant__ MvParams P) {
  constexpr int D3P = NC / 4;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_base = sbase + MV_STAGES * MV_STAGE_BYTES;
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto empty_bar = [&](int s) { return bar_base + 8u * (MV_STAGES + s); };
  auto tfull_bar = [&](int b) { return bar_base + 8u * (2 * MV_STAGES + b); };
  auto tempty_bar = [&](int b) { return bar_base + 8u * (2 * MV_STAGES + 2 + b); };
  const uint32_t tmem_slot = bar_base + 8u * (2 * MV_STAGES + 4);
  uint8_t* bar_ptr = smem + MV_STAGES * MV_STAGE_BYTES;
  uint32_t* tmem_slot_ptr = reinterpret_cast<uint32_t*>(bar_ptr + 8 * (2 * MV_STAGES + 4));
  uint32_t* ticket_ptr = reinterpret_cast<uint32_t*>(bar_ptr + 8 * (2 * MV_STAGES + 5));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int32_t num_units = P.num_tiles * P.splits;
  constexpr int32_t B_bytes = NC * MV_BLOCK_K;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmX);
    tma_prefetch(&tmUe);
    for (int s = 0; s < MV_STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull_bar(b), 1);
      mbar_init(tempty_bar(b), 128);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;

  auto kb_range = [&](int32_t split, int32_t& k0, int32_t& k1) {
    k0 = static_cast<int32_t>(static_cast<int64_t>(P.num_kb) * split / P.splits);
    k1 = static_cast<int32_t>(static_cast<int64_t>(P.num_kb) * (split + 1) / P.splits);
  };

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int32_t u = blockIdx.x; u < num_units; u += gridDim.x) {
        const int32_t tile = u / P.splits, split = u % P.splits;
        int32_t k0, k1;
        kb_range(split, k0, k1);
        for (int32_t kb = k0; kb < k1; ++kb) {
          mbar_wait(empty_bar(stage), phase ^ 1);
          const uint32_t sa = sbase + stage * MV_STAGE_BYTES;
          mbar_arrive_expect_tx(full_bar(stage), MV_A_BYTES + B_bytes);
          tma_load_3d(sa, &tmX, full_bar(stage), kb * MV_BLOCK_K, tile * MV_BLOCK_R, 0);
          tma_load_3d(sa + MV_A_BYTES, &tmUe, full_bar(stage), kb * MV_BLOCK_K, 0, 0);
          if (++stage == MV_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      // A = raw X bytes (unsigned), B = U_exp (U digits: signed, or unsigned plane)
      const uint32_t idesc = idesc_i8(MV_BLOCK_R, NC, /*a_signed=*/false, /*b_signed=*/!P.u_unsigned);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int32_t u = blockIdx.x; u < num_units; u += gridDim.x) {
        int32_t k0, k1;
        kb_range(u % P.splits, k0, k1);
        mbar_wait(tempty_bar(acc), acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * MV_MAX_N;
        for (int32_t kb = k0; kb < k1; ++kb) {
          mbar_wait(full_bar(stage), phase);
          tc_fence_after();
          const uint32_t sa = sbase + stage * MV_STAGE_BYTES;
#pragma unroll
          for (int kk = 0; kk < MV_BLOCK_K / 32; ++kk)
            mma_i8(d_tmem, umma_desc_sw128(sa + kk * 32), umma_desc_sw128(sa + MV_A_BYTES + kk * 32), idesc,
                   (kb != k0 || kk != 0));
          mma_commit(empty_bar(stage));
          if (++stage == MV_STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(tfull_bar(acc));
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue (128 threads)
    const int quad = warp & 3;
    const int r_in = quad * 32 + lane;  // TMEM lane = row of the tile
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int32_t u = blockIdx.x; u < num_units; u += gridDim.x) {
      const int32_t tile = u / P.splits;
      mbar_wait(tfull_bar(acc), acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * MV_MAX_N;
      int32_t c[NC];
#pragma unroll
      for (int q = 0; q < NC / 16; ++q) {
        uint32_t v[16];
        tmem_ld16(t_row + q * 16, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) c[q * 16 + i] = static_cast<int32_t>(v[i]);
      }
      tc_fence_before();
      mbar_arrive(tempty_bar(acc));  // the accumulator is in registers: let the MMA reuse it
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }

      bool last = true;
      if (P.splits > 1) {
        int32_t* mine = P.partial + (static_cast<int64_t>(u) * NC) * MV_BLOCK_R;
#pragma unroll
        for (int n = 0; n < NC; ++n) mine[n * MV_BLOCK_R + r_in] = c[n];
        __threadfence();
        named_bar_sync(1, 128);
        if (threadIdx.x == 128) *ticket_ptr = atomicAdd(P.tickets + tile, 1u);
        named_bar_sync(1, 128);
        last = (*ticket_ptr == static_cast<uint32_t>(P.splits - 1));
        if (last) {
          __threadfence();
          for (int32_t s = 0; s < P.splits; ++s) {
            const int32_t uu = tile * P.splits + s;
            if (uu == u) continue;
            const int32_t* other = P.partial + (static_cast<int64_t>(uu) * NC) * MV_BLOCK_R;
#pragma unroll
            for (int n = 0; n < NC; ++n) c[n] += __ldcg(other + n * MV_BLOCK_R + r_in);
          }
          if (threadIdx.x == 128) P.tickets[tile] = 0;  // ready for the next launch
        }
        named_bar_sync(1, 128);  // ticket_ptr is reused by the next unit
      }
      if (last) {
        const int64_t r = static_cast<int64_t>(tile) * MV_BLOCK_R + r_in;
        if (r < P.o.R) {
#pragma unroll
          for (int j = 0; j < D3P; ++j) {
            if (j < P.o.d3_loc) {
              const uint32_t res = recombine_mod(c[j], c[D3P + j], c[2 * D3P + j], c[3 * D3P + j], P.m);
              store_out(P.o, P.m, j, r, res);
            }
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<256>(tmem_base);
  }
}

// U_exp[ℓ·d3p + jj][4k + ℓ'] = (ℓ' == ℓ && jj < d3_loc) ? plane[j_off + jj][k] : 0, as bytes;
// [N][4·d2p].  One thread per 4 output bytes (one k): 32-bit stores.
__global__ void k_expand_u(const int8_t* __restrict__ plane, int64_t d2p, int32_t j_off, int32_t d3_loc, int32_t d3p,
                           uint32_t* __restrict__ ue) {
  const int n = blockIdx.y;  // row of U_exp
  const int l = n / d3p, jj = n % d3p;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < d2p;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t b = (jj < d3_loc) ? static_cast<uint8_t>(plane[static_cast<int64_t>(j_off + jj) * d2p + k]) : 0u;
    ue[static_cast<int64_t>(n) * d2p + k] = b << (8 * l);
  }
}

}  // namespace ctpt
