// gemm_fused_t.cuh — the skinny-U limb GEMM with the limb split fused into its load path and the
// byte limbs kept in TENSOR MEMORY (d3 ≤ 256, CP-Mv at d3 = 1 included;
// Table 4's d3 ∈ {1, 2^6, 2^7}; CP-Mv).
//
// Same contraction and epilogue arithmetic as gemm_tc.cuh (C_ℓ = X_ℓ·U over Z, out = Σ 2^{8ℓ} C_ℓ
// mod p).  Below the ridge (≈ d3 limb MACs per byte of X) the step is HBM-bound, so
// the schedule reads X exactly once: a tile is 64 (or 32) rows of X × ALL of U's d3_loc columns ×
// the full K loop, and the int32 residues are split into their four base-2^8 digits on the way in
// (no limb workspace: 4 B of HBM per residue instead of split + GEMM's 4 + 4 + 4).  Round 1's
// kernel kept the limbs in shared memory as the MMA's B operand with U^T as A (M = 128 columns
// of U); this one swaps the operand roles so that the limbs never touch shared memory:
//   MMA A = the limb tile in TMEM (tcgen05.mma …, [a-tmem]): M = 128 lanes = 32 rows of X × 4
//           limbs — lane 16h + 8ℓ' + r of quadrant q holds limb 2h + ℓ' of row 8q + r of the
//           tile, its 32-bit columns 4 consecutive residues' bytes (K-major);
//   MMA B = U^T (N = d3_loc rounded up to 16, ≤ 256 rows × 128 B per K-block, TMA, SWIZZLE_128B);
//   D     = 128 lanes × N columns, same lane mapping: C_ℓ[row][j] for every j.
// So the converters store their PRMT byte transposes with tcgen05.st (STTM) instead of STS into
// a swizzled shared-memory image that the MMA then re-reads, and N is d3 itself (no M = 128 group
// padded to 128 columns of U).  The .16x256b TMEM access shape (thread 4r + c ↔ lanes r, r + 8 ×
// column pair c) matches that lane mapping: a converter thread that loaded 8 residues of row r
// stores all four of their limbs, and an epilogue thread gets all four limb sums of its outputs —
// no cross-lane exchange on either side (an earlier version with lane = 4r + ℓ needed shuffles
// and selects for a 4×4 word transpose and was issue-bound: 51 % issue slots at d3 = 64).
//
// Converter data path per K-block (32 rows × 128 residues, 16 KB per sub-tile): TMA raw tiles
// (4 boxes of 32 rows × 32 residues, SWIZZLE_128B) → LDS.128 → PRMT 4×4 byte transpose → STTM.
// Two converter groups (warps 8–11, 12–15) take alternate K-blocks for 32-row tiles; every ring
// length is then even so a stage always meets the same group (round 1's parity lesson: a group
// two phases behind once passed a barrier of the other group's fill).
// Unsigned-U plane (U' = U + u_offset): the converters also form Σ_k X[r][k] (IDP4A byte sums of
// the limb words), flushed per tile through shared memory; the epilogue subtracts
// u_offset·Σ_k X[r][k] mod p.
// Warp roles (512 threads): w0 U^T TMA, w1 MMA issuer, w2 TMEM allocator, w3 raw X TMA,
// w4–7 epilogue, w8–15 converters.
#pragma once
#include <cstdint>

#include "kernels.cuh"
#include "ptx.cuh"

namespace ctpt {

constexpr int FT_SUB_ROWS = 32;      // rows of X per MMA (× 4 limbs = MMA M = 128)
constexpr int FT_BK = 128;           // residues (K bytes of each limb row) per K-block
constexpr int FT_MMA_K = 32;
constexpr int FT_BOX_BYTES = 4096;   // one raw TMA box: 32 rows × 32 residues
constexpr int FT_THREADS = 512;
// Shapes (template <NPMAX, SUB>):
//   SUB = 2 (d3_loc ≤ 224): a tile is 64 rows = two 32-row sub-tiles that share each U^T stage
//     (U^T is read from L2 once per 64 rows); one D buffer of 2 × NPMAX columns and the rest of
//     TMEM as A stages of 2 × AW columns, AW = 32 (a K-block, 128 residues) or 16 (half a
//     K-block): NPMAX = 128 / 160 / 192 / 224 → 4 / 3 / 2 / 2 stages of AW = 32 / 32 / 32 / 16;
//     the 8 converter warps split every K-block (warp 8 + 4s + q: sub-tile s, quadrant q);
//   SUB = 1, NPMAX = 256 (224 < d3_loc ≤ 256): 32-row tiles (a 64-row D would need all 512 TMEM
//     columns), one D buffer of 256 columns + 8 A stages of 32 columns; two converter groups of 4
//     warps take alternate K-blocks; U^T is read from L2 once per 32 rows.
__host__ __device__ constexpr int ft_rows(int sub) { return 32 * sub; }
__host__ __device__ constexpr int ft_raw_bytes(int sub) { return sub * 4 * FT_BOX_BYTES; }
__host__ __device__ constexpr int ft_u_bytes(int npmax) { return npmax * 128; }
// U^T stages in shared memory; raw X stages (≥ 128 KB in flight per SM where it fits beside U^T)
__host__ __device__ constexpr int ft_us(int npmax, int sub) { return (sub == 2 && npmax >= 160 && npmax != 192) ? 3 : 4; }
__host__ __device__ constexpr int ft_raw_stages(int npmax, int sub) {
  return sub == 2 ? (npmax >= 192 ? 4 : 5) : (npmax == 256 ? 6 : 10);
}
#ifndef CTPT_FT_AW_FROM
#define CTPT_FT_AW_FROM 224  // narrowest NPMAX with half-K-block limb stages (A/B builds)
#endif
// TMEM columns per sub-tile in one limb stage: 32 = a whole K-block, 16 = half of one
__host__ __device__ constexpr int ft_aw(int npmax, int sub) { return (sub == 2 && npmax >= CTPT_FT_AW_FROM) ? 16 : 32; }
__host__ __device__ constexpr int ft_ast(int npmax, int sub) {
  return sub == 2 ? ((512 - 2 * npmax) / (2 * ft_aw(npmax, sub)) < 4 ? (512 - 2 * npmax) / (2 * ft_aw(npmax, sub)) : 4)
                  : 8;
}
// + 512 B of barriers, 1 KB of row-sum partials (unsigned-U row correction), 1 KB of alignment slack
__host__ __device__ constexpr int ft_smem_bytes(int npmax, int sub) {
  return ft_us(npmax, sub) * ft_u_bytes(npmax) + ft_raw_stages(npmax, sub) * ft_raw_bytes(sub) + 512 + 1024 + 1024;
}

struct FusedTParams {
  int64_t R;
  int32_t j_off;       // first U column (col_begin)
  int32_t plane;       // U digit plane (3rd TMA coordinate)
  int32_t num_kb;      // ceil(d2p / 128)
  int32_t num_tiles;   // ceil(R / (32·SUB))
  int32_t np;          // MMA N = d3_loc rounded up to 16 (≤ NPMAX)
  int32_t u_unsigned;  // U plane is u8 (U' = U + u_offset) instead of balanced s8 digits
  uint32_t off_mod;    // u_offset mod p: the epilogue subtracts u_offset·Σ_k X[r][k] (row sums formed by the
                       // converters while they split X); 0: no correction
  ModP m;
  OutParams o;         // o.rowcorr is not used (the row sums are formed in-kernel)
};

// D[tmem] (+)= A[tmem] · B[smem]^T, kind::i8 (A from tensor memory).
__device__ __forceinline__ void mma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 32 lanes × 32 bit, 32 consecutive columns per thread: registers → TMEM.
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// .16x256b.x4: 16 TMEM lanes × 32 columns; thread t = 4r + c holds, for repetition k, the words
// (lane r, column 8k + 2c), (lane r, 8k + 2c + 1), (lane r + 8, 8k + 2c), (lane r + 8, 8k + 2c + 1)
// in registers 4k .. 4k + 3 (the mma accumulator-fragment pattern).
__device__ __forceinline__ void tmem_st16x256_x4(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st16x256_x2(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x2.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void tmem_ld16x256_x4(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

template <int NPMAX, int SUB>
__global__ void __launch_bounds__(FT_THREADS, 1)
    k_gemm_fused_t(const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmX,
                   const __grid_constant__ FusedTParams P) {
  constexpr int U_BYTES = ft_u_bytes(NPMAX);
  constexpr int RAW = ft_raw_stages(NPMAX, SUB);
  constexpr int RAW_BYTES = ft_raw_bytes(SUB);
  constexpr int FT_AST = ft_ast(NPMAX, SUB);
  constexpr int FT_US = ft_us(NPMAX, SUB);
  static_assert(ft_smem_bytes(NPMAX, SUB) <= 232448, "shared memory per CTA");
  static_assert(FT_AST >= 2, "at least two limb stages (convert one while the MMA reads the other)");
  constexpr int ROWS = ft_rows(SUB);
  constexpr int NBUF = 1;                      // D: SUB × NPMAX columns (one buffer)
  constexpr int D_COLS = SUB * NPMAX;
  constexpr int AW = ft_aw(NPMAX, SUB);          // columns per sub-tile of one A stage (4 residues each)
  constexpr int HPK = 32 / AW;                   // A stages per K-block
  constexpr int ASTAGE_COLS = SUB * AW;          // one A stage: SUB sub-tiles × AW columns
  constexpr uint32_t A_COL0 = D_COLS;           // TMEM columns [A_COL0, 512) hold the limb stages
  constexpr int GROUPS = SUB == 1 ? 2 : 1;      // converter groups taking alternate K-blocks
  static_assert(A_COL0 + ASTAGE_COLS * FT_AST <= 512, "TMEM budget");
  static_assert(RAW % GROUPS == 0 && FT_AST % GROUPS == 0, "ring lengths must be multiples of the group count");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t raw_base = sbase + FT_US * U_BYTES;
  const uint32_t bar_base = raw_base + RAW * RAW_BYTES;
  auto u_full = [&](int s) { return bar_base + 8u * s; };
  auto u_empty = [&](int s) { return bar_base + 8u * (FT_US + s); };
  auto raw_full = [&](int s) { return bar_base + 8u * (2 * FT_US + s); };
  auto raw_empty = [&](int s) { return bar_base + 8u * (2 * FT_US + RAW + s); };
  auto a_full = [&](int s) { return bar_base + 8u * (2 * FT_US + 2 * RAW + s); };
  auto a_empty = [&](int s) { return bar_base + 8u * (2 * FT_US + 2 * RAW + FT_AST + s); };
  auto d_full = [&](int b) { return bar_base + 8u * (2 * FT_US + 2 * RAW + 2 * FT_AST + b); };
  auto d_empty = [&](int b) { return bar_base + 8u * (2 * FT_US + 2 * RAW + 2 * FT_AST + 2 + b); };
  // row-sum partials of tile t live in buffer t & 1: full = every converter warp wrote its partials,
  // empty = every epilogue thread read them
  auto rows_full = [&](int b) { return bar_base + 8u * (2 * FT_US + 2 * RAW + 2 * FT_AST + 4 + b); };
  auto rows_empty = [&](int b) { return bar_base + 8u * (2 * FT_US + 2 * RAW + 2 * FT_AST + 6 + b); };
  constexpr int NBAR = 2 * FT_US + 2 * RAW + 2 * FT_AST + 8;
  static_assert(8 * NBAR + 8 <= 512, "barrier area");
  // rsum[buf][sub-tile][group][32 rows] u64 partial row sums (1 KB)
  uint64_t* rsum = reinterpret_cast<uint64_t*>(smem + FT_US * U_BYTES + RAW * RAW_BYTES + 512);
  static_assert(2 * SUB * GROUPS * 32 * 8 <= 1024, "row-sum area");
  const uint32_t tmem_slot = bar_base + 8u * NBAR;
  uint32_t* tmem_slot_ptr = reinterpret_cast<uint32_t*>(smem + FT_US * U_BYTES + RAW * RAW_BYTES + 8 * NBAR);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int32_t my_tiles =
      (P.num_tiles > static_cast<int32_t>(blockIdx.x)) ? (P.num_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t n_it = static_cast<int64_t>(my_tiles) * P.num_kb;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmU);
    tma_prefetch(&tmX);
    for (int s = 0; s < FT_US; ++s) {
      mbar_init(u_full(s), 1);
      mbar_init(u_empty(s), 1);
    }
    for (int s = 0; s < RAW; ++s) {
      mbar_init(raw_full(s), 1);
      mbar_init(raw_empty(s), 8 / GROUPS);  // the converter warps that consumed it
    }
    for (int s = 0; s < FT_AST; ++s) {
      mbar_init(a_full(s), 8 / GROUPS);
      mbar_init(a_empty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(d_full(b), 1);
      mbar_init(d_empty(b), 128);
      mbar_init(rows_full(b), 8);    // the 8 converter warps
      mbar_init(rows_empty(b), 128); // the 128 epilogue threads
    }
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
      const uint32_t ubytes = static_cast<uint32_t>(P.np) * 128u;
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t it = 0; it < n_it; ++it) {
        const int32_t kb = static_cast<int32_t>(it % P.num_kb);
        mbar_wait(u_empty(stage), phase ^ 1);
        mbar_arrive_expect_tx(u_full(stage), ubytes);
        tma_load_3d(sbase + stage * U_BYTES, &tmU, u_full(stage), kb * FT_BK, P.j_off, P.plane);
        if (++stage == FT_US) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      // A = u8 limbs, B = U^T digits (s8, or u8 in the unsigned-plane mode), D = s32
      const uint32_t idesc = idesc_i8(128, static_cast<uint32_t>(P.np), /*a_signed=*/false, /*b_signed=*/!P.u_unsigned);
      int us = 0, as = 0, acc = 0;
      uint32_t uph = 0, aph = 0, acc_phase = 0;
      for (int32_t t = 0; t < my_tiles; ++t) {
        mbar_wait(d_empty(acc), acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * D_COLS;
        for (int32_t kb = 0; kb < P.num_kb; ++kb) {
          mbar_wait(u_full(us), uph);
          const uint32_t su = sbase + us * U_BYTES;
#pragma unroll
          for (int hh = 0; hh < HPK; ++hh) {
            mbar_wait(a_full(as), aph);
            tc_fence_after();
#pragma unroll
            for (int k2 = 0; k2 < AW / 8; ++k2) {  // MMA K = 32 residues = 8 columns
              const int kk = hh * (AW / 8) + k2;
              const uint64_t bd = umma_desc_sw128(su + kk * FT_MMA_K);
#pragma unroll
              for (int sb = 0; sb < SUB; ++sb)  // the sub-tiles share the U^T stage
                mma_i8_ts(d_tmem + sb * NPMAX, tmem_base + A_COL0 + as * ASTAGE_COLS + sb * AW + k2 * (FT_MMA_K / 4), bd,
                          idesc, (kb | kk) != 0);
            }
            mma_commit(a_empty(as));  // the limb stage is free once these MMAs are done
            if (++as == FT_AST) { as = 0; aph ^= 1; }
          }
          mma_commit(u_empty(us));  // and the U^T stage once the whole K-block's are
          if (++us == FT_US) { us = 0; uph ^= 1; }
        }
        mma_commit(d_full(acc));
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
        const uint32_t dst = raw_base + rs * RAW_BYTES;
#pragma unroll
        for (int sb = 0; sb < SUB; ++sb)
#pragma unroll
          for (int b = 0; b < 4; ++b)  // box (sub-tile sb, residues 32b..): 32 rows × 128 B, SWIZZLE_128B
            tma_load_2d(dst + (sb * 4 + b) * FT_BOX_BYTES, &tmX, raw_full(rs), kb * FT_BK + 32 * b,
                        tr * ROWS + sb * FT_SUB_ROWS);
        if (++rs == RAW) { rs = 0; rphase ^= 1; }
      }
    }
  } else if (warp >= 4 && warp < 8) {  // (warp 2, the TMEM allocator, idles until the dealloc)
    // ---------------------------------------------------------------- epilogue (warps 4–7)
    // Quadrant q's lanes: 16h + 8ℓ' + r = limb 2h + ℓ' of tile row 8q + r.  Two .16x256b loads
    // (lane blocks h = 0, 1) give thread t = 4r + c all four limb sums of row 8q + r for the
    // columns 8k + 2c + {0, 1} of the 32-column chunk: the recombination is thread-local.
    const int q = warp & 3;
    const int r = lane >> 2, c = lane & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    const int nchunk = (P.np + 31) / 32;
    for (int32_t t = 0; t < my_tiles; ++t) {
      const int64_t tr = static_cast<int64_t>(blockIdx.x) + static_cast<int64_t>(t) * gridDim.x;
      // unsigned-U plane: X·U = X·U' − u_offset·Σ_k X[r][k]; this thread's rows' corrections
      uint32_t corr[SUB];
      if (P.off_mod) {
        mbar_wait(rows_full(t & 1), static_cast<uint32_t>((t >> 1) & 1));
#pragma unroll
        for (int sb = 0; sb < SUB; ++sb) {
          uint64_t sum = 0;
#pragma unroll
          for (int g = 0; g < GROUPS; ++g) sum += rsum[(((t & 1) * SUB + sb) * GROUPS + g) * 32 + 8 * q + r];
          corr[sb] = static_cast<uint32_t>(static_cast<uint64_t>(barrett64(sum, P.m)) * P.off_mod % P.m.p);
        }
        mbar_arrive(rows_empty(t & 1));
      }
      mbar_wait(d_full(acc), acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int chunk = 0; chunk < SUB * nchunk; ++chunk) {
        const int sb = chunk / nchunk, c0 = 32 * (chunk % nchunk);
        const int64_t row = tr * ROWS + sb * FT_SUB_ROWS + 8 * q + r;
        const uint32_t t_col = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * D_COLS + sb * NPMAX + c0;
        uint32_t lo[16], hi[16];  // limbs 0, 1 and limbs 2, 3
        tmem_ld16x256_x4(t_col, lo);
        tmem_ld16x256_x4(t_col + (16u << 16), hi);
        tmem_ld_wait();
        if (chunk + 1 == SUB * nchunk) {  // every column read: hand D back before the last stores
          tc_fence_before();
          mbar_arrive(d_empty(acc));
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            uint32_t res = recombine_mod(static_cast<int32_t>(lo[4 * k + e]), static_cast<int32_t>(lo[4 * k + 2 + e]),
                                         static_cast<int32_t>(hi[4 * k + e]), static_cast<int32_t>(hi[4 * k + 2 + e]), P.m);
            if (P.off_mod) res = sub_mod(res, sb == 0 ? corr[0] : corr[SUB - 1], P.m.p);
            const int64_t j = static_cast<int64_t>(c0) + 8 * k + 2 * c + e;
            if (j < P.o.d3_loc && row < P.o.R) store_out(P.o, P.m, j, row, res);  // (+ the Rescale epilogue)
          }
      }
      if (++acc == NBUF) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp >= 8) {
    // ---------------------------------------------------------------- converters (warps 8–15)
    // TMEM quadrant q (warp % 4 == q, as tcgen05.st requires) holds tile rows 8q .. 8q + 7: lane
    // 16h + 8ℓ' + r = limb 2h + ℓ' of row 8q + r.  Thread t = 4r + c loads residues 32k + 8c .. +7
    // of row 8q + r (two LDS.128 per repetition k; consecutive rows in an 8-lane phase differ in the
    // swizzle's bit 0, so the 8 lanes hit 8 distinct 16-B bank groups), byte-transposes them
    // (PRMT) into limb words and stores limbs 0–1 / 2–3 with two .16x256b.x4 STTMs whose fragment
    // pattern is exactly (lane r | r + 8, columns 8k + 2c | + 1): no cross-lane exchange.
    const int cw = warp - 8;
    // hi = the K-block parity (SUB = 1: two groups on alternate K-blocks) or the sub-tile (SUB = 2)
    const int q = cw & 3, hi = cw >> 2;
    const int grp = SUB == 1 ? hi : 0, sb = SUB == 1 ? 0 : hi;
    const int r = lane >> 2, c = lane & 3;
    const int row = 8 * q + r;            // row of the 32-row sub-tile
    const uint32_t t_lane = static_cast<uint32_t>(q * 32) << 16;
    // Global iterations it ≡ grp (mod GROUPS), walked tile by tile so that every tile's row-sum
    // partials are flushed — also by a group that has no K-block in the tile (num_kb = 1)
    for (int32_t t = 0; t < my_tiles; ++t) {
      const int64_t it0 = static_cast<int64_t>(t) * P.num_kb;
      uint32_t lsum[4] = {0u, 0u, 0u, 0u};  // Σ of each limb over this thread's residues of the tile
      for (int64_t it = it0 + ((grp - it0 % GROUPS) + GROUPS) % GROUPS; it < it0 + P.num_kb; it += GROUPS) {
        const int rs = static_cast<int>(it % RAW);
        mbar_wait(raw_full(rs), static_cast<uint32_t>((it / RAW) & 1));
        const uint32_t raw = raw_base + rs * RAW_BYTES + sb * 4 * FT_BOX_BYTES;
        uint32_t l01[16], l23[16];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            // residues 32k + 8c + 4e .. +3: box k, 16-B chunk 2c + e of row `row`
            const int cb = 2 * c + e;
            const uint32_t a = raw + k * FT_BOX_BYTES + row * 128 + ((cb ^ (row & 7)) << 4);
            CTPT_CHECK(a >= raw_base && a + 16 <= raw_base + RAW * RAW_BYTES);
            const uint4 x = lds128(a);
            uint32_t w0, w1, w2, w3;
            byte_transpose4(x.x, x.y, x.z, x.w, w0, w1, w2, w3);  // wm = limb m of the 4 residues
            l01[4 * k + e] = w0;
            l01[4 * k + 2 + e] = w1;
            l23[4 * k + e] = w2;
            l23[4 * k + 2 + e] = w3;
            if (P.off_mod) {  // byte sums of each limb (IDP4A): Σ_k x[k] = Σ_ℓ 2^{8ℓ} Σ_k x_ℓ[k]
              lsum[0] = __dp4a(w0, 0x01010101u, lsum[0]);
              lsum[1] = __dp4a(w1, 0x01010101u, lsum[1]);
              lsum[2] = __dp4a(w2, 0x01010101u, lsum[2]);
              lsum[3] = __dp4a(w3, 0x01010101u, lsum[3]);
            }
          }
        }
        if constexpr (HPK == 1) {
          const int as = static_cast<int>(it % FT_AST);
          mbar_wait(a_empty(as), static_cast<uint32_t>(((it / FT_AST) & 1) ^ 1));
          tc_fence_after();
          const uint32_t ta = tmem_base + t_lane + A_COL0 + as * ASTAGE_COLS + sb * 32;
          CTPT_CHECK(A_COL0 + as * ASTAGE_COLS + sb * 32 + 32 <= 512);
          tmem_st16x256_x4(ta, l01);
          tmem_st16x256_x4(ta + (16u << 16), l23);
          // The raw tile is handed back only here: the STTMs take every limb word as an operand, so
          // every LDS of the tile has completed (register computations such as the PRMTs may be
          // scheduled past a fence; an asm operand may not), then a proxy fence orders the generic
          // reads before the TMA's async-proxy refill.
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(raw_empty(rs));
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(a_full(as));
        } else {
          // half-K-block stages (AW = 16): repetitions 0–1 (residues 0..63) into stage n = 2·it,
          // 2–3 into stage 2·it + 1 — the .x2 fragment of each half is registers 0..7 / 8..15
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int64_t n = it * 2 + hh;
            const int as = static_cast<int>(n % FT_AST);
            mbar_wait(a_empty(as), static_cast<uint32_t>(((n / FT_AST) & 1) ^ 1));
            tc_fence_after();
            const uint32_t ta = tmem_base + t_lane + A_COL0 + as * ASTAGE_COLS + sb * AW;
            CTPT_CHECK(A_COL0 + as * ASTAGE_COLS + sb * AW + AW <= 512);
            uint32_t h01[8], h23[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              h01[i] = l01[8 * hh + i];
              h23[i] = l23[8 * hh + i];
            }
            tmem_st16x256_x2(ta, h01);
            tmem_st16x256_x2(ta + (16u << 16), h23);
            if (hh == 1) {  // every limb word of the K-block is an STTM operand by now: release the raw tile
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) mbar_arrive(raw_empty(rs));
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(a_full(as));
          }
        }
      }
      if (P.off_mod) {
        // this warp's partial row sums of tile t: Σ_ℓ 2^{8ℓ}·lsum_ℓ, summed over the 4 threads of a row
        uint64_t part = static_cast<uint64_t>(lsum[0]) + (static_cast<uint64_t>(lsum[1]) << 8) +
                        (static_cast<uint64_t>(lsum[2]) << 16) + (static_cast<uint64_t>(lsum[3]) << 24);
        part += __shfl_xor_sync(0xffffffffu, part, 1);
        part += __shfl_xor_sync(0xffffffffu, part, 2);
        mbar_wait(rows_empty(t & 1), static_cast<uint32_t>(((t >> 1) & 1) ^ 1));
        if (c == 0) rsum[(((t & 1) * SUB + sb) * GROUPS + grp) * 32 + row] = part;
        __syncwarp();
        if (lane == 0) mbar_arrive(rows_full(t & 1));
      }
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
