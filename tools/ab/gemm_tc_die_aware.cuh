// gemm_tc.cuh — the limb GEMM on the 5th-generation tensor cores (SURVEY.md §8(a) a4 + a5).
//
// Per prime p, with X = [A; B] ∈ Z_p^{R×d2} split into four u8 limb planes X_ℓ and U0's
// balanced s8 digit plane U (k_U = 1 per pass):
//     C_ℓ = X_ℓ · U   over Z (int32, exact: d2·255·128 < 2^31),
//     out = (C_0 + 2^8 C_1 + 2^16 C_2 + 2^24 C_3) mod p
//
// Mapping onto tcgen05.mma.cta_group::1.kind::i8 (D[M×N] += A[M×K]·B[N×K]^T, K-major both):
//   MMA "A" = U^T tile: 128 output columns j × K        (s8, TMEM lanes = j)
//   MMA "B" = 4 limb tiles stacked: (ℓ, r) = ℓ·64 + r, 256 × K   (u8)
//   D = 128 lanes × 256 int32 columns: lane j holds C_ℓ[r][j] at column ℓ·64 + r, so one
//   epilogue thread owns all four limb sums of its 64 outputs — recombination needs no
//   data exchange.  One MMA (M=128, N=256, K=32) per 32-byte K step.
// Tiles: 128 (j) × 64 (r) outputs, K-block 128 bytes, 4-stage TMA→SMEM ring (48 KB/stage),
// double-buffered TMEM accumulators (2 × 256 columns = all 512).
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM allocator, w4–7 epilogue.
// Persistent: grid = min(#tiles, #SMs); tiles visited in groups of GROUP_J j-tiles so the
// U panels of a group stay in L2 while the X panels stream.
#pragma once
#include <cstdint>

#include "kernels.cuh"
#include "ptx.cuh"

namespace ctpt {

constexpr int TC_BLOCK_J = 128;   // MMA M (output columns per tile)
constexpr int TC_BLOCK_R = 64;    // rows of X per tile (× 4 limbs = MMA N = 256)
constexpr int TC_BLOCK_K = 128;   // bytes of K per stage (one 128-B swizzle row)
constexpr int TC_STAGES = 4;
constexpr int TC_MMA_K = 32;      // K per kind::i8 MMA
constexpr int TC_U_BYTES = TC_BLOCK_J * TC_BLOCK_K;            // 16 KB
constexpr int TC_X_BYTES = 4 * TC_BLOCK_R * TC_BLOCK_K;        // 32 KB
constexpr int TC_STAGE_BYTES = TC_U_BYTES + TC_X_BYTES;        // 48 KB
constexpr int TC_ACC_COLS = 4 * TC_BLOCK_R;                    // 256
constexpr int TC_THREADS = 256;
// TMA-store epilogue: per epilogue warp two 4-KB staging halves ([32 columns j][32 rows r] uint32,
// SWIZZLE_128B), one TMA store per half
constexpr int TC_OUT_HALF_BYTES = 32 * 32 * 4;
constexpr int TC_OUT_BYTES = 4 * 2 * TC_OUT_HALF_BYTES;         // 32 KB
constexpr int TC_SMEM_BYTES = TC_STAGES * TC_STAGE_BYTES + TC_OUT_BYTES + 256 + 1024;
constexpr int TC_GROUP_J_DEFAULT = 16;  // measured best of {8,16,32,64,128} on c3 (profiles/r01)

// The limb split of the NEXT prime, run by the GEMM's two otherwise idle warps (2 and 3) while
// this prime's MMAs run (ctpt_problem.split_overlap): x = Σ_{ℓ<4} x_ℓ 2^{8ℓ} byte transpose as in
// k_split / k_split_rows (+ the unsigned-U row correction), streaming loads and stores
// (evict-first) so the GEMM's L2-resident operand panels stay put.
struct SplitJob {
  const uint4* x;      // next prime's X, [R][d2p] int32 as uint4 (nullptr: no side split)
  uint8_t* limbs;      // its byte limbs in 32-KB tiles (limb_tile_off, kernels.cuh)
  uint32_t* rowcorr;   // u_offset·Σ_k X[r][k] mod p per row (unsigned-U mode), or nullptr
  int64_t R, d2p16;    // rows; 16-residue groups per row of X
  int64_t nkb;         // 128-byte k-blocks per limb tile row (⌈d2p / 128⌉)
  uint32_t p, off_mod; // next prime; u_offset mod p
};

__device__ __forceinline__ void side_split_rows(const SplitJob& J, int64_t worker, int64_t nworkers, int lane) {
  const int64_t kp16 = J.nkb * 8;
  for (int64_t r = worker; r < J.R; r += nworkers) {
    uint64_t sum = 0;
    for (int64_t c = lane; c < kp16; c += 32) {
      uint4 w[4] = {};
      if (c < J.d2p16) {
#pragma unroll
        for (int i = 0; i < 4; ++i) w[i] = __ldcs(J.x + 4 * (r * J.d2p16 + c) + i);
      }
      uint32_t o[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        sum += static_cast<uint64_t>(w[i].x) + w[i].y + w[i].z + w[i].w;
        byte_transpose4(w[i].x, w[i].y, w[i].z, w[i].w, o[0][i], o[1][i], o[2][i], o[3][i]);
      }
      uint8_t* t = J.limbs + limb_tile_off(r, 16 * c, J.nkb);
#pragma unroll
      for (int l = 0; l < 4; ++l)
        __stcs(reinterpret_cast<uint4*>(t + l * 8192), make_uint4(o[l][0], o[l][1], o[l][2], o[l][3]));
    }
    if (J.rowcorr) {
#pragma unroll
      for (int s = 16; s; s >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, s);
      if (lane == 0) J.rowcorr[r] = static_cast<uint32_t>((sum % J.p) * J.off_mod % J.p);
    }
  }
}

struct TcParams {
  int64_t R, d2;
  int32_t j_off;      // first U column (col_begin)
  int32_t plane;      // U digit plane index (3rd TMA coordinate)
  int32_t num_kb;     // k-blocks of 128 B (ceil(d2 / 128))
  int32_t tiles_j, tiles_r;
  int32_t num_tiles;
  int32_t group_j;    // tiles visited in groups of group_j j-tiles (L2 reuse of U panels)
  int32_t u_unsigned; // U plane is u8 (U + u_offset) instead of balanced s8 digits
  int32_t serpentine; // odd waves (tile iteration (tile − blockIdx) / grid) walk K backwards, so the U^T
                      // panel lines a wave touched last are the next wave's first reads (L2 reuse when
                      // the group's U^T panel + a wave's X rows exceed L2, e.g. K = 32768)
  int32_t tma_store;  // epilogue stages each 32 × 32 output block in shared memory and writes it with
                      // one TMA store (tmAU / tmBU); needs rows_A and d1 multiples of 64 (a tile's 64
                      // rows lie inside A' or B') and device-local outputs; else 16-byte STG stores
  ModP m;
  OutParams o;
  SplitJob sj;        // the next prime's limb split (warps 2–3), or sj.x = nullptr
};

__device__ __forceinline__ void tc_tile_coords(int32_t tile, const TcParams& P, int32_t& tj, int32_t& tr) {
  const int32_t per_group = P.group_j * P.tiles_r;
  const int32_t g = tile / per_group;
  const int32_t rem = tile - g * per_group;
  const int32_t gj = min(P.group_j, P.tiles_j - g * P.group_j);
  tj = g * P.group_j + rem % gj;
  tr = rem / gj;
}

// ---- EXPERIMENT (tools/ab/gemm_tc_die_aware.cuh): die-aware raster -------------------------------
// The L2 is two per-die partitions and a line read from both dies is cached in both
// (tools/l2_probe): a U^T panel read by every SM costs twice its size.  Here each die's CTAs take
// their own part of a 32-j-tile super-group (widths ∝ the dies' SM counts), so a panel is read from
// one die only, and both dies walk the r-tiles at the same rate, so an X tile is fetched once for
// 32 j-tiles instead of 16.  The SM → die map is probed by L2 latency on the first launch (which
// runs the ordinary raster) and cached in device globals.  Assumes one CTA on every SM
// (grid = #SMs, idle GPU): a measurement build, not a product path.
__device__ int g_sm_die[256];          // 0 = unknown, 1 / 2 = die
__device__ unsigned g_probe_count;
__device__ volatile unsigned g_die_ready;
__device__ unsigned g_die_printed;

struct DieSched {
  int32_t on;      // die-aware schedule in use
  int32_t start, stride, total;  // this CTA's walk: T = start, start + stride, … < total
  int32_t g, joff; // this die's j-tiles per super-group and their offset inside it
};

__device__ __forceinline__ void sched_coords(int32_t T, const TcParams& P, const DieSched& S, int32_t& tj, int32_t& tr) {
  if (!S.on) {
    tc_tile_coords(T, P, tj, tr);
    return;
  }
  const int32_t per_sg = P.tiles_r * S.g;
  const int32_t sg = T / per_sg;
  const int32_t t = T - sg * per_sg;
  tr = t / S.g;
  tj = sg * 32 + S.joff + (t - tr * S.g);
}

__device__ __forceinline__ uint64_t die_timer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t smid_u32() {
  uint32_t v;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(v));
  return v;
}

// thread 0 of the CTA: probe (first launch) or read the cached map and build this CTA's schedule
__device__ void die_sched_setup(const TcParams& P, DieSched& S) {
  S.on = 0;
  S.start = static_cast<int32_t>(blockIdx.x);
  S.stride = static_cast<int32_t>(gridDim.x);
  S.total = P.num_tiles;
  S.g = 0;
  S.joff = 0;
  const uint32_t sm = smid_u32();
  if (sm >= 256) return;
  if (!g_die_ready) {
    if (g_sm_die[sm] != 0) return;  // (a second CTA on this SM)
    const uint64_t t0 = die_timer_ns();
    while (die_timer_ns() - t0 < static_cast<uint64_t>(blockIdx.x) * 10000ull) {}
    const char* base = reinterpret_cast<const char*>(P.o.BU);
    uint32_t lat[16];
    uint32_t sum = 0;
    for (int k = 0; k < 16; ++k) {
      const char* p = base + static_cast<size_t>(k) * 4096 * 5;  // distinct 2-KB hash grains
      uint32_t v = 0;
      for (int w = 0; w < 2; ++w) {
        // the next access depends on this one's result: bit 31 of an output residue (< p < 2^31) is 0 in
        // practice, which ptxas cannot know (it folded `and v, 0` and issued the atomics without waiting)
        const uint32_t z = (v >> 31) << 2;
        // an atomic is performed in the line's HOME partition (a plain load would hit the copy the
        // first read left in this die's partition: every SM measured the same latency that way)
        asm volatile("atom.global.add.u32 %0, [%1], 0;" : "=r"(v) : "l"(p + z) : "memory");
      }
      const long long c0 = clock64();
      for (int w = 0; w < 8; ++w) {
        // the next access depends on this one's result: bit 31 of an output residue (< p < 2^31) is 0 in
        // practice, which ptxas cannot know (it folded `and v, 0` and issued the atomics without waiting)
        const uint32_t z = (v >> 31) << 2;
        // an atomic is performed in the line's HOME partition (a plain load would hit the copy the
        // first read left in this die's partition: every SM measured the same latency that way)
        asm volatile("atom.global.add.u32 %0, [%1], 0;" : "=r"(v) : "l"(p + z) : "memory");
      }
      const long long c1 = clock64();
      lat[k] = static_cast<uint32_t>(c1 - c0) + (v >> 31);
      sum += lat[k];
    }
    g_sm_die[sm] = lat[0] * 16u > sum ? 2 : 1;
    if (blockIdx.x < 3 || blockIdx.x > gridDim.x - 3)
      printf("ctpt die probe: cta %d sm %u lat/8 = %u %u %u %u %u %u %u %u | %u %u %u %u %u %u %u %u\n", blockIdx.x, sm,
             lat[0] / 8, lat[1] / 8, lat[2] / 8, lat[3] / 8, lat[4] / 8, lat[5] / 8, lat[6] / 8, lat[7] / 8, lat[8] / 8,
             lat[9] / 8, lat[10] / 8, lat[11] / 8, lat[12] / 8, lat[13] / 8, lat[14] / 8, lat[15] / 8);
    __threadfence();
    // everyone waits for the end of the stagger window before the GEMM's traffic starts
    while (die_timer_ns() - t0 < static_cast<uint64_t>(gridDim.x + 4) * 10000ull) {}
    if (atomicAdd(&g_probe_count, 1u) == gridDim.x - 1) g_die_ready = 1;
    return;
  }
  const int d = g_sm_die[sm];
  if (d == 0 || (P.tiles_j % 32) != 0) return;
  int n[2] = {0, 0}, rank = 0;
  for (int i = 0; i < 256; ++i) {
    const int di = g_sm_die[i];
    if (di == 0) continue;
    ++n[di - 1];
    if (di == d && i < static_cast<int>(sm)) ++rank;
  }
  if (n[0] + n[1] != static_cast<int>(gridDim.x)) return;  // not one CTA per probed SM
  int g0 = (32 * n[0] + (n[0] + n[1]) / 2) / (n[0] + n[1]);
  if (n[0] > 0 && g0 == 0) g0 = 1;
  if (n[1] > 0 && g0 == 32) g0 = 31;
  S.on = 1;
  S.g = d == 1 ? g0 : 32 - g0;
  S.joff = d == 1 ? 0 : g0;
  S.start = rank;
  S.stride = n[d - 1];
  S.total = (P.tiles_j / 32) * P.tiles_r * S.g;
  if (blockIdx.x == 0 && atomicAdd(&g_die_printed, 1u) == 0)
    printf("ctpt die-aware raster: %d + %d SMs, j-tiles %d + %d per super-group\n", n[0], n[1], g0, 32 - g0);
}

__global__ void __launch_bounds__(TC_THREADS, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmX,
              const __grid_constant__ CUtensorMap tmAU, const __grid_constant__ CUtensorMap tmBU,
              const __grid_constant__ TcParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t out_base = sbase + TC_STAGES * TC_STAGE_BYTES;  // 1024-B aligned (SWIZZLE_128B atoms)
  const uint32_t bar_base = out_base + TC_OUT_BYTES;
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto empty_bar = [&](int s) { return bar_base + 8u * (TC_STAGES + s); };
  auto tfull_bar = [&](int b) { return bar_base + 8u * (2 * TC_STAGES + b); };
  auto tempty_bar = [&](int b) { return bar_base + 8u * (2 * TC_STAGES + 2 + b); };
  const uint32_t tmem_slot = bar_base + 8u * (2 * TC_STAGES + 4);
  uint32_t* tmem_slot_ptr =
      reinterpret_cast<uint32_t*>(smem + TC_STAGES * TC_STAGE_BYTES + TC_OUT_BYTES + 8 * (2 * TC_STAGES + 4));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmU);
    tma_prefetch(&tmX);
    if (P.tma_store) {
      tma_prefetch(&tmAU);
      tma_prefetch(&tmBU);
    }
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull_bar(b), 1);
      mbar_init(tempty_bar(b), 128);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  DieSched* sched_smem = reinterpret_cast<DieSched*>(smem + TC_STAGES * TC_STAGE_BYTES + TC_OUT_BYTES + 128);
  if (threadIdx.x == 96) {  // warp 3 (idle unless the side split runs)
    DieSched tmp;
    die_sched_setup(P, tmp);
    *sched_smem = tmp;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;
  const DieSched S = *sched_smem;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int32_t wave = 0;
      for (int32_t tile = S.start; tile < S.total; tile += S.stride, ++wave) {
        int32_t tj, tr;
        sched_coords(tile, P, S, tj, tr);
        const bool back = P.serpentine && (wave & 1);
        for (int32_t kb0 = 0; kb0 < P.num_kb; ++kb0) {
          // the MMA warp accumulates in stage order; integer sums do not depend on the K order
          const int32_t kb = back ? P.num_kb - 1 - kb0 : kb0;
          mbar_wait(empty_bar(stage), phase ^ 1);
          const uint32_t su = sbase + stage * TC_STAGE_BYTES;
          mbar_arrive_expect_tx(full_bar(stage), TC_STAGE_BYTES);
          tma_load_3d(su, &tmU, full_bar(stage), kb * TC_BLOCK_K, P.j_off + tj * TC_BLOCK_J, P.plane);
          tma_load_5d(su + TC_U_BYTES, &tmX, full_bar(stage), 0, 0, 0, kb, tr);  // one 32-KB limb tile
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
      for (int32_t tile = S.start; tile < S.total; tile += S.stride) {
        mbar_wait(tempty_bar(acc), acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * TC_ACC_COLS;
        for (int32_t kb = 0; kb < P.num_kb; ++kb) {
          mbar_wait(full_bar(stage), phase);
          tc_fence_after();
          const uint32_t su = sbase + stage * TC_STAGE_BYTES;
#pragma unroll
          for (int kk = 0; kk < TC_BLOCK_K / TC_MMA_K; ++kk) {
            const uint64_t ad = umma_desc_sw128(su + kk * TC_MMA_K);
            const uint64_t bd = umma_desc_sw128(su + TC_U_BYTES + kk * TC_MMA_K);
            mma_i8(d_tmem, ad, bd, idesc, (kb | kk) != 0);
          }
          mma_commit(empty_bar(stage));  // frees the SMEM stage once these MMAs have read it
          if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(tfull_bar(acc));  // accumulator ready for the epilogue
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp == 2 || warp == 3) {
    // ---------------------------------------------------------------- next prime's limb split
    if (P.sj.x) side_split_rows(P.sj, 2 * static_cast<int64_t>(blockIdx.x) + (warp - 2), 2 * static_cast<int64_t>(gridDim.x), lane);
  } else {
    // ---------------------------------------------------------------- epilogue (warps 4–7)
    const int quad = warp & 3;  // TMEM lanes [32·quad, 32·quad + 32)
    const uint32_t stg = out_base + quad * 2 * TC_OUT_HALF_BYTES;  // this warp's two staging halves
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int32_t tile = S.start; tile < S.total; tile += S.stride) {
      int32_t tj, tr;
      sched_coords(tile, P, S, tj, tr);
      mbar_wait(tfull_bar(acc), acc_phase);
      tc_fence_after();
      const int64_t j = static_cast<int64_t>(tj) * TC_BLOCK_J + quad * 32 + lane;
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * TC_ACC_COLS;
      const int64_t r_tile = static_cast<int64_t>(tr) * TC_BLOCK_R;
      // two halves of 32 rows: four 32-column TMEM loads (one per limb) each; the accumulator is
      // handed back to the MMA warp as soon as the last loads have landed, before the last stores
      // (c3 3.709 vs 3.694e14 against 16-column loads, profiles/r01/gemm_epilogue_ld32/)
#pragma unroll 1
      for (int h = 0; h < TC_BLOCK_R / 32; ++h) {
        uint32_t v0[32], v1[32], v2[32], v3[32];
        tmem_ld32(t_row + 0 * TC_BLOCK_R + h * 32, v0);
        tmem_ld32(t_row + 1 * TC_BLOCK_R + h * 32, v1);
        tmem_ld32(t_row + 2 * TC_BLOCK_R + h * 32, v2);
        tmem_ld32(t_row + 3 * TC_BLOCK_R + h * 32, v3);
        tmem_ld_wait();
        if (h == TC_BLOCK_R / 32 - 1) {
          tc_fence_before();
          mbar_arrive(tempty_bar(acc));
        }
        if (P.tma_store) {
          // the 32 × 32 block (columns j of this warp, rows r_tile + 32h ..) through shared memory:
          // lane = column j holds 32 consecutive rows = one 128-B row of the staging image, its 16-B
          // chunk c at position c ^ (j & 7) (SWIZZLE_128B; conflict-free STS.128)
          uint32_t res[32];
#pragma unroll
          for (int i = 0; i < 32; ++i)
            res[i] = recombine_mod(static_cast<int32_t>(v0[i]), static_cast<int32_t>(v1[i]),
                                   static_cast<int32_t>(v2[i]), static_cast<int32_t>(v3[i]), P.m);
          const int64_t r0 = r_tile + h * 32;
          finish_rows<32>(P.o, P.m, j, r0, res, j < P.o.d3_loc);
          const uint32_t buf = stg + h * TC_OUT_HALF_BYTES;
          CTPT_CHECK(buf >= out_base && buf + TC_OUT_HALF_BYTES <= out_base + TC_OUT_BYTES);
          CTPT_CHECK(r0 + 32 <= (r0 < P.o.rows_A ? P.o.rows_A : P.o.rows_A + P.o.d1));  // inside A' or B
          if (lane == 0) bulk_wait_read<1>();  // this half's previous store has read its buffer
          __syncwarp();
#pragma unroll
          for (int c = 0; c < 8; ++c)
            sts128(buf + lane * 128 + ((c ^ (lane & 7)) << 4), res[4 * c], res[4 * c + 1], res[4 * c + 2],
                   res[4 * c + 3]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const int32_t jc = static_cast<int32_t>(tj) * TC_BLOCK_J + quad * 32;
            if (r0 < P.o.rows_A)
              tma_store_2d(&tmAU, buf, static_cast<int32_t>(r0), jc);
            else
              tma_store_2d(&tmBU, buf, static_cast<int32_t>(r0 - P.o.rows_A), jc);
            bulk_commit();
          }
          continue;
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          uint32_t res[16];
#pragma unroll
          for (int i = 0; i < 16; ++i)
            res[i] = recombine_mod(static_cast<int32_t>(v0[q * 16 + i]), static_cast<int32_t>(v1[q * 16 + i]),
                                   static_cast<int32_t>(v2[q * 16 + i]), static_cast<int32_t>(v3[q * 16 + i]), P.m);
          if (j < P.o.d3_loc) store16(P.o, P.m, j, r_tile + h * 32 + q * 16, res);
        }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (P.tma_store && lane == 0) bulk_wait<0>();  // every store performed before the CTA exits
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

}  // namespace ctpt
