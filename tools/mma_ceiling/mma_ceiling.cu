// mma_ceiling.cu — the measured INT8 roofline for k_gemm_tc (a probe, not part of the product
// library): how many tcgen05.mma.cta_group::1.kind::i8 (M = 128, N = 256, K = 32) a B200 sustains
// when NOTHING but the MMA runs — operands resident in shared memory, no TMA, no epilogue, no
// DRAM — with operand bytes of a chosen distribution.  Under the 1000 W cap the rate depends on
// the operand bits, so the probe fills the A tile (k_gemm_tc's U^T side) and the
// B tile (its X-limb side) with the same statistics as the real GEMM: A = U + 8 ∈ [0, 16] (u8
// plane), B = uniform bytes.  k_gemm_tc's achieved TOP/s ÷ this rate is the fraction of the
// tensor pipe's power-limited ceiling it reaches.
//
// extern "C" int mma_ceiling_run(int blocks, long long iters, int a_max, int b_max, unsigned seed,
//                                float* ms_out, void* stream);
//   a_max / b_max: operand bytes uniform in [0, a_max] / [0, b_max] (0 = all zero).
//   Each CTA issues `iters` K-blocks of 4 MMAs (K = 128) into two alternating TMEM accumulators.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../paper_2503_16080_b200/csrc/ptx.cuh"

using namespace ctpt;

namespace {

constexpr int kA = 128 * 128;  // A tile: 128 rows × 128 K bytes (SWIZZLE_128B K-major image)
constexpr int kB = 256 * 128;  // B tile: 256 rows × 128 K bytes

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__global__ void __launch_bounds__(128, 1) k_mma_ceiling(long long iters, int a_max, int b_max, unsigned seed) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar = sbase + kA + kB;
  const uint32_t tmem_slot = bar + 8;
  uint32_t* tmem_slot_ptr = reinterpret_cast<uint32_t*>(smem + kA + kB + 8);
  // operands: bytes uniform in [0, max] (the swizzle permutes bytes within a row, so any
  // i.i.d. fill is a valid operand image with the same statistics)
  for (int i = threadIdx.x; i < (kA + kB) / 4; i += blockDim.x) {
    const int lim = (4 * i < kA) ? a_max : b_max;
    uint32_t w = 0;
    for (int b = 0; b < 4; ++b) {
      const uint32_t h = hash32(seed ^ (blockIdx.x * 0x9E3779B9u) ^ static_cast<uint32_t>(4 * i + b) * 0x85EBCA6Bu);
      w |= (lim > 0 ? (h % static_cast<uint32_t>(lim + 1)) : 0u) << (8 * b);
    }
    reinterpret_cast<uint32_t*>(smem)[i] = w;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_i8(128, 256, /*a_signed=*/false, /*b_signed=*/false);
    for (long long it = 0; it < iters; ++it) {
      const uint32_t d = tmem_base + static_cast<uint32_t>(it & 1) * 256;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_i8(d, umma_desc_sw128(sbase + kk * 32), umma_desc_sw128(sbase + kA + kk * 32), idesc, (it >= 2) || kk);
    }
    mma_commit(bar);
    mbar_wait(bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

// A-operand reuse probe: per K slice two MMAs share A (M = 128) against two different B tiles
// (N = 256 each) into two accumulators; with `reuse` the first is issued with
// .collector::a::fill and the second with .collector::a::lastuse, so the second MMA need not
// read A from shared memory again.  Same MACs and operand statistics either way.
__device__ __forceinline__ void mma_i8_col(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc, int mode) {
  if (mode == 1)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8.collector::a::fill [%0], %1, %2, %3, p;\n}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else if (mode == 2)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8.collector::a::lastuse [%0], %1, %2, %3, p;\n}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else
    mma_i8(d, a, b, idesc, acc);
}

__global__ void __launch_bounds__(128, 1) k_mma_reuse(long long iters, int a_max, int b_max, unsigned seed, int reuse) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar = sbase + kA + 2 * kB;
  const uint32_t tmem_slot = bar + 8;
  uint32_t* tmem_slot_ptr = reinterpret_cast<uint32_t*>(smem + kA + 2 * kB + 8);
  for (int i = threadIdx.x; i < (kA + 2 * kB) / 4; i += blockDim.x) {
    const int lim = (4 * i < kA) ? a_max : b_max;
    uint32_t w = 0;
    for (int b = 0; b < 4; ++b) {
      const uint32_t h = hash32(seed ^ (blockIdx.x * 0x9E3779B9u) ^ static_cast<uint32_t>(4 * i + b) * 0x85EBCA6Bu);
      w |= (lim > 0 ? (h % static_cast<uint32_t>(lim + 1)) : 0u) << (8 * b);
    }
    reinterpret_cast<uint32_t*>(smem)[i] = w;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_i8(128, 256, false, false);
    for (long long it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t a = umma_desc_sw128(sbase + kk * 32);
        const uint32_t acc = (it >= 1) || kk;
        mma_i8_col(tmem_base, a, umma_desc_sw128(sbase + kA + kk * 32), idesc, acc, reuse ? 1 : 0);
        mma_i8_col(tmem_base + 256, a, umma_desc_sw128(sbase + kA + kB + kk * 32), idesc, acc, reuse ? 2 : 0);
      }
    }
    mma_commit(bar);
    mbar_wait(bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

}  // namespace

extern "C" int mma_reuse_run(int blocks, long long iters, int a_max, int b_max, unsigned seed, int reuse, float* ms_out,
                             void* stream) {
  const int smem = kA + 2 * kB + 64 + 1024;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaFuncSetAttribute(k_mma_reuse, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  k_mma_reuse<<<blocks, 128, smem, st>>>(iters, a_max, b_max, seed, reuse);
  cudaEventRecord(e1, st);
  if (cudaGetLastError() != cudaSuccess) return 2;
  if (cudaEventSynchronize(e1) != cudaSuccess) return 3;
  cudaEventElapsedTime(ms_out, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return 0;
}

namespace {
}  // namespace

extern "C" int mma_ceiling_run(int blocks, long long iters, int a_max, int b_max, unsigned seed, float* ms_out,
                               void* stream) {
  const int smem = kA + kB + 64 + 1024;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaFuncSetAttribute(k_mma_ceiling, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  k_mma_ceiling<<<blocks, 128, smem, st>>>(iters, a_max, b_max, seed);
  cudaEventRecord(e1, st);
  if (cudaGetLastError() != cudaSuccess) return 2;
  if (cudaEventSynchronize(e1) != cudaSuccess) return 3;
  cudaEventElapsedTime(ms_out, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return 0;
}

// ---------------------------------------------------------------------------------------------
// Main-loop probe: k_gemm_tc's TMA → SMEM ring → tcgen05.mma pipeline WITHOUT its epilogue
// (accumulators are never read), to split the gap between the pure-MMA ceiling above and the
// real GEMM into data movement and epilogue.  mode 0: the real (tile, k-block) coordinates over
// the caller's U^T plane and X limbs (DRAM + L2 traffic as in the GEMM); mode 1: every load
// re-reads the SAME (tile 0, k-block 0) operands (L2-resident: L2 → SMEM traffic, no DRAM).
// Same tile order, raster group and ring as gemm_tc.cuh.
// ---------------------------------------------------------------------------------------------
namespace {

__device__ __forceinline__ void tma_load_5d(uint32_t dst, const CUtensorMap* m, uint32_t bar, int32_t c0, int32_t c1,
                                            int32_t c2, int32_t c3, int32_t c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
      : "memory");
}

constexpr int PB_BLOCK_J = 128, PB_BLOCK_R = 64, PB_BLOCK_K = 128, PB_STAGES = 4;
constexpr int PB_U = PB_BLOCK_J * PB_BLOCK_K, PB_X = 4 * PB_BLOCK_R * PB_BLOCK_K, PB_STAGE = PB_U + PB_X;

struct ProbeParams {
  int32_t num_kb, tiles_j, tiles_r, num_tiles, group_j, mode;
};

__global__ void __launch_bounds__(256, 1) k_mainloop_probe(const __grid_constant__ CUtensorMap tmU,
                                                           const __grid_constant__ CUtensorMap tmX,
                                                           const __grid_constant__ ProbeParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_base = sbase + PB_STAGES * PB_STAGE;
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto empty_bar = [&](int s) { return bar_base + 8u * (PB_STAGES + s); };
  auto tfull_bar = [&](int b) { return bar_base + 8u * (2 * PB_STAGES + b); };
  auto tempty_bar = [&](int b) { return bar_base + 8u * (2 * PB_STAGES + 2 + b); };
  const uint32_t tmem_slot = bar_base + 8u * (2 * PB_STAGES + 4);
  uint32_t* tmem_slot_ptr = reinterpret_cast<uint32_t*>(smem + PB_STAGES * PB_STAGE + 8 * (2 * PB_STAGES + 4));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < PB_STAGES; ++s) {
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
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;
  auto coords = [&](int32_t tile, int32_t& tj, int32_t& tr) {
    const int32_t per_group = P.group_j * P.tiles_r;
    const int32_t g = tile / per_group, rem = tile - g * per_group;
    const int32_t gj = min(P.group_j, P.tiles_j - g * P.group_j);
    tj = g * P.group_j + rem % gj;
    tr = rem / gj;
  };
  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int32_t tile = blockIdx.x; tile < P.num_tiles; tile += gridDim.x) {
        int32_t tj, tr;
        coords(tile, tj, tr);
        if (P.mode & 1) tj = tr = 0;
        for (int32_t kb = 0; kb < P.num_kb; ++kb) {
          mbar_wait(empty_bar(stage), phase ^ 1);
          const uint32_t su = sbase + stage * PB_STAGE;
          const int32_t k = (P.mode & 1) ? 0 : kb;
          mbar_arrive_expect_tx(full_bar(stage), PB_STAGE);
          if (P.mode & 4)
            tma_load_5d(su, &tmU, full_bar(stage), 0, 0, 0, k, tj);
          else
            tma_load_3d(su, &tmU, full_bar(stage), k * PB_BLOCK_K, tj * PB_BLOCK_J, 0);
          if (P.mode & 2)
            tma_load_5d(su + PB_U, &tmX, full_bar(stage), 0, 0, 0, k, tr);
          else
            tma_load_3d(su + PB_U, &tmX, full_bar(stage), k * PB_BLOCK_K, tr * PB_BLOCK_R, 0);
          if (++stage == PB_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_i8(128, 256, false, false);
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int32_t tile = blockIdx.x; tile < P.num_tiles; tile += gridDim.x) {
        mbar_wait(tempty_bar(acc), acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * 256;
        for (int32_t kb = 0; kb < P.num_kb; ++kb) {
          mbar_wait(full_bar(stage), phase);
          tc_fence_after();
          const uint32_t su = sbase + stage * PB_STAGE;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_i8(d, umma_desc_sw128(su + kk * 32), umma_desc_sw128(su + PB_U + kk * 32), idesc, (kb | kk) != 0);
          mma_commit(empty_bar(stage));
          if (++stage == PB_STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(tfull_bar(acc));
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int32_t tile = blockIdx.x; tile < P.num_tiles; tile += gridDim.x) {  // no epilogue: hand back
      mbar_wait(tfull_bar(acc), acc_phase);
      tc_fence_after();
      tc_fence_before();
      mbar_arrive(tempty_bar(acc));
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int tmap3(EncodeFn enc, CUtensorMap* m, void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0, uint32_t b1,
          uint32_t b2) {
  cuuint64_t dims[3] = {d0, d1, d2}, strides[2] = {d0, d0 * d1};
  cuuint32_t box[3] = {b0, b1, b2}, es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
                 CUDA_SUCCESS
             ? 0
             : 1;
}

}  // namespace

// u_plane: [d3][K] u8 (U^T), limbs: [4][R][K] u8, K a multiple of 128.  Runs `launches` launches
// back to back; *ms_out = mean ms per launch.
extern "C" int mainloop_probe_run(const void* u_plane, const void* limbs, long long R, long long K, long long d3,
                                  int group_j, int mode, int launches, float* ms_out, void* stream) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return 1;
  EncodeFn enc = reinterpret_cast<EncodeFn>(fn);
  CUtensorMap tmU, tmX;
  if (mode & 4) {  // U^T viewed as tiles [d3/128][K/128][1][128 j][128 B], 16 KB each
    cuuint64_t dims[5] = {128, 128, 1, static_cast<cuuint64_t>(K / 128), static_cast<cuuint64_t>(d3 / 128)};
    cuuint64_t strides[4] = {128, 128 * 128, 128 * 128, static_cast<cuuint64_t>(K / 128) * 128 * 128};
    cuuint32_t box[5] = {128, 128, 1, 1, 1}, es[5] = {1, 1, 1, 1, 1};
    if (enc(&tmU, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, const_cast<void*>(u_plane), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return 2;
  } else if (tmap3(enc, &tmU, const_cast<void*>(u_plane), K, d3, 1, PB_BLOCK_K, PB_BLOCK_J, 1)) {
    return 2;
  }
  if (mode & 2) {  // the same bytes viewed as tiles [R/64][K/128][4 limbs][64 rows][128 B], 32 KB each
    cuuint64_t dims[5] = {128, 64, 4, static_cast<cuuint64_t>(K / 128), static_cast<cuuint64_t>(R / 64)};
    cuuint64_t strides[4] = {128, 64 * 128, 4 * 64 * 128, static_cast<cuuint64_t>(K / 128) * 4 * 64 * 128};
    cuuint32_t box[5] = {128, 64, 4, 1, 1}, es[5] = {1, 1, 1, 1, 1};
    if (enc(&tmX, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, const_cast<void*>(limbs), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return 3;
  } else if (tmap3(enc, &tmX, const_cast<void*>(limbs), K, R, 4, PB_BLOCK_K, PB_BLOCK_R, 4)) {
    return 3;
  }
  ProbeParams P;
  P.num_kb = static_cast<int32_t>(K / PB_BLOCK_K);
  P.tiles_j = static_cast<int32_t>((d3 + PB_BLOCK_J - 1) / PB_BLOCK_J);
  P.tiles_r = static_cast<int32_t>((R + PB_BLOCK_R - 1) / PB_BLOCK_R);
  P.num_tiles = P.tiles_j * P.tiles_r;
  P.group_j = group_j;
  P.mode = mode;
  const int smem = PB_STAGES * PB_STAGE + 256 + 1024;
  if (cudaFuncSetAttribute(k_mainloop_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return 4;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  for (int i = 0; i < launches; ++i)
    k_mainloop_probe<<<sms < P.num_tiles ? sms : P.num_tiles, 256, smem, st>>>(tmU, tmX, P);
  cudaEventRecord(e1, st);
  if (cudaGetLastError() != cudaSuccess) return 5;
  if (cudaEventSynchronize(e1) != cudaSuccess) return 6;
  cudaEventElapsedTime(ms_out, e0, e1);
  *ms_out /= launches;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return 0;
}
