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
