// l2_probe.cu — how much data SHARED BY ALL SMs does the B200's L2 hold?
//
// k_gemm_tc keeps a U^T panel of G·128·d2 bytes resident in L2 while X streams; G = 16 (33.5 MB on
// c3) is the measured optimum and G = 32 (67 MB + a 19-MB X stream) thrashes, although the L2 is
// 126 MB.  Hypothesis: the L2 is two per-die partitions and a line read by SMs of both dies ends up
// in both, so data shared by every SM has about half the capacity.  Probe: every CTA (one per SM)
// reads the WHOLE buffer of S bytes, repeatedly, each CTA starting at its own offset (so the CTAs do
// not walk in lockstep and the working set is all S bytes at any moment); aggregate bandwidth vs S
// shows where the buffer stops fitting.  Second mode: each CTA reads only its own 1/148 slice
// (data private to one SM): the capacity for unshared data.  Third mode: CTAs read the half of the
// buffer selected by (smid parity is NOT the die) — not attempted: the SM→die map is per-GPU.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_probe l2_probe.cu && ./l2_probe
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(1024, 1) k_read(const uint4* __restrict__ buf, size_t n16, int iters, int shared_mode,
                                                   unsigned long long* sink) {
  // shared_mode 1: every CTA reads all n16 vectors, starting at blockIdx·n16/grid
  // shared_mode 0: CTA b reads only its slice [b·n16/grid, (b+1)·n16/grid)
  const size_t per = n16 / gridDim.x;
  const size_t start = static_cast<size_t>(blockIdx.x) * per;
  const size_t len = shared_mode ? n16 : per;
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
    for (size_t i = threadIdx.x; i < len; i += blockDim.x) {
      size_t j = start + i;
      if (j >= n16) j -= n16;
      uint4 v;
      asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(buf + j));
      acc += v.x ^ v.w;
    }
  }
  if (acc == 0x1234567887654321ull) *sink = acc;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  const size_t maxb = 320ull << 20;
  uint4* buf;
  unsigned long long* sink;
  cudaMalloc(&buf, maxb);
  cudaMalloc(&sink, 8);
  cudaMemset(buf, 1, maxb);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int sizes_mb[] = {8, 16, 24, 32, 40, 48, 56, 64, 72, 80, 96, 112, 128, 160, 192, 256};
  for (int mode = 1; mode >= 0; --mode) {
    for (int mb : sizes_mb) {
      const size_t bytes = static_cast<size_t>(mb) << 20;
      const size_t n16 = bytes / 16 / sms * sms;
      // shared: each CTA reads `bytes` per iteration; private: bytes / sms
      const double per_iter = mode ? static_cast<double>(n16) * 16 * sms : static_cast<double>(n16) * 16;
      int iters = static_cast<int>(4e11 / per_iter);  // ≈ 0.4 TB of loads per case
      if (iters < 4) iters = 4;
      if (iters > 4000) iters = 4000;
      k_read<<<sms, 1024>>>(buf, n16, 2, mode, sink);  // warm the cache
      cudaEventRecord(e0);
      k_read<<<sms, 1024>>>(buf, n16, iters, mode, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaError_t err = cudaGetLastError();
      if (err != cudaSuccess) {
        printf("{\"error\": \"%s\"}\n", cudaGetErrorString(err));
        return 1;
      }
      printf("{\"mode\": \"%s\", \"buffer_mb\": %d, \"iters\": %d, \"ms\": %.3f, \"load_gbs\": %.1f}\n",
             mode ? "every CTA reads the whole buffer" : "each CTA reads its own 1/148 slice", mb, iters, ms,
             per_iter * iters / (ms / 1e3) / 1e9);
      fflush(stdout);
    }
  }
  return 0;
}
