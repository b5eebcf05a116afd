/* ctpt_client.c — a plain C client of the C ABI (include/ctpt.h): no torch, no Python.
 *
 * Shows the boundary is usable on its own: the caller owns every device buffer (cudaMalloc),
 * passes plain pointers and a stream, and reads the status / ctpt_last_error() of each call.
 *
 *   ctpt_client sizes                    host-only checks (no GPU): ctpt_query_sizes on the
 *                                        BASELINE configs and every documented refusal
 *   ctpt_client run <in.bin> <out.bin>   layout → plain precompute → ctpt_matmul on the GPU
 *
 * in.bin (little-endian): int32 fmt, L; int64 N, d1, d2, d3; uint32 primes[L];
 *   uint32 a_polys[L][n_a][N] (n_a = d2·k for shared-s, d2 otherwise, 0 for structured-A);
 *   uint32 b_polys[L][d2·k][N]; int64 U[d2][d3].
 * out.bin: uint32 AU[L][d3][rows_A], uint32 BU[L][d3][d1].
 * Exit code 0 on success, 1 on a usage / IO error, 2 on a non-OK library status. */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ctpt.h"

#define CK(call)                                                                                 \
  do {                                                                                           \
    ctpt_status s_ = (call);                                                                     \
    if (s_ != CTPT_OK) {                                                                         \
      fprintf(stderr, "%s:%d %s -> status %d: %s\n", __FILE__, __LINE__, #call, (int)s_,         \
              ctpt_last_error());                                                                \
      return 2;                                                                                  \
    }                                                                                            \
  } while (0)
#define CU(call)                                                                                 \
  do {                                                                                           \
    cudaError_t e_ = (call);                                                                     \
    if (e_ != cudaSuccess) {                                                                     \
      fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #call, cudaGetErrorString(e_));    \
      return 2;                                                                                  \
    }                                                                                            \
  } while (0)

static int expect(const char* what, ctpt_status got, ctpt_status want) {
  printf("%-48s status %d (want %d)%s\n", what, (int)got, (int)want, got == want ? "" : "  MISMATCH");
  return got == want ? 0 : 1;
}

static int cmd_sizes(void) {
  static const uint32_t P3[3] = {2147352577u, 2146959361u, 2146041857u}; /* ctgen.primes(3) */
  ctpt_problem pb;
  ctpt_sizes sz;
  int bad = 0;
  printf("%s\n", ctpt_version());
  /* c3: shared-a, N = 4096, d1 = d2 = d3 = 16384, L = 3 */
  memset(&pb, 0, sizeof(pb));
  pb.fmt = CTPT_SHARED_A;
  pb.L = 3;
  pb.N = 4096;
  pb.d1 = pb.d2 = pb.d3 = 16384;
  pb.primes = P3;
  pb.kU = 1;
  bad |= expect("c3 query_sizes", ctpt_query_sizes(&pb, &sz), CTPT_OK);
  printf("c3: R=%lld d2p=%lld ctmat=%zu plain=%zu ws=%zu outAU=%zu outBU=%zu\n", (long long)sz.R,
         (long long)sz.d2p, sz.ctmat_bytes, sz.plain_bytes, sz.workspace_bytes, sz.out_AU_bytes, sz.out_BU_bytes);
  if (sz.R != 20480 || sz.d2p != 16384 || sz.ctmat_bytes != 256 + (size_t)3 * 20480 * 16384 * 4 ||
      sz.out_AU_bytes != (size_t)3 * 16384 * 4096 * 4 || sz.out_BU_bytes != (size_t)3 * 16384 * 16384 * 4) {
    printf("c3 sizes MISMATCH\n");
    bad = 1;
  }
  /* refusals (include/ctpt.h) */
  ctpt_problem q = pb;
  q.fmt = CTPT_RLWE;
  bad |= expect("RLWE with d1 != N", ctpt_query_sizes(&q, &sz), CTPT_ERR_SHAPE);
  q = pb;
  q.N = 3000;
  bad |= expect("N not a power of two", ctpt_query_sizes(&q, &sz), CTPT_ERR_SHAPE);
  q = pb;
  q.d1 = 4096 * 4 + 1;
  bad |= expect("N does not divide d1", ctpt_query_sizes(&q, &sz), CTPT_ERR_SHAPE);
  static const uint32_t PC[1] = {2147352575u}; /* odd, composite */
  q = pb;
  q.L = 1;
  q.primes = PC;
  bad |= expect("composite modulus", ctpt_query_sizes(&q, &sz), CTPT_ERR_MODULUS);
  static const uint32_t PR[2] = {2147352577u, 2147352577u};
  q = pb;
  q.L = 2;
  q.primes = PR;
  bad |= expect("repeated prime", ctpt_query_sizes(&q, &sz), CTPT_ERR_MODULUS);
  q = pb;
  q.d2 = 65794;
  bad |= expect("d2 beyond the int32 exactness bound", ctpt_query_sizes(&q, &sz), CTPT_ERR_OVERFLOW);
  q = pb;
  q.u_unsigned = 1;
  q.d2 = 33026;
  bad |= expect("d2 beyond the u8 x u8 bound", ctpt_query_sizes(&q, &sz), CTPT_ERR_OVERFLOW);
  q = pb;
  q.col_begin = 10;
  q.col_end = 5;
  bad |= expect("empty column shard", ctpt_query_sizes(&q, &sz), CTPT_ERR_SHAPE);
  q = pb;
  q.fmt = 7;
  bad |= expect("unknown format", ctpt_query_sizes(&q, &sz), CTPT_ERR_UNSUPPORTED);
  bad |= expect("NULL problem", ctpt_query_sizes(NULL, &sz), CTPT_ERR_ARG);
  printf("%s\n", bad ? "FAILED" : "all refusals as documented");
  return bad;
}

static int read_all(FILE* f, void* p, size_t n) { return fread(p, 1, n, f) == n ? 0 : 1; }

static int cmd_run(const char* in_path, const char* out_path) {
  FILE* f = fopen(in_path, "rb");
  if (!f) return 1;
  int32_t hdr32[2];
  int64_t hdr64[4];
  if (read_all(f, hdr32, sizeof hdr32) || read_all(f, hdr64, sizeof hdr64)) return 1;
  ctpt_problem pb;
  memset(&pb, 0, sizeof(pb));
  pb.fmt = hdr32[0];
  pb.L = hdr32[1];
  pb.N = hdr64[0];
  pb.d1 = hdr64[1];
  pb.d2 = hdr64[2];
  pb.d3 = hdr64[3];
  uint32_t* primes = (uint32_t*)malloc(sizeof(uint32_t) * pb.L);
  if (read_all(f, primes, sizeof(uint32_t) * pb.L)) return 1;
  pb.primes = primes;
  const int64_t k = pb.d1 / pb.N;
  const int64_t n_a = pb.fmt == CTPT_STRUCT_A ? 0 : (pb.fmt == CTPT_SHARED_S ? pb.d2 * k : pb.d2);
  const size_t a_bytes = sizeof(uint32_t) * pb.L * n_a * pb.N, b_bytes = sizeof(uint32_t) * pb.L * pb.d2 * k * pb.N;
  const size_t u_bytes = sizeof(int64_t) * pb.d2 * pb.d3;
  void* h_a = malloc(a_bytes ? a_bytes : 1);
  void* h_b = malloc(b_bytes);
  void* h_u = malloc(u_bytes);
  if (read_all(f, h_a, a_bytes) || read_all(f, h_b, b_bytes) || read_all(f, h_u, u_bytes)) return 1;
  fclose(f);

  ctpt_sizes sz;
  pb.kU = 4; /* size the plain buffer for the worst case; precompute returns the real kU */
  CK(ctpt_query_sizes(&pb, &sz));
  cudaStream_t st;
  CU(cudaStreamCreate(&st));
  void *d_a = NULL, *d_b, *d_u, *d_ctmat, *d_plain, *d_ws, *d_AU = NULL, *d_BU;
  if (a_bytes) CU(cudaMalloc(&d_a, a_bytes));
  CU(cudaMalloc(&d_b, b_bytes));
  CU(cudaMalloc(&d_u, u_bytes));
  CU(cudaMalloc(&d_ctmat, sz.ctmat_bytes));
  CU(cudaMalloc(&d_plain, sz.plain_bytes));
  if (a_bytes) CU(cudaMemcpy(d_a, h_a, a_bytes, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_b, h_b, b_bytes, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_u, h_u, u_bytes, cudaMemcpyHostToDevice));

  CK(ctpt_layout(&pb, (const uint32_t*)d_a, (const uint32_t*)d_b, d_ctmat, 1, st));
  int32_t kU = 0;
  CK(ctpt_plain_precompute(&pb, (const int64_t*)d_u, d_plain, &kU, st));
  pb.kU = kU;
  CK(ctpt_query_sizes(&pb, &sz)); /* the workspace depends on kU */
  CU(cudaMalloc(&d_ws, sz.workspace_bytes ? sz.workspace_bytes : 1));
  if (sz.out_AU_bytes) CU(cudaMalloc(&d_AU, sz.out_AU_bytes));
  CU(cudaMalloc(&d_BU, sz.out_BU_bytes));
  CK(ctpt_matmul(&pb, d_ctmat, d_plain, (uint32_t*)d_AU, (uint32_t*)d_BU, d_ws, sz.workspace_bytes, st));
  CU(cudaStreamSynchronize(st));

  void* h_AU = malloc(sz.out_AU_bytes ? sz.out_AU_bytes : 1);
  void* h_BU = malloc(sz.out_BU_bytes);
  if (sz.out_AU_bytes) CU(cudaMemcpy(h_AU, d_AU, sz.out_AU_bytes, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(h_BU, d_BU, sz.out_BU_bytes, cudaMemcpyDeviceToHost));
  FILE* o = fopen(out_path, "wb");
  if (!o) return 1;
  if (sz.out_AU_bytes) fwrite(h_AU, 1, sz.out_AU_bytes, o);
  fwrite(h_BU, 1, sz.out_BU_bytes, o);
  fclose(o);
  printf("ok: kU=%d R=%lld d2p=%lld\n", kU, (long long)sz.R, (long long)sz.d2p);
  cudaFree(d_a);
  cudaFree(d_b);
  cudaFree(d_u);
  cudaFree(d_ctmat);
  cudaFree(d_plain);
  cudaFree(d_ws);
  cudaFree(d_AU);
  cudaFree(d_BU);
  cudaStreamDestroy(st);
  return 0;
}

int main(int argc, char** argv) {
  if (argc >= 2 && strcmp(argv[1], "sizes") == 0) return cmd_sizes();
  if (argc >= 4 && strcmp(argv[1], "run") == 0) return cmd_run(argv[2], argv[3]);
  fprintf(stderr, "usage: %s sizes | run <in.bin> <out.bin>\n", argv[0]);
  return 1;
}
