// ctpt.cu — C ABI (include/ctpt.h): validation, size queries, TMA descriptor encoding and
// kernel launches for the CP-MM hot path on sm_100a.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/ctpt.h"
#include "gemm_tc.cuh"
#include "gemm_fused_t.cuh"
#include "gemm_mv.cuh"
#include "kernels.cuh"

using namespace ctpt;

namespace {

thread_local char g_err[512] = "ok";

ctpt_status fail(ctpt_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

#define CUDA_TRY_L(label, expr)                                                                 \
  do {                                                                                          \
    cudaError_t e_ = (expr);                                                                    \
    if (e_ != cudaSuccess) return fail(CTPT_ERR_CUDA, "%s: %s", label, cudaGetErrorString(e_)); \
  } while (0)

#define CUDA_TRY(expr)                                                                          \
  do {                                                                                          \
    cudaError_t e_ = (expr);                                                                    \
    if (e_ != cudaSuccess) return fail(CTPT_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

constexpr int kMaxPrimes = 64;
constexpr size_t kHeader = 256;

struct Dims {
  int64_t N, d1, d2, d3, k, rows_A, R, d2p, j0, j1, d3_loc;
  int L;
  int L_out;  // primes in the outputs: L, or L − 1 after an RNS Rescale by the last prime
};

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// Deterministic Miller–Rabin for n < 2^32 (witnesses 2, 7, 61 suffice below 4,759,123,141):
// the moduli must be primes — the Rescale inverts q_1 modulo each of them (Fermat), and the RNS
// result is only meaningful for pairwise coprime moduli.
bool is_prime_u32(uint32_t n) {
  if (n < 2) return false;
  for (uint32_t q : {2u, 3u, 5u, 7u, 11u, 13u}) {
    if (n == q) return true;
    if (n % q == 0) return false;
  }
  auto mulmod = [n](uint64_t a, uint64_t b) { return a * b % n; };
  uint32_t d = n - 1;
  int r = 0;
  while (!(d & 1)) { d >>= 1; ++r; }
  for (uint64_t a : {2ull, 7ull, 61ull}) {
    if (a % n == 0) continue;
    uint64_t x = 1, b = a % n;
    for (uint32_t e = d; e; e >>= 1, b = mulmod(b, b))
      if (e & 1) x = mulmod(x, b);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int i = 1; i < r && comp; ++i) {
      x = mulmod(x, x);
      if (x == n - 1) comp = false;
    }
    if (comp) return false;
  }
  return true;
}

ctpt_status check_problem(const ctpt_problem* pb, Dims& d) {
  if (!pb) return fail(CTPT_ERR_ARG, "problem is NULL");
  if (pb->fmt < CTPT_RLWE || pb->fmt > CTPT_STRUCT_A) return fail(CTPT_ERR_UNSUPPORTED, "unknown format %d", pb->fmt);
  if (pb->L < 1 || pb->L > kMaxPrimes) return fail(CTPT_ERR_ARG, "L = %d outside 1..%d", pb->L, kMaxPrimes);
  if (!pb->primes) return fail(CTPT_ERR_ARG, "primes is NULL");
  if (pb->N < 1 || (pb->N & (pb->N - 1))) return fail(CTPT_ERR_SHAPE, "N = %lld is not a power of two", (long long)pb->N);
  if (pb->d1 < 1 || pb->d2 < 1 || pb->d3 < 1) return fail(CTPT_ERR_SHAPE, "d1, d2, d3 must be >= 1");
  // Table 1: RLWE needs d1 = N; shared-s and shared-a need N | d1.
  if (pb->fmt == CTPT_RLWE && pb->d1 != pb->N) return fail(CTPT_ERR_SHAPE, "RLWE format requires d1 = N");
  if (pb->d1 % pb->N) return fail(CTPT_ERR_SHAPE, "shared-s / shared-a / structured-A formats require N | d1");
  for (int i = 0; i < pb->L; ++i) {
    const uint32_t p = pb->primes[i];
    if (p < 3 || !(p & 1u) || p >= (1u << 31)) return fail(CTPT_ERR_MODULUS, "prime %u must be odd and in (2, 2^31)", p);
    if (!is_prime_u32(p)) return fail(CTPT_ERR_MODULUS, "modulus %u is not prime", p);
    for (int j = 0; j < i; ++j)
      if (pb->primes[j] == p) return fail(CTPT_ERR_MODULUS, "prime %u repeated", p);
  }
  const int64_t c0 = pb->col_begin, c1 = pb->col_end == 0 ? pb->d3 : pb->col_end;
  if (c0 < 0 || c1 > pb->d3 || c0 >= c1) return fail(CTPT_ERR_SHAPE, "column shard [%lld, %lld) invalid", (long long)c0, (long long)c1);
  const int kU = pb->kU <= 0 ? 1 : pb->kU;
  if (kU > 4) return fail(CTPT_ERR_ARG, "kU = %d > 4", kU);
  // Exactness (Lemma le:strategy1 with K = 2^8): |C_ℓ| ≤ d2 · 255 · 128 must stay < 2^31.
  if (pb->d2 * 255LL * 128LL >= (1LL << 31)) return fail(CTPT_ERR_OVERFLOW, "d2 = %lld too large for exact int32 limb accumulation (d2 <= 65793)", (long long)pb->d2);
  d.N = pb->N; d.d1 = pb->d1; d.d2 = pb->d2; d.d3 = pb->d3; d.L = pb->L;
  d.k = pb->d1 / pb->N;
  // structured-A shared-a (Algorithm 7): only B·U is computed, Ã passes through
  d.rows_A = (pb->fmt == CTPT_SHARED_S) ? pb->d1 : (pb->fmt == CTPT_STRUCT_A ? 0 : pb->N);
  d.R = d.rows_A + d.d1;
  d.d2p = round_up(d.d2, 16);
  d.j0 = c0; d.j1 = c1; d.d3_loc = c1 - c0;
  if (pb->rescale != 0 && pb->rescale != 1) return fail(CTPT_ERR_ARG, "rescale must be 0 or 1");
  if (pb->split_overlap != 0 && pb->split_overlap != 1) return fail(CTPT_ERR_ARG, "split_overlap must be 0 or 1");
  if (pb->kernel < CTPT_KERNEL_AUTO || pb->kernel > CTPT_KERNEL_MV) return fail(CTPT_ERR_ARG, "unknown kernel choice %d", pb->kernel);
  if (pb->raster_group < 0 || pb->max_ctas < 0) return fail(CTPT_ERR_ARG, "raster_group and max_ctas must be >= 0");
  if (pb->rescale && pb->L < 2) return fail(CTPT_ERR_ARG, "Rescale by the last prime needs L >= 2 primes");
  d.L_out = pb->rescale ? pb->L - 1 : pb->L;
  if (pb->u_unsigned) {
    // u8 × u8 limb products: |C_ℓ| ≤ d2·255·255 must stay < 2^31 (the int32 accumulator)
    if (kU != 1 || pb->plain_per_prime) return fail(CTPT_ERR_ARG, "unsigned-U planes need kU = 1 and shared planes");
    if (pb->d2 * 255LL * 255LL >= (1LL << 31)) return fail(CTPT_ERR_OVERFLOW, "d2 = %lld too large for unsigned-U planes (d2 <= 33025)", (long long)pb->d2);
  }
  if (d.R > INT32_MAX / 2 || d.d3 > INT32_MAX / 2) return fail(CTPT_ERR_SHAPE, "dimension exceeds TMA coordinate range");
  return CTPT_OK;
}

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

// The 16-byte layout kernel needs 4-row chunks that never straddle A and B (and aligned vectors):
// rows_A and d1 multiples of 4; other shapes take the 4-byte kernel.
bool layout_vec_ok(int64_t rows_A, int64_t d1) { return rows_A % 4 == 0 && d1 % 4 == 0; }

// d_ws of ctpt_matmul / ctpt_split / ctpt_gemm, in this order:
//   limbs   [4][R][d2p] u8                      (one prime's byte-limb planes)
//   rowcorr [R] u32        (unsigned-U mode with u_offset ≠ 0: u_offset·Σ_k X[r][k] mod p)
//   xlast   [d3_loc][R] u32 (rescale: the last prime's product)
//   mv      U_exp + K-split partials + tickets   (d3_loc ≤ 32: the raw-byte kernel, MvPlan)
bool needs_rowcorr(const ctpt_problem* pb) { return pb->u_unsigned && pb->u_offset != 0; }
// the byte limbs of R rows in 32-KB tiles (limb_tile_off): rows padded to 64, K to 128
int64_t limb_nkb(int64_t d2p) { return (d2p + 127) / 128; }
size_t limb_tile_bytes(int64_t rows, int64_t d2p) {
  return static_cast<size_t>(4) * round_up(rows, 64) * (limb_nkb(d2p) * 128);
}
size_t ws_limb_bytes(const Dims& d) { return limb_tile_bytes(d.R, d.d2p); }
size_t ws_corr_off(const Dims& d) { return align256(ws_limb_bytes(d)); }
size_t ws_xlast_off(const ctpt_problem* pb, const Dims& d) {
  return ws_corr_off(d) + (needs_rowcorr(pb) ? align256(static_cast<size_t>(4) * d.R) : 0);
}
size_t mv_ws_bytes(const Dims& d);
size_t ws_base_bytes(const ctpt_problem* pb, const Dims& d) {
  if (needs_rowcorr(pb) || pb->rescale)
    return ws_xlast_off(pb, d) + (pb->rescale ? static_cast<size_t>(4) * d.R * d.d3_loc : 0);
  return ws_limb_bytes(d);
}
// the very-skinny kernel's U_exp + split partials + tickets live after everything else
// split_overlap: a second limb + rowcorr buffer after the base region; prime l uses buffer l & 1
bool overlap_on(const ctpt_problem* pb, const Dims& d) { return pb->split_overlap && !pb->rescale && d.L >= 2; }
size_t ws_ovl_off(const ctpt_problem* pb, const Dims& d) { return align256(ws_base_bytes(pb, d)); }
size_t ws_ovl_bytes(const ctpt_problem* pb, const Dims& d) {
  return overlap_on(pb, d) ? align256(ws_limb_bytes(d)) + align256(static_cast<size_t>(4) * d.R) : 0;
}
void* ws_limbs(const ctpt_problem* pb, const Dims& d, void* ws, int l) {
  return (overlap_on(pb, d) && (l & 1)) ? static_cast<uint8_t*>(ws) + ws_ovl_off(pb, d) : ws;
}
uint32_t* ws_corr(const ctpt_problem* pb, const Dims& d, void* ws, int l) {
  uint8_t* w = static_cast<uint8_t*>(ws);
  return reinterpret_cast<uint32_t*>((overlap_on(pb, d) && (l & 1)) ? w + ws_ovl_off(pb, d) + align256(ws_limb_bytes(d))
                                                                     : w + ws_corr_off(d));
}
size_t ws_mv_off(const ctpt_problem* pb, const Dims& d) { return align256(ws_base_bytes(pb, d)) + ws_ovl_bytes(pb, d); }
// prime l's limb split as a job for the previous prime's GEMM kernel (warps 2–3, gemm_tc.cuh)
SplitJob make_split_job(const ctpt_problem* pb, const Dims& d, const uint32_t* X0, void* ws, int l) {
  SplitJob J{};
  const uint32_t p = pb->primes[l];
  J.x = reinterpret_cast<const uint4*>(X0 + static_cast<int64_t>(l) * d.R * d.d2p);
  J.limbs = static_cast<uint8_t*>(ws_limbs(pb, d, ws, l));
  J.rowcorr = needs_rowcorr(pb) ? ws_corr(pb, d, ws, l) : nullptr;
  J.R = d.R;
  J.d2p16 = d.d2p / 16;
  J.nkb = limb_nkb(d.d2p);
  J.p = p;
  J.off_mod = static_cast<uint32_t>(((static_cast<int64_t>(pb->u_offset) % p) + p) % p);
  return J;
}
size_t ws_bytes_needed(const ctpt_problem* pb, const Dims& d) {
  if (d.d3_loc <= 32) return ws_mv_off(pb, d) + mv_ws_bytes(d);
  return overlap_on(pb, d) ? ws_ovl_off(pb, d) + ws_ovl_bytes(pb, d) : ws_base_bytes(pb, d);
}

// Barrett constants for p; with nonneg_limbs (u8 limbs × the u8 U plane: every limb sum C_ℓ ≥ 0)
// also the Montgomery recombination of kernels.cuh recombine_mod (redc = 2 when d2·255·255 < 2^30
// bounds every C_ℓ below 2^30, else 1).
ModP make_modp(uint32_t p, bool nonneg_limbs = false, int64_t d2 = 0) {
  ModP m;
  memset(&m, 0, sizeof(m));
  m.p = p;
  m.mu = static_cast<uint64_t>((static_cast<unsigned __int128>(1) << 64) / p);
  const uint64_t two56 = 1ULL << 56;
  m.off = ((two56 + p - 1) / p) * static_cast<uint64_t>(p);
#ifdef CTPT_NO_REDC  // A/B build switch (tools/ab_build.py): Barrett on the int64 recombination everywhere
  nonneg_limbs = false;
#endif
  if (nonneg_limbs && d2 * 255LL * 255LL < (1LL << 31)) {
    m.redc = (d2 * 255LL * 255LL < (1LL << 30)) ? 2 : 1;
    uint32_t inv = p;  // p·inv ≡ 1 (mod 2^k), Newton doubling k = 3 → 48
    for (int i = 0; i < 5; ++i) inv *= 2u - p * inv;
    m.pinv = 0u - inv;
    for (int l = 0; l < 4; ++l)
      m.w[l] = static_cast<uint32_t>((static_cast<unsigned __int128>(1) << (8 * l + 32)) % p);
    m.p32 = static_cast<uint64_t>(p) << 32;
  }
  return m;
}

uint32_t powmod_u32(uint32_t b, uint32_t e, uint32_t p) {
  uint64_t r = 1 % p, x = b % p;
  while (e) {
    if (e & 1) r = r * x % p;
    x = x * x % p;
    e >>= 1;
  }
  return static_cast<uint32_t>(r);
}

uint32_t pow2mod(int e, uint32_t p) {
  uint64_t r = 1 % p;
  for (int i = 0; i < e; ++i) r = (r * 2) % p;
  return static_cast<uint32_t>(r);
}

// ---------------------------------------------------------------- TMA descriptors
PFN_cuMemGetAddressRange_v3020 get_addr_range() {
  static PFN_cuMemGetAddressRange_v3020 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(p);
  });
  return fn;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 3-D uint8 tensor [dim2][dim1][dim0] with row pitch `pitch1` bytes and plane pitch `pitch2`.
ctpt_status make_tmap_u8(CUtensorMap* m, const void* base, uint64_t dim0, uint64_t dim1, uint64_t dim2,
                         uint64_t pitch1, uint64_t pitch2, uint32_t box0, uint32_t box1, uint32_t box2) {
  auto enc = get_encode();
  if (!enc) return fail(CTPT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {dim0, dim1, dim2};
  cuuint64_t strides[2] = {pitch1, pitch2};
  cuuint32_t box[3] = {box0, box1, box2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CTPT_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return CTPT_OK;
}

// The byte limbs in 32-KB tiles as a 5-D tensor {128 B, 64 rows, 4 limbs, k-block, row tile}:
// one box of {128, 64, box_limbs, 1, 1} is (part of) one contiguous tile (limb_tile_off).
ctpt_status make_tmap_limb_tiles(CUtensorMap* m, const void* base, int64_t rows, int64_t d2p, uint32_t box_limbs) {
  auto enc = get_encode();
  if (!enc) return fail(CTPT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const uint64_t nkb = static_cast<uint64_t>((d2p + 127) / 128), ntr = static_cast<uint64_t>((rows + 63) / 64);
  cuuint64_t dims[5] = {128, 64, 4, nkb, ntr};
  cuuint64_t strides[4] = {128, 64 * 128, 4 * 64 * 128, nkb * 4 * 64 * 128};
  cuuint32_t box[5] = {128, 64, box_limbs, 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CTPT_ERR_CUDA, "cuTensorMapEncodeTiled (limb tiles) failed (%d)", static_cast<int>(r));
  return CTPT_OK;
}

// 2-D tensor [dim1][dim0] of `esize`-byte elements, row pitch dim0·esize, no swizzle.
ctpt_status make_tmap_2d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, uint32_t esize, uint64_t dim0,
                         uint64_t dim1, uint32_t box0, uint32_t box1) {
  auto enc = get_encode();
  if (!enc) return fail(CTPT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {dim0, dim1};
  cuuint64_t strides[1] = {dim0 * esize};
  cuuint32_t box[2] = {box0, box1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CTPT_ERR_CUDA, "cuTensorMapEncodeTiled (2d) failed (%d)", static_cast<int>(r));
  return CTPT_OK;
}

// 2-D uint32 output tensor [cols][rows] (an output matrix in per-column layout: column j contiguous)
// for the TMA-store epilogue: box {32 rows, 32 columns}, SWIZZLE_128B.
ctpt_status make_tmap_out(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols) {
  auto enc = get_encode();
  if (!enc) return fail(CTPT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {rows, cols};
  cuuint64_t strides[1] = {rows * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CTPT_ERR_CUDA, "cuTensorMapEncodeTiled (outputs) failed (%d)", static_cast<int>(r));
  return CTPT_OK;
}

// Memory of the CURRENT device (not a peer / IPC mapping of another GPU's memory, nor host memory):
// the TMA-store epilogue is used only there; stores into a peer's buffer (the fused multi-GPU
// gather) keep the plain 16-byte STG path.
bool on_current_device(const void* p) {
  int dev = -1;
  cudaPointerAttributes a;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();  // clear a sticky "invalid value" from an unregistered pointer
    return false;
  }
  return a.type == cudaMemoryTypeDevice && a.device == dev;
}

// 2-D uint32 tensor [dim1][dim0] (the stacked int32 X of one prime) read in boxes of 32 rows × 32
// residues (128 B) with SWIZZLE_128B: the raw tiles of the limbs-in-TMEM skinny kernel.
ctpt_status make_tmap_u32_sw128(CUtensorMap* m, const void* base, uint64_t dim0, uint64_t dim1) {
  auto enc = get_encode();
  if (!enc) return fail(CTPT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {dim0, dim1};
  cuuint64_t strides[1] = {dim0 * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CTPT_ERR_CUDA, "cuTensorMapEncodeTiled (raw X) failed (%d)", static_cast<int>(r));
  return CTPT_OK;
}

int num_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
    n = 148;
  return n;
}

// cudaFuncSetAttribute applies to the CURRENT device only: run the set-up once per device (a
// process may drive several GPUs from different threads).
constexpr int kMaxDevices = 64;
ctpt_status tc_setup() {
  static cudaError_t errs[kMaxDevices];
  static std::once_flag onces[kMaxDevices];
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return fail(CTPT_ERR_CUDA, "device ordinal %d out of range", dev);
  cudaError_t& e = errs[dev];
  std::call_once(onces[dev], [&e] {
    e = cudaFuncSetAttribute(k_gemm_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM_BYTES);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_gemm_fused_t<128, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, ft_smem_bytes(128, 2));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_gemm_fused_t<160, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, ft_smem_bytes(160, 2));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_gemm_fused_t<192, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, ft_smem_bytes(192, 2));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_gemm_fused_t<224, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, ft_smem_bytes(224, 2));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_gemm_fused_t<256, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, ft_smem_bytes(256, 1));
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_gemm_mv<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, MV_SMEM_BYTES);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_gemm_mv<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, MV_SMEM_BYTES);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_gemm_mv<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, MV_SMEM_BYTES);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_gemm_mv<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, MV_SMEM_BYTES);
  });
  if (e != cudaSuccess) return fail(CTPT_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  return CTPT_OK;
}

int plane_index(const ctpt_problem* pb, int l, int i) {
  const int kU = pb->kU <= 0 ? 1 : pb->kU;
  return pb->plain_per_prime ? l * kU + i : i;
}

// One prime's limb GEMM (all kU passes) over R rows of byte limbs.
struct GemmArgs {
  const void* limbs;     // [4][R][d2p] u8
  int64_t R;             // rows of X in `limbs` (the problem's R, or a chunk's)
  Dims d;                // d2, d2p, d3, j0, d3_loc
  const int8_t* planes;  // U^T digit planes [nplanes][d3][d2p]
  int nplanes, plane0, kU;
  int u_unsigned;        // U plane is u8 (U + u_offset)
  uint32_t p;
  OutParams o;           // accumulate / w are set per pass
  SplitJob sj;           // the next prime's limb split, run inside the first pass (sj.x = nullptr: none)
  int raster_group;      // k_gemm_tc raster group (0: automatic)
  int max_ctas;          // cap on the persistent grids (0: one CTA per SM)
  int64_t u_offset;      // unsigned-U plane offset (the fused skinny kernel forms the row sums itself)
};
// GemmArgs fields that come straight from the problem
void gemm_args_from_problem(GemmArgs& g, const ctpt_problem* pb) {
  g.raster_group = pb->raster_group;
  g.max_ctas = pb->max_ctas;
  g.u_offset = pb->u_unsigned ? pb->u_offset : 0;
}
// persistent grid size: one CTA per SM (or the caller's cap, e.g. SMs left to a concurrent
// communication kernel), never more than the work units
int64_t grid_cap(int max_ctas) {
  const int sms = num_sms();
  return max_ctas > 0 ? std::min(max_ctas, sms) : sms;
}
ctpt_status launch_split(const uint32_t* x, int64_t rows, int64_t d2p, void* limbs, cudaStream_t st);
// the limb split of `rows` rows of X for prime p; in the unsigned-U mode it also writes rowcorr
ctpt_status launch_split_prime(const ctpt_problem* pb, const uint32_t* x, int64_t rows, int64_t d2p, uint32_t p,
                               void* limbs, uint32_t* rowcorr, cudaStream_t st);
ctpt_status launch_gemm(const GemmArgs& g, cudaStream_t st, bool simt);
ctpt_status launch_split_job(const SplitJob& J, cudaStream_t st);
ctpt_status launch_fused(const GemmArgs& g, const uint32_t* x, cudaStream_t st);

// Kernel choice per prime (ctpt_problem.kernel):
//  * the skinny regime: d3_loc ≤ 256 columns and one U digit plane — the
//    step is HBM-bound and the fused kernel (split inside the GEMM's load path, X read once)
//    replaces split + GEMM;
//  * the very-skinny regime (d3_loc ≤ 32): raw residue bytes straight into the MMA (gemm_mv.cuh);
//  * otherwise the limb split + k_gemm_tc.
// CTPT_KERNEL_AUTO takes the first that applies; a forced choice that does not apply is refused.
constexpr int64_t kFusedMaxD3 = 256;
constexpr int64_t kMvMaxD3 = 32;
int mv_nc(const Dims& d) {  // N = 4·d3p, d3p ∈ {4, 8, 16, 32}
  int d3p = 4;
  while (d3p < d.d3_loc) d3p *= 2;
  return 4 * d3p;
}
struct MvPlan {
  int nc, splits;
  int32_t tiles, num_kb;
  size_t ue_off, part_off, ticket_off, total;
};
MvPlan mv_plan(const Dims& d) {
  MvPlan m;
  m.nc = mv_nc(d);
  m.tiles = static_cast<int32_t>((d.R + MV_BLOCK_R - 1) / MV_BLOCK_R);
  m.num_kb = static_cast<int32_t>(4 * d.d2p / MV_BLOCK_K + ((4 * d.d2p) % MV_BLOCK_K ? 1 : 0));
  // K-split units: ≈ 12 per SM for balance, but never shorter than 32 k-blocks (512 KB of X per
  // 128-row unit) — shorter units were dominated by their fixed cost (pipeline fill, the exact
  // int32 partials and the ticket): at R = 8192, d2 = 4096, 8-k-block units ran at 0.29 of HBM
  // and half the fused kernel's speed (tools/table4.py rows 1, 4)
  const int target = 12 * num_sms();
  int s = static_cast<int>((target + m.tiles - 1) / m.tiles);
  s = std::max(1, std::min(s, std::max(1, m.num_kb / 32)));
  m.splits = s;
  m.ue_off = 0;
  m.part_off = align256(static_cast<size_t>(m.nc) * 4 * d.d2p);
  const size_t part = m.splits > 1 ? static_cast<size_t>(m.tiles) * m.splits * m.nc * MV_BLOCK_R * 4 : 0;
  m.ticket_off = m.part_off + align256(part);
  m.total = m.ticket_off + align256(static_cast<size_t>(m.tiles) * 4);
  return m;
}
// the limbs-in-TMEM kernel forms the unsigned-U row sums itself; the other skinny kernels need u_offset = 0
bool fused_applies(const Dims& d, int kU, const ctpt_problem* pb) {
  (void)pb;
  return kU == 1 && d.d3_loc <= kFusedMaxD3;
}
bool mv_applies(const Dims& d, int kU, const ctpt_problem* pb) {
  return kU == 1 && d.d3_loc <= kMvMaxD3 && !needs_rowcorr(pb);
}
enum class Path { SplitGemm, Fused, Mv };
ctpt_status choose_path(const ctpt_problem* pb, const Dims& d, Path& path) {
  const int kU = pb->kU <= 0 ? 1 : pb->kU;
  switch (pb->kernel) {
    case CTPT_KERNEL_SPLIT_GEMM: path = Path::SplitGemm; return CTPT_OK;
    case CTPT_KERNEL_FUSED:
      if (!fused_applies(d, kU, pb)) return fail(CTPT_ERR_UNSUPPORTED, "the fused kernel needs kU = 1 and d3_loc <= 256");
      path = Path::Fused;
      return CTPT_OK;
    case CTPT_KERNEL_MV:
      if (!mv_applies(d, kU, pb)) return fail(CTPT_ERR_UNSUPPORTED, "raw-byte kernel needs kU = 1, d3_loc <= 32 and u_offset = 0");
      path = Path::Mv;
      return CTPT_OK;
    default:
      // d3_loc ≤ 32: the raw-byte kernel only when there are fewer 64-row tiles than SMs (it splits
      // the K loop across CTAs); with enough rows the limbs-in-TMEM kernel streams faster (c4's
      // ciphertexts, d3 = 1 / 8 / 16 / 32: 1.06 / 1.06 / 1.05 / 1.04 vs 1.01 / 0.99 / 0.96 / 0.92
      // of HBM, profiles/r02/fused_tmem_v3_ab2/)
      path = (mv_applies(d, kU, pb) && (d.R + 63) / 64 < num_sms()) ? Path::Mv
             : fused_applies(d, kU, pb)                          ? Path::Fused
                                                                 : Path::SplitGemm;
      return CTPT_OK;
  }
}
size_t mv_ws_bytes(const Dims& d) { return mv_plan(d).total; }

}  // namespace

extern "C" {

const char* ctpt_last_error(void) { return g_err; }

// CTPT_SRC_HASH: sha256 prefix of csrc/ + include/ at build time (__graft_entry__.build_ctpt), so a
// run's records show which source the loaded binary was built from.
#ifndef CTPT_SRC_HASH
#define CTPT_SRC_HASH "unknown"
#endif
const char* ctpt_version(void) { return "ctpt 0.2 sm_100a tcgen05 kind::i8 src=" CTPT_SRC_HASH; }

ctpt_status ctpt_query_sizes(const ctpt_problem* pb, ctpt_sizes* out) {
  Dims d;
  ctpt_status s = check_problem(pb, d);
  if (s != CTPT_OK) return s;
  if (!out) return fail(CTPT_ERR_ARG, "out is NULL");
  const int kU = pb->kU <= 0 ? 1 : pb->kU;
  out->ctmat_bytes = kHeader + static_cast<size_t>(d.L) * d.R * d.d2p * 4;
  out->plain_bytes = kHeader + static_cast<size_t>(kU) * d.d3 * d.d2p;
  out->plain_rns_bytes = kHeader + static_cast<size_t>(d.L) * 4 * d.d3 * d.d2p;
  out->workspace_bytes = ws_bytes_needed(pb, d);
  out->out_AU_bytes = static_cast<size_t>(d.L_out) * d.d3_loc * d.rows_A * 4;
  out->out_BU_bytes = static_cast<size_t>(d.L_out) * d.d3_loc * d.d1 * 4;
  out->rows_A = d.rows_A;
  out->R = d.R;
  out->d2p = d.d2p;
  out->d3_loc = d.d3_loc;
  return CTPT_OK;
}

ctpt_status ctpt_layout(const ctpt_problem* pb, const uint32_t* d_a, const uint32_t* d_b, void* d_ctmat, int validate,
                        void* stream) {
  Dims d;
  ctpt_status s = check_problem(pb, d);
  if (s != CTPT_OK) return s;
  if ((!d_a && d.rows_A > 0) || !d_b || !d_ctmat) return fail(CTPT_ERR_ARG, "null device pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* hdr = static_cast<uint8_t*>(d_ctmat);
  LayoutParams P;
  memset(&P, 0, sizeof(P));
  P.a = d_a;
  P.b = d_b;
  P.x = reinterpret_cast<uint32_t*>(hdr + kHeader);
  P.rows_A = d.rows_A;
  P.d1 = d.d1;
  P.R = d.R;
  P.d2 = d.d2;
  P.d2p = d.d2p;
  for (int i = 0; i < d.L; ++i) P.p_arr[i] = pb->primes[i];
  P.validate = validate ? 1 : 0;
  P.bad_flag = reinterpret_cast<uint32_t*>(hdr);  // header word 0
  if (validate) CUDA_TRY(cudaMemsetAsync(hdr, 0, 4, st));
  dim3 grid(static_cast<unsigned>((d.R + 63) / 64), static_cast<unsigned>((d.d2p + 63) / 64), d.L);
  if (grid.y > 65535) return fail(CTPT_ERR_SHAPE, "d2 too large for the layout grid");
  if (layout_vec_ok(d.rows_A, d.d1))
    k_layout_v4<<<grid, 256, 0, st>>>(P);
  else
    k_layout<<<grid, 256, 0, st>>>(P);
  CUDA_TRY(cudaGetLastError());
  if (validate) {
    uint32_t flag = 0;
    CUDA_TRY(cudaMemcpyAsync(&flag, hdr, 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (flag) return fail(CTPT_ERR_RANGE, "an input residue is >= its prime");
  }
  return CTPT_OK;
}

static ctpt_status plain_common(const ctpt_problem* pb, const int64_t* d_U, const uint32_t* d_Ures, void* d_plain,
                                int32_t* kU_out, void* stream, int32_t* u_offset_out = nullptr) {
  Dims d;
  ctpt_status s = check_problem(pb, d);
  if (s != CTPT_OK) return s;
  if ((!d_U && !d_Ures) || !d_plain || !kU_out) return fail(CTPT_ERR_ARG, "null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* hdr = static_cast<uint8_t*>(d_plain);
  PlainParams P;
  memset(&P, 0, sizeof(P));
  P.planes = reinterpret_cast<int8_t*>(hdr + kHeader);
  P.d2 = d.d2;
  P.d3 = d.d3;
  P.d2p = d.d2p;
  int nblk_z = 1;
  if (d_U) {
    // max|U| decides k_U (minimal balanced int8 digit count) and whether U's centred
    // residue is U itself for every prime (needs |U| < p/2).
    long long init[2] = {LLONG_MAX, LLONG_MIN};
    CUDA_TRY(cudaMemcpyAsync(hdr, init, 16, cudaMemcpyHostToDevice, st));
    const int64_t n = d.d2 * d.d3;
    k_minmax_i64<<<static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((n + 2047) / 2048, 8LL * num_sms()))), 256, 0, st>>>(
        d_U, n, reinterpret_cast<long long*>(hdr));
    CUDA_TRY(cudaGetLastError());
    long long mm[2];
    CUDA_TRY(cudaMemcpyAsync(mm, hdr, 16, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (u_offset_out) {
      // unsigned-U plane: U' = U + u_offset ∈ [0, 255], u_offset = max(0, −min U)
      const long long off = mm[0] < 0 ? -mm[0] : 0;
      if (mm[1] + off > 255)
        return fail(CTPT_ERR_RANGE, "max(U) - min(U, 0) = %lld > 255: no single unsigned plane", mm[1] + off);
      if (d.d2 * 255LL * 255LL >= (1LL << 31))
        return fail(CTPT_ERR_OVERFLOW, "d2 = %lld too large for unsigned-U planes (d2 <= 33025)", (long long)d.d2);
      P.u = d_U;
      P.kU = 1;
      P.rns = 0;
      P.unsigned_plane = 1;
      P.u_offset = off;
      *u_offset_out = static_cast<int32_t>(off);
    }
    uint32_t pmin = pb->primes[0];
    for (int i = 1; i < d.L; ++i) pmin = std::min(pmin, pb->primes[i]);
    const long long amax = std::max(mm[1], -mm[0]);
    if (!u_offset_out && amax >= static_cast<long long>(pmin / 2))
      return fail(CTPT_ERR_RANGE, "max|U| = %lld >= min(p)/2: use ctpt_plain_precompute_rns", amax);
    int kU = 1;
    // k balanced digits cover [-128·(256^k-1)/255, 127·(256^k-1)/255]
    while (kU < 4) {
      const long long span = ((1LL << (8 * kU)) - 1) / 255;
      if (mm[0] >= -128 * span && mm[1] <= 127 * span) break;
      ++kU;
    }
    if (!u_offset_out) {
      P.u = d_U;
      P.kU = kU;
      P.rns = 0;
    }
  } else {
    P.ures = d_Ures;
    P.kU = 4;
    P.rns = 1;
    for (int i = 0; i < d.L; ++i) P.p_arr[i] = pb->primes[i];
    nblk_z = d.L;
  }
  dim3 grid(static_cast<unsigned>((d.d2p + PLAIN_TK - 1) / PLAIN_TK), static_cast<unsigned>((d.d3 + PLAIN_TJ - 1) / PLAIN_TJ),
           nblk_z);
  if (grid.y > 65535) return fail(CTPT_ERR_SHAPE, "d3 too large for the precompute grid");
  k_plain<<<grid, 256, 0, st>>>(P);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(st));
  *kU_out = P.kU;
  return CTPT_OK;
}

ctpt_status ctpt_plain_precompute(const ctpt_problem* pb, const int64_t* d_U, void* d_plain, int32_t* kU_out,
                                  void* stream) {
  if (!d_U) return fail(CTPT_ERR_ARG, "d_U is NULL");
  return plain_common(pb, d_U, nullptr, d_plain, kU_out, stream);
}

ctpt_status ctpt_plain_precompute_unsigned(const ctpt_problem* pb, const int64_t* d_U, void* d_plain,
                                           int32_t* u_offset_out, void* stream) {
  if (!d_U || !u_offset_out) return fail(CTPT_ERR_ARG, "null pointer");
  int32_t kU = 0;
  return plain_common(pb, d_U, nullptr, d_plain, &kU, stream, u_offset_out);
}

ctpt_status ctpt_plain_precompute_rns(const ctpt_problem* pb, const uint32_t* d_Ures, void* d_plain, int32_t* kU_out,
                                      void* stream) {
  if (!d_Ures) return fail(CTPT_ERR_ARG, "d_Ures is NULL");
  return plain_common(pb, nullptr, d_Ures, d_plain, kU_out, stream);
}

ctpt_status ctpt_split(const ctpt_problem* pb, int32_t l, const void* d_ctmat, void* d_ws, size_t ws_bytes,
                       void* stream) {
  Dims d;
  ctpt_status s = check_problem(pb, d);
  if (s != CTPT_OK) return s;
  if (l < 0 || l >= d.L) return fail(CTPT_ERR_ARG, "prime index %d out of range", l);
  if (!d_ctmat || !d_ws) return fail(CTPT_ERR_ARG, "null device pointer");
  if (ws_bytes < ws_bytes_needed(pb, d)) return fail(CTPT_ERR_ARG, "workspace too small");
  const int64_t n = d.R * d.d2p;  // multiple of 16
  const uint32_t* x = reinterpret_cast<const uint32_t*>(static_cast<const uint8_t*>(d_ctmat) + kHeader) + l * n;
  return launch_split_prime(pb, x, d.R, d.d2p, pb->primes[l], ws_limbs(pb, d, d_ws, l), ws_corr(pb, d, d_ws, l),
                            static_cast<cudaStream_t>(stream));
}

static ctpt_status gemm_common(const ctpt_problem* pb, int32_t l, const void* d_ws, size_t ws_bytes,
                               const void* d_plain, uint32_t* d_AU_l, uint32_t* d_BU_l, void* stream, bool simt,
                               const void* d_ctmat_next = nullptr) {
  Dims d;
  ctpt_status s = check_problem(pb, d);
  if (s != CTPT_OK) return s;
  if (pb->rescale) return fail(CTPT_ERR_UNSUPPORTED, "Rescale needs every prime: use ctpt_matmul");
  if (l < 0 || l >= d.L) return fail(CTPT_ERR_ARG, "prime index %d out of range", l);
  if (!d_ws || !d_plain || (!d_AU_l && d.rows_A > 0) || !d_BU_l) return fail(CTPT_ERR_ARG, "null device pointer");
  if (ws_bytes < ws_bytes_needed(pb, d)) return fail(CTPT_ERR_ARG, "workspace too small");
  GemmArgs g{};
  gemm_args_from_problem(g, pb);
  g.limbs = ws_limbs(pb, d, const_cast<void*>(d_ws), l);
  g.u_unsigned = pb->u_unsigned;
  if (needs_rowcorr(pb)) g.o.rowcorr = ws_corr(pb, d, const_cast<void*>(d_ws), l);
  g.R = d.R;
  g.d = d;
  g.kU = pb->kU <= 0 ? 1 : pb->kU;
  g.planes = reinterpret_cast<const int8_t*>(static_cast<const uint8_t*>(d_plain) + kHeader);
  g.nplanes = pb->plain_per_prime ? d.L * g.kU : g.kU;
  g.plane0 = plane_index(pb, l, 0);
  g.p = pb->primes[l];
  g.o.AU = d_AU_l;
  g.o.BU = d_BU_l;
  g.o.rows_A = d.rows_A;
  g.o.d1 = d.d1;
  g.o.R = d.R;
  g.o.d3_loc = d.d3_loc;
  if (d_ctmat_next && l + 1 < d.L)
    g.sj = make_split_job(pb, d, reinterpret_cast<const uint32_t*>(static_cast<const uint8_t*>(d_ctmat_next) + kHeader),
                          const_cast<void*>(d_ws), l + 1);
  return launch_gemm(g, static_cast<cudaStream_t>(stream), simt);
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// Internal launchers (shared by the per-stage entry points and the host-pipelined executor)
// ---------------------------------------------------------------------------------------------
namespace {

ctpt_status launch_split_prime(const ctpt_problem* pb, const uint32_t* x, int64_t rows, int64_t d2p, uint32_t p,
                               void* limbs, uint32_t* rowcorr, cudaStream_t st) {
  if (!needs_rowcorr(pb)) return launch_split(x, rows, d2p, limbs, st);
  const int64_t off = pb->u_offset;
  const uint32_t off_mod = static_cast<uint32_t>(((off % static_cast<int64_t>(p)) + p) % p);
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(rows, INT32_MAX)));
  k_split_rows<<<blocks, 256, 0, st>>>(reinterpret_cast<const uint4*>(x), static_cast<uint8_t*>(limbs), rowcorr, rows,
                                        d2p / 16, limb_nkb(d2p), p, off_mod);
  CUDA_TRY(cudaGetLastError());
  return CTPT_OK;
}

ctpt_status launch_split_job(const SplitJob& J, cudaStream_t st) {
  if (!J.rowcorr) return launch_split(reinterpret_cast<const uint32_t*>(J.x), J.R, J.d2p16 * 16, J.limbs, st);
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(J.R, INT32_MAX)));
  k_split_rows<<<blocks, 256, 0, st>>>(J.x, J.limbs, J.rowcorr, J.R, J.d2p16, J.nkb, J.p, J.off_mod);
  CUDA_TRY(cudaGetLastError());
  return CTPT_OK;
}

ctpt_status launch_split(const uint32_t* x, int64_t rows, int64_t d2p, void* limbs, cudaStream_t st) {
  const int64_t nkb = limb_nkb(d2p), groups = rows * nkb * 8;  // 16-residue groups incl. K padding
  const int blocks = static_cast<int>(std::min<int64_t>((groups + 255) / 256, static_cast<int64_t>(num_sms()) * 16));
  if (blocks > 0)
    k_split<<<blocks, 256, 0, st>>>(reinterpret_cast<const uint4*>(x), static_cast<uint8_t*>(limbs), rows, d2p / 16, nkb);
  CUDA_TRY(cudaGetLastError());
  return CTPT_OK;
}

ctpt_status launch_gemm(const GemmArgs& g, cudaStream_t st, bool simt) {
  const Dims& d = g.d;
  const ModP m = make_modp(g.p, g.u_unsigned != 0, d.d2);
  if (simt) {
    for (int i = 0; i < g.kU; ++i) {
      SimtParams S;
      S.limbs = static_cast<const uint8_t*>(g.limbs);
      S.uplane = g.planes + static_cast<int64_t>(g.plane0 + i) * d.d3 * d.d2p;
      S.R = g.R;
      S.d2 = d.d2;
      S.d2p = d.d2p;
      S.j_off = d.j0;
      S.u_unsigned = g.u_unsigned;
      S.m = m;
      S.o = g.o;
      S.o.accumulate = i > 0;
      S.o.w = pow2mod(8 * i, g.p);
      if (i < g.kU - 1) S.o.xlast = nullptr;
      dim3 grid(static_cast<unsigned>((g.R + 15) / 16), static_cast<unsigned>((d.d3_loc + 15) / 16));
      k_gemm_simt<<<grid, 256, 0, st>>>(S);
      CUDA_TRY(cudaGetLastError());
    }
    return g.sj.x ? launch_split_job(g.sj, st) : CTPT_OK;
  }
  ctpt_status s = tc_setup();
  if (s != CTPT_OK) return s;
  // (A CTA-pair kernel — cta_group::2, M = 256 — and a 2-CTA multicast cluster were measured
  // against this single-CTA kernel under the 1000 W cap and lost: they keep the tensor pipe busier
  // per clock but clock lower, profiles/r01/gemm_1cta_vs_2cta_final/, gemm_mc_vs_tc/; removed.)
  CUtensorMap tmU, tmX;
  s = make_tmap_u8(&tmU, g.planes, d.d2, d.d3, g.nplanes, d.d2p, d.d3 * d.d2p, TC_BLOCK_K, 128, 1);
  if (s != CTPT_OK) return s;
  s = make_tmap_limb_tiles(&tmX, g.limbs, g.R, d.d2p, 4);
  if (s != CTPT_OK) return s;
  TcParams P;
  P.R = g.R;
  P.d2 = d.d2;
  P.j_off = static_cast<int32_t>(d.j0);
  P.num_kb = static_cast<int32_t>((d.d2 + TC_BLOCK_K - 1) / TC_BLOCK_K);
  P.tiles_j = static_cast<int32_t>((d.d3_loc + TC_BLOCK_J - 1) / TC_BLOCK_J);
  P.tiles_r = static_cast<int32_t>((g.R + TC_BLOCK_R - 1) / TC_BLOCK_R);
  const int64_t nt = static_cast<int64_t>(P.tiles_j) * P.tiles_r;
  if (nt > INT32_MAX) return fail(CTPT_ERR_SHAPE, "too many tiles");
  P.num_tiles = static_cast<int32_t>(nt);
  // raster group: keep a group's U^T panels within ≈ 32 MB of L2 but never below the measured best
  // of 16 j-tiles: short-K problems (c2: 0.5 MB per panel) take every j-tile in one group, so each
  // X panel is read from DRAM once (c2: +2.4 %; c3, c4: 16 measured best, profiles/r01/raster_group_*)
  const int64_t per_panel = static_cast<int64_t>(TC_BLOCK_J) * P.num_kb * TC_BLOCK_K;
  const int64_t fit = (32LL << 20) / std::max<int64_t>(per_panel, 1);
  P.group_j = static_cast<int32_t>(std::min<int64_t>(std::max<int64_t>(fit, TC_GROUP_J_DEFAULT), P.tiles_j));
  if (g.raster_group > 0) P.group_j = g.raster_group;
  // Serpentine K order when one wave's operand footprint exceeds L2: per K byte a wave touches the
  // group's U^T panel (128·group_j B) and the X limb rows of ≈ SMs / group_j r-tiles (256 B each).
  // c4 / c5 (K = 32768): 144 MB per wave, the next wave would re-read the whole panel from DRAM —
  // reversing K on odd waves starts it on the lines the last wave touched (c4 GEMM: 33.4 → 27.9 GB
  // of DRAM reads per launch, bench +1.0 %); c3 (72 MB, fits) loses 1.5 % with it, so it stays off
  // there (profiles/r02/serpentine/).
  {
    const double wave_bytes = static_cast<double>(P.num_kb) * TC_BLOCK_K *
                              (static_cast<double>(TC_BLOCK_J) * P.group_j +
                               4.0 * TC_BLOCK_R * static_cast<double>(num_sms()) / P.group_j);
    P.serpentine = wave_bytes > 100.0e6 ? 1 : 0;
  }
#ifdef CTPT_TC_NO_SERPENTINE  // A/B measurement build only (tools/ab_build.py): K always ascending
  P.serpentine = 0;
#endif
#ifdef CTPT_TC_SERPENTINE_ALWAYS  // A/B measurement build only
  P.serpentine = 1;
#endif
  P.u_unsigned = g.u_unsigned;
  P.m = m;
  // TMA-store epilogue: a tile's 64 rows must lie inside A' or inside B' (rows_A, d1 multiples of
  // 64; then every row pitch is 16-B aligned) and the outputs must be this device's memory
  const OutParams& o0 = g.o;
  const bool has_a = o0.rows_A > 0, has_b = o0.d1 > 0;
  P.tma_store = o0.rows_A % 64 == 0 && o0.d1 % 64 == 0 && (has_a || has_b) &&
                (!has_a || (reinterpret_cast<uintptr_t>(o0.AU) % 16 == 0 && on_current_device(o0.AU))) &&
                (!has_b || (reinterpret_cast<uintptr_t>(o0.BU) % 16 == 0 && on_current_device(o0.BU)));
#ifdef CTPT_NO_TMA_STORE  // A/B measurement build only (tools/ab_build.py): the 16-byte STG epilogue
  P.tma_store = 0;
#endif
  CUtensorMap tmAU = tmU, tmBU = tmU;  // unused placeholders unless tma_store
  if (P.tma_store) {
    if (has_a && (s = make_tmap_out(&tmAU, o0.AU, o0.rows_A, d.d3_loc)) != CTPT_OK) return s;
    if (has_b && (s = make_tmap_out(&tmBU, o0.BU, o0.d1, d.d3_loc)) != CTPT_OK) return s;
  }
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(nt, grid_cap(g.max_ctas)));
  // k_U > 1 digit planes (Rescale's real U, general Mod-PP-MM): one launch per digit whose epilogue
  // accumulates Σ_i 2^{8i}·(digit i's product mod p) through the outputs.  (All digits in one launch
  // with register accumulation was measured slower: the tile's k_U U^T panels crowd L2,
  // profiles/r01/gemm_multi_digit/; removed.)
  for (int i = 0; i < g.kU; ++i) {
    const bool first = i == 0, last = i == g.kU - 1;
    P.plane = g.plane0 + i;
    P.o = g.o;
    P.o.accumulate = !first;
    P.o.w = pow2mod(8 * i, g.p);
    if (!last) P.o.xlast = nullptr;     // Rescale on the final pass only
    if (!first) P.o.rowcorr = nullptr;  // the unsigned-U row correction exactly once
    P.sj = first ? g.sj : SplitJob{};   // the next prime's split rides on the first pass
    k_gemm_tc<<<grid, TC_THREADS, TC_SMEM_BYTES, st>>>(tmU, tmX, tmAU, tmBU, P);
    CUDA_TRY(cudaGetLastError());
  }
  return CTPT_OK;
}

ctpt_status launch_fused(const GemmArgs& g, const uint32_t* x, cudaStream_t st) {
  const Dims& d = g.d;
  if (g.kU != 1 || d.d3_loc > kFusedMaxD3) return fail(CTPT_ERR_UNSUPPORTED, "fused kernel needs kU = 1 and d3_loc <= 256");
  ctpt_status s = tc_setup();
  if (s != CTPT_OK) return s;
  // limbs in tensor memory (gemm_fused_t.cuh): 64-row tiles (two 32-row sub-tiles sharing each U^T
  // stage) up to 224 columns, 32-row tiles above; MMA N = d3_loc rounded up to 16; the unsigned-U
  // row sums formed in the converters.  (The round-1 limbs-in-shared-memory kernel lost at every
  // width: profiles/r02/fused_tmem_v3*/, fused_rowsum/; removed.)
  FusedTParams T;
  T.R = g.R;
  T.j_off = static_cast<int32_t>(d.j0);
  T.plane = g.plane0;
  T.num_kb = static_cast<int32_t>((d.d2p + FT_BK - 1) / FT_BK);
#ifndef CTPT_FT_SUB2_MAX
#define CTPT_FT_SUB2_MAX 224  // widest d3_loc on 64-row tiles (A/B builds: 192 = 32-row tiles above)
#endif
  const int sub = d.d3_loc <= CTPT_FT_SUB2_MAX ? 2 : 1;
  const int64_t ntt = (g.R + ft_rows(sub) - 1) / ft_rows(sub);
  if (ntt > INT32_MAX) return fail(CTPT_ERR_SHAPE, "too many tiles");
  T.num_tiles = static_cast<int32_t>(ntt);
  T.np = static_cast<int32_t>((d.d3_loc + 15) / 16 * 16);
  T.u_unsigned = g.u_unsigned;
  T.off_mod = static_cast<uint32_t>(((g.u_offset % static_cast<int64_t>(g.p)) + g.p) % g.p);
  T.m = make_modp(g.p, g.u_unsigned != 0, d.d2);
  T.o = g.o;
  T.o.accumulate = 0;
  T.o.w = 1;
  T.o.rowcorr = nullptr;  // the kernel forms the row sums while it splits X
  CUtensorMap tmU, tmX;
  s = make_tmap_u8(&tmU, g.planes, d.d2, d.d3, g.nplanes, d.d2p, d.d3 * d.d2p, FT_BK, static_cast<uint32_t>(T.np), 1);
  if (s != CTPT_OK) return s;
  s = make_tmap_u32_sw128(&tmX, x, d.d2p, g.R);
  if (s != CTPT_OK) return s;
  // balanced persistent grid: the same number of rounds as min(tiles, SMs) CTAs would take, spread
  // over as few CTAs as that needs, so no round ends with most SMs idle behind a few stragglers
  // (an HBM-bound CTA can pull more than 1/148 of the bandwidth; profiles/r01/fused_balanced_grid/)
  const int64_t cap = grid_cap(g.max_ctas);
  const int64_t rounds = (ntt + cap - 1) / cap;
  const unsigned grid = static_cast<unsigned>((ntt + rounds - 1) / rounds);
  if (sub == 2 && d.d3_loc <= 128)
    k_gemm_fused_t<128, 2><<<grid, FT_THREADS, ft_smem_bytes(128, 2), st>>>(tmU, tmX, T);
  else if (sub == 2 && d.d3_loc <= 160)
    k_gemm_fused_t<160, 2><<<grid, FT_THREADS, ft_smem_bytes(160, 2), st>>>(tmU, tmX, T);
  else if (sub == 2 && d.d3_loc <= 192)
    k_gemm_fused_t<192, 2><<<grid, FT_THREADS, ft_smem_bytes(192, 2), st>>>(tmU, tmX, T);
  else if (sub == 2)
    k_gemm_fused_t<224, 2><<<grid, FT_THREADS, ft_smem_bytes(224, 2), st>>>(tmU, tmX, T);
  else
    k_gemm_fused_t<256, 1><<<grid, FT_THREADS, ft_smem_bytes(256, 1), st>>>(tmU, tmX, T);
  CUDA_TRY(cudaGetLastError());
  return CTPT_OK;
}

// The very-skinny kernel for one prime: expand U into U_exp in the workspace, zero the tickets,
// run k_gemm_mv<NC>.  `mv_ws` points at the MvPlan region of the workspace.
ctpt_status launch_mv(const GemmArgs& g, const uint32_t* x, void* mv_ws, cudaStream_t st) {
  const Dims& d = g.d;
  if (g.kU != 1 || d.d3_loc > kMvMaxD3) return fail(CTPT_ERR_UNSUPPORTED, "mv kernel needs kU = 1 and d3_loc <= 32");
  ctpt_status s = tc_setup();
  if (s != CTPT_OK) return s;
  Dims dd = d;
  dd.R = g.R;
  const MvPlan mp = mv_plan(dd);
  uint8_t* w = static_cast<uint8_t*>(mv_ws);
  uint32_t* ue = reinterpret_cast<uint32_t*>(w + mp.ue_off);
  const int8_t* plane = g.planes + static_cast<int64_t>(g.plane0) * d.d3 * d.d2p;
  const int d3p = mp.nc / 4;
  dim3 eg(static_cast<unsigned>(std::min<int64_t>((d.d2p + 255) / 256, 1024)), static_cast<unsigned>(mp.nc));
  k_expand_u<<<eg, 256, 0, st>>>(plane, d.d2p, static_cast<int32_t>(d.j0), static_cast<int32_t>(d.d3_loc), d3p, ue);
  CUDA_TRY_L("k_expand_u launch", cudaGetLastError());
  if (mp.splits > 1) CUDA_TRY(cudaMemsetAsync(w + mp.ticket_off, 0, static_cast<size_t>(mp.tiles) * 4, st));
  CUtensorMap tmX, tmUe;
  const uint64_t kbytes = static_cast<uint64_t>(4) * d.d2p;
  s = make_tmap_u8(&tmX, x, kbytes, g.R, 1, kbytes, kbytes * g.R, MV_BLOCK_K, MV_BLOCK_R, 1);
  if (s != CTPT_OK) return s;
  s = make_tmap_u8(&tmUe, ue, kbytes, mp.nc, 1, kbytes, kbytes * mp.nc, MV_BLOCK_K, mp.nc, 1);
  if (s != CTPT_OK) return s;
  MvParams P{};
  P.num_kb = mp.num_kb;
  P.num_tiles = mp.tiles;
  P.splits = mp.splits;
  P.u_unsigned = g.u_unsigned;
  P.partial = reinterpret_cast<int32_t*>(w + mp.part_off);
  P.tickets = reinterpret_cast<uint32_t*>(w + mp.ticket_off);
  P.m = make_modp(g.p, g.u_unsigned != 0, d.d2);
  P.o = g.o;
  P.o.accumulate = 0;
  P.o.w = 1;
  const int64_t units = static_cast<int64_t>(mp.tiles) * mp.splits;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(units, grid_cap(g.max_ctas)));
  switch (mp.nc) {
    case 16: k_gemm_mv<16><<<grid, MV_THREADS, MV_SMEM_BYTES, st>>>(tmX, tmUe, P); break;
    case 32: k_gemm_mv<32><<<grid, MV_THREADS, MV_SMEM_BYTES, st>>>(tmX, tmUe, P); break;
    case 64: k_gemm_mv<64><<<grid, MV_THREADS, MV_SMEM_BYTES, st>>>(tmX, tmUe, P); break;
    default: k_gemm_mv<128><<<grid, MV_THREADS, MV_SMEM_BYTES, st>>>(tmX, tmUe, P); break;
  }
  CUDA_TRY_L("k_gemm_mv launch", cudaGetLastError());
  return CTPT_OK;
}

}  // namespace

extern "C" {

ctpt_status ctpt_gemm_mv(const ctpt_problem* pb, int32_t l, const void* d_ctmat, const void* d_plain,
                         uint32_t* d_AU_l, uint32_t* d_BU_l, void* d_ws, size_t ws_bytes, void* stream) {
  Dims d;
  ctpt_status s = check_problem(pb, d);
  if (s != CTPT_OK) return s;
  if (pb->rescale) return fail(CTPT_ERR_UNSUPPORTED, "Rescale needs every prime: use ctpt_matmul");
  if (needs_rowcorr(pb)) return fail(CTPT_ERR_UNSUPPORTED, "the mv kernel does not form row sums (u_offset != 0)");
  if (l < 0 || l >= d.L) return fail(CTPT_ERR_ARG, "prime index %d out of range", l);
  if (!d_ctmat || !d_plain || (!d_AU_l && d.rows_A > 0) || !d_BU_l || !d_ws) return fail(CTPT_ERR_ARG, "null pointer");
  if (ws_bytes < ws_bytes_needed(pb, d)) return fail(CTPT_ERR_ARG, "workspace too small");
  GemmArgs g{};
  gemm_args_from_problem(g, pb);
  g.R = d.R;
  g.d = d;
  g.kU = pb->kU <= 0 ? 1 : pb->kU;
  g.u_unsigned = pb->u_unsigned;
  g.planes = reinterpret_cast<const int8_t*>(static_cast<const uint8_t*>(d_plain) + kHeader);
  g.nplanes = pb->plain_per_prime ? d.L * g.kU : g.kU;
  g.plane0 = plane_index(pb, l, 0);
  g.p = pb->primes[l];
  g.o.AU = d_AU_l;
  g.o.BU = d_BU_l;
  g.o.rows_A = d.rows_A;
  g.o.d1 = d.d1;
  g.o.R = d.R;
  g.o.d3_loc = d.d3_loc;
  const uint32_t* x =
      reinterpret_cast<const uint32_t*>(static_cast<const uint8_t*>(d_ctmat) + kHeader) + l * d.R * d.d2p;
  return launch_mv(g, x, static_cast<uint8_t*>(d_ws) + ws_mv_off(pb, d), static_cast<cudaStream_t>(stream));
}

ctpt_status ctpt_gemm_fused(const ctpt_problem* pb, int32_t l, const void* d_ctmat, const void* d_plain,
                            uint32_t* d_AU_l, uint32_t* d_BU_l, void* stream) {
  Dims d;
  ctpt_status s = check_problem(pb, d);
  if (s != CTPT_OK) return s;
  if (pb->rescale) return fail(CTPT_ERR_UNSUPPORTED, "Rescale needs every prime: use ctpt_matmul");
  if (l < 0 || l >= d.L) return fail(CTPT_ERR_ARG, "prime index %d out of range", l);
  if (!d_ctmat || !d_plain || (!d_AU_l && d.rows_A > 0) || !d_BU_l) return fail(CTPT_ERR_ARG, "null device pointer");
  GemmArgs g{};
  gemm_args_from_problem(g, pb);
  g.limbs = nullptr;
  g.u_unsigned = pb->u_unsigned;
  g.R = d.R;
  g.d = d;
  g.kU = pb->kU <= 0 ? 1 : pb->kU;
  g.planes = reinterpret_cast<const int8_t*>(static_cast<const uint8_t*>(d_plain) + kHeader);
  g.nplanes = pb->plain_per_prime ? d.L * g.kU : g.kU;
  g.plane0 = plane_index(pb, l, 0);
  g.p = pb->primes[l];
  g.o.AU = d_AU_l;
  g.o.BU = d_BU_l;
  g.o.rows_A = d.rows_A;
  g.o.d1 = d.d1;
  g.o.R = d.R;
  g.o.d3_loc = d.d3_loc;
  const uint32_t* x =
      reinterpret_cast<const uint32_t*>(static_cast<const uint8_t*>(d_ctmat) + kHeader) + l * d.R * d.d2p;
  return launch_fused(g, x, static_cast<cudaStream_t>(stream));
}

ctpt_status ctpt_gemm(const ctpt_problem* pb, int32_t l, const void* d_ws, size_t ws_bytes, const void* d_plain,
                      uint32_t* d_AU_l, uint32_t* d_BU_l, void* stream) {
  return gemm_common(pb, l, d_ws, ws_bytes, d_plain, d_AU_l, d_BU_l, stream, false);
}

ctpt_status ctpt_gemm_next(const ctpt_problem* pb, int32_t l, const void* d_ctmat, void* d_ws, size_t ws_bytes,
                           const void* d_plain, uint32_t* d_AU_l, uint32_t* d_BU_l, void* stream) {
  Dims d;
  ctpt_status s = check_problem(pb, d);
  if (s != CTPT_OK) return s;
  if (!overlap_on(pb, d)) return fail(CTPT_ERR_ARG, "ctpt_gemm_next needs split_overlap = 1, no rescale and L >= 2");
  if (!d_ctmat) return fail(CTPT_ERR_ARG, "null device pointer");
  return gemm_common(pb, l, d_ws, ws_bytes, d_plain, d_AU_l, d_BU_l, stream, false, d_ctmat);
}

ctpt_status ctpt_gemm_simt(const ctpt_problem* pb, int32_t l, const void* d_ws, size_t ws_bytes, const void* d_plain,
                           uint32_t* d_AU_l, uint32_t* d_BU_l, void* stream) {
  return gemm_common(pb, l, d_ws, ws_bytes, d_plain, d_AU_l, d_BU_l, stream, true);
}

static ctpt_status matmul_impl(const ctpt_problem* pb, const Dims& d, const uint32_t* X0, const void* d_plain,
                               uint32_t* d_AU, uint32_t* d_BU, void* d_ws, size_t ws_bytes, void* stream);

ctpt_status ctpt_matmul(const ctpt_problem* pb, const void* d_ctmat, const void* d_plain, uint32_t* d_AU,
                        uint32_t* d_BU, void* d_ws, size_t ws_bytes, void* stream) {
  Dims d;
  ctpt_status s = check_problem(pb, d);
  if (s != CTPT_OK) return s;
  if ((!d_AU && d.rows_A > 0) || !d_BU || !d_ctmat || !d_plain) return fail(CTPT_ERR_ARG, "null pointer");
  const uint32_t* X0 = reinterpret_cast<const uint32_t*>(static_cast<const uint8_t*>(d_ctmat) + kHeader);
  return matmul_impl(pb, d, X0, d_plain, d_AU, d_BU, d_ws, ws_bytes, stream);
}

ctpt_status ctpt_rescale(int32_t L, const uint32_t* primes, int64_t n, const uint32_t* d_in, uint32_t* d_out,
                         void* stream) {
  if (L < 2 || L > kMaxPrimes) return fail(CTPT_ERR_ARG, "Rescale needs 2 <= L <= %d", kMaxPrimes);
  if (!primes || (n > 0 && (!d_in || !d_out))) return fail(CTPT_ERR_ARG, "null pointer");
  if (n < 0) return fail(CTPT_ERR_SHAPE, "n < 0");
  for (int i = 0; i < L; ++i) {
    const uint32_t p = primes[i];
    if (p < 3 || !(p & 1u) || p >= (1u << 31) || !is_prime_u32(p)) return fail(CTPT_ERR_MODULUS, "bad prime %u", p);
    for (int j = 0; j < i; ++j)
      if (primes[j] == p) return fail(CTPT_ERR_MODULUS, "prime %u repeated", p);
  }
  if (n == 0) return CTPT_OK;
  RescaleParams P{};
  P.in = d_in;
  P.out = d_out;
  P.n = n;
  P.L = L;
  P.p_last = primes[L - 1];
  for (int l = 0; l < L - 1; ++l) {
    P.m[l] = make_modp(primes[l]);
    P.inv[l] = powmod_u32(P.p_last % primes[l], primes[l] - 2, primes[l]);
  }
  dim3 grid(static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 4096)), static_cast<unsigned>(L - 1));
  k_rescale<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(P);
  CUDA_TRY(cudaGetLastError());
  return CTPT_OK;
}

// Mod-PP-MM_{q; M, K, Nc} in RNS as the degenerate problem "structured-A with N = 1": rows_A = 0,
// d1 = M, d2 = K, d3 = Nc, general per-prime Y planes (k_U = 4).
static ctpt_problem modmm_problem(int32_t L, const uint32_t* primes, int64_t M, int64_t K, int64_t Nc) {
  ctpt_problem pb{};
  pb.fmt = CTPT_STRUCT_A;
  pb.L = L;
  pb.N = 1;
  pb.d1 = M;
  pb.d2 = K;
  pb.d3 = Nc;
  pb.primes = primes;
  pb.kU = 4;
  pb.plain_per_prime = 1;
  return pb;
}

ctpt_status ctpt_modmatmul_sizes(int32_t L, const uint32_t* primes, int64_t M, int64_t K, int64_t Nc,
                                 int64_t* ldx, size_t* plain_bytes, size_t* ws_bytes) {
  ctpt_problem pb = modmm_problem(L, primes, M, K, Nc);
  Dims d;
  ctpt_status s = check_problem(&pb, d);
  if (s != CTPT_OK) return s;
  if (!ldx || !plain_bytes || !ws_bytes) return fail(CTPT_ERR_ARG, "null pointer");
  *ldx = d.d2p;
  *plain_bytes = kHeader + static_cast<size_t>(d.L) * 4 * d.d3 * d.d2p;
  *ws_bytes = ws_bytes_needed(&pb, d);
  return CTPT_OK;
}

ctpt_status ctpt_modmatmul_precompute(int32_t L, const uint32_t* primes, int64_t M, int64_t K, int64_t Nc,
                                      const uint32_t* d_Y, void* d_plain, void* stream) {
  ctpt_problem pb = modmm_problem(L, primes, M, K, Nc);
  int32_t kU = 0;
  return ctpt_plain_precompute_rns(&pb, d_Y, d_plain, &kU, stream);
}

ctpt_status ctpt_modmatmul(int32_t L, const uint32_t* primes, int64_t M, int64_t K, int64_t Nc, const uint32_t* d_X,
                           int64_t ldx, const void* d_plain, uint32_t* d_ZT, void* d_ws, size_t ws_bytes,
                           void* stream) {
  ctpt_problem pb = modmm_problem(L, primes, M, K, Nc);
  Dims d;
  ctpt_status s = check_problem(&pb, d);
  if (s != CTPT_OK) return s;
  if (!d_X || !d_plain || !d_ZT) return fail(CTPT_ERR_ARG, "null pointer");
  if (ldx != d.d2p) return fail(CTPT_ERR_SHAPE, "ldx = %lld must be K rounded up to 16 (%lld)", (long long)ldx, (long long)d.d2p);
  return matmul_impl(&pb, d, d_X, d_plain, nullptr, d_ZT, d_ws, ws_bytes, stream);
}

static ctpt_status matmul_impl(const ctpt_problem* pb, const Dims& d, const uint32_t* X0, const void* d_plain,
                               uint32_t* d_AU, uint32_t* d_BU, void* d_ws, size_t ws_bytes, void* stream) {
  Path path;
  ctpt_status s = choose_path(pb, d, path);
  if (s != CTPT_OK) return s;
  const bool fused = path != Path::SplitGemm;
  const bool mv = path == Path::Mv;
  if ((!fused || mv) && !d_ws) return fail(CTPT_ERR_ARG, "null workspace");
  if (!fused || mv || pb->rescale) {
    const size_t need = ws_bytes_needed(pb, d);
    if (ws_bytes < need) return fail(CTPT_ERR_ARG, "workspace too small (%zu < %zu)", ws_bytes, need);
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool ovl = overlap_on(pb, d) && !fused && !mv;  // primes run in order 0..L−1 (no rescale)
  uint32_t* xlast = pb->rescale
                        ? reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(d_ws) + ws_xlast_off(pb, d))
                        : nullptr;
  // one prime's product (fused skinny kernel, or split + limb GEMM) into the outputs `o`
  auto run = [&](int l, const OutParams& o) -> ctpt_status {
    GemmArgs g{};
    gemm_args_from_problem(g, pb);
  gemm_args_from_problem(g, pb);
    g.d = d;
    g.R = d.R;
    g.kU = pb->kU <= 0 ? 1 : pb->kU;
    g.planes = reinterpret_cast<const int8_t*>(static_cast<const uint8_t*>(d_plain) + kHeader);
    g.nplanes = pb->plain_per_prime ? d.L * g.kU : g.kU;
    g.plane0 = plane_index(pb, l, 0);
    g.p = pb->primes[l];
    g.u_unsigned = pb->u_unsigned;
    g.o = o;
    const uint32_t* x = X0 + static_cast<int64_t>(l) * d.R * d.d2p;
    if (mv) return launch_mv(g, x, static_cast<uint8_t*>(d_ws) + ws_mv_off(pb, d), st);
    if (fused) return launch_fused(g, x, st);
    uint32_t* corr = ws_corr(pb, d, d_ws, l);
    if (!ovl || l == 0) {  // with split_overlap only the first prime is split on its own
      ctpt_status s2 = launch_split_prime(pb, x, d.R, d.d2p, g.p, ws_limbs(pb, d, d_ws, l), corr, st);
      if (s2 != CTPT_OK) return s2;
    }
    g.limbs = ws_limbs(pb, d, d_ws, l);
    if (needs_rowcorr(pb)) g.o.rowcorr = corr;
    if (ovl && l + 1 < d.L) g.sj = make_split_job(pb, d, X0, d_ws, l + 1);
    return launch_gemm(g, st, false);
  };
  if (pb->rescale) {
    // RNS Rescale by q_1 = p_{L−1} (Alg. 6 step 2 / Alg. 7 step 2): the last
    // prime's product first, kept per column [d3_loc][R] in the workspace; the other primes'
    // epilogues then emit ⌊x / p_{L−1}⌉ mod p_l directly.
    OutParams o{};
    o.AU = xlast;
    o.BU = xlast;
    o.rows_A = d.R;
    o.d1 = 0;
    o.R = d.R;
    o.d3_loc = d.d3_loc;
    s = run(d.L - 1, o);
    if (s != CTPT_OK) return s;
  }
  for (int l = 0; l < d.L_out; ++l) {
    OutParams o{};
    o.AU = d_AU ? d_AU + static_cast<int64_t>(l) * d.d3_loc * d.rows_A : nullptr;
    o.BU = d_BU + static_cast<int64_t>(l) * d.d3_loc * d.d1;
    o.rows_A = d.rows_A;
    o.d1 = d.d1;
    o.R = d.R;
    o.d3_loc = d.d3_loc;
    if (pb->rescale) {
      const uint32_t pl = pb->primes[d.L - 1], p = pb->primes[l];
      o.xlast = xlast;
      o.p_last = pl;
      o.p_last_inv = powmod_u32(pl % p, p - 2, p);  // p prime (Fermat)
    }
    s = run(l, o);
    if (s != CTPT_OK) return s;
  }
  return CTPT_OK;
}

}  // extern "C"

// =============================================================================================
// Host-pipelined executor: per-column ciphertexts in HOST memory → (A·U, B·U) in HOST memory.
// The stacked X of each prime is cut into row chunks; chunk i's host→device copy, chunk i−1's
// layout + split + GEMM and chunk i−2's device→host copy run concurrently on three streams
// (copy engines in both directions + the SMs), with two staging buffers per direction.
// =============================================================================================
namespace {

struct HostPlan {
  int64_t chunk;  // rows of X per chunk (multiple of 64)
  size_t in_bytes, cm_bytes, limb_bytes, out_bytes, corr_bytes, mv_bytes, total;
  std::vector<std::pair<int64_t, int64_t>> pieces;  // the row chunks [r0, r1) of one prime, in order
};

HostPlan host_plan(const Dims& d, int64_t chunk_rows) {
  HostPlan h;
  const int64_t Rr = (d.R + 63) / 64 * 64;
  if (chunk_rows > 0) {  // fixed chunks of chunk_rows (rounded to 64); a chunk may straddle A / B
    const int64_t c = std::max<int64_t>(64, std::min<int64_t>((chunk_rows + 63) / 64 * 64, Rr));
    for (int64_t r0 = 0; r0 < d.R; r0 += c) h.pieces.emplace_back(r0, std::min(d.R, r0 + c));
  } else {
    // default: ~6 chunks per prime (c3: 97 ms/step = 86 % of the concurrent-PCIe floor, vs 110 ms
    // with 4 chunks; profiles/r01/e2e_chunk_sweep.txt), cut separately within A's rows and B's rows
    // (a chunk up to 5/4 of the target is not split), so no copy carries a few-hundred-row sliver
    // of the other part: every 2-D copy moves the chunk's full width (an A part of rows_A ≤ 1.25 ×
    // target rows is one copy whose width is the whole host pitch)
    const int64_t target = std::max<int64_t>(64, ((d.R + 5) / 6 + 63) / 64 * 64);
    const int64_t seg[2][2] = {{0, d.rows_A}, {d.rows_A, d.R}};
    for (const auto& sg : seg) {
      const int64_t len = sg[1] - sg[0];
      if (len <= 0) continue;
      const int64_t n = len * 4 <= target * 5 ? 1 : (len + target - 1) / target;
      const int64_t piece = ((len + n - 1) / n + 63) / 64 * 64;
      for (int64_t r0 = sg[0]; r0 < sg[1]; r0 += piece) h.pieces.emplace_back(r0, std::min(sg[1], r0 + piece));
    }
  }
  int64_t c = 64;
  for (const auto& pc : h.pieces) c = std::max(c, pc.second - pc.first);
  h.chunk = c;
  h.in_bytes = align256(static_cast<size_t>(d.d2) * c * 4);
  h.cm_bytes = align256(static_cast<size_t>(c) * d.d2p * 4);
  h.limb_bytes = align256(limb_tile_bytes(c, d.d2p));
  h.out_bytes = align256(static_cast<size_t>(d.d3_loc) * c * 4);
  h.corr_bytes = align256(static_cast<size_t>(c) * 4);  // rowcorr of a chunk (unsigned-U mode)
  Dims dc = d;
  dc.R = c;
  h.mv_bytes = d.d3_loc <= kMvMaxD3 ? align256(mv_plan(dc).total) : 0;  // very-skinny kernel, per chunk
  h.total = 2 * h.in_bytes + h.cm_bytes + h.limb_bytes + 2 * h.out_bytes + h.corr_bytes + h.mv_bytes;
  return h;
}

ctpt_status launch_layout_cols(const uint32_t* a_colmajor, uint32_t* x, int64_t rows, int64_t d2, int64_t d2p,
                               cudaStream_t st) {
  LayoutParams P;
  memset(&P, 0, sizeof(P));
  P.a = a_colmajor;
  P.b = a_colmajor;  // never read: every row is an "A" row
  P.x = x;
  P.rows_A = rows;
  P.d1 = 0;
  P.R = rows;
  P.d2 = d2;
  P.d2p = d2p;
  dim3 grid(static_cast<unsigned>((rows + 63) / 64), static_cast<unsigned>((d2p + 63) / 64), 1);
  if (layout_vec_ok(rows, 0))
    k_layout_v4<<<grid, 256, 0, st>>>(P);
  else
    k_layout<<<grid, 256, 0, st>>>(P);
  CUDA_TRY(cudaGetLastError());
  return CTPT_OK;
}

struct StreamSet {
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev[10] = {};
  ~StreamSet() {  // resources are released once the enqueued work completes
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (h2d) cudaStreamDestroy(h2d);
    if (d2h) cudaStreamDestroy(d2h);
  }
};

#ifdef CTPT_HOST_TRACE
// Diagnostic build only (tools/ab_build.py OUT.so -DCTPT_HOST_TRACE): timing events around every
// chunk's H2D, compute and D2H; the call synchronises at the end and prints the timeline (ms from
// the fork) to stderr.  The release library never synchronises in ctpt_matmul_host*.
struct HostTrace {
  std::vector<cudaEvent_t> ev;
  cudaEvent_t rec(cudaStream_t st) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    ev.push_back(e);
    return e;
  }
};
#endif

// The staging buffers of one pipeline serve every unit of a batch: each region is sized for the
// largest unit.
struct HostWs {
  size_t in_bytes = 0, cm_bytes = 0, limb_bytes = 0, out_bytes = 0, corr_bytes = 0, mv_bytes = 0;
  size_t total() const { return 2 * in_bytes + cm_bytes + limb_bytes + 2 * out_bytes + corr_bytes + mv_bytes; }
  void cover(const HostPlan& h) {
    in_bytes = std::max(in_bytes, h.in_bytes);
    cm_bytes = std::max(cm_bytes, h.cm_bytes);
    limb_bytes = std::max(limb_bytes, h.limb_bytes);
    out_bytes = std::max(out_bytes, h.out_bytes);
    corr_bytes = std::max(corr_bytes, h.corr_bytes);
    mv_bytes = std::max(mv_bytes, h.mv_bytes);
  }
};

ctpt_status host_ws_units(int32_t n, const ctpt_problem* probs, int64_t chunk_rows, HostWs& ws) {
  if (n < 1 || !probs) return fail(CTPT_ERR_ARG, "need n >= 1 problems");
  for (int32_t u = 0; u < n; ++u) {
    Dims d;
    ctpt_status s = check_problem(probs + u, d);
    if (s != CTPT_OK) return s;
    if (probs[u].rescale) return fail(CTPT_ERR_UNSUPPORTED, "ctpt_matmul_host does not Rescale (use ctpt_matmul)");
    ws.cover(host_plan(d, chunk_rows));
  }
  return CTPT_OK;
}

}  // namespace

extern "C" {

ctpt_status ctpt_host_workspace_bytes(const ctpt_problem* pb, int64_t chunk_rows, size_t* bytes) {
  return ctpt_host_workspace_bytes_units(1, pb, chunk_rows, bytes);
}

ctpt_status ctpt_host_workspace_bytes_units(int32_t n, const ctpt_problem* probs, int64_t chunk_rows, size_t* bytes) {
  if (!bytes) return fail(CTPT_ERR_ARG, "bytes is NULL");
  HostWs ws;
  ctpt_status s = host_ws_units(n, probs, chunk_rows, ws);
  if (s != CTPT_OK) return s;
  *bytes = ws.total();
  return CTPT_OK;
}

ctpt_status ctpt_matmul_host(const ctpt_problem* pb, const uint32_t* h_a, const uint32_t* h_b, const void* d_plain,
                             uint32_t* h_AU, uint32_t* h_BU, void* d_ws, size_t ws_bytes, int64_t chunk_rows,
                             void* stream) {
  return ctpt_matmul_host_units(1, pb, &h_a, &h_b, &d_plain, &h_AU, &h_BU, d_ws, ws_bytes, chunk_rows, stream);
}

ctpt_status ctpt_matmul_host_units(int32_t n, const ctpt_problem* probs, const uint32_t* const* h_as,
                                   const uint32_t* const* h_bs, const void* const* d_plains, uint32_t* const* h_AUs,
                                   uint32_t* const* h_BUs, void* d_ws, size_t ws_bytes, int64_t chunk_rows,
                                   void* stream) {
  HostWs hw;
  ctpt_status s = host_ws_units(n, probs, chunk_rows, hw);
  if (s != CTPT_OK) return s;
  if (!h_as || !h_bs || !d_plains || !h_AUs || !h_BUs || !d_ws) return fail(CTPT_ERR_ARG, "null pointer");
  if (ws_bytes < hw.total()) return fail(CTPT_ERR_ARG, "workspace too small (%zu < %zu)", ws_bytes, hw.total());
  for (int32_t u = 0; u < n; ++u) {  // validate every unit before enqueueing anything
    Dims d;
    check_problem(probs + u, d);
    if (((!h_as[u] || !h_AUs[u]) && d.rows_A > 0) || !h_bs[u] || !d_plains[u] || !h_BUs[u])
      return fail(CTPT_ERR_ARG, "null pointer (unit %d)", u);
  }
  std::vector<Path> paths(static_cast<size_t>(n));
  for (int32_t u = 0; u < n; ++u) {
    Dims d;
    check_problem(probs + u, d);
    s = choose_path(probs + u, d, paths[static_cast<size_t>(u)]);
    if (s != CTPT_OK) return s;
  }
  cudaStream_t sc = static_cast<cudaStream_t>(stream);
  uint8_t* w = static_cast<uint8_t*>(d_ws);
  uint32_t* in[2] = {reinterpret_cast<uint32_t*>(w), reinterpret_cast<uint32_t*>(w + hw.in_bytes)};
  uint32_t* cm = reinterpret_cast<uint32_t*>(w + 2 * hw.in_bytes);
  void* limbs = w + 2 * hw.in_bytes + hw.cm_bytes;
  uint32_t* ob[2] = {reinterpret_cast<uint32_t*>(w + 2 * hw.in_bytes + hw.cm_bytes + hw.limb_bytes),
                     reinterpret_cast<uint32_t*>(w + 2 * hw.in_bytes + hw.cm_bytes + hw.limb_bytes + hw.out_bytes)};
  uint32_t* corr = reinterpret_cast<uint32_t*>(w + 2 * hw.in_bytes + hw.cm_bytes + hw.limb_bytes + 2 * hw.out_bytes);
  uint8_t* mvws = w + 2 * hw.in_bytes + hw.cm_bytes + hw.limb_bytes + 2 * hw.out_bytes + hw.corr_bytes;

  StreamSet ss;
  CUDA_TRY(cudaStreamCreateWithFlags(&ss.h2d, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&ss.d2h, cudaStreamNonBlocking));
  for (auto& e : ss.ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaEvent_t ev_start = ss.ev[0], ev_end = ss.ev[1];
  cudaEvent_t* in_ready = ss.ev + 2;  // [2]
  cudaEvent_t* in_free = ss.ev + 4;   // [2]
  cudaEvent_t* out_ready = ss.ev + 6; // [2]
  cudaEvent_t* out_free = ss.ev + 8;  // [2]

  // fork: copies start only after prior work on the caller's stream (e.g. the precompute)
  CUDA_TRY(cudaEventRecord(ev_start, sc));
  CUDA_TRY(cudaStreamWaitEvent(ss.h2d, ev_start, 0));
  CUDA_TRY(cudaStreamWaitEvent(ss.d2h, ev_start, 0));
#ifdef CTPT_HOST_TRACE
  HostTrace tr;
  tr.rec(sc);
#define CTPT_TRACE(st) tr.rec(st)
#else
#define CTPT_TRACE(st) ((void)0)
#endif

  // One pipeline over every (unit, prime, row chunk): the chunk counter `it` and the staging
  // buffers run on across unit boundaries, so unit u+1's first copies overlap unit u's last GEMMs
  // and copies (one fill and one drain per call, not per unit).
  int64_t it = 0;
  for (int32_t u = 0; u < n; ++u) {
    const ctpt_problem* pb = probs + u;
    Dims d;
    check_problem(pb, d);
    const HostPlan hp = host_plan(d, chunk_rows);
    const Path path = paths[static_cast<size_t>(u)];
    GemmArgs g{};
    gemm_args_from_problem(g, pb);
    g.d = d;
    g.kU = pb->kU <= 0 ? 1 : pb->kU;
    g.planes = reinterpret_cast<const int8_t*>(static_cast<const uint8_t*>(d_plains[u]) + kHeader);
    g.nplanes = pb->plain_per_prime ? d.L * g.kU : g.kU;
    g.limbs = limbs;
    g.u_unsigned = pb->u_unsigned;
    if (needs_rowcorr(pb)) g.o.rowcorr = corr;
    const bool fused = path != Path::SplitGemm;
    const bool mv = path == Path::Mv;

    for (int l = 0; l < d.L; ++l) {
      const uint32_t* a_l = h_as[u] + static_cast<int64_t>(l) * d.d2 * d.rows_A;
      const uint32_t* b_l = h_bs[u] + static_cast<int64_t>(l) * d.d2 * d.d1;
      uint32_t* AU_l = h_AUs[u] + static_cast<int64_t>(l) * d.d3_loc * d.rows_A;
      uint32_t* BU_l = h_BUs[u] + static_cast<int64_t>(l) * d.d3_loc * d.d1;
      for (size_t pi = 0; pi < hp.pieces.size(); ++pi, ++it) {
        const int b = static_cast<int>(it & 1);
        const int64_t r0 = hp.pieces[pi].first, r1 = hp.pieces[pi].second, rows = r1 - r0;
        const int64_t na = std::max<int64_t>(0, std::min(r1, d.rows_A) - r0), nb = rows - na;
        const int64_t rb0 = r0 + na - d.rows_A;  // first B row of the chunk (if nb > 0)
        // 1. host → device: the chunk's rows of every ciphertext column, packed col-major [d2][rows]
        if (it >= 2) CUDA_TRY(cudaStreamWaitEvent(ss.h2d, in_free[b], 0));
        CTPT_TRACE(ss.h2d);
        if (na)
          CUDA_TRY(cudaMemcpy2DAsync(in[b], rows * 4, a_l + r0, d.rows_A * 4, na * 4, d.d2, cudaMemcpyHostToDevice,
                                     ss.h2d));
        if (nb)
          CUDA_TRY(cudaMemcpy2DAsync(in[b] + na, rows * 4, b_l + rb0, d.d1 * 4, nb * 4, d.d2, cudaMemcpyHostToDevice,
                                     ss.h2d));
        CUDA_TRY(cudaEventRecord(in_ready[b], ss.h2d));
        CTPT_TRACE(ss.h2d);
        // 2. layout + split + GEMM on the caller's stream
        CUDA_TRY(cudaStreamWaitEvent(sc, in_ready[b], 0));
        CTPT_TRACE(sc);
        s = launch_layout_cols(in[b], cm, rows, d.d2, d.d2p, sc);
        if (s != CTPT_OK) return s;
        CUDA_TRY(cudaEventRecord(in_free[b], sc));
        if (!fused) {
          s = launch_split_prime(pb, cm, rows, d.d2p, pb->primes[l], limbs, corr, sc);
          if (s != CTPT_OK) return s;
        }
        if (it >= 2) CUDA_TRY(cudaStreamWaitEvent(sc, out_free[b], 0));
        CTPT_TRACE(sc);
        g.R = rows;
        g.p = pb->primes[l];
        g.plane0 = plane_index(pb, l, 0);
        g.o.AU = ob[b];
        g.o.BU = ob[b];
        g.o.rows_A = rows;
        g.o.d1 = 0;
        g.o.R = rows;
        g.o.d3_loc = d.d3_loc;
        s = mv ? launch_mv(g, cm, mvws, sc) : fused ? launch_fused(g, cm, sc) : launch_gemm(g, sc, false);
        if (s != CTPT_OK) return s;
        CUDA_TRY(cudaEventRecord(out_ready[b], sc));
        CTPT_TRACE(sc);
        // 3. device → host: rows [r0, r1) of every output column
        CUDA_TRY(cudaStreamWaitEvent(ss.d2h, out_ready[b], 0));
        CTPT_TRACE(ss.d2h);
        if (na)
          CUDA_TRY(cudaMemcpy2DAsync(AU_l + r0, d.rows_A * 4, ob[b], rows * 4, na * 4, d.d3_loc,
                                     cudaMemcpyDeviceToHost, ss.d2h));
        if (nb)
          CUDA_TRY(cudaMemcpy2DAsync(BU_l + rb0, d.d1 * 4, ob[b] + na, rows * 4, nb * 4, d.d3_loc,
                                     cudaMemcpyDeviceToHost, ss.d2h));
        CUDA_TRY(cudaEventRecord(out_free[b], ss.d2h));
        CTPT_TRACE(ss.d2h);
      }
    }
  }
  // join: the caller's stream completes only after the last device→host copy
  CUDA_TRY(cudaEventRecord(ev_end, ss.d2h));
  CUDA_TRY(cudaStreamWaitEvent(sc, ev_end, 0));
#ifdef CTPT_HOST_TRACE
  // per chunk: h2d start, h2d end, compute start (input ready), GEMM start (output buffer free),
  // compute end, d2h start, d2h end — ms from the fork
  cudaStreamSynchronize(sc);
  for (size_t i = 1; i + 7 <= tr.ev.size(); i += 7) {
    float t[7];
    for (int k = 0; k < 7; ++k) cudaEventElapsedTime(&t[k], tr.ev[0], tr.ev[i + k]);
    fprintf(stderr, "trace chunk %zu h2d %.3f %.3f comp %.3f %.3f %.3f d2h %.3f %.3f\n", (i - 1) / 7, t[0], t[1], t[2],
            t[3], t[4], t[5], t[6]);
  }
  for (auto e : tr.ev) cudaEventDestroy(e);
#endif
#undef CTPT_TRACE
  return CTPT_OK;
}

}  // extern "C"

// =============================================================================================
// Multi-GPU gather over peer memory: CUDA IPC plumbing so a rank's ctpt_matmul
// can store its unit's outputs straight into rank 0's gathered [L][d3][rows] buffers.
// =============================================================================================
extern "C" {

ctpt_status ctpt_ipc_export(const void* d_ptr, void* handle, uint64_t* offset) {
  if (!d_ptr || !handle || !offset) return fail(CTPT_ERR_ARG, "null pointer");
  static_assert(sizeof(cudaIpcMemHandle_t) == CTPT_IPC_HANDLE_BYTES, "IPC handle size");
  auto range = get_addr_range();
  if (!range) return fail(CTPT_ERR_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  const CUresult r = range(&base, &size, reinterpret_cast<CUdeviceptr>(d_ptr));
  if (r != CUDA_SUCCESS) return fail(CTPT_ERR_CUDA, "cuMemGetAddressRange failed (%d)", static_cast<int>(r));
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  memcpy(handle, &h, sizeof(h));
  *offset = static_cast<uint64_t>(reinterpret_cast<CUdeviceptr>(d_ptr) - base);
  return CTPT_OK;
}

ctpt_status ctpt_ipc_open(const void* handle, uint64_t offset, void** d_base, void** d_ptr) {
  if (!handle || !d_base || !d_ptr) return fail(CTPT_ERR_ARG, "null pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  // opened in the calling thread's CURRENT device context: the mapping is usable by that device's
  // kernels, with peer access to the owning GPU enabled on demand
  CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *d_base = base;
  *d_ptr = static_cast<uint8_t*>(base) + offset;
  return CTPT_OK;
}

ctpt_status ctpt_ipc_close(void* d_base) {
  if (!d_base) return fail(CTPT_ERR_ARG, "null pointer");
  CUDA_TRY(cudaIpcCloseMemHandle(d_base));
  return CTPT_OK;
}

ctpt_status ctpt_peer_access(int32_t device, int32_t peer, int32_t* can) {
  if (!can) return fail(CTPT_ERR_ARG, "null pointer");
  if (device == peer) {
    *can = 1;
    return CTPT_OK;
  }
  int c = 0;
  CUDA_TRY(cudaDeviceCanAccessPeer(&c, device, peer));
  *can = c;
  return CTPT_OK;
}

}  // extern "C"
