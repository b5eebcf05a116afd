// kernels.cuh — the memory-bound kernels of the CP-MM path (layout, plaintext precompute,
// limb split) and the shared epilogue arithmetic (limb recombination + Barrett reduction).
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace ctpt {

// ------------------------------------------------------------------------------------------
// Epilogue arithmetic ("compute their sum using integer arithmetic …
// then reduce it modulo the modulus").
// ------------------------------------------------------------------------------------------
struct ModP {
  uint32_t p;
  uint64_t mu;   // floor(2^64 / p)
  uint64_t off;  // p * ceil(2^56 / p): makes t + off non-negative for |t| < 2^56
  // Montgomery form of the recombination (limb sums known non-negative: u8 limbs × the u8 U plane)
  int32_t redc;  // 0: Barrett on the int64 sum; 1: Montgomery, sums < 2^31; 2: Montgomery, sums < 2^30
  uint32_t pinv; // −p^{−1} mod 2^32
  uint32_t w[4]; // 2^{8ℓ + 32} mod p
  uint64_t p32;  // p · 2^32
};

// r = x mod p for x < 2^64 (Barrett with a 64-bit reciprocal; q_est ∈ {q-1, q}).
__device__ __forceinline__ uint32_t barrett64(uint64_t x, const ModP& m) {
  uint64_t q = __umul64hi(x, m.mu);
  uint64_t r = x - q * m.p;
  r = (r >= m.p) ? r - m.p : r;
  r = (r >= m.p) ? r - m.p : r;
  return static_cast<uint32_t>(r);
}

// t = C0 + 2^8 C1 + 2^16 C2 + 2^24 C3 (the exact limb recombination), reduced to [0, p).
//  * redc = 0 (general, C_ℓ signed): t in int64, Barrett — ≈ 30 instructions per output;
//  * redc > 0 (C_ℓ ≥ 0: u8 limbs × the u8 U plane, C_ℓ < 2^31 by the d2 ≤ 33025 refusal):
//    x = Σ_ℓ C_ℓ·w_ℓ with w_ℓ = 2^{8ℓ+32} mod p (four IMAD.WIDE.U32), so x ≡ t·2^32 (mod p), then
//    one Montgomery reduction REDC(x) = x·2^{−32} mod p ≡ t: q = x·(−p^{−1}) mod 2^32,
//    y = (x + q·p) / 2^32 < 2p, one min-subtract — ≈ 8 instructions.  REDC needs x < p·2^32:
//    redc = 2 when every C_ℓ < 2^30 (then x < 4·2^30·p), redc = 1 subtracts p·2^32 once
//    (x < 4·2^31·p = 2·p·2^32).  The epilogue's ALU work is the issue-rate limit of the
//    k_gemm_tc epilogue warps, which drain a tile in the time the MMAs compute the next.
__device__ __forceinline__ uint32_t recombine_mod(int32_t c0, int32_t c1, int32_t c2, int32_t c3, const ModP& m) {
  if (m.redc) {
    uint64_t x = static_cast<uint64_t>(static_cast<uint32_t>(c0)) * m.w[0];
    x += static_cast<uint64_t>(static_cast<uint32_t>(c1)) * m.w[1];
    x += static_cast<uint64_t>(static_cast<uint32_t>(c2)) * m.w[2];
    x += static_cast<uint64_t>(static_cast<uint32_t>(c3)) * m.w[3];
    if (m.redc == 1) x = (x >= m.p32) ? x - m.p32 : x;
    const uint32_t q = static_cast<uint32_t>(x) * m.pinv;
    const uint32_t y = static_cast<uint32_t>((x + static_cast<uint64_t>(q) * m.p) >> 32);  // < 2p
    return min(y, y - m.p);  // y − p wraps above y when y < p
  }
  int64_t t = static_cast<int64_t>(c0) + (static_cast<int64_t>(c1) << 8) + (static_cast<int64_t>(c2) << 16) +
              (static_cast<int64_t>(c3) << 24);
  return barrett64(static_cast<uint64_t>(t + static_cast<int64_t>(m.off)), m);
}

// (prev + w·r) mod p for the k_U > 1 accumulation passes (Σ_i 2^{8i} (A·U_i) mod p).
__device__ __forceinline__ uint32_t accum_mod(uint32_t prev, uint32_t r, uint32_t w, const ModP& m) {
  uint64_t x = static_cast<uint64_t>(r) * w + prev;  // < 2^62 + 2^31
  return barrett64(x, m);
}

// ------------------------------------------------------------------------------------------
// Layout: per-column ciphertexts (column-major A [d2][rows_A], B [d2][d1] per prime) →
// stacked K-major X = [A; B] int32 [R][d2p].  Pure permutation (§8(a) a1).
// 64x64 tiles through shared memory so both the reads (along r) and writes (along k) coalesce.
// ------------------------------------------------------------------------------------------
struct LayoutParams {
  const uint32_t* a;  // [L][d2][rows_A]
  const uint32_t* b;  // [L][d2][d1]
  uint32_t* x;        // [L][R][d2p]
  int64_t rows_A, d1, R, d2, d2p;
  uint32_t p_arr[64];
  int32_t validate;
  uint32_t* bad_flag;  // device word, OR-ed with 1 on a residue ≥ p
};

__global__ void __launch_bounds__(256) k_layout(const __grid_constant__ LayoutParams P) {
  __shared__ uint32_t tile[64][65];
  const int l = blockIdx.z;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 64;
  const int64_t k0 = static_cast<int64_t>(blockIdx.y) * 64;
  const uint32_t p = P.p_arr[l];
  const uint32_t* a = P.a + static_cast<int64_t>(l) * P.d2 * P.rows_A;
  const uint32_t* b = P.b + static_cast<int64_t>(l) * P.d2 * P.d1;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 64 x 4
  bool bad = false;
  // read: element (k, r) with r fastest
  for (int kk = ty; kk < 64; kk += 4) {
    const int64_t k = k0 + kk, r = r0 + tx;
    uint32_t v = 0;
    if (k < P.d2 && r < P.R) {
      v = (r < P.rows_A) ? a[k * P.rows_A + r] : b[k * P.d1 + (r - P.rows_A)];
      bad |= (v >= p);
    }
    tile[kk][tx] = v;
  }
  __syncthreads();
  uint32_t* x = P.x + static_cast<int64_t>(l) * P.R * P.d2p;
  for (int rr = ty; rr < 64; rr += 4) {
    const int64_t r = r0 + rr, k = k0 + tx;
    if (r < P.R && k < P.d2p) x[r * P.d2p + k] = tile[tx][rr];  // zero for k >= d2
  }
  if (P.validate && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(P.bad_flag, 1u);
}

// The same permutation with 16-byte accesses on both sides (rows_A and d1 multiples of 4, so a
// 4-row chunk never straddles A and B and every vector is aligned).  One 64 (k) × 64 (r) tile
// per block: 4 LDG.128 per thread (16 r-chunks × 64 k), stored into shared memory with the
// 16-byte chunk c of row k at position c ^ ((k >> 2) & 7); then each thread owns a 4 (k) × 4 (r)
// block — 4 LDS.128 (conflict-free under that swizzle), a register transpose, 4 STG.128 that
// 16 lanes turn into one 256-byte row segment of X.
__global__ void __launch_bounds__(256) k_layout_v4(const __grid_constant__ LayoutParams P) {
  __shared__ __align__(16) uint32_t tile[64 * 64];
  const int l = blockIdx.z;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 64;
  const int64_t k0 = static_cast<int64_t>(blockIdx.y) * 64;
  const uint32_t p = P.p_arr[l];
  const uint32_t* a = P.a + static_cast<int64_t>(l) * P.d2 * P.rows_A;
  const uint32_t* b = P.b + static_cast<int64_t>(l) * P.d2 * P.d1;
  const int c = threadIdx.x & 15;  // 4-row chunk of the tile
  const int kq0 = threadIdx.x >> 4;  // 0..15
  const int64_t r = r0 + 4 * c;
  bool bad = false;
  uint4 v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t k = k0 + kq0 + 16 * i;
    v[i] = make_uint4(0u, 0u, 0u, 0u);
    if (k < P.d2 && r < P.R)
      v[i] = (r < P.rows_A) ? __ldcs(reinterpret_cast<const uint4*>(a + k * P.rows_A + r))
                            : __ldcs(reinterpret_cast<const uint4*>(b + k * P.d1 + (r - P.rows_A)));
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int kk = kq0 + 16 * i;
    bad |= (v[i].x >= p) | (v[i].y >= p) | (v[i].z >= p) | (v[i].w >= p);
    *reinterpret_cast<uint4*>(&tile[kk * 64 + ((c ^ ((kk >> 2) & 7)) << 2)]) = v[i];
  }
  __syncthreads();
  const int kq = threadIdx.x & 15;  // k = 4kq .. 4kq+3
  const int rq = threadIdx.x >> 4;  // r = 4rq .. 4rq+3
  uint4 w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int kk = 4 * kq + i;
    w[i] = *reinterpret_cast<const uint4*>(&tile[kk * 64 + ((rq ^ ((kk >> 2) & 7)) << 2)]);
  }
  uint32_t* x = P.x + static_cast<int64_t>(l) * P.R * P.d2p;
  const int64_t k = k0 + 4 * kq;
  if (k < P.d2p) {  // d2p is a multiple of 16: a 4-k quad is all in or all out
    const uint4 o0 = make_uint4(w[0].x, w[1].x, w[2].x, w[3].x), o1 = make_uint4(w[0].y, w[1].y, w[2].y, w[3].y),
                o2 = make_uint4(w[0].z, w[1].z, w[2].z, w[3].z), o3 = make_uint4(w[0].w, w[1].w, w[2].w, w[3].w);
    const int64_t rr = r0 + 4 * rq;
    if (rr + 0 < P.R) __stcs(reinterpret_cast<uint4*>(x + (rr + 0) * P.d2p + k), o0);
    if (rr + 1 < P.R) __stcs(reinterpret_cast<uint4*>(x + (rr + 1) * P.d2p + k), o1);
    if (rr + 2 < P.R) __stcs(reinterpret_cast<uint4*>(x + (rr + 2) * P.d2p + k), o2);
    if (rr + 3 < P.R) __stcs(reinterpret_cast<uint4*>(x + (rr + 3) * P.d2p + k), o3);
  }
  if (P.validate && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(P.bad_flag, 1u);
}

// ------------------------------------------------------------------------------------------
// Limb split (inside the timed ctpt_matmul): x = Σ_{ℓ<4} x_ℓ 2^{8ℓ},
// x_ℓ ∈ [0,255] — the digits of Lemma le:strategy1's decomposition with
// K = 2^8 for a canonical (non-negative) residue.  int32 [n] → uint8 [4][n]; 16 elements per
// thread: 4 × 16-B loads, an 8-PRMT 4×4 byte transpose per 4 words, 4 × 16-B stores.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void byte_transpose4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t& l0,
                                                uint32_t& l1, uint32_t& l2, uint32_t& l3) {
  const uint32_t t0 = __byte_perm(w0, w1, 0x5140), t1 = __byte_perm(w0, w1, 0x7362);
  const uint32_t t2 = __byte_perm(w2, w3, 0x5140), t3 = __byte_perm(w2, w3, 0x7362);
  l0 = __byte_perm(t0, t2, 0x5410);
  l1 = __byte_perm(t0, t2, 0x7632);
  l2 = __byte_perm(t1, t3, 0x5410);
  l3 = __byte_perm(t1, t3, 0x7632);
}

// Limb planes in 32-KB tiles: limb ℓ of X[r][k] lives at byte
//   ((r / 64) · nkb + k / 128) · 32768 + ℓ · 8192 + (r % 64) · 128 + k % 128,   nkb = ⌈d2p / 128⌉,
// i.e. each (64-row, 128-K) tile of all four limbs — one TMA box of the GEMM — is one contiguous
// 32-KB block (measured: the GEMM's main loop +3.9 %, fewer DRAM-latency bubbles than 256 strided
// 128-B rows; profiles/r01/gemm_breakdown/).  K columns d2p .. 128·nkb are written as zeros (they
// enter every output's K sum); rows R .. 64·⌈R/64⌉ are never written (they only reach outputs
// that are not stored).
__device__ __forceinline__ int64_t limb_tile_off(int64_t r, int64_t k, int64_t nkb) {
  return (((r >> 6) * nkb + (k >> 7)) << 15) + ((r & 63) << 7) + (k & 127);
}

__global__ void __launch_bounds__(256) k_split(const uint4* __restrict__ x, uint8_t* __restrict__ limbs, int64_t R,
                                               int64_t d2p16, int64_t nkb) {
  // one thread per 16 consecutive residues (16 | 128, so they share a tile); x row stride d2p
  const int64_t kp16 = nkb * 8;
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < R * kp16;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = g / kp16, c = g - r * kp16;
    uint4 w[4] = {};
    if (c < d2p16) {
#pragma unroll
      for (int i = 0; i < 4; ++i) w[i] = __ldcs(x + 4 * (r * d2p16 + c) + i);  // streaming: read once
    }
    uint32_t o[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) byte_transpose4(w[i].x, w[i].y, w[i].z, w[i].w, o[0][i], o[1][i], o[2][i], o[3][i]);
    uint8_t* t = limbs + limb_tile_off(r, 16 * c, nkb);
#pragma unroll
    for (int l = 0; l < 4; ++l) *reinterpret_cast<uint4*>(t + l * 8192) = make_uint4(o[l][0], o[l][1], o[l][2], o[l][3]);
  }
}
__global__ void __launch_bounds__(256) k_split_rows(const uint4* __restrict__ x, uint8_t* __restrict__ limbs,
                                                   uint32_t* __restrict__ rowcorr, int64_t R, int64_t d2p16,
                                                   int64_t nkb, uint32_t p, uint32_t off_mod_p) {
  __shared__ uint64_t part[8];
  const int64_t kp16 = nkb * 8;
  for (int64_t r = blockIdx.x; r < R; r += gridDim.x) {
    uint64_t sum = 0;
    for (int64_t c = threadIdx.x; c < kp16; c += blockDim.x) {
      uint4 w[4] = {};
      if (c < d2p16) {
#pragma unroll
        for (int i = 0; i < 4; ++i) w[i] = __ldcs(x + 4 * (r * d2p16 + c) + i);
      }
      uint32_t o[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        sum += static_cast<uint64_t>(w[i].x) + w[i].y + w[i].z + w[i].w;
        byte_transpose4(w[i].x, w[i].y, w[i].z, w[i].w, o[0][i], o[1][i], o[2][i], o[3][i]);
      }
      uint8_t* t = limbs + limb_tile_off(r, 16 * c, nkb);
#pragma unroll
      for (int l = 0; l < 4; ++l) *reinterpret_cast<uint4*>(t + l * 8192) = make_uint4(o[l][0], o[l][1], o[l][2], o[l][3]);
    }
#pragma unroll
    for (int s = 16; s; s >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, s);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t t = 0;
      for (int w = 0; w < (blockDim.x >> 5); ++w) t += part[w];
      rowcorr[r] = static_cast<uint32_t>((t % p) * off_mod_p % p);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------
// Plaintext precompute (§8(a) a2): U int64 [d2][d3] → balanced int8 digits of the centred
// residue, written transposed (U^T, K-major) as planes [kU][d3][d2p].
// ------------------------------------------------------------------------------------------
// min / max of n int64 values: 16-byte loads, four in flight per thread per iteration (a grid of a
// few CTAs per SM streams 2 GB at HBM speed), warp shuffles, one atomic pair per warp.
__global__ void __launch_bounds__(256) k_minmax_i64(const int64_t* __restrict__ u, int64_t n, long long* mm /*[2]: min, max*/) {
  long long lo = LLONG_MAX, hi = LLONG_MIN;
  auto take = [&](long long v) {
    lo = v < lo ? v : lo;
    hi = v > hi ? v : hi;
  };
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nthr = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const bool vec = (reinterpret_cast<uintptr_t>(u) & 15) == 0;
  const int64_t n2 = vec ? n / 2 : 0;  // 16-byte pairs
  const longlong2* u2 = reinterpret_cast<const longlong2*>(u);
  int64_t i = tid;
  for (; i + 3 * nthr < n2; i += 4 * nthr) {
    longlong2 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = __ldcs(u2 + i + q * nthr);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      take(v[q].x);
      take(v[q].y);
    }
  }
  for (; i < n2; i += nthr) {
    const longlong2 v = __ldcs(u2 + i);
    take(v.x);
    take(v.y);
  }
  for (int64_t k = 2 * n2 + tid; k < n; k += nthr) take(u[k]);
  for (int o = 16; o; o >>= 1) {
    long long a = __shfl_xor_sync(0xffffffffu, lo, o), b = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
  }
}

// balanced digit: d = ((x + 128) mod 256) - 128, x <- (x - d) / 256
__device__ __forceinline__ int8_t balanced_digit(int64_t& x) {
  const int64_t d = ((x + 128) & 255) - 128;
  x = (x - d) >> 8;
  return static_cast<int8_t>(d);
}

struct PlainParams {
  const int64_t* u;     // [d2][d3] (int64 mode)
  const uint32_t* ures; // [L][d2][d3] (rns mode)
  int8_t* planes;       // [nplanes][d3][d2p]
  int64_t d2, d3, d2p;
  int32_t kU;
  int32_t rns;          // 0: shared planes from int64 U; 1: per-prime planes from residues
  int32_t unsigned_plane;  // 1: one u8 plane holding U + u_offset ∈ [0, 255] (int64 mode, kU = 1)
  int64_t u_offset;
  uint32_t p_arr[64];
};

// Tile: 128 k × 32 j; grid: (ceil(d2p/128), ceil(d3/32), L or 1); block 256 = 32 (j) × 8.  Reads
// coalesce along j (a warp reads 32 consecutive entries of U's row k); the digits are transposed
// through shared memory ([32 j][132 B]: the 33-word row pitch makes the byte writes of a warp hit
// 32 distinct banks) and written as one 16-byte store per thread (a warp writes 4 rows j of
// 128 contiguous k bytes).
constexpr int PLAIN_TK = 128, PLAIN_TJ = 32, PLAIN_PITCH = PLAIN_TK + 4;
__global__ void __launch_bounds__(256) k_plain(const __grid_constant__ PlainParams P) {
  __shared__ __align__(16) uint8_t t[4][PLAIN_TJ][PLAIN_PITCH];
  const int l = blockIdx.z;
  const int64_t k0 = static_cast<int64_t>(blockIdx.x) * PLAIN_TK, j0 = static_cast<int64_t>(blockIdx.y) * PLAIN_TJ;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t j = j0 + tx;
  for (int kk = ty; kk < PLAIN_TK; kk += 8) {
    const int64_t k = k0 + kk;
    const bool in = k < P.d2 && j < P.d3;
    int64_t x = 0;
    if (in) {
      if (P.rns) {
        const uint32_t p = P.p_arr[l];
        const uint32_t v = P.ures[(static_cast<int64_t>(l) * P.d2 + k) * P.d3 + j];
        x = (v > p / 2) ? static_cast<int64_t>(v) - p : static_cast<int64_t>(v);  // centred residue
      } else {
        x = P.u[k * P.d3 + j];
      }
    }
    if (P.unsigned_plane) {
      t[0][tx][kk] = in ? static_cast<uint8_t>(x + P.u_offset) : 0;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) t[i][tx][kk] = (i < P.kU) ? static_cast<uint8_t>(balanced_digit(x)) : 0;
    }
  }
  __syncthreads();
  // thread → row jj = threadIdx / 8, 16-byte chunk c = threadIdx % 8 (k = k0 + 16c .. +15)
  const int jj = threadIdx.x >> 3, c = threadIdx.x & 7;
  const int64_t jw = j0 + jj, kw = k0 + 16 * c;
  if (jw < P.d3 && kw < P.d2p) {  // d2p is a multiple of 16 (of 128), so a chunk never straddles it
    for (int i = 0; i < P.kU; ++i) {
      const uint32_t* src = reinterpret_cast<const uint32_t*>(&t[i][jj][16 * c]);
      const int64_t plane = static_cast<int64_t>(l) * P.kU + i;
      *reinterpret_cast<uint4*>(P.planes + (plane * P.d3 + jw) * P.d2p + kw) = make_uint4(src[0], src[1], src[2], src[3]);
    }
  }
}

// ------------------------------------------------------------------------------------------
// Epilogue output routing shared by both GEMMs: row r of the stacked X is row r of A'
// (r < rows_A) or row r - rows_A of B'; output column j is contiguous (per-column layout).
// ------------------------------------------------------------------------------------------
struct OutParams {
  uint32_t* AU;  // [d3_loc][rows_A]
  uint32_t* BU;  // [d3_loc][d1]
  int64_t rows_A, d1, R, d3_loc;
  uint32_t w;          // 2^{8i} mod p for pass i
  int32_t accumulate;  // pass i > 0: out = (out + w·r) mod p
  // RNS Rescale by the last prime q_1 = p_L of the basis (Alg. 6/7 step 2),
  // applied on the final pass when xlast != nullptr: xlast = the product's residues mod p_L,
  // per column [d3_loc][R] (stacked rows); out = (x − [x]_{p_L}) · p_L^{-1} mod p.
  const uint32_t* xlast;
  uint32_t p_last, p_last_inv;
  // Unsigned-U mode (planes hold U' = U + u_offset ≥ 0): X·U = X·U' − u_offset·Σ_k X[r][k], so
  // the epilogue subtracts rowcorr[r] = u_offset·Σ_k X[r][k] mod p (nullptr: nothing to subtract).
  const uint32_t* rowcorr;
};

__device__ __forceinline__ uint32_t* out_ptr(const OutParams& o, int64_t j, int64_t r) {
  CTPT_CHECK(j >= 0 && j < o.d3_loc && r >= 0 && r < o.R);
  return (r < o.rows_A) ? o.AU + j * o.rows_A + r : o.BU + j * o.d1 + (r - o.rows_A);
}

// y = ⌊x / p_L⌉ mod p from x mod p (v) and x mod p_L (xl): with c the centred residue of x mod
// p_L, (x − c)/p_L is the rounded quotient (p_L odd: no ties) and ≡ (v − c)·p_L^{-1} (mod p).
__device__ __forceinline__ uint32_t rescale_last(uint32_t v, uint32_t xl, const OutParams& o, const ModP& m) {
  const int64_t c = (xl > (o.p_last >> 1)) ? static_cast<int64_t>(xl) - o.p_last : static_cast<int64_t>(xl);
  const uint32_t cm = barrett64(static_cast<uint64_t>(c + (static_cast<int64_t>(m.p) << 32)), m);
  uint32_t d = v + (m.p - cm);
  d = (d >= m.p) ? d - m.p : d;
  return barrett64(static_cast<uint64_t>(d) * o.p_last_inv, m);
}

// (a − b) mod p for a, b ∈ [0, p): d = a − b wraps above p exactly when a < b
__device__ __forceinline__ uint32_t sub_mod(uint32_t a, uint32_t b, uint32_t p) {
  const uint32_t d = a - b;
  return min(d, d + p);
}

// Standalone RNS Rescale of residue arrays (Alg. 7 step 2 on Ã's polynomials):
// in [L][n] canonical residues → out [L−1][n] = ⌊x / p_{L−1}⌉ mod p_l.
struct RescaleParams {
  const uint32_t* in;
  uint32_t* out;
  int64_t n;
  int32_t L;
  uint32_t p_last;
  ModP m[64];
  uint32_t inv[64];  // p_last^{-1} mod p_l
};

__global__ void __launch_bounds__(256) k_rescale(const __grid_constant__ RescaleParams P) {
  const int l = blockIdx.y;
  OutParams o{};
  o.p_last = P.p_last;
  o.p_last_inv = P.inv[l];
  const uint32_t* xl = P.in + static_cast<int64_t>(P.L - 1) * P.n;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < P.n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    P.out[static_cast<int64_t>(l) * P.n + i] = rescale_last(P.in[static_cast<int64_t>(l) * P.n + i], xl[i], o, P.m[l]);
}

__device__ __forceinline__ void store_out(const OutParams& o, const ModP& m, int64_t j, int64_t r, uint32_t v) {
  uint32_t* q = out_ptr(o, j, r);
  if (o.rowcorr) v = sub_mod(v, o.rowcorr[r], m.p);
  if (o.accumulate) v = accum_mod(*q, v, o.w, m);
  if (o.xlast) v = rescale_last(v, o.xlast[j * o.R + r], o, m);
  *q = v;
}

// The output transforms of store16 without the store, for NR consecutive rows r0.. of column j that
// lie inside A' or inside B' with 4-aligned vectors (the TMA-store epilogue stages the results in
// shared memory): the unsigned-U row correction, the k_U > 1 accumulation of the previous pass's
// outputs and the Rescale.  j_ok = false (a column past d3_loc, clipped by the TMA store) skips the
// reads of the previous outputs / xlast.
template <int NR>
__device__ __forceinline__ void finish_rows(const OutParams& o, const ModP& m, int64_t j, int64_t r0, uint32_t (&res)[NR],
                                            bool j_ok) {
  static_assert(NR % 4 == 0, "vector rows");
  if (o.rowcorr) {
    const uint4* rc = reinterpret_cast<const uint4*>(o.rowcorr + r0);
#pragma unroll
    for (int i = 0; i < NR / 4; ++i) {
      const uint4 c = rc[i];
      res[4 * i] = sub_mod(res[4 * i], c.x, m.p);
      res[4 * i + 1] = sub_mod(res[4 * i + 1], c.y, m.p);
      res[4 * i + 2] = sub_mod(res[4 * i + 2], c.z, m.p);
      res[4 * i + 3] = sub_mod(res[4 * i + 3], c.w, m.p);
    }
  }
  if (!j_ok) return;
  if (o.accumulate) {
    const uint4* q = reinterpret_cast<const uint4*>(out_ptr(o, j, r0));
#pragma unroll
    for (int i = 0; i < NR / 4; ++i) {
      const uint4 pv = q[i];
      res[4 * i] = accum_mod(pv.x, res[4 * i], o.w, m);
      res[4 * i + 1] = accum_mod(pv.y, res[4 * i + 1], o.w, m);
      res[4 * i + 2] = accum_mod(pv.z, res[4 * i + 2], o.w, m);
      res[4 * i + 3] = accum_mod(pv.w, res[4 * i + 3], o.w, m);
    }
  }
  if (o.xlast) {
    const uint4* xl = reinterpret_cast<const uint4*>(o.xlast + j * o.R + r0);
#pragma unroll
    for (int i = 0; i < NR / 4; ++i) {
      const uint4 x = xl[i];
      res[4 * i] = rescale_last(res[4 * i], x.x, o, m);
      res[4 * i + 1] = rescale_last(res[4 * i + 1], x.y, o, m);
      res[4 * i + 2] = rescale_last(res[4 * i + 2], x.z, o, m);
      res[4 * i + 3] = rescale_last(res[4 * i + 3], x.w, o, m);
    }
  }
}

// Store 16 consecutive rows r0..r0+15 of output column j (one epilogue thread's TMEM chunk):
// 4 × 16-byte stores when the 16 rows lie inside A' or inside B' and both are 4-aligned.
__device__ __forceinline__ void store16(const OutParams& o, const ModP& m, int64_t j, int64_t r0, uint32_t (&res)[16]) {
  const bool in_a = (r0 + 15 < o.rows_A), in_b = (r0 >= o.rows_A);
  if (((o.rows_A & 3) == 0) && ((o.d1 & 3) == 0) && r0 + 15 < o.R && (in_a || in_b)) {
    CTPT_CHECK(out_ptr(o, j, r0 + 15) == out_ptr(o, j, r0) + 15);
    uint4* q = reinterpret_cast<uint4*>(out_ptr(o, j, r0));
    if (o.rowcorr) {
      const uint4* rc = reinterpret_cast<const uint4*>(o.rowcorr + r0);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint4 c = rc[i];
        res[4 * i] = sub_mod(res[4 * i], c.x, m.p);
        res[4 * i + 1] = sub_mod(res[4 * i + 1], c.y, m.p);
        res[4 * i + 2] = sub_mod(res[4 * i + 2], c.z, m.p);
        res[4 * i + 3] = sub_mod(res[4 * i + 3], c.w, m.p);
      }
    }
    if (o.accumulate) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint4 pv = q[i];
        res[4 * i] = accum_mod(pv.x, res[4 * i], o.w, m);
        res[4 * i + 1] = accum_mod(pv.y, res[4 * i + 1], o.w, m);
        res[4 * i + 2] = accum_mod(pv.z, res[4 * i + 2], o.w, m);
        res[4 * i + 3] = accum_mod(pv.w, res[4 * i + 3], o.w, m);
      }
    }
    if (o.xlast) {
      const uint4* xl = reinterpret_cast<const uint4*>(o.xlast + j * o.R + r0);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint4 x = xl[i];
        res[4 * i] = rescale_last(res[4 * i], x.x, o, m);
        res[4 * i + 1] = rescale_last(res[4 * i + 1], x.y, o, m);
        res[4 * i + 2] = rescale_last(res[4 * i + 2], x.z, o, m);
        res[4 * i + 3] = rescale_last(res[4 * i + 3], x.w, o, m);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) q[i] = make_uint4(res[4 * i], res[4 * i + 1], res[4 * i + 2], res[4 * i + 3]);
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (r0 + i < o.R) store_out(o, m, j, r0 + i, res[i]);
  }
}

// ------------------------------------------------------------------------------------------
// CUDA-core bring-up GEMM (diagnostics only): same limb planes, same epilogue.
// One thread per (j, r) output; block 16 (r) x 16 (j).
// ------------------------------------------------------------------------------------------
struct SimtParams {
  const uint8_t* limbs;  // 32-KB limb tiles (limb_tile_off)
  const int8_t* uplane;  // [d3_total][d2p] plane for this pass
  int64_t R, d2, d2p, j_off;
  int32_t u_unsigned;    // plane holds u8 values (U + u_offset)
  ModP m;
  OutParams o;
};

__global__ void k_gemm_simt(const __grid_constant__ SimtParams P) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * 16 + (threadIdx.x & 15);
  const int64_t j = static_cast<int64_t>(blockIdx.y) * 16 + (threadIdx.x >> 4);
  if (r >= P.R || j >= P.o.d3_loc) return;
  int32_t c[4] = {0, 0, 0, 0};
  const int8_t* u = P.uplane + (P.j_off + j) * P.d2p;
  const int64_t nkb = (P.d2p + 127) / 128;
  for (int64_t k = 0; k < P.d2; ++k) {
    const int32_t uk = P.u_unsigned ? static_cast<int32_t>(static_cast<uint8_t>(u[k])) : static_cast<int32_t>(u[k]);
    const uint8_t* t = P.limbs + limb_tile_off(r, k, nkb);
#pragma unroll
    for (int l = 0; l < 4; ++l) c[l] += static_cast<int32_t>(t[l * 8192]) * uk;
  }
  store_out(P.o, P.m, j, r, recombine_mod(c[0], c[1], c[2], c[3], P.m));
}

}  // namespace ctpt
