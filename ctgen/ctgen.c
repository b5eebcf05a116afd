/*
 * ctgen.c — seeded synthetic-input generator for the CP-MM hot path.
 *
 * This module is INPUT SYNTHESIS ONLY.  It serves both sides (the CUDA product
 * path via bench.py / the binding's users, and the CPU oracle via tests) and it
 * holds none of the arithmetic of the method under test (Algorithm 6's modular
 * products A·U, B·U mod p, the limb split, the reduction).  It produces the
 * method's INPUT: per-column RLWE ciphertexts in one of the three structured-S
 * formats of PAPER.md §3, plus the plaintext matrix U.
 *
 * Random numbers (readings Q5–Q13):
 *   draw64(seed, tag, idx) = splitmix64(splitmix64(seed ^ tag) + idx)
 * Counter-based, so generation is order-independent and parallel.
 *
 * Streams (tag = kind << 56 | fields):
 *   SK   (key t)                    idx = coefficient            ternary {-1,0,1}
 *   A    (prime value p, poly)      idx = coefficient            uniform mod p
 *   E    (poly)                     idx = coefficient            discrete Gaussian σ=3.2 on [-20,20]
 *   M    (-)                        idx = j*d1 + i (column-major) uniform 53-bit grid on [-1,1)
 *   U    (-)                        idx = k*d3 + j                uniform integers {-B..B}
 *
 * Encryption (symmetric; b = m + e − a·sk, reading Q25) uses a
 * negacyclic NTT per prime (all primes are ≡ 1 mod 2^16).  The oracle checks
 * this generator with its own schoolbook negacyclic product (tests/).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define CTGEN_RLWE 0
#define CTGEN_SHARED_S 1
#define CTGEN_SHARED_A 2
#define CTGEN_STRUCT_A 3 /* structured-A shared-a: a_i shared by row block i, sk_j per column */

#define K_SK 1ULL
#define K_A 2ULL
#define K_E 3ULL
#define K_M 4ULL
#define K_U 5ULL
#define K_R 6ULL /* generic stream for test vectors (Freivalds r, etc.) */
#define K_UR 7ULL /* real-valued U for the Rescale workloads (uniform 53-bit grid on [-1,1)) */

static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

uint64_t ctgen_draw64(uint64_t seed, uint64_t tag, uint64_t idx) {
  return splitmix64(splitmix64(seed ^ tag) + idx);
}

static inline uint64_t tag_sk(uint64_t t) { return (K_SK << 56) | t; }
static inline uint64_t tag_a(uint64_t p, uint64_t poly) { return (K_A << 56) | (p << 24) | poly; }
static inline uint64_t tag_e(uint64_t poly) { return (K_E << 56) | poly; }
static inline uint64_t tag_m(void) { return K_M << 56; }
static inline uint64_t tag_u(void) { return K_U << 56; }

/* ---------------- primes (reading Q5) ---------------- */
static uint64_t powmod64(uint64_t b, uint64_t e, uint64_t m) {
  unsigned __int128 r = 1, x = b % m;
  while (e) {
    if (e & 1) r = (r * x) % m;
    x = (x * x) % m;
    e >>= 1;
  }
  return (uint64_t)r;
}

static int is_prime_mr(uint64_t n) {
  /* deterministic Miller–Rabin for n < 4,759,123,141 with bases {2,7,61} */
  if (n < 2) return 0;
  static const uint64_t small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61};
  for (unsigned i = 0; i < sizeof(small) / sizeof(small[0]); ++i) {
    if (n == small[i]) return 1;
    if (n % small[i] == 0) return 0;
  }
  uint64_t d = n - 1;
  int s = 0;
  while ((d & 1) == 0) { d >>= 1; ++s; }
  static const uint64_t bases[] = {2, 7, 61};
  for (int i = 0; i < 3; ++i) {
    uint64_t x = powmod64(bases[i], d, n);
    if (x == 1 || x == n - 1) continue;
    int comp = 1;
    for (int r = 1; r < s; ++r) {
      x = (uint64_t)(((unsigned __int128)x * x) % n);
      if (x == n - 1) { comp = 0; break; }
    }
    if (comp) return 0;
  }
  return 1;
}

/* The L largest primes p < 2^31 with p ≡ 1 (mod 2^16), descending. */
int ctgen_primes(int L, uint32_t* out) {
  int n = 0;
  for (uint64_t c = ((1ULL << 31) - 1) >> 16; c >= 1 && n < L; --c) {
    uint64_t p = (c << 16) + 1;
    if (p >= (1ULL << 31)) continue;
    if (is_prime_mr(p)) out[n++] = (uint32_t)p;
  }
  return n;
}

int ctgen_is_prime(uint64_t n) { return is_prime_mr(n); }

/* ---------------- samplers ---------------- */
/* CDT of the discrete Gaussian rho(x) ∝ exp(-x^2/(2σ^2)), σ=3.2, x ∈ [-20,20].
 * CDT[i] = round(2^64 · P(X ≤ i-20)) for i = 0..39; P(X ≤ 20) = 1.
 * Generated once with 60-digit decimal arithmetic (reading Q7). */
static const uint64_t CDT[40] = {
    0x00000001c37cd27fULL, 0x0000000d9b159a02ULL, 0x00000055b95f064eULL, 0x000001e40f062e35ULL,
    0x000009af7ff5b13dULL, 0x00002d198d9a6df4ULL, 0x0000bf07c2f15f98ULL, 0x0002e06a072ea65fULL,
    0x000a1907f127e4aeULL, 0x00204c0fb022221fULL, 0x005e3165c1f6eb47ULL, 0x00fab6a9a61d5e1dULL,
    0x0261b17054d25dbdULL, 0x054c69363c89057aULL, 0x0acd2766d6a8f360ULL, 0x143796b53f652e74ULL,
    0x22d43df1e68717d9ULL, 0x37651d97aa683b5bULL, 0x51a5da2be47094ccULL, 0x700ad4bf92b7e709ULL,
    0x8ff52b406d4818f7ULL, 0xae5a25d41b8f6b34ULL, 0xc89ae2685597c4a5ULL, 0xdd2bc20e1978e827ULL,
    0xebc8694ac09ad18cULL, 0xf532d89929570ca0ULL, 0xfab396c9c376fa86ULL, 0xfd9e4e8fab2da243ULL,
    0xff05495659e2a1e3ULL, 0xffa1ce9a3e0914b9ULL, 0xffdfb3f04fdddde1ULL, 0xfff5e6f80ed81b52ULL,
    0xfffd1f95f8d159a1ULL, 0xffff40f83d0ea068ULL, 0xffffd2e67265920cULL, 0xfffff650800a4ec3ULL,
    0xfffffe1bf0f9d1cbULL, 0xffffffaa46a0f9b2ULL, 0xfffffff264ea65feULL, 0xfffffffe3c832d81ULL};

static inline int32_t gauss_from_u64(uint64_t u) {
  int i = 0;
  while (i < 40 && u >= CDT[i]) ++i;
  return i - 20;
}

int32_t ctgen_err(uint64_t seed, uint64_t poly, uint64_t coeff) {
  return gauss_from_u64(ctgen_draw64(seed, tag_e(poly), coeff));
}

int32_t ctgen_sk_coeff(uint64_t seed, uint64_t t, uint64_t i) {
  return (int32_t)(ctgen_draw64(seed, tag_sk(t), i) % 3ULL) - 1;
}

void ctgen_sk(uint64_t seed, uint64_t t, int64_t N, int8_t* out) {
  for (int64_t i = 0; i < N; ++i) out[i] = (int8_t)ctgen_sk_coeff(seed, t, (uint64_t)i);
}

uint32_t ctgen_a_coeff(uint64_t seed, uint32_t p, uint64_t poly, uint64_t i) {
  return (uint32_t)(ctgen_draw64(seed, tag_a(p, poly), i) % p);
}

/* m = 2*(r53/2^53) - 1 = (r53 - 2^52) * 2^-52, exactly representable (reading Q10). */
double ctgen_msg(uint64_t seed, int64_t d1, int64_t i, int64_t j) {
  uint64_t r53 = ctgen_draw64(seed, tag_m(), (uint64_t)(j * d1 + i)) >> 11;
  return ldexp((double)((int64_t)r53 - (1LL << 52)), -52);
}

/* ⌊Δ·m⌉ = ⌊Δ·m + 1/2⌋ computed in exact integer arithmetic from the draw (Q9).
 * Δ·m = v · 2^(logΔ-52) with v = r53 - 2^52. */
int64_t ctgen_encoded(uint64_t seed, int64_t d1, int64_t i, int64_t j, int log_delta) {
  uint64_t r53 = ctgen_draw64(seed, tag_m(), (uint64_t)(j * d1 + i)) >> 11;
  int64_t v = (int64_t)r53 - (1LL << 52);
  int s = 52 - log_delta;
  if (s <= 0) return v * (1LL << (-s));
  return (v + (1LL << (s - 1))) >> s; /* arithmetic shift = floor */
}

/* plaintext coefficient P = ⌊ΔM⌉ + E for entry (i, j) of the d1 x d2 matrix, where
 * (i, j) lives in b-poly j*k + t, coefficient i - t*N. */
int64_t ctgen_plain(uint64_t seed, int64_t N, int64_t d1, int64_t i, int64_t j, int log_delta) {
  int64_t k = d1 / N;
  int64_t t = i / N;
  return ctgen_encoded(seed, d1, i, j, log_delta) + ctgen_err(seed, (uint64_t)(j * k + t), (uint64_t)(i - t * N));
}

int64_t ctgen_u(uint64_t seed, int64_t d3, int64_t k, int64_t j, int64_t bound) {
  uint64_t w = 2ULL * (uint64_t)bound + 1ULL;
  return (int64_t)(ctgen_draw64(seed, tag_u(), (uint64_t)(k * d3 + j)) % w) - bound;
}

void ctgen_U(uint64_t seed, int64_t d2, int64_t d3, int64_t bound, int64_t* out, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
  for (int64_t k = 0; k < d2; ++k)
    for (int64_t j = 0; j < d3; ++j) out[k * d3 + j] = ctgen_u(seed, d3, k, j, bound);
}

/* Real U ∈ [-1,1)^{d2×d3} on the 53-bit grid (stream K_UR, idx k*d3 + j), and its encoding
 * U0 = ⌊scale · U⌉ (Alg. 6 REQUIRE: U0 = ⌊Δ·U⌉; ties up) for an arbitrary
 * integer scale < 2^62 (e.g. Δ_U = the rescaling prime), computed exactly in 128-bit:
 * scale·U = scale·v·2^-52 with v = r53 - 2^52, so ⌊scale·U + 1/2⌋ = (scale·v + 2^51) >> 52. */
double ctgen_u_real(uint64_t seed, int64_t d3, int64_t k, int64_t j) {
  uint64_t r53 = ctgen_draw64(seed, K_UR << 56, (uint64_t)(k * d3 + j)) >> 11;
  return ldexp((double)((int64_t)r53 - (1LL << 52)), -52);
}

void ctgen_U_real(uint64_t seed, int64_t d2, int64_t d3, uint64_t scale, double* out_real, int64_t* out_enc,
                  int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
  for (int64_t k = 0; k < d2; ++k)
    for (int64_t j = 0; j < d3; ++j) {
      uint64_t r53 = ctgen_draw64(seed, K_UR << 56, (uint64_t)(k * d3 + j)) >> 11;
      int64_t v = (int64_t)r53 - (1LL << 52);
      if (out_real) out_real[k * d3 + j] = ldexp((double)v, -52);
      if (out_enc) {
        __int128 t = (__int128)scale * v + ((__int128)1 << 51);
        out_enc[k * d3 + j] = (int64_t)(t >> 52); /* arithmetic shift = floor */
      }
    }
}

uint64_t ctgen_uniform(uint64_t seed, uint64_t stream, uint64_t idx, uint64_t mod) {
  return ctgen_draw64(seed, (K_R << 56) | stream, idx) % mod;
}

/* ---------------- negacyclic NTT (generator-internal) ---------------- */
typedef struct {
  uint32_t p;
  int64_t N;
  int logN;
  uint32_t* psi_pow;      /* ψ^bitrev(i), forward twiddles (merged negacyclic form) */
  uint32_t* psi_pow_sh;   /* Shoup companions floor(w·2^32/p) */
  uint32_t* ipsi_pow;     /* ψ^-bitrev(i) */
  uint32_t* ipsi_pow_sh;
  uint32_t n_inv, n_inv_sh;
} ntt_plan;

static inline uint32_t mul_shoup(uint32_t a, uint32_t w, uint32_t wsh, uint32_t p) {
  uint32_t q = (uint32_t)(((uint64_t)a * wsh) >> 32);
  uint64_t r = (uint64_t)a * w - (uint64_t)q * p;
  uint32_t rr = (uint32_t)r;
  return rr >= p ? rr - p : rr;
}
static inline uint32_t shoup_of(uint32_t w, uint32_t p) { return (uint32_t)(((uint64_t)w << 32) / p); }

static uint32_t bitrev(uint32_t x, int bits) {
  uint32_t r = 0;
  for (int i = 0; i < bits; ++i) { r = (r << 1) | (x & 1); x >>= 1; }
  return r;
}

static int ntt_plan_init(ntt_plan* pl, uint32_t p, int64_t N) {
  pl->p = p;
  pl->N = N;
  pl->logN = 0;
  while ((1LL << pl->logN) < N) pl->logN++;
  if ((1LL << pl->logN) != N) return -1;
  if (((uint64_t)p - 1) % (uint64_t)(2 * N) != 0) return -2;
  /* primitive 2N-th root of unity ψ: ψ^N ≡ -1 */
  uint64_t psi = 0;
  for (uint64_t x = 2; x < p; ++x) {
    uint64_t c = powmod64(x, (p - 1) / (uint64_t)(2 * N), p);
    if (powmod64(c, (uint64_t)N, p) == p - 1) { psi = c; break; }
  }
  if (!psi) return -3;
  uint64_t ipsi = powmod64(psi, p - 2, p);
  pl->psi_pow = (uint32_t*)malloc(sizeof(uint32_t) * N);
  pl->psi_pow_sh = (uint32_t*)malloc(sizeof(uint32_t) * N);
  pl->ipsi_pow = (uint32_t*)malloc(sizeof(uint32_t) * N);
  pl->ipsi_pow_sh = (uint32_t*)malloc(sizeof(uint32_t) * N);
  uint64_t pw = 1, ipw = 1;
  uint32_t* tmp = (uint32_t*)malloc(sizeof(uint32_t) * N);
  uint32_t* itmp = (uint32_t*)malloc(sizeof(uint32_t) * N);
  for (int64_t i = 0; i < N; ++i) {
    tmp[i] = (uint32_t)pw;
    itmp[i] = (uint32_t)ipw;
    pw = pw * psi % p;
    ipw = ipw * ipsi % p;
  }
  for (int64_t i = 0; i < N; ++i) {
    uint32_t r = bitrev((uint32_t)i, pl->logN);
    pl->psi_pow[i] = tmp[r];
    pl->ipsi_pow[i] = itmp[r];
    pl->psi_pow_sh[i] = shoup_of(tmp[r], p);
    pl->ipsi_pow_sh[i] = shoup_of(itmp[r], p);
  }
  free(tmp);
  free(itmp);
  pl->n_inv = (uint32_t)powmod64((uint64_t)N, p - 2, p);
  pl->n_inv_sh = shoup_of(pl->n_inv, p);
  return 0;
}

static void ntt_plan_free(ntt_plan* pl) {
  free(pl->psi_pow);
  free(pl->psi_pow_sh);
  free(pl->ipsi_pow);
  free(pl->ipsi_pow_sh);
}

/* In-place forward negacyclic NTT (Cooley–Tukey, standard→bit-reversed). */
static void ntt_fwd(const ntt_plan* pl, uint32_t* a) {
  const uint32_t p = pl->p;
  int64_t N = pl->N;
  int64_t t = N;
  for (int64_t m = 1; m < N; m <<= 1) {
    t >>= 1;
    for (int64_t i = 0; i < m; ++i) {
      uint32_t w = pl->psi_pow[m + i], wsh = pl->psi_pow_sh[m + i];
      int64_t j1 = 2 * i * t;
      for (int64_t j = j1; j < j1 + t; ++j) {
        uint32_t u = a[j];
        uint32_t v = mul_shoup(a[j + t], w, wsh, p);
        uint32_t s = u + v;
        a[j] = s >= p ? s - p : s;
        a[j + t] = u >= v ? u - v : u + p - v;
      }
    }
  }
}

/* In-place inverse negacyclic NTT (Gentleman–Sande, bit-reversed→standard), scaled by 1/N. */
static void ntt_inv(const ntt_plan* pl, uint32_t* a) {
  const uint32_t p = pl->p;
  int64_t N = pl->N;
  int64_t t = 1;
  for (int64_t m = N >> 1; m >= 1; m >>= 1) {
    int64_t j1 = 0;
    for (int64_t i = 0; i < m; ++i) {
      uint32_t w = pl->ipsi_pow[m + i], wsh = pl->ipsi_pow_sh[m + i];
      for (int64_t j = j1; j < j1 + t; ++j) {
        uint32_t u = a[j], v = a[j + t];
        uint32_t s = u + v;
        a[j] = s >= p ? s - p : s;
        uint32_t d = u >= v ? u - v : u + p - v;
        a[j + t] = mul_shoup(d, w, wsh, p);
      }
      j1 += 2 * t;
    }
    t <<= 1;
  }
  for (int64_t j = 0; j < N; ++j) a[j] = mul_shoup(a[j], pl->n_inv, pl->n_inv_sh, p);
}

static inline uint32_t mulmod(uint32_t a, uint32_t b, uint32_t p) { return (uint32_t)((uint64_t)a * b % p); }

/* Negacyclic product c = a·s mod (p, X^N+1) via the NTT (exported for the test that
 * compares it with the oracle's schoolbook product). */
int ctgen_negacyclic_ntt(const uint32_t* a, const int8_t* s, int64_t N, uint32_t p, uint32_t* out) {
  ntt_plan pl;
  if (ntt_plan_init(&pl, p, N)) return -1;
  uint32_t* x = (uint32_t*)malloc(sizeof(uint32_t) * N);
  uint32_t* y = (uint32_t*)malloc(sizeof(uint32_t) * N);
  for (int64_t i = 0; i < N; ++i) {
    x[i] = a[i] % p;
    y[i] = s[i] >= 0 ? (uint32_t)s[i] : p - (uint32_t)(-s[i]);
  }
  ntt_fwd(&pl, x);
  ntt_fwd(&pl, y);
  for (int64_t i = 0; i < N; ++i) x[i] = mulmod(x[i], y[i], p);
  ntt_inv(&pl, x);
  memcpy(out, x, sizeof(uint32_t) * N);
  free(x);
  free(y);
  ntt_plan_free(&pl);
  return 0;
}

/* ---------------- encryption of a matrix in a structured-S column format ----------------
 *
 * M ∈ R^{d1×d2} (column j encrypted separately), k = d1/N chunks per column.
 *   RLWE     (k = 1):  a_j, b_j with  a_j·sk + b_j = P_j
 *   shared-s (k ≥ 1):  a_{t,j}, b_{t,j} with a_{t,j}·sk + b_{t,j} = P_{t,j}
 *   shared-a (k ≥ 1):  a_j, b_{t,j} with a_j·sk_t + b_{t,j} = P_{t,j}
 * P_{t,j} = Pol(⌊Δ M_{tN.., j}⌉ + e_{t,j}).
 *
 * Output layout (per-column ciphertexts, canonical residues in [0,p)):
 *   a_polys[l][n_a_loc][N], n_a_loc = ncols * (fmt == SHARED_S ? k : 1)
 *   b_polys[l][ncols * k][N]
 * with local column c = j - col_begin, poly index c*k + t (a: c or c*k+t).
 * Streams use the GLOBAL column index j, so a column range reproduces the same values.
 */
static int encrypt_struct_a(int64_t N, int64_t d1, uint64_t seed, int log_delta, int L, const uint32_t* primes,
                            int64_t col_begin, int64_t col_end, uint32_t* a_polys, uint32_t* b_polys);

int ctgen_encrypt(int fmt, int64_t N, int64_t d1, int64_t d2, uint64_t seed, int log_delta, int L,
                  const uint32_t* primes, int64_t col_begin, int64_t col_end, uint32_t* a_polys,
                  uint32_t* b_polys, int nthreads) {
  if (N <= 0 || (N & (N - 1))) return -1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  if (fmt == CTGEN_STRUCT_A) {
    if (d1 % N) return -2;
    if (col_begin < 0 || col_end > d2 || col_begin > col_end) return -4;
    return encrypt_struct_a(N, d1, seed, log_delta, L, primes, col_begin, col_end, a_polys, b_polys);
  }
  if (d1 % N) return -2;
  if (fmt == CTGEN_RLWE && d1 != N) return -3;
  if (col_begin < 0 || col_end > d2 || col_begin > col_end) return -4;
  const int64_t k = d1 / N;
  const int64_t ncols = col_end - col_begin;
  const int64_t n_a_per_col = (fmt == CTGEN_SHARED_S) ? k : 1;
  const int nkeys = (fmt == CTGEN_SHARED_A) ? (int)k : 1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  for (int l = 0; l < L; ++l) {
    const uint32_t p = primes[l];
    ntt_plan pl;
    if (ntt_plan_init(&pl, p, N)) return -5;
    /* NTT of every key */
    uint32_t* sk_hat = (uint32_t*)malloc(sizeof(uint32_t) * N * nkeys);
    for (int t = 0; t < nkeys; ++t) {
      for (int64_t i = 0; i < N; ++i) {
        int32_t s = ctgen_sk_coeff(seed, (uint64_t)t, (uint64_t)i);
        sk_hat[t * N + i] = s >= 0 ? (uint32_t)s : p - (uint32_t)(-s);
      }
      ntt_fwd(&pl, sk_hat + t * N);
    }
    uint32_t* A = a_polys + (int64_t)l * ncols * n_a_per_col * N;
    uint32_t* B = b_polys + (int64_t)l * ncols * k * N;
#ifdef _OPENMP
#pragma omp parallel
#endif
    {
      uint32_t* ahat = (uint32_t*)malloc(sizeof(uint32_t) * N);
      uint32_t* prod = (uint32_t*)malloc(sizeof(uint32_t) * N);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 4)
#endif
      for (int64_t c = 0; c < ncols; ++c) {
        const int64_t j = col_begin + c;
        for (int64_t t = 0; t < k; ++t) {
          /* the a-part for (column j, chunk t) */
          const int64_t apoly_global = (fmt == CTGEN_SHARED_S) ? j * k + t : j;
          uint32_t* a_out = A + (c * n_a_per_col + ((fmt == CTGEN_SHARED_S) ? t : 0)) * N;
          if (fmt == CTGEN_SHARED_S || t == 0) {
            for (int64_t i = 0; i < N; ++i) a_out[i] = ctgen_a_coeff(seed, p, (uint64_t)apoly_global, (uint64_t)i);
            memcpy(ahat, a_out, sizeof(uint32_t) * N);
            ntt_fwd(&pl, ahat);
          }
          const uint32_t* skh = sk_hat + ((fmt == CTGEN_SHARED_A) ? t : 0) * N;
          for (int64_t i = 0; i < N; ++i) prod[i] = mulmod(ahat[i], skh[i], p);
          ntt_inv(&pl, prod); /* prod = a·sk mod (p, X^N+1) */
          uint32_t* b_out = B + (c * k + t) * N;
          for (int64_t i = 0; i < N; ++i) {
            int64_t P = ctgen_plain(seed, N, d1, t * N + i, j, log_delta);
            int64_t pm = P % (int64_t)p;
            if (pm < 0) pm += p;
            uint32_t v = (uint32_t)pm;
            b_out[i] = v >= prod[i] ? v - prod[i] : v + p - prod[i];
          }
        }
      }
      free(ahat);
      free(prod);
    }
    free(sk_hat);
    ntt_plan_free(&pl);
  }
  return 0;
}

/* Fill uniformly random canonical residues (for bandwidth-only sweeps that do not
 * decrypt).  Stream K_A with poly index offset 2^23 to stay disjoint from real a-parts. */
void ctgen_uniform_residues(uint64_t seed, uint32_t p, int64_t n, uint32_t* out, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
  for (int64_t i = 0; i < n; ++i) out[i] = (uint32_t)(ctgen_draw64(seed, tag_a(p, 1ULL << 23), (uint64_t)i) % p);
}

/* Bulk versions (row-major [nrows][ncols] blocks of the d1 x d2 matrices, rows [r0,r0+nrows),
 * columns [c0,c0+ncols)) for the large-config tests. */
void ctgen_msg_block(uint64_t seed, int64_t d1, int64_t r0, int64_t nrows, int64_t c0, int64_t ncols, double* out,
                     int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
  for (int64_t i = 0; i < nrows; ++i)
    for (int64_t j = 0; j < ncols; ++j) out[i * ncols + j] = ctgen_msg(seed, d1, r0 + i, c0 + j);
}

void ctgen_plain_block(uint64_t seed, int64_t N, int64_t d1, int log_delta, int64_t r0, int64_t nrows, int64_t c0,
                       int64_t ncols, int64_t* out, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
  for (int64_t i = 0; i < nrows; ++i)
    for (int64_t j = 0; j < ncols; ++j) out[i * ncols + j] = ctgen_plain(seed, N, d1, r0 + i, c0 + j, log_delta);
}

/* ---------------- structured-A shared-a (Algorithm 7) ----------------
 *   a_i · sk_j + b_{i,j} = P_{i,j}   (i < k = d1/N row blocks, j < d2 columns)
 * i.e. Ã·S + B = P with Ã = [toep(a_0); …; toep(a_{k−1})] ∈ Z_q^{d1×N} and S = [Vec(sk_j)]_j.
 * One a-poly per row block (stream A, poly index 2^22 + i: disjoint from the column-indexed
 * a-parts of the other formats) shared by every column; one ternary key per GLOBAL column j
 * (stream SK, t = j).  Output: a_polys[l][k][N], b_polys[l][ncols·k][N] (poly c·k + i). */
static int encrypt_struct_a(int64_t N, int64_t d1, uint64_t seed, int log_delta, int L, const uint32_t* primes,
                            int64_t col_begin, int64_t col_end, uint32_t* a_polys, uint32_t* b_polys) {
  const int64_t k = d1 / N;
  const int64_t ncols = col_end - col_begin;
  for (int l = 0; l < L; ++l) {
    const uint32_t p = primes[l];
    ntt_plan pl;
    if (ntt_plan_init(&pl, p, N)) return -5;
    uint32_t* A = a_polys + (int64_t)l * k * N;
    uint32_t* B = b_polys + (int64_t)l * ncols * k * N;
    uint32_t* a_hat = (uint32_t*)malloc(sizeof(uint32_t) * N * k);
    for (int64_t i = 0; i < k; ++i) {
      for (int64_t c = 0; c < N; ++c) A[i * N + c] = ctgen_a_coeff(seed, p, (1ULL << 22) + (uint64_t)i, (uint64_t)c);
      memcpy(a_hat + i * N, A + i * N, sizeof(uint32_t) * N);
      ntt_fwd(&pl, a_hat + i * N);
    }
#ifdef _OPENMP
#pragma omp parallel
#endif
    {
      uint32_t* skh = (uint32_t*)malloc(sizeof(uint32_t) * N);
      uint32_t* prod = (uint32_t*)malloc(sizeof(uint32_t) * N);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 4)
#endif
      for (int64_t c = 0; c < ncols; ++c) {
        const int64_t j = col_begin + c;
        for (int64_t x = 0; x < N; ++x) {
          int32_t s = ctgen_sk_coeff(seed, (uint64_t)j, (uint64_t)x);
          skh[x] = s >= 0 ? (uint32_t)s : p - (uint32_t)(-s);
        }
        ntt_fwd(&pl, skh);
        for (int64_t i = 0; i < k; ++i) {
          for (int64_t x = 0; x < N; ++x) prod[x] = mulmod(a_hat[i * N + x], skh[x], p);
          ntt_inv(&pl, prod); /* a_i · sk_j */
          uint32_t* b_out = B + (c * k + i) * N;
          for (int64_t x = 0; x < N; ++x) {
            int64_t P = ctgen_plain(seed, N, d1, i * N + x, j, log_delta);
            int64_t pm = P % (int64_t)p;
            if (pm < 0) pm += p;
            uint32_t v = (uint32_t)pm;
            b_out[x] = v >= prod[x] ? v - prod[x] : v + p - prod[x];
          }
        }
      }
      free(skh);
      free(prod);
    }
    free(a_hat);
    ntt_plan_free(&pl);
  }
  return 0;
}
