/*
 * oracle.c — TEST INFRASTRUCTURE.  A plain, slow, obviously-correct CPU
 * implementation of what the CP-MM hot path computes (Algorithm 6,
 * P:1693–1707, step 1: (A', B') <- (A·U0, B·U0) mod q, per RNS prime p).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load this library.  It shares no code with the CUDA path
 * (paper_2503_16080_b200/csrc): no limbs, no centred digits, no Barrett, no
 * tiling.  Every product is the textbook definition with one `% p` at the end.
 *
 * Operand conventions (readings Q1, Q2, Q14):
 *   X is a ciphertext matrix (A or B) given column by column, exactly as the
 *   per-column ciphertexts store it: X_colmajor[k*rows + r] = X[r][k], canonical
 *   residues in [0, p).  U is an integer matrix, row-major U[k*d3 + j]; negative
 *   entries are taken mod p (U0 mod p, canonical).  Outputs are per-column:
 *   out[c*rows + r] = (X·U)[r][j_c] mod p.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

static inline uint64_t canon(int64_t x, uint32_t p) {
  int64_t r = x % (int64_t)p;
  return (uint64_t)(r < 0 ? r + p : r);
}

static void set_threads(int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
}

/* Schoolbook modular matmul on a list of output columns (Alg. 6 step 1):
 *   out[c][r] = ( Σ_{k<d2} X[r][k] · (U[k][cols[c]] mod p) ) mod p
 * The sum is accumulated exactly in unsigned 128-bit (products < 2^62, d2 < 2^17
 * terms < 2^79), with a single reduction at the end. */
void orc_modmatmul_cols(const uint32_t* X, int64_t rows, int64_t d2, const int64_t* U, int64_t d3,
                        const int64_t* cols, int64_t ncols, uint32_t p, uint32_t* out, int nthreads) {
  set_threads(nthreads);
  /* work items = (output column, block of rows); each row's sum is still taken over k in order */
  const int64_t RB = 2048;
  const int64_t nrb = (rows + RB - 1) / RB;
#ifdef _OPENMP
#pragma omp parallel
#endif
  {
    u128* acc = (u128*)malloc(sizeof(u128) * (size_t)RB);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
    for (int64_t w = 0; w < ncols * nrb; ++w) {
      const int64_t c = w / nrb, r0 = (w % nrb) * RB;
      const int64_t r1 = r0 + RB < rows ? r0 + RB : rows;
      const int64_t j = cols[c];
      memset(acc, 0, sizeof(u128) * (size_t)RB);
      for (int64_t k = 0; k < d2; ++k) {
        const uint64_t u = canon(U[k * d3 + j], p);
        const uint32_t* xk = X + k * rows;
        for (int64_t r = r0; r < r1; ++r) acc[r - r0] += (u128)((uint64_t)xk[r] * u);
      }
      for (int64_t r = r0; r < r1; ++r) out[c * rows + r] = (uint32_t)(acc[r - r0] % p);
    }
    free(acc);
  }
}

/* The same definition evaluated on a list of single entries (r_idx[e], j_idx[e]). */
void orc_modmatmul_entries(const uint32_t* X, int64_t rows, int64_t d2, const int64_t* U, int64_t d3,
                           const int64_t* r_idx, const int64_t* j_idx, int64_t n, uint32_t p, uint32_t* out,
                           int nthreads) {
  set_threads(nthreads);
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
  for (int64_t e = 0; e < n; ++e) {
    const int64_t r = r_idx[e], j = j_idx[e];
    u128 acc = 0;
    for (int64_t k = 0; k < d2; ++k) acc += (u128)((uint64_t)X[k * rows + r] * canon(U[k * d3 + j], p));
    out[e] = (uint32_t)(acc % p);
  }
}

/* Freivalds' check of C = X·U mod p with a vector v ∈ Z_p^{d3}:
 *   lhs = C·v mod p   (C given per column: C[c*rows + r] for c < d3)
 *   rhs = X·(U·v) mod p
 * Returns the number of rows where lhs != rhs. */
int64_t orc_freivalds(const uint32_t* X, int64_t rows, int64_t d2, const int64_t* U, int64_t d3,
                      const uint32_t* C, uint32_t p, const uint64_t* v, uint32_t* lhs_out, uint32_t* rhs_out,
                      int nthreads) {
  set_threads(nthreads);
  uint64_t* w = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)d2);
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
  for (int64_t k = 0; k < d2; ++k) {
    u128 acc = 0;
    for (int64_t j = 0; j < d3; ++j) acc += (u128)(canon(U[k * d3 + j], p) * (v[j] % p));
    w[k] = (uint64_t)(acc % p);
  }
  int64_t bad = 0;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) reduction(+ : bad)
#endif
  for (int64_t r = 0; r < rows; ++r) {
    u128 a = 0, b = 0;
    for (int64_t j = 0; j < d3; ++j) a += (u128)((uint64_t)C[j * rows + r] * (v[j] % p));
    for (int64_t k = 0; k < d2; ++k) b += (u128)((uint64_t)X[k * rows + r] * w[k]);
    uint32_t la = (uint32_t)(a % p), rb = (uint32_t)(b % p);
    if (lhs_out) lhs_out[r] = la;
    if (rhs_out) rhs_out[r] = rb;
    bad += (la != rb);
  }
  free(w);
  return bad;
}

/* Negacyclic product by the Toeplitz definition: c = toep(s)·Vec(a), i.e.
 *   c_i = Σ_{j ≤ i} s_{i-j} a_j  −  Σ_{j > i} s_{N+i-j} a_j   (mod p). */
static uint32_t negacyclic_coeff(const uint32_t* a, const int64_t* s, int64_t N, uint32_t p, int64_t i) {
  u128 pos = 0, neg = 0;
  for (int64_t j = 0; j < N; ++j) {
    if (j <= i) {
      int64_t sv = s[i - j];
      if (sv >= 0) pos += (u128)((uint64_t)a[j] * (uint64_t)sv);
      else neg += (u128)((uint64_t)a[j] * (uint64_t)(-sv));
    } else {
      int64_t sv = s[N + i - j];
      if (sv >= 0) neg += (u128)((uint64_t)a[j] * (uint64_t)sv);
      else pos += (u128)((uint64_t)a[j] * (uint64_t)(-sv));
    }
  }
  uint64_t P = (uint64_t)(pos % p), Q = (uint64_t)(neg % p);
  return (uint32_t)((P + p - Q) % p);
}

void orc_negacyclic_mul(const uint32_t* a, const int64_t* s, int64_t N, uint32_t p, uint32_t* out) {
  for (int64_t i = 0; i < N; ++i) out[i] = negacyclic_coeff(a, s, N, p, i);
}

/* Decryption of one output column in a structured-S format (P:852 Dec; P:1688 identity
 * S·(A·U0) + B·U0 = M·U0 mod q):  out = S·a_col + b_col mod p, chunk by chunk:
 *   RLWE / shared-a:  out[tN+i] = (toep(sk_t)·a)_i + b[tN+i]   (a has N entries; t=0 for RLWE)
 *   shared-s:         out[tN+i] = (toep(sk)·a_t)_i + b[tN+i]   (a has d1 entries, chunk t)
 *   structured-A:     out[tN+i] = (toep(a_t)·key)_i + b[tN+i]  (Ã·S + B; a holds the
 *                     k = d1/N shared polys a_t, key is the column's secret Vec(sk_j) — or, for an
 *                     Algorithm 7 output column, the column (S·U)_j of the new key, P:1751–1757;
 *                     toep(a)·Vec(s) = Vec(a·s) = toep(s)·Vec(a), so the same coefficient formula)
 * fmt: 0 RLWE, 1 shared-s, 2 shared-a, 3 structured-A.  sks: nkeys × N integer keys (int64;
 * |key| < 2^31 so every product stays below 2^62). */
int orc_decrypt_col(int fmt, int64_t N, int64_t d1, const int64_t* sks, const uint32_t* a_col,
                    const uint32_t* b_col, uint32_t p, uint32_t* out, int nthreads) {
  if (N <= 0 || d1 % N || fmt < 0 || fmt > 3) return -1;
  set_threads(nthreads);
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 64)
#endif
  for (int64_t r = 0; r < d1; ++r) {
    const int64_t t = r / N, i = r % N;
    const int64_t* key = sks + ((fmt == 2) ? t : 0) * N;
    const uint32_t* a = a_col + ((fmt == 1 || fmt == 3) ? t * N : 0);
    out[r] = (uint32_t)(((uint64_t)negacyclic_coeff(a, key, N, p, i) + b_col[r]) % p);
  }
  return 0;
}
