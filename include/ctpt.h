/*
 * ctpt.h — C ABI of the B200 (sm_100a) ciphertext × plaintext matmul library
 *          (libctpt.so, built from paper_2503_16080_b200/csrc/).
 *
 * What it computes.  arXiv 2503.16080, Algorithm 6 step 1:
 * a matrix M ∈ R^{d1×d2} encrypted column by column in a structured-S format,
 *     S·A + B ≈ Δ·M (mod q)                  (Lemma le:mat_struct_s),
 * is multiplied by a known integer plaintext U0 ∈ Z^{d2×d3} as
 *     (A', B') = (A·U0 mod q, B·U0 mod q),    so that S·A' + B' ≈ Δ·M·U0,
 * i.e. one Mod-PP-MM_{rows_A,d2,d3} plus one Mod-PP-MM_{d1,d2,d3} (Thm th:pcmm P:1711,
 * th:pcmm-shs P:1722).  q = p_0·…·p_{L-1} is held in RNS: every product is computed
 * independently per prime p < 2^31 (the one-product-per-prime structure of Strategy 3,
 * P:1444–1448).  Rescale (Alg. 6 step 2) is not performed: U is an integer matrix
 * (scale 1), so the output keeps scale Δ (reading Q3).
 *
 * How.  Each 31-bit residue x ∈ [0,p) is split into its four base-2^8 digits (the
 * signed-digit decomposition of Lemma le:strategy1, with K = 2^8 and
 * non-negative digits since x ≥ 0); U0's centred residues into balanced int8 digits.
 * The limb products run on the tcgen05 tensor cores (kind::i8, u8 × s8 → s32 in TMEM);
 * limb recombination Σ 2^{8ℓ} C_ℓ and the reduction mod p are fused into the epilogue
 * (P:1385–1388), so only reduced residues are written.
 *
 * Formats (Table 1):
 *   CTPT_RLWE      d1 = N, one key,                  A ∈ Z_q^{N×d2}
 *   CTPT_SHARED_S  N | d1, one key, S = I ⊗ toep(sk), A ∈ Z_q^{d1×d2}
 *   CTPT_SHARED_A  N | d1, k = d1/N keys, shared a,  A ∈ Z_q^{N×d2}
 *   CTPT_STRUCT_A  N | d1, structured-A shared-a: Ã·S + B ≈ Δ·M with
 *                  Ã = [toep(a_0); …; toep(a_{k−1})] (k = d1/N polynomials shared by all
 *                  columns) and a general S = [Vec(sk_j)]_j.  Algorithm 7 (CP-MM with
 *                  precomputation) step 1 computes only B' = B·U:
 *                  the output (Ã, B') encrypts M·U under S·U; Ã passes through unchanged
 *                  (no Rescale, reading Q3), so the library never reads the a-polynomials.
 * rows_A = N (RLWE, shared-a), d1 (shared-s) or 0 (structured-A).  R = rows_A + d1.
 * With rows_A = 0 every A-side pointer (d_a_polys, d_AU, h_a_polys, h_AU) may be NULL.
 *
 * Conventions for every entry point:
 *  - Residues at the boundary are canonical uint32 in [0, p) (reading Q14).
 *  - All device memory is allocated and owned by the caller; sizes come from
 *    ctpt_query_sizes.  The library never allocates or frees device memory and keeps
 *    no global state besides a per-thread error string.
 *  - `stream` is a cudaStream_t passed as void*.  All device work is enqueued on it.
 *    ctpt_layout(validate=0), ctpt_split and ctpt_gemm / ctpt_matmul never synchronise;
 *    ctpt_plain_precompute* and ctpt_layout(validate=1) synchronise `stream` (they read
 *    a device-computed value back).
 *  - Argument validation is synchronous; on a non-OK status nothing was enqueued and
 *    ctpt_last_error() describes the problem.  Asynchronous CUDA faults surface as
 *    CTPT_ERR_CUDA on a later call.
 *  - Calls on distinct streams and distinct buffers may run concurrently.
 *  - The library reads no environment variables.  Kernel choice, raster group and grid cap are
 *    explicit ctpt_problem fields: kernel, raster_group and max_ctas.  Every choice gives the same
 *    residues (tests/test_gpu_parity.py runs each).  Variants that were measured and lost in
 *    round 1 (CTA-pair and multicast GEMMs, K split, L2 prefetch/hints, register-fed converters,
 *    …) were removed; DESIGN.md §6 keeps what each measured.
 */
#ifndef CTPT_H_
#define CTPT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CTPT_OK = 0,
  CTPT_ERR_ARG = 1,         /* null pointer, bad enum, bad buffer size                              */
  CTPT_ERR_SHAPE = 2,       /* Table 1 dimension rules violated, or d2/d3 < 1          */
  CTPT_ERR_MODULUS = 3,     /* moduli must be distinct odd primes, 2 < p < 2^31                       */
  CTPT_ERR_OVERFLOW = 4,    /* exactness bound of the int8 limb products would fail (refuse, never
                               round: Lemma le:strategy1's d2·‖limb‖·‖limb‖ bound, K = 2^8)          */
  CTPT_ERR_RANGE = 5,       /* an input residue ≥ p (validate=1), or |U| too large for a shared plane */
  CTPT_ERR_UNSUPPORTED = 6, /* format / option not implemented (MLWE, MLWE structured-A)             */
  CTPT_ERR_CUDA = 7         /* a CUDA runtime/driver error (see ctpt_last_error)                    */
} ctpt_status;

typedef enum { CTPT_RLWE = 0, CTPT_SHARED_S = 1, CTPT_SHARED_A = 2, CTPT_STRUCT_A = 3 } ctpt_format;

/* Which kernel path ctpt_matmul / ctpt_matmul_host run per prime (ctpt_problem.kernel).  AUTO:
 * the raw-byte kernel k_gemm_mv when d3_loc ≤ 32 and R has fewer 64-row tiles than the GPU has
 * SMs, the fused skinny kernels when d3_loc ≤ 256, else the limb split + k_gemm_tc.  The first two
 * need kU = 1; k_gemm_mv also needs u_offset = 0 (k_gemm_fused_t forms the unsigned-U row sums
 * itself).  A forced choice that does not apply returns CTPT_ERR_UNSUPPORTED. */
typedef enum {
  CTPT_KERNEL_AUTO = 0,
  CTPT_KERNEL_SPLIT_GEMM = 1, /* k_split[_rows] + k_gemm_tc (tcgen05, any d3, any kU)            */
  CTPT_KERNEL_FUSED = 2,      /* k_gemm_fused_t: split in the GEMM's load path, X read once, the
                                 limbs in tensor memory as the MMA's A operand (d3_loc ≤ 256)      */
  CTPT_KERNEL_MV = 3          /* k_gemm_mv: raw residue bytes × expanded U (d3_loc ≤ 32)          */
} ctpt_kernel;

/* One CP-MM problem, possibly a shard of a larger one:
 * `primes` may be any subset of the RNS basis and [col_begin, col_end) any block of U's
 * columns; outputs then hold exactly that shard. */
typedef struct {
  int32_t fmt;              /* ctpt_format                                                   */
  int32_t L;                /* number of primes in `primes` (1..64)                           */
  int64_t N;                /* ring degree, a power of two                                    */
  int64_t d1, d2, d3;       /* M ∈ R^{d1×d2}, U ∈ Z^{d2×d3}                                   */
  const uint32_t* primes;   /* HOST array of L primes                                         */
  int64_t col_begin;        /* first column of U to multiply (0)                              */
  int64_t col_end;          /* one past the last column; 0 means d3                          */
  int32_t kU;               /* int8 digits per U entry, as returned by ctpt_plain_precompute* */
  int32_t plain_per_prime;  /* 0: one U digit set shared by all primes (ctpt_plain_precompute)
                               1: per-prime digit sets (ctpt_plain_precompute_rns)            */
  int32_t rescale;          /* 0: outputs are (A·U, B·U) mod every prime (Alg. 6 step 1).
                               1: ctpt_matmul also performs Alg. 6 / Alg. 7 step 2, Rescale
                               (P:1681), dividing by q_1 = primes[L−1] (the paper's
                               "q_1 ≈ Δ that divides q"): outputs hold ⌊x / q_1⌉ mod
                               p_l for the first L−1 primes only, x ∈ Z_q the exact product.
                               Needs L ≥ 2 and the whole prime set; the per-prime entry points
                               and ctpt_matmul_host return CTPT_ERR_UNSUPPORTED.            */
  int32_t u_unsigned;       /* 1: the digit plane holds U' = U + u_offset ∈ [0, 255] as u8
                               (ctpt_plain_precompute_unsigned; kU = 1, shared plane, d2 ≤ 33025)
                               and the limb MMAs run u8 × u8; 0: balanced s8 digits.          */
  int32_t u_offset;         /* the offset ctpt_plain_precompute_unsigned returned (≥ 0)        */
  int32_t split_overlap;    /* 1: ctpt_matmul splits prime l+1's residues into limbs INSIDE
                               prime l's GEMM kernel (two otherwise idle warps per CTA), into a
                               second limb workspace — only the first prime's split runs on its
                               own.  Applies to the split + GEMM path (d3_loc > 256, no
                               rescale, kU = 1); the workspace doubles its limb planes.
                               0: split, GEMM, split, GEMM …                                   */
  int32_t kernel;           /* a ctpt_kernel value; 0 = CTPT_KERNEL_AUTO                       */
  int32_t raster_group;     /* k_gemm_tc: j-tiles (128 output columns each) per raster group, so
                               a group's U^T panels stay in L2 while the X panels stream;
                               0: automatic (≈ 32 MB of U^T panels, at least 16)             */
  int32_t max_ctas;         /* cap on the persistent kernels' CTA count; 0: one CTA per SM.  Set
                               it when a concurrent kernel (e.g. an NCCL receive posted before
                               the compute) must keep SMs of its own.         */
} ctpt_problem;

typedef struct {
  size_t ctmat_bytes;       /* d_ctmat: 256-byte header + L·R·d2p int32 (K-major stacked [A;B]) */
  size_t plain_bytes;       /* d_plain for ctpt_plain_precompute: 256 + kU·d3·d2p int8          */
  size_t plain_rns_bytes;   /* d_plain for ctpt_plain_precompute_rns: 256 + L·4·d3·d2p int8     */
  size_t workspace_bytes;   /* d_ws for ctpt_matmul / ctpt_split / ctpt_gemm: the byte limbs of
                               one prime in 32-KB tiles, 4·⌈R/64⌉·64·⌈d2p/128⌉·128 (+ row sums in
                               the unsigned-U mode, + 4·R·d3_loc with rescale, + a second limb
                               buffer with split_overlap, + the raw-byte kernel's U_exp and
                               partials when d3_loc ≤ 32)                                       */
  size_t out_AU_bytes;      /* L_out·d3_loc·rows_A uint32 (L_out = L, or L − 1 with rescale)    */
  size_t out_BU_bytes;      /* L_out·d3_loc·d1 uint32                                          */
  int64_t rows_A, R, d2p, d3_loc;
} ctpt_sizes;

/* Thread-local description of the last non-OK status (never NULL). */
const char* ctpt_last_error(void);

/* Library version / build string, including "src=<hash>": a sha256 prefix of the csrc/ and
 * include/ sources the binary was built from (__graft_entry__.py computes the same hash). */
const char* ctpt_version(void);

/* Validate `prob` (Table 1 rules, primes, exactness bound for prob->kU; kU=0 is treated as 1)
 * and fill `out`.  Host only; needs no GPU. */
ctpt_status ctpt_query_sizes(const ctpt_problem* prob, ctpt_sizes* out);

/* Format layout (column j of A / B are the
 * coefficients of ciphertext j).  Inputs are the per-column ciphertexts of `prob`'s L primes:
 *   d_a_polys: uint32 [L][n_a][N], n_a = d2·(k for shared-s, else 1), poly j·k+t = column j chunk t
 *              (not read, may be NULL, for CTPT_STRUCT_A)
 *   d_b_polys: uint32 [L][d2·k][N]
 * i.e. per prime A and B in column-major order [d2][rows_A] and [d2][d1].
 * Output d_ctmat (ctmat_bytes): a 256-byte header, then for each prime the stacked matrix
 * X = [A; B] ∈ Z_p^{R×d2} in row-major (K-major) int32 with row stride d2p = ⌈d2/16⌉·16 and
 * zero padding.  A pure permutation of int32 values (no limb split; SURVEY.md §8(a) note 2).
 * validate=1 additionally checks every residue is < p (synchronises; CTPT_ERR_RANGE). */
ctpt_status ctpt_layout(const ctpt_problem* prob, const uint32_t* d_a_polys, const uint32_t* d_b_polys,
                        void* d_ctmat, int validate, void* stream);

/* Plaintext precompute ("pre-computation … can be amortized", P:954;
 * k2 = 1 "when U is low-precision").  d_U: int64 [d2][d3] row-major on the device.
 * Requires max|U| < min(p)/2 so the centred residue of U is U itself for every prime (else
 * CTPT_ERR_RANGE: use ctpt_plain_precompute_rns).  Writes kU balanced int8 digit planes
 * (U^T, K-major, [kU][d3][d2p]) into d_plain and the digit count to *kU_out.  Synchronises. */
ctpt_status ctpt_plain_precompute(const ctpt_problem* prob, const int64_t* d_U, void* d_plain, int32_t* kU_out,
                                  void* stream);

/* Unsigned-U plaintext precompute: the same U as ctpt_plain_precompute, stored as ONE u8 plane
 * U' = U + u_offset ∈ [0, 255] with u_offset = max(0, −min U) (*u_offset_out).  The product is
 * unchanged — X·U = X·U' − u_offset·(Σ_k X[r][k]) — and ctpt_split (or, in the skinny regime, the
 * limbs-in-TMEM kernel's converters) forms the per-row sums while it reads X, so the epilogue
 * subtracts u_offset·Σ_k X[r][k] mod p (an O(R) correction, the
 * same bookkeeping as the paper's chop with digits of one sign).  Why: the tensor
 * cores' switching energy depends on the operand bits, and at the 1000 W cap a non-negative
 * small U (no sign-extended high bits) sustains ≈ 5 % more int8 ops
 * (profiles/r01/power_operands_c3gemm.jsonl).  Then set prob->kU = 1, prob->u_unsigned = 1,
 * prob->u_offset = *u_offset_out.  CTPT_ERR_RANGE when max U + u_offset > 255,
 * CTPT_ERR_OVERFLOW when d2 > 33025 (u8·u8 limb products).  Synchronises. */
ctpt_status ctpt_plain_precompute_unsigned(const ctpt_problem* prob, const int64_t* d_U, void* d_plain,
                                           int32_t* u_offset_out, void* stream);

/* General plaintext U ∈ Z_q given as canonical residues d_Ures: uint32 [L][d2][d3].
 * Writes 4 balanced int8 digit planes of each centred residue per prime ([L][4][d3][d2p]),
 * *kU_out = 4; set prob->plain_per_prime = 1 for the matmul.  Synchronises. */
ctpt_status ctpt_plain_precompute_rns(const ctpt_problem* prob, const uint32_t* d_Ures, void* d_plain,
                                      int32_t* kU_out, void* stream);

/* The hot path: (A·U0 mod p, B·U0 mod p) for every prime of `prob` and U columns
 * [col_begin, col_end) (Alg. 6 step 1), and with prob->rescale = 1 the RNS Rescale by
 * the last prime fused into the other primes' epilogues (step 2).  Per prime: the limb split of X into the
 * workspace (timed here by design), then the tcgen05 limb GEMM with
 * the fused recombine + Barrett epilogue (a4, a5).  Outputs in per-column ciphertext layout:
 *   d_AU: uint32 [L][d3_loc][rows_A], d_BU: uint32 [L][d3_loc][d1]   (output column j is
 *   ciphertext j of M·U under the same S).
 * d_ws: workspace_bytes, ws_bytes its size.  Never synchronises. */
ctpt_status ctpt_matmul(const ctpt_problem* prob, const void* d_ctmat, const void* d_plain, uint32_t* d_AU,
                        uint32_t* d_BU, void* d_ws, size_t ws_bytes, void* stream);

/* The two stages of ctpt_matmul for prime index l alone (so callers can time them apart):
 * ctpt_split writes the 4 limb planes of prime l into d_ws; ctpt_gemm consumes them. */
ctpt_status ctpt_split(const ctpt_problem* prob, int32_t l, const void* d_ctmat, void* d_ws, size_t ws_bytes,
                       void* stream);
ctpt_status ctpt_gemm(const ctpt_problem* prob, int32_t l, const void* d_ws, size_t ws_bytes, const void* d_plain,
                      uint32_t* d_AU_l, uint32_t* d_BU_l, void* stream);

/* The skinny-U regime (d3_loc ≤ 256 and kU = 1, CP-Mv at d3 = 1,
 * P:982; Table 4's d3 ∈ {1, 2^6, 2^7}).  For prime index l: the same
 * (A·U mod p, B·U mod p) as ctpt_split + ctpt_gemm, but the limb split runs inside the GEMM's
 * load path, reading the int32 residues of d_ctmat exactly once (no workspace): the regime is
 * HBM-bound and this saves the split's write + re-read.  The kernel (k_gemm_fused_t) keeps the
 * limbs in tensor memory as the MMA's A operand (U^T is B) and, with the unsigned-U plane, forms
 * the row sums Σ_k X[r][k] for the u_offset correction while it splits X.  ctpt_matmul (and
 * ctpt_matmul_host) choose it automatically when d3_loc ≤ 256 and kU = 1 (see ctpt_kernel;
 * ctpt_problem.kernel overrides).  Outputs as for ctpt_gemm.
 * CTPT_ERR_UNSUPPORTED when kU ≠ 1 or d3_loc > 256.  Never synchronises. */
ctpt_status ctpt_gemm_fused(const ctpt_problem* prob, int32_t l, const void* d_ctmat, const void* d_plain,
                            uint32_t* d_AU_l, uint32_t* d_BU_l, void* stream);

/* RNS Rescale of residue arrays by the last prime: d_in uint32 [L][n] canonical
 * residues of elements x ∈ Z_q → d_out uint32 [L−1][n] with ⌊x / primes[L−1]⌉ mod primes[l].
 * Algorithm 7 step 2 rescales BOTH output parts: ctpt_matmul with rescale = 1
 * does B', and this call does Ã (its d1/N polynomials, O(d1) work — "Rescale should be performed
 * on this polynomial representation of Ã"), e.g. d_in = the a_polys of a structured-A
 * ciphertext.  Never synchronises. */
ctpt_status ctpt_rescale(int32_t L, const uint32_t* primes, int64_t n, const uint32_t* d_in, uint32_t* d_out,
                         void* stream);

/* Mod-PP-MM_{q; M, K, Nc} in RNS — the paper's plaintext modular product (notation P:1685,
 * "Mod-PP-MM_{q; d1,d2,d3}"), which CC-MM (Alg. 8: "≈ 12 fp-PP-MM calls",
 * P:1599) and the RGSW product (Alg. 9) reduce to, with operands that are full
 * residues on BOTH sides:  Z = X·Y mod p for every prime p of `primes` (q = Π p).
 *   d_X:   uint32 [L][M][ldx] row-major canonical residues, ldx = K rounded up to 16 (from
 *          ctpt_modmatmul_sizes), the padding columns zero.  Read directly (no layout pass).
 *   d_Y:   uint32 [L][K][Nc] row-major canonical residues; ctpt_modmatmul_precompute turns it
 *          into per-prime balanced-digit planes in d_plain (4 digits: 16 limb MACs per residue
 *          MAC) — done once when Y is reused (synchronises).
 *   d_ZT:  uint32 [L][Nc][M]: Z TRANSPOSED (column j of Z contiguous), like every output here.
 *   d_ws:  ws_bytes from ctpt_modmatmul_sizes.
 * Exact (Lemma le:strategy1 with K = 2^8): K ≤ 65793, else CTPT_ERR_OVERFLOW.  Never
 * synchronises.  Same kernels as ctpt_matmul (the degenerate format "structured-A, N = 1"). */
ctpt_status ctpt_modmatmul_sizes(int32_t L, const uint32_t* primes, int64_t M, int64_t K, int64_t Nc, int64_t* ldx,
                                 size_t* plain_bytes, size_t* ws_bytes);
ctpt_status ctpt_modmatmul_precompute(int32_t L, const uint32_t* primes, int64_t M, int64_t K, int64_t Nc,
                                      const uint32_t* d_Y, void* d_plain, void* stream);
ctpt_status ctpt_modmatmul(int32_t L, const uint32_t* primes, int64_t M, int64_t K, int64_t Nc, const uint32_t* d_X,
                           int64_t ldx, const void* d_plain, uint32_t* d_ZT, void* d_ws, size_t ws_bytes,
                           void* stream);

/* The very-skinny regime (d3_loc ≤ 32, kU = 1; CP-Mv at d3 = 1) for prime l:
 * the int32 residues of d_ctmat are fed to the tensor cores as raw bytes against an expanded
 * U_exp (U's digits spread to byte position ℓ of every 4-byte group, built in d_ws), so every
 * limb product comes out of ONE byte-level contraction with no limb split at all; work is split
 * over K with exact int32 partials in d_ws (ws_bytes from ctpt_query_sizes).  ctpt_matmul
 * takes this kernel automatically when d3_loc ≤ 32 (ctpt_problem.kernel overrides that).  Outputs as for
 * ctpt_gemm.  CTPT_ERR_UNSUPPORTED when kU ≠ 1, d3_loc > 32 or u_offset ≠ 0.  Never synchronises. */
ctpt_status ctpt_gemm_mv(const ctpt_problem* prob, int32_t l, const void* d_ctmat, const void* d_plain,
                         uint32_t* d_AU_l, uint32_t* d_BU_l, void* d_ws, size_t ws_bytes, void* stream);

/* End-to-end executor from HOST buffers (the e2e path): the same computation as
 * ctpt_layout + ctpt_matmul, but the per-column ciphertexts h_a_polys / h_b_polys (layouts as
 * for ctpt_layout) and the outputs h_AU / h_BU (layouts as for ctpt_matmul) live in host
 * memory.  The stacked X of each prime is processed in row chunks of `chunk_rows` (≤ 0: about
 * R/6 rows, rounded to 64 and cut separately within A's and within B's rows, so no chunk straddles
 * the two parts); the host→device copy of one chunk, the layout + split + GEMM of the
 * previous one and the device→host copy of the one before run concurrently (two internal
 * copy streams forked from and joined back into `stream`).  Host buffers must be page-locked
 * (cudaHostAlloc / cudaHostRegister) for the copies to overlap.  d_plain as for ctpt_matmul;
 * d_ws: at least ctpt_host_workspace_bytes(prob, chunk_rows) bytes.  Returns once everything
 * is enqueued; the results are in host memory after `stream` completes.  No validation of
 * residue ranges (use ctpt_layout with validate=1 for that). */
ctpt_status ctpt_host_workspace_bytes(const ctpt_problem* prob, int64_t chunk_rows, size_t* bytes);
ctpt_status ctpt_matmul_host(const ctpt_problem* prob, const uint32_t* h_a_polys, const uint32_t* h_b_polys,
                             const void* d_plain, uint32_t* h_AU, uint32_t* h_BU, void* d_ws, size_t ws_bytes,
                             int64_t chunk_rows, void* stream);

/* The host executor over n UNITS in one pipeline (e.g. a rank's (prime, column-block) units of
 * the multi-GPU plan, or the primes of one problem held in separate host
 * buffers): unit u is problem probs[u] with host inputs h_a_polys[u] / h_b_polys[u], plaintext
 * d_plains[u] and host outputs h_AUs[u] / h_BUs[u], each exactly as for ctpt_matmul_host.  The
 * chunks of all units flow through one set of staging buffers and copy streams, so unit u+1's
 * first copies overlap unit u's last GEMMs and copies: one pipeline fill and one drain per call
 * instead of one per unit (n calls of ctpt_matmul_host on one stream serialise, since each joins
 * its device→host stream back into `stream` before the next forks).  d_ws: at least
 * ctpt_host_workspace_bytes_units(n, probs, chunk_rows) bytes (each staging region sized for the
 * largest unit).  Every unit is validated before anything is enqueued; errors as for
 * ctpt_matmul_host (CTPT_ERR_ARG for n < 1).  ctpt_matmul_host(p, …) ≡ the n = 1 case. */
ctpt_status ctpt_host_workspace_bytes_units(int32_t n, const ctpt_problem* probs, int64_t chunk_rows,
                                            size_t* bytes);
ctpt_status ctpt_matmul_host_units(int32_t n, const ctpt_problem* probs, const uint32_t* const* h_a_polys,
                                   const uint32_t* const* h_b_polys, const void* const* d_plains,
                                   uint32_t* const* h_AUs, uint32_t* const* h_BUs, void* d_ws, size_t ws_bytes,
                                   int64_t chunk_rows, void* stream);

/* ctpt_gemm for prime l with the limb split of prime l+1 fused in (prob->split_overlap = 1,
 * no rescale, L ≥ 2): while prime l's MMAs run, two otherwise idle warps of every CTA split
 * prime l+1's residues of d_ctmat into the OTHER limb buffer of d_ws (prime l uses buffer l & 1;
 * ctpt_split(prob, l, …) fills buffer l & 1 too), so a step is ctpt_split(0), then
 * ctpt_gemm_next(l) for l = 0 … L−1 (the last one splits nothing).  Outputs, errors and
 * synchronisation as for ctpt_gemm; CTPT_ERR_ARG without split_overlap. */
ctpt_status ctpt_gemm_next(const ctpt_problem* prob, int32_t l, const void* d_ctmat, void* d_ws, size_t ws_bytes,
                           const void* d_plain, uint32_t* d_AU_l, uint32_t* d_BU_l, void* stream);

/* ---- Multi-GPU gather over peer memory (output column j is ciphertext j,
 * P:1688–1690, so a (prime, column-block) unit's outputs are one contiguous block of the gathered
 * [L][d3][rows] layout and a remote rank's ctpt_matmul can store them there directly).
 *
 * ctpt_ipc_export: a CUDA IPC handle (CTPT_IPC_HANDLE_BYTES opaque bytes written to `handle`) for
 *   the device allocation containing d_ptr, and d_ptr's byte offset in it (the allocation may be a
 *   block of a caching allocator's larger segment).  Host only, no stream work.
 * ctpt_ipc_open: map a handle exported by another process into the CALLING thread's current
 *   device (the owner may be another GPU: peer access is enabled as needed,
 *   cudaIpcMemLazyEnablePeerAccess), so the current device's kernels can store into it over
 *   NVLink.  *d_base receives the mapping's base (for ctpt_ipc_close), *d_ptr = base + offset.
 *   Errors: CTPT_ERR_CUDA (e.g. no peer access between the two devices: use an NCCL gather).
 * ctpt_ipc_close: unmap a base returned by ctpt_ipc_open.
 * ctpt_peer_access: *can = 1 if `device` can read and write `peer`'s memory (1 when device ==
 *   peer).  Does not enable anything. */
#define CTPT_IPC_HANDLE_BYTES 64
ctpt_status ctpt_ipc_export(const void* d_ptr, void* handle, uint64_t* offset);
ctpt_status ctpt_ipc_open(const void* handle, uint64_t offset, void** d_base, void** d_ptr);
ctpt_status ctpt_ipc_close(void* d_base);
ctpt_status ctpt_peer_access(int32_t device, int32_t peer, int32_t* can);

/* Bring-up / diagnostics only (not a product path): the same limb GEMM and epilogue on
 * CUDA cores, reading the same workspace and plain planes.  Used by the tests to tell a
 * layout/split bug from a tensor-core descriptor bug. */
ctpt_status ctpt_gemm_simt(const ctpt_problem* prob, int32_t l, const void* d_ws, size_t ws_bytes,
                           const void* d_plain, uint32_t* d_AU_l, uint32_t* d_BU_l, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CTPT_H_ */
