"""CPU oracle for the CP-MM hot path — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2503_16080_b200``) never imports it and shares no code with it.

What it computes, and where the paper defines it (``P:n`` = PAPER.md line n):

* ``encode``            ⌊Δ·m⌉ = ⌊Δ·m + ½⌋
* ``toeplitz``          toep(m), the matrix of u ↦ u·m in R_N
* ``negacyclic_mul``    c = toep(s)·Vec(a) mod p, C schoolbook
* ``secret_matrix``     S_RLWE = toep(sk), S_sh-s = I ⊗ toep(sk),
                        S_sh-a = [toep(sk_0); …; toep(sk_{k-1})]
* ``struct_a_matrices`` structured-A shared-a: Ã = [toep(a_0); …; toep(a_{k-1})] and
                        S = [Vec(sk_j)]_j with Ã·S + B ≈ M
* ``su_column``         column j of S·U, the Algorithm 7 output key
* ``format_matrices``   (A, B) with column j = the coefficients of ciphertext j
                        
* ``encrypt_small``     b = P − S-part, so that a·sk + b = P
* ``modmatmul``         (X·U0) mod p, schoolbook with 128-bit accumulation
                        (Alg. 6 step 1; Thm th:pcmm P:1711, th:pcmm-shs P:1722)
* ``decrypt_cols``      S·A' + B' mod p (identity at P:1688)
* ``crt_centred``       centred CRT over the RNS basis (reading Q14)
* ``rescale_last``      Rescale(x) = ⌊x / q_1⌉ mod q/q_1 with q_1 the last prime
                        (Alg. 6 step 2 P:1705), exact integers
* ``precision_bits``    log‖M‖∞ − log‖M − M̃‖∞
* ``freivalds``         probabilistic check of C = X·U mod p (test protocol)

Every function is pinned by tests/test_oracle_pins.py against things the paper
or mathematics fix (closed forms, SPEC/paper examples, brute force in exact
Python integers).  The paper prints no numeric worked example for CP-MM
(SURVEY.md §8(c) c4), so no function pins against a printed CP-MM output: against printed
values the CP-MM functions are "parity unpinned"; each is pinned by the
identities and brute-force cases listed in the tests instead.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

RLWE, SHARED_S, SHARED_A, STRUCT_A = 0, 1, 2, 3


def build(force: bool = False) -> str:
    import subprocess

    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c11", "-o", _LIB_PATH, src])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, u32, P = ctypes.c_int64, ctypes.c_uint32, ctypes.c_void_p
        L.orc_modmatmul_cols.restype = None
        L.orc_modmatmul_cols.argtypes = [P, i64, i64, P, i64, P, i64, u32, P, ctypes.c_int]
        L.orc_modmatmul_entries.restype = None
        L.orc_modmatmul_entries.argtypes = [P, i64, i64, P, i64, P, P, i64, u32, P, ctypes.c_int]
        L.orc_freivalds.restype = i64
        L.orc_freivalds.argtypes = [P, i64, i64, P, i64, P, u32, P, P, P, ctypes.c_int]
        L.orc_negacyclic_mul.restype = None
        L.orc_negacyclic_mul.argtypes = [P, P, i64, u32, P]
        L.orc_decrypt_col.restype = ctypes.c_int
        L.orc_decrypt_col.argtypes = [ctypes.c_int, i64, i64, P, P, P, u32, P, ctypes.c_int]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle expects C-contiguous arrays"
    return ctypes.c_void_p(a.ctypes.data)


# ----------------------------------------------------------------------------------
# L0 arithmetic: rounding, Toeplitz, negacyclic ring
# ----------------------------------------------------------------------------------
def round_half_up(x: float) -> int:
    """⌊x⌉ = integer part of x + 1/2, evaluated exactly: r = floor(x);
    r += (x - r >= 0.5).  x - r is exact for |x| < 2^52 (Sterbenz), and x is an
    integer already when |x| >= 2^52 (reading Q9)."""
    r = math.floor(x)
    if x - r >= 0.5:
        r += 1
    return int(r)


def encode(m, log_delta: int):
    """CKKS coefficient encoding of reals: ⌊Δ·m⌉ with Δ = 2^log_delta.
    Δ is a power of two, so Δ·m is exact (ldexp)."""
    if np.isscalar(m):
        return round_half_up(math.ldexp(float(m), log_delta))
    m = np.asarray(m, dtype=np.float64)
    return np.array([round_half_up(math.ldexp(float(v), log_delta)) for v in m.ravel()],
                    dtype=np.int64).reshape(m.shape)


def decode(p_int, log_delta: int):
    """Dcd_coeff(p) = p_i / Δ."""
    return np.asarray(p_int, dtype=np.float64) / float(2 ** log_delta) if not np.isscalar(p_int) \
        else float(p_int) / float(2 ** log_delta)


def toeplitz(m) -> np.ndarray:
    """toep(m) ∈ Z^{N×N}: entry (i, j) = m_{i-j} if i ≥ j else −m_{N+i-j}.
    Returned as an int64 (object when entries are Python ints) matrix over Z (not reduced)."""
    m = list(m)
    N = len(m)
    T = np.empty((N, N), dtype=object)
    for i in range(N):
        for j in range(N):
            T[i, j] = m[i - j] if i >= j else -m[N + i - j]
    try:
        return T.astype(np.int64)
    except OverflowError:
        return T


def negacyclic_mul(a: np.ndarray, s: np.ndarray, p: int) -> np.ndarray:
    """Vec(a·s mod (p, X^N+1)) = toep(s)·Vec(a) mod p, schoolbook in C.
    a: canonical residues (uint32), s: small signed integers (int64)."""
    a = np.ascontiguousarray(a, dtype=np.uint32)
    s = np.ascontiguousarray(s, dtype=np.int64)
    out = np.empty_like(a)
    lib().orc_negacyclic_mul(_ptr(a), _ptr(s), a.shape[0], p, _ptr(out))
    return out


# ----------------------------------------------------------------------------------
# L2 formats with structured S (Table 1)
# ----------------------------------------------------------------------------------
def rows_A(fmt: int, N: int, d1: int) -> int:
    """Row count of the A the CP-MM multiplies: N for RLWE and shared-a (A ∈ Z_q^{N×d2},
    Lemma le:mat_struct_s), d1 for shared-s (A ∈ Z_q^{d1×d2}), and 0
    for structured-A shared-a, where Algorithm 7 multiplies only B."""
    if fmt == STRUCT_A:
        return 0
    return d1 if fmt == SHARED_S else N


def check_dims(fmt: int, N: int, d1: int) -> None:
    """Table 1: RLWE needs d1 = N; shared-s / shared-a need N | d1; N a power of two."""
    if N <= 0 or N & (N - 1):
        raise ValueError("N must be a power of two")
    if fmt == RLWE and d1 != N:
        raise ValueError("RLWE format requires d1 = N")
    if d1 % N:
        raise ValueError("shared-s / shared-a / structured-A formats require N | d1")


def secret_matrix(fmt: int, sks, N: int, d1: int) -> np.ndarray:
    """Dense structured secret S over Z (small N only):
    S_RLWE = toep(sk); S_sh-s = I_{d1/N} ⊗ toep(sk);
    S_sh-a = vertical stack of toep(sk_t), t < k."""
    check_dims(fmt, N, d1)
    k = d1 // N
    if fmt == RLWE:
        return toeplitz(sks[0])
    if fmt == SHARED_S:
        return np.kron(np.eye(k, dtype=np.int64), toeplitz(sks[0]))
    return np.vstack([toeplitz(sks[t]) for t in range(k)])


def format_matrices(fmt: int, N: int, d1: int, a_polys: np.ndarray, b_polys: np.ndarray):
    """(A, B) for ONE prime from per-column ciphertexts (column j of A
    holds the coefficients of a_j).  a_polys: [n_a][N], b_polys: [ncols*k][N] (uint32).
    Chunk t of column j is poly j*k + t and occupies rows [tN, (t+1)N) (reading Q18).
    Returns dense A [rows_A][ncols], B [d1][ncols]."""
    check_dims(fmt, N, d1)
    k = d1 // N
    ncols = b_polys.shape[0] // k
    B = np.empty((d1, ncols), dtype=np.uint32)
    for j in range(ncols):
        for t in range(k):
            B[t * N:(t + 1) * N, j] = b_polys[j * k + t]
    if fmt == STRUCT_A:  # Ã is not a per-column matrix; Algorithm 7 multiplies B only
        A = np.empty((0, ncols), dtype=np.uint32)
    elif fmt == SHARED_S:
        A = np.empty((d1, ncols), dtype=np.uint32)
        for j in range(ncols):
            for t in range(k):
                A[t * N:(t + 1) * N, j] = a_polys[j * k + t]
    else:
        A = np.empty((N, ncols), dtype=np.uint32)
        for j in range(ncols):
            A[:, j] = a_polys[j]
    return A, B


def struct_a_matrices(a_polys, sks):
    """Structured-A shared-a: Ã = (toep(a_0)^t | … | toep(a_{k-1})^t)^t ∈ Z^{d1×N}
    from the k row-block polynomials a_i, and S ∈ Z^{N×d2} the horizontal concatenation of
    Vec(sk_j), so that Ã·S + B ≈ M (mod q).  Small sizes only (dense, object entries)."""
    At = np.vstack([toeplitz([int(v) for v in a]) for a in a_polys]).astype(object)
    S = np.stack([np.asarray(s, dtype=np.int64) for s in sks], axis=1).astype(object)
    return At, S


def su_column(sks, U: np.ndarray, j: int) -> np.ndarray:
    """Column j of S·U with S = [Vec(sk_0) | … | Vec(sk_{d2-1})]: Σ_k U[k][j]·sk_k over Z —
    the secret of output column j of Algorithm 7 (the key S·U)."""
    acc = np.zeros(len(sks[0]), dtype=np.int64)
    for k in range(U.shape[0]):
        u = int(U[k, j])
        if u:
            acc += u * np.asarray(sks[k], dtype=np.int64)
    return acc


def encrypt_small(fmt: int, sks, P: np.ndarray, a_cols: np.ndarray, p: int) -> np.ndarray:
    """b-parts of a structured-S encryption of the integer plaintext P ∈ Z^{d1×d2}
    given the a-parts (dense A), by the matrix identity S·A + B = P mod p
    (Lemma le:mat_struct_s; Dec P:852; reading Q25: b = P − a·sk).
    Small sizes only (dense S, exact Python integers)."""
    d1 = P.shape[0]
    N = len(sks[0])
    S = secret_matrix(fmt, sks, N, d1).astype(object)
    SA = S.dot(a_cols.astype(object))
    B = (P.astype(object) - SA) % p
    return B.astype(np.uint32)


# ----------------------------------------------------------------------------------
# L4/L5: Alg. 6 step 1 — the two Mod-PP-MMs
# ----------------------------------------------------------------------------------
def modmatmul(X_colmajor: np.ndarray, U: np.ndarray, p: int, cols=None, nthreads: int = 0) -> np.ndarray:
    """(X·U0) mod p on output columns `cols` (default: all), schoolbook.
    X_colmajor: uint32 [d2][rows] (column k of X contiguous, as the ciphertexts store it);
    U: int64 [d2][d3].  Returns uint32 [ncols][rows] (output column j contiguous)."""
    X = np.ascontiguousarray(X_colmajor, dtype=np.uint32)
    U = np.ascontiguousarray(U, dtype=np.int64)
    d2, rows = X.shape
    assert U.shape[0] == d2
    d3 = U.shape[1]
    cols = np.arange(d3, dtype=np.int64) if cols is None else np.ascontiguousarray(cols, dtype=np.int64)
    out = np.empty((cols.shape[0], rows), dtype=np.uint32)
    lib().orc_modmatmul_cols(_ptr(X), rows, d2, _ptr(U), d3, _ptr(cols), cols.shape[0], p, _ptr(out), nthreads)
    return out


def modmatmul_entries(X_colmajor: np.ndarray, U: np.ndarray, p: int, r_idx, j_idx, nthreads: int = 0):
    X = np.ascontiguousarray(X_colmajor, dtype=np.uint32)
    U = np.ascontiguousarray(U, dtype=np.int64)
    d2, rows = X.shape
    r_idx = np.ascontiguousarray(r_idx, dtype=np.int64)
    j_idx = np.ascontiguousarray(j_idx, dtype=np.int64)
    out = np.empty(r_idx.shape[0], dtype=np.uint32)
    lib().orc_modmatmul_entries(_ptr(X), rows, d2, _ptr(U), U.shape[1], _ptr(r_idx), _ptr(j_idx),
                                r_idx.shape[0], p, _ptr(out), nthreads)
    return out


def freivalds(X_colmajor: np.ndarray, U: np.ndarray, C: np.ndarray, p: int, v: np.ndarray,
              nthreads: int = 0) -> int:
    """Number of rows r where (C·v)[r] != (X·(U·v))[r] mod p.  C: uint32 [d3][rows]."""
    X = np.ascontiguousarray(X_colmajor, dtype=np.uint32)
    U = np.ascontiguousarray(U, dtype=np.int64)
    C = np.ascontiguousarray(C, dtype=np.uint32)
    v = np.ascontiguousarray(v, dtype=np.uint64)
    d2, rows = X.shape
    assert C.shape == (U.shape[1], rows)
    return int(lib().orc_freivalds(_ptr(X), rows, d2, _ptr(U), U.shape[1], _ptr(C), p, _ptr(v), None, None,
                                   nthreads))


def decrypt_col(fmt: int, N: int, d1: int, sks, a_col: np.ndarray, b_col: np.ndarray, p: int,
                nthreads: int = 0) -> np.ndarray:
    """S·a + b mod p for one column in a structured-S format.  For
    structured-A shared-a (fmt 3) it is Ã·key + b: `a_col` holds the k = d1/N shared
    polynomials a_t (k·N entries) and sks = [key], the column's Vec(sk_j) — or (S·U)_j for an
    Algorithm 7 output column."""
    k = d1 // N
    nkeys = k if fmt == SHARED_A else 1
    S = np.ascontiguousarray(np.stack([np.asarray(sks[t], dtype=np.int64) for t in range(nkeys)]))
    a = np.ascontiguousarray(a_col, dtype=np.uint32).ravel()
    b = np.ascontiguousarray(b_col, dtype=np.uint32)
    want_a = d1 if fmt == STRUCT_A else rows_A(fmt, N, d1)
    assert a.shape[0] == want_a and b.shape[0] == d1
    out = np.empty(d1, dtype=np.uint32)
    rc = lib().orc_decrypt_col(fmt, N, d1, _ptr(S), _ptr(a), _ptr(b), p, _ptr(out), nthreads)
    assert rc == 0
    return out


# ----------------------------------------------------------------------------------
# Decode: CRT over the RNS basis and precision
# ----------------------------------------------------------------------------------
def crt_centred(residues, primes) -> int:
    """The unique x ∈ (−q/2, q/2] with x ≡ residues[i] (mod primes[i]), q = Π primes
    (Strategy 3's CRT step; centred representative P:4, reading Q14).
    Exact Python integers: x = Σ r_i·(q/p_i)·((q/p_i)^{-1} mod p_i) mod q."""
    q = 1
    for p in primes:
        q *= int(p)
    x = 0
    for r, p in zip(residues, primes):
        p = int(p)
        qi = q // p
        x += int(r) * qi * pow(qi, -1, p)
    x %= q
    if x > q // 2:
        x -= q
    return x


def crt_centred_array(res: np.ndarray, primes) -> list:
    """res: [L][n] residues → list of n exact centred integers."""
    res = np.asarray(res)
    return [crt_centred([int(res[l, i]) for l in range(res.shape[0])], primes) for i in range(res.shape[1])]


def round_div(x: int, d: int) -> int:
    """⌊x/d⌉ = ⌊x/d + 1/2⌋ for integers, d > 0, exactly: ⌊(2x + d) / (2d)⌋."""
    return (2 * int(x) + int(d)) // (2 * int(d))


def rescale_last(res: np.ndarray, primes) -> np.ndarray:
    """Rescale: (A, B) ↦ (⌊A/Δ⌉, ⌊B/Δ⌉) with Δ replaced by q_1 = primes[-1], a
    divisor of q ("choose q_1 ≈ Δ that divides q and replace q/Δ by q/q_1").
    res: canonical residues [L][n] of elements x ∈ Z_q; returns the residues [L−1][n] of
    ⌊x/q_1⌉ mod q/q_1 — the plain definition: CRT to the exact integer, divide, round.
    (The result does not depend on the representative of x: x + q gives + q/q_1.)"""
    res = np.asarray(res)
    L, n = res.shape
    q1 = int(primes[-1])
    out = np.empty((L - 1, n), dtype=np.uint32)
    for i in range(n):
        x = crt_centred([int(res[l, i]) for l in range(L)], primes)
        y = round_div(x, q1)
        for l in range(L - 1):
            out[l, i] = y % int(primes[l])
    return out


def precision_bits(M_ref: np.ndarray, M_approx: np.ndarray) -> float:
    """prec = log2‖M‖∞ − log2‖M − M̃‖∞; +inf when exact."""
    num = float(np.max(np.abs(M_ref)))
    den = float(np.max(np.abs(np.asarray(M_ref, dtype=np.float64) - np.asarray(M_approx, dtype=np.float64))))
    if den == 0.0:
        return math.inf
    return math.log2(num) - math.log2(den)


# ----------------------------------------------------------------------------------
# Strategy 1 bookkeeping (Lemma le:strategy1) — used to pin limb counts
# ----------------------------------------------------------------------------------
def strategy1_counts(theta1: float, theta2: float, d2: int, K: int | None = None):
    """K = ⌊√(2^53/d2)⌋ and k_i = ⌈log θ_i / log K⌉ (Lemma le:strategy1).
    With K given explicitly (e.g. 2^8 for an int8 tensor-core analogue) only the k_i change."""
    if K is None:
        K = math.isqrt(2 ** 53 // d2)
    k1 = max(1, math.ceil(math.log(theta1) / math.log(K)))
    k2 = max(1, math.ceil(math.log(theta2) / math.log(K)))
    return k1, k2


def chop(r: int, K: int) -> list:
    """Signed base-K decomposition r = Σ r_i K^i with r_i of the sign of r and |r_i| < K
    (proof of Lemma le:strategy1)."""
    sgn = -1 if r < 0 else 1
    m = abs(int(r))
    digits = []
    while m:
        digits.append(sgn * (m % K))
        m //= K
    return digits or [0]
