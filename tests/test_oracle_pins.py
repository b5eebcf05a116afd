"""Pins for the CPU oracle (oracle/), -m "not gpu".

Every oracle function is checked here against something other than itself:
values the paper (or the SPEC written from it) prints (tests/golden/), closed
forms, special cases, and brute force in exact Python integers.  Each test
names the plausible oracle mistake it would catch.
"""
import json
import math
import os
import random
from fractions import Fraction

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_fixtures.json")))
P31 = 2147352577  # a prime < 2^31, ≡ 1 mod 2^16 (checked in test_ctgen)


# ------------------------------------------------------------------ rounding / encoding
def test_round_ties_golden():
    # catches floor(x+0.5)-style double rounding and ties-to-even
    for x, r in GOLD["round_ties"]["cases"]:
        assert oracle.round_half_up(x) == r, x


def test_encode_golden():
    for key in ("encode_half_at_2_20", "encode_zero"):
        g = GOLD[key]
        assert oracle.encode(g["z"], g["log_delta"]) == g["encoded"]


@pytest.mark.parametrize("log_delta", [10, 20, 40, 45, 50, 52, 53, 60])
def test_encode_matches_exact_rational(log_delta):
    # ⌊Δm⌉ = floor(Δm + 1/2) in exact rationals; catches a wrong tie or a lost bit
    rng = random.Random(log_delta)
    for _ in range(2000):
        m = rng.uniform(-1, 1)
        want = math.floor(Fraction(m) * 2 ** log_delta + Fraction(1, 2))
        assert oracle.encode(m, log_delta) == want
    # exact ties
    for n in range(-5, 6):
        m = (n + 0.5) / 2 ** log_delta
        assert oracle.encode(m, log_delta) == math.floor(Fraction(m) * 2 ** log_delta + Fraction(1, 2))


# ------------------------------------------------------------------ Toeplitz / ring
def test_toeplitz_golden():
    for key in ("toeplitz_1_plus_2X_N2", "toeplitz_general_N4"):
        g = GOLD[key]
        assert oracle.toeplitz(g["m"]).tolist() == g["toep"]


def _polymul_negacyclic_bruteforce(x, y):
    """x·y in Z[X]/(X^N+1) by explicit polynomial multiplication and X^N = -1 folding."""
    N = len(x)
    full = [0] * (2 * N)
    for i in range(N):
        for j in range(N):
            full[i + j] += int(x[i]) * int(y[j])
    return [full[i] - full[i + N] for i in range(N)]


def test_toeplitz_columns_are_shifted_products():
    # column j of toep(m) = Vec(X^j · m) (P:1072 definition of rotmtx); catches a sign or index slip
    rng = random.Random(1)
    N = 8
    m = [rng.randint(-9, 9) for _ in range(N)]
    T = oracle.toeplitz(m)
    for j in range(N):
        xj = [0] * N
        xj[j] = 1
        assert T[:, j].tolist() == _polymul_negacyclic_bruteforce(xj, m)


@pytest.mark.parametrize("N", [8, 64])
def test_toeplitz_times_vec_is_ring_product(N):
    # toep(x)·Vec(y) = Vec(x·y) (SPEC acceptance 1)
    rng = random.Random(N)
    for _ in range(20 if N == 64 else 100):
        x = [rng.randint(-50, 50) for _ in range(N)]
        y = [rng.randint(-50, 50) for _ in range(N)]
        assert oracle.toeplitz(x).dot(np.array(y, dtype=np.int64)).tolist() == _polymul_negacyclic_bruteforce(x, y)


def test_x_pow_n_minus_one():
    N = GOLD["X_pow_N_is_minus_one"]["N"]
    a = np.zeros(N, dtype=np.uint32)
    a[N - 1] = 1  # X^{N-1}
    s = np.zeros(N, dtype=np.int64)
    s[1] = 1  # X
    out = oracle.negacyclic_mul(a, s, P31)
    want = np.zeros(N, dtype=np.uint32)
    want[0] = P31 - 1  # -1 mod p
    assert (out == want).all()


@pytest.mark.parametrize("N", [1, 2, 8, 16, 64])
def test_negacyclic_mul_bruteforce(N):
    rng = np.random.default_rng(N)
    for _ in range(10):
        a = rng.integers(0, P31, N, dtype=np.uint64).astype(np.uint32)
        s = rng.integers(-1, 2, N).astype(np.int64)
        want = [v % P31 for v in _polymul_negacyclic_bruteforce(a.tolist(), s.tolist())]
        assert oracle.negacyclic_mul(a, s, P31).tolist() == want


# ------------------------------------------------------------------ structured S
def test_secret_matrices_structure():
    N, k = 4, 3
    rng = random.Random(3)
    sks = [[rng.randint(-1, 1) for _ in range(N)] for _ in range(k)]
    S = oracle.secret_matrix(oracle.RLWE, sks, N, N)
    assert S.shape == (N, N) and (S == oracle.toeplitz(sks[0])).all()
    Ss = oracle.secret_matrix(oracle.SHARED_S, sks, N, k * N)  # I ⊗ toep(sk): block diagonal, identical blocks
    assert Ss.shape == (k * N, k * N)
    for t in range(k):
        for u in range(k):
            blk = Ss[t * N:(t + 1) * N, u * N:(u + 1) * N]
            assert (blk == (oracle.toeplitz(sks[0]) if t == u else 0)).all()
    Sa = oracle.secret_matrix(oracle.SHARED_A, sks, N, k * N)  # vertical stack of k Toeplitz blocks
    assert Sa.shape == (k * N, N)
    for t in range(k):
        assert (Sa[t * N:(t + 1) * N] == oracle.toeplitz(sks[t])).all()


def test_dims_rules_table1():
    with pytest.raises(ValueError):
        oracle.check_dims(oracle.RLWE, 16, 32)
    with pytest.raises(ValueError):
        oracle.check_dims(oracle.SHARED_S, 16, 40)
    with pytest.raises(ValueError):
        oracle.check_dims(oracle.SHARED_A, 12, 24)
    oracle.check_dims(oracle.SHARED_A, 16, 64)
    assert oracle.rows_A(oracle.SHARED_A, 16, 64) == 16  # shared-a stores N·d2 a-entries
    assert oracle.rows_A(oracle.SHARED_S, 16, 64) == 64
    assert oracle.rows_A(oracle.RLWE, 16, 16) == 16


def test_format_matrices_layout():
    # A[tN+i][j] = coefficient i of a_{t,j} (shared-s), B likewise (reading Q18)
    N, k, ncols = 4, 2, 3
    a = np.arange(ncols * k * N, dtype=np.uint32).reshape(ncols * k, N)
    b = 1000 + np.arange(ncols * k * N, dtype=np.uint32).reshape(ncols * k, N)
    A, B = oracle.format_matrices(oracle.SHARED_S, N, k * N, a, b)
    for j in range(ncols):
        for t in range(k):
            for i in range(N):
                assert A[t * N + i, j] == a[j * k + t, i]
                assert B[t * N + i, j] == b[j * k + t, i]
    a2 = np.arange(ncols * N, dtype=np.uint32).reshape(ncols, N)
    A2, B2 = oracle.format_matrices(oracle.SHARED_A, N, k * N, a2, b)
    assert A2.shape == (N, ncols) and (A2[:, 1] == a2[1]).all()


# ------------------------------------------------------------------ modular matmul (Alg. 6 step 1)
def _brute_modmatmul(X, U, p):
    """exact Python-integer (X · (U mod p)) mod p, X: [rows][d2]."""
    Xo = X.astype(object)
    Uo = (U.astype(object)) % p
    return Xo.dot(Uo) % p


def test_modmatmul_golden_1x1():
    g = GOLD["modmatmul_1x1"]
    X = np.array([[g["X"]]], dtype=np.uint32)
    U = np.array([[g["U"]]], dtype=np.int64)
    assert oracle.modmatmul(X, U, g["p"])[0, 0] == g["out"]


@pytest.mark.parametrize("rows,d2,d3", [(1, 1, 1), (7, 5, 3), (33, 64, 9), (64, 129, 17)])
def test_modmatmul_bruteforce(rows, d2, d3):
    rng = np.random.default_rng(rows * 1000 + d2)
    X = rng.integers(0, P31, (rows, d2), dtype=np.uint64).astype(np.uint32)
    X[0, :] = P31 - 1  # extreme residues
    U = rng.integers(-8, 9, (d2, d3)).astype(np.int64)
    U[:, 0] = -8
    C = oracle.modmatmul(np.ascontiguousarray(X.T), U, P31)  # [d3][rows]
    want = _brute_modmatmul(X, U, P31)
    assert (C.T.astype(object) == want).all()


def test_modmatmul_large_U_residues():
    # U entries near ±p/2 and beyond (the general U ∈ Z_q case of precompute_rns)
    rng = np.random.default_rng(5)
    import ctgen

    p = ctgen.primes(3)[2]
    X = rng.integers(0, p, (9, 40), dtype=np.uint64).astype(np.uint32)
    U = rng.integers(-(2 ** 40), 2 ** 40, (40, 6)).astype(np.int64)
    C = oracle.modmatmul(np.ascontiguousarray(X.T), U, p)
    assert (C.T.astype(object) == _brute_modmatmul(X, U, p)).all()


def test_modmatmul_special_cases():
    rng = np.random.default_rng(7)
    rows, d2 = 12, 10
    Xc = rng.integers(0, P31, (d2, rows), dtype=np.uint64).astype(np.uint32)  # col-major
    I = np.eye(d2, dtype=np.int64)
    assert (oracle.modmatmul(Xc, I, P31) == Xc).all()  # U = I → A
    assert (oracle.modmatmul(Xc, np.zeros((d2, 3), np.int64), P31) == 0).all()  # U = 0 → 0
    E = np.zeros((d2, 4), dtype=np.int64)
    E[3, 2] = -1  # U = -e_3 e_2^T copies the negated column 3 into output column 2
    C = oracle.modmatmul(Xc, E, P31)
    assert (C[2] == (P31 - Xc[3].astype(np.int64)) % P31).all()
    assert (C[0] == 0).all()


def test_modmatmul_linear_in_U():
    rng = np.random.default_rng(9)
    Xc = rng.integers(0, P31, (20, 16), dtype=np.uint64).astype(np.uint32)
    U1 = rng.integers(-8, 9, (20, 5)).astype(np.int64)
    U2 = rng.integers(-8, 9, (20, 5)).astype(np.int64)
    C1 = oracle.modmatmul(Xc, U1, P31).astype(np.int64)
    C2 = oracle.modmatmul(Xc, U2, P31).astype(np.int64)
    C12 = oracle.modmatmul(Xc, U1 + U2, P31).astype(np.int64)
    assert ((C1 + C2) % P31 == C12).all()


def test_modmatmul_entries_and_freivalds():
    rng = np.random.default_rng(11)
    d2, rows, d3 = 50, 40, 30
    Xc = rng.integers(0, P31, (d2, rows), dtype=np.uint64).astype(np.uint32)
    U = rng.integers(-8, 9, (d2, d3)).astype(np.int64)
    C = oracle.modmatmul(Xc, U, P31)
    r_idx = rng.integers(0, rows, 100)
    j_idx = rng.integers(0, d3, 100)
    assert (oracle.modmatmul_entries(Xc, U, P31, r_idx, j_idx) == C[j_idx, r_idx]).all()
    v = rng.integers(0, P31, d3, dtype=np.uint64)
    assert oracle.freivalds(Xc, U, C, P31, v) == 0
    Cbad = C.copy()
    Cbad[4, 7] = (int(Cbad[4, 7]) + 1) % P31
    assert oracle.freivalds(Xc, U, Cbad, P31, v) == 1


# ------------------------------------------------------------------ decryption
@pytest.mark.parametrize("fmt,N,k", [(oracle.RLWE, 8, 1), (oracle.SHARED_S, 8, 3), (oracle.SHARED_A, 8, 3)])
def test_decrypt_col_matches_dense_S(fmt, N, k):
    rng = np.random.default_rng(fmt * 10 + N)
    d1 = N * k
    nkeys = k if fmt == oracle.SHARED_A else 1
    sks = [rng.integers(-1, 2, N).tolist() for _ in range(nkeys)]
    ra = oracle.rows_A(fmt, N, d1)
    a = rng.integers(0, P31, ra, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, P31, d1, dtype=np.uint64).astype(np.uint32)
    S = oracle.secret_matrix(fmt, sks, N, d1).astype(object)
    want = (S.dot(a.astype(object)) + b.astype(object)) % P31
    assert oracle.decrypt_col(fmt, N, d1, sks, a, b, P31).tolist() == want.tolist()


# ------------------------------------------------------------------ CRT / precision
def test_crt_small_bruteforce():
    primes = [3, 5, 7]
    q = 105
    for x in range(-52, 53):  # (−q/2, q/2]
        res = [x % p for p in primes]
        assert oracle.crt_centred(res, primes) == x
    # the SPEC's {3,5}, 7 → residues (1,2) → 7 example
    assert oracle.crt_centred([1, 2], [3, 5]) == 7


def test_crt_big():
    import ctgen

    ps = ctgen.primes(8)
    q = math.prod(ps)
    rng = random.Random(5)
    for _ in range(200):
        x = rng.randrange(-(q // 2) + 1, q // 2 + 1)
        assert oracle.crt_centred([x % p for p in ps], ps) == x


def test_precision_golden():
    g = GOLD["precision_metric"]
    assert oracle.precision_bits(np.array(g["M"]), np.array(g["Mt"])) == pytest.approx(g["bits"])


def test_strategy1_counts_golden():
    # Lemma le:strategy1: K = ⌊√(2^53/d2)⌋, k_i = ⌈log θ_i / log K⌉; paper: k1=3, k2=1
    g = GOLD["strategy1_k1_k2"]
    for d2 in g["d2"]:
        k1, k2 = oracle.strategy1_counts(2.0 ** (g["q_bits"] - 1), 2.0 ** g["u_bits"], d2)
        assert (k1, k2) == (g["k1"], g["k2"])


def test_chop_reconstructs():
    # Eq. (decomp): r = Σ r_i K^i with digits of the sign of r and |r_i| < K
    rng = random.Random(4)
    for K in (2, 10, 256, 1482910):
        for _ in range(300):
            r = rng.randint(-(2 ** 62), 2 ** 62)
            digits = oracle.chop(r, K)
            assert sum(d * K ** i for i, d in enumerate(digits)) == r
            assert all(abs(d) < K for d in digits)
            assert all(d == 0 or (d > 0) == (r > 0) for d in digits)
