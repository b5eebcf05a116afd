"""Structured-A shared-a format and Algorithm 7 (CP-MM with precomputation), -m "not gpu".

SURVEY.md §8(f) row 2.  The format: a_i · sk_j + b_{ij} ≈ Σ_k m_{Ni+k, j} X^k, i.e.
Ã·S + B ≈ M (mod q) with Ã = [toep(a_0); …; toep(a_{k−1})] ∈ Z_q^{d1×N} and S = [Vec(sk_j)]_j.
Algorithm 7 step 1: B' = B·U; then Ã·(S·U) + B' ≈ M·U, i.e. (Ã, B')
encrypts M·U under the secret S·U.  Pins: the generator against the dense matrix identity built
from the paper's Toeplitz definition; the oracle's Algorithm-7 decryption against dense exact
integer arithmetic; brute force over Z_q (q = p0·p1, not RNS) after CRT.
"""
import numpy as np
import pytest

import ctgen
import oracle

SA = ctgen.STRUCT_A


def _ct(N=16, k=3, d2=5, L=2, seed=4, log_delta=20):
    d1 = N * k
    ps = ctgen.primes(L)
    ct = ctgen.encrypt(SA, N, d1, d2, seed, log_delta, ps)
    sks = [ctgen.sk(seed, j, N) for j in range(d2)]
    P = ctgen.plain_matrix(seed, N, d1, range(d1), range(d2), log_delta)
    return ct, ps, sks, P


def test_layout_of_struct_a_ciphertexts():
    ct, ps, sks, P = _ct()
    assert ct.a_polys.shape == (2, 3, 16)  # k row-block polys per prime, shared by all columns
    assert ct.b_polys.shape == (2, 5 * 3, 16)
    assert oracle.rows_A(SA, 16, 48) == 0 and ctgen.rows_A_of(SA, 16, 48) == 0
    A, B = oracle.format_matrices(SA, 16, 48, ct.a_polys[0], ct.b_polys[0])
    assert A.shape == (0, 5) and B.shape == (48, 5)


def test_generator_satisfies_struct_a_identity():
    """Ã·S + B ≡ ⌊ΔM⌉ + E (mod p), every entry, dense Ã and S from P:143–160."""
    ct, ps, sks, P = _ct()
    for l, p in enumerate(ps):
        At, S = oracle.struct_a_matrices(ct.a_polys[l], sks)
        assert At.shape == (48, 16) and S.shape == (16, 5)
        _, B = oracle.format_matrices(SA, 16, 48, ct.a_polys[l], ct.b_polys[l])
        lhs = (At.dot(S) + B.astype(object)) % p
        assert (lhs == (P.astype(object) % p)).all()


def test_shared_key_across_row_blocks():
    """sk_j does not depend on the row block i: the same key decrypts every chunk."""
    ct, ps, sks, P = _ct(N=8, k=4, d2=3)
    p = ps[0]
    _, B = oracle.format_matrices(SA, 8, 32, ct.a_polys[0], ct.b_polys[0])
    for j in range(3):
        dec = oracle.decrypt_col(SA, 8, 32, [sks[j]], ct.a_polys[0], B[:, j], p)
        assert np.array_equal(dec.astype(np.int64), P[:, j] % p)


def test_decrypt_col_fmt3_matches_dense_with_large_key():
    """The oracle's structured-A decryption Ã·key + b against the dense product for a key with
    entries up to 2^20 (an S·U column is no longer ternary)."""
    rng = np.random.default_rng(1)
    N, k, p = 16, 2, ctgen.primes(1)[0]
    a = rng.integers(0, p, (k, N)).astype(np.uint32)
    key = rng.integers(-(2 ** 20), 2 ** 20, N)
    b = rng.integers(0, p, N * k).astype(np.uint32)
    At, _ = oracle.struct_a_matrices(a, [np.zeros(N, np.int64)])
    want = (At.dot(key.astype(object)) + b.astype(object)) % p
    got = oracle.decrypt_col(SA, N, N * k, [key], a, b, p)
    assert [int(x) for x in got] == list(want)


def test_algorithm7_identity_small():
    """B' = B·U mod p; Ã·(S·U) + B' ≡ (⌊ΔM⌉+E)·U (mod p) on every output column."""
    ct, ps, sks, P = _ct(N=16, k=3, d2=20, L=2)
    U = ctgen.U_matrix(4, 20, 7, 8)
    PU = P.astype(object).dot(U.astype(object))
    for l, p in enumerate(ps):
        _, B = oracle.format_matrices(SA, 16, 48, ct.a_polys[l], ct.b_polys[l])
        Bp = oracle.modmatmul(np.ascontiguousarray(B.T), U, p)  # [d3][d1]
        At, S = oracle.struct_a_matrices(ct.a_polys[l], sks)
        SU = S.dot(U.astype(object))
        for j in range(7):
            w = oracle.su_column(sks, U, j)
            assert [int(x) for x in w] == list(SU[:, j])
            dec = oracle.decrypt_col(SA, 16, 48, [w], ct.a_polys[l], Bp[j], p)
            assert [int(x) for x in dec] == [int(v) % p for v in PU[:, j]]


def test_algorithm7_brute_force_over_Zq():
    """B·U over Z_q with q = p0·p1 (exact Python integers, not RNS) equals the per-prime oracle
    products after CRT — the one-product-per-prime reduction (Strategy 3)."""
    ct, ps, sks, P = _ct(N=8, k=2, d2=6, L=2)
    q = ps[0] * ps[1]
    U = ctgen.U_matrix(9, 6, 4, 8)
    Bs = [oracle.format_matrices(SA, 8, 16, ct.a_polys[l], ct.b_polys[l])[1] for l in range(2)]
    outs = [oracle.modmatmul(np.ascontiguousarray(Bs[l].T), U, ps[l]) for l in range(2)]
    Bq = np.empty(Bs[0].shape, dtype=object)
    for i in range(Bq.shape[0]):
        for j in range(Bq.shape[1]):
            Bq[i, j] = oracle.crt_centred([int(Bs[0][i, j]), int(Bs[1][i, j])], ps) % q
    want = Bq.dot(U.astype(object)) % q
    for j in range(4):
        for i in range(16):
            got = oracle.crt_centred([int(outs[0][j, i]), int(outs[1][j, i])], ps) % q
            assert got == want[i, j]


@pytest.mark.parametrize("bad", [(0, 64, 64), (3, 16, 40)])
def test_dims(bad):
    fmt, N, d1 = bad
    if fmt == 0:
        oracle.check_dims(SA, 16, 64)  # N | d1 is enough for structured-A
        return
    with pytest.raises(ValueError):
        oracle.check_dims(SA, N, d1)
