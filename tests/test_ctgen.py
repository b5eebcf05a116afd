"""Pins for the seeded input generator (ctgen/), -m "not gpu".

The generator is checked against the oracle's independent implementations
(schoolbook negacyclic product, float-based encoder, dense structured S) and
against the distributions DESIGN.md §Inputs states.
"""
import math

import numpy as np
import pytest

import ctgen
import oracle


def _is_prime_trial(n: int) -> bool:
    if n < 2:
        return False
    if n % 2 == 0:
        return n == 2
    f = 3
    while f * f <= n:
        if n % f == 0:
            return False
        f += 2
    return True


def test_primes_reading_q5():
    ps = ctgen.primes(8)
    assert ps == sorted(ps, reverse=True)
    assert len(set(ps)) == 8
    for p in ps:
        assert 2 ** 30 < p < 2 ** 31 and p % 2 ** 16 == 1 and _is_prime_trial(p)
    # no candidate c·2^16+1 between 2^31 and the smallest chosen prime was skipped
    c = (2 ** 31 - 1) >> 16
    expect = []
    while len(expect) < 8:
        n = (c << 16) + 1
        if n < 2 ** 31 and _is_prime_trial(n):
            expect.append(n)
        c -= 1
    assert ps == expect


def test_draw64_counter_based():
    a = [ctgen.draw64(0, 7, i) for i in range(100)]
    b = [ctgen.draw64(0, 7, i) for i in reversed(range(100))][::-1]
    assert a == b
    assert ctgen.draw64(1, 7, 0) != ctgen.draw64(0, 7, 0)
    assert len(set(a)) == 100


def test_secret_ternary_frequencies():
    s = ctgen.sk(0, 0, 30000)
    assert set(np.unique(s).tolist()) <= {-1, 0, 1}
    for v in (-1, 0, 1):
        assert abs(np.mean(s == v) - 1 / 3) < 0.015
    assert not np.array_equal(ctgen.sk(0, 1, 1000), ctgen.sk(0, 0, 1000))  # shared-a keys independent


def test_gaussian_moments_reading_q7():
    e = ctgen.err(0, 5, range(100000))
    assert np.abs(e).max() <= 20
    assert abs(e.mean()) < 0.05
    assert abs(e.var() - 3.2 ** 2) < 0.25  # σ = 3.2 is the standard deviation


def test_U_range_reading_q11():
    U = ctgen.U_matrix(0, 300, 200, 8)
    assert U.min() == -8 and U.max() == 8
    assert set(np.unique(U).tolist()) == set(range(-8, 9))
    U4 = ctgen.U_matrix(0, 64, 64, 4)
    assert U4.min() >= -4 and U4.max() <= 4


def test_msg_grid_reading_q10():
    vals = [ctgen.msg(0, 64, i, j) for i in range(40) for j in range(40)]
    assert all(-1.0 <= v < 1.0 for v in vals)
    assert all(math.ldexp(v, 52) == int(math.ldexp(v, 52)) for v in vals)  # 53-bit grid


@pytest.mark.parametrize("log_delta", [10, 20, 40, 45, 50, 52, 53, 60])
def test_generator_encoder_equals_oracle_encoder(log_delta):
    # generator's integer encoder vs the oracle's float encoder (two implementations of P:803/P:838)
    d1 = 128
    L = ctgen.lib()
    for i in range(0, 128, 3):
        for j in range(0, 50, 7):
            m = ctgen.msg(3, d1, i, j)
            assert L.ctgen_encoded(3, d1, i, j, log_delta) == oracle.encode(m, log_delta)


@pytest.mark.parametrize("N", [1, 2, 8, 64, 1024])
def test_ntt_equals_oracle_schoolbook(N):
    p = ctgen.primes(2)[1]
    rng = np.random.default_rng(N)
    a = rng.integers(0, p, N, dtype=np.uint64).astype(np.uint32)
    s = rng.integers(-1, 2, N).astype(np.int8)
    assert (ctgen.negacyclic_ntt(a, s, p) == oracle.negacyclic_mul(a, s.astype(np.int64), p)).all()


def _keys(fmt, N, k, seed=0):
    nk = k if fmt == ctgen.SHARED_A else 1
    return [ctgen.sk(seed, t, N).astype(np.int64).tolist() for t in range(nk)]


@pytest.mark.parametrize("fmt,N,k", [(ctgen.RLWE, 16, 1), (ctgen.SHARED_S, 16, 3), (ctgen.SHARED_A, 16, 3),
                                     (ctgen.SHARED_A, 8, 4), (ctgen.SHARED_S, 4, 2)])
def test_encryption_equals_oracle_small(fmt, N, k):
    """Generator ciphertexts == oracle's dense-S encryption of the same plaintext and a-parts,
    and S·A + B ≡ ⌊ΔM⌉ + E (mod p) exactly (Lemma le:mat_struct_s)."""
    d1, d2, log_delta = N * k, 12, 20
    ps = ctgen.primes(2)
    ct = ctgen.encrypt(fmt, N, d1, d2, 0, log_delta, ps)
    sks = _keys(fmt, N, k)
    M = ctgen.msg_matrix(0, d1, range(d1), range(d2))
    E = ctgen.err_matrix(0, N, d1, range(d1), range(d2))
    P = oracle.encode(M, log_delta) + E
    assert (P == ctgen.plain_matrix(0, N, d1, range(d1), range(d2), log_delta)).all()
    for l, p in enumerate(ps):
        A, B = oracle.format_matrices(fmt, N, d1, ct.a_polys[l], ct.b_polys[l])
        assert A.shape == (oracle.rows_A(fmt, N, d1), d2)
        assert (oracle.encrypt_small(fmt, sks, P, A, p) == B).all()
        S = oracle.secret_matrix(fmt, sks, N, d1).astype(object)
        assert ((S.dot(A.astype(object)) + B.astype(object) - P.astype(object)) % p == 0).all()


def test_encryption_column_range_reproducible():
    ps = ctgen.primes(1)
    full = ctgen.encrypt(ctgen.SHARED_A, 16, 64, 20, 0, 30, ps)
    part = ctgen.encrypt(ctgen.SHARED_A, 16, 64, 20, 0, 30, ps, col_begin=5, col_end=9)
    assert (part.a_polys[0] == full.a_polys[0][5:9]).all()
    assert (part.b_polys[0] == full.b_polys[0][5 * 4:9 * 4]).all()


def test_encryption_large_N_decrypts():
    """N=4096 shared-a (config 3's format and ring): the oracle's schoolbook decryption of
    sampled columns recovers P = ⌊ΔM⌉ + E exactly."""
    N, k, log_delta = 4096, 2, 45
    d1, d2 = N * k, 3
    ps = ctgen.primes(2)
    ct = ctgen.encrypt(ctgen.SHARED_A, N, d1, d2, 0, log_delta, ps)
    sks = _keys(ctgen.SHARED_A, N, k)
    j = 1
    P = ctgen.plain_matrix(0, N, d1, range(d1), [j], log_delta)[:, 0]
    for l, p in enumerate(ps):
        A, B = oracle.format_matrices(ctgen.SHARED_A, N, d1, ct.a_polys[l], ct.b_polys[l])
        dec = oracle.decrypt_col(ctgen.SHARED_A, N, d1, sks, A[:, j], B[:, j], p)
        assert (dec.astype(np.int64) == P % p).all()


def test_config_table():
    c = ctgen.CONFIGS
    assert c["c3"].R == 20480 and c["c3"].residue_macs == 3 * 20480 * 16384 * 16384
    assert c["c5"].R == 65536 and c["c5"].k == 2
    assert c["c4"].rows_A == 32768 and c["c2"].rows_A == 4096


def test_bulk_blocks_match_scalar():
    N, d1, ld = 16, 64, 30
    Mb = ctgen.msg_block(4, d1, 3, 10, 2, 5)
    Pb = ctgen.plain_block(4, N, d1, ld, 3, 10, 2, 5)
    assert (Mb == ctgen.msg_matrix(4, d1, range(3, 13), range(2, 7))).all()
    assert (Pb == ctgen.plain_matrix(4, N, d1, range(3, 13), range(2, 7), ld)).all()


def test_colmajor_views_equal_format_matrices():
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from gpu_helpers import colmajor_views

    for fmt, N, k in [(ctgen.RLWE, 16, 1), (ctgen.SHARED_S, 8, 3), (ctgen.SHARED_A, 8, 3)]:
        d1, d2 = N * k, 7
        ct = ctgen.encrypt(fmt, N, d1, d2, 0, 20, ctgen.primes(1))
        A, B = oracle.format_matrices(fmt, N, d1, ct.a_polys[0], ct.b_polys[0])
        Av, Bv = colmajor_views(fmt, N, d1, d2, ct.a_polys[0], ct.b_polys[0])
        assert (Av == A.T).all() and (Bv == B.T).all()
