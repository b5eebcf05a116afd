"""Oracle end-to-end CP-MM (Algorithm 6 without Rescale; reading Q3), -m "not gpu".

Pins the oracle's Alg. 6 step 1 against:
* brute force over Z_q with q = Π p (NOT per prime), for N ≤ 16, compared after CRT;
* the decryption identity S·(A·U) + B·U ≡ (⌊ΔM⌉+E)·U (mod p), exact (reading Q16);
* the error bound |Dec − Δ·M·U| ≤ ‖U‖∞·d2·(B_e + ½) (north star; reading Q16);
* config 1 end to end (reading Q15 for its precision).
"""
import math

import numpy as np
import pytest

import ctgen
import oracle


def _cpmm_oracle(ct, U, p_index):
    """(A·U mod p, B·U mod p) per column for prime p_index, via the oracle's schoolbook."""
    p = ct.primes[p_index]
    A, B = oracle.format_matrices(ct.fmt, ct.N, ct.d1, ct.a_polys[p_index], ct.b_polys[p_index])
    AU = oracle.modmatmul(np.ascontiguousarray(A.T), U, p)  # [d3][rows_A]
    BU = oracle.modmatmul(np.ascontiguousarray(B.T), U, p)  # [d3][d1]
    return A, B, AU, BU


@pytest.mark.parametrize("fmt,N,k", [(ctgen.RLWE, 16, 1), (ctgen.SHARED_S, 8, 2), (ctgen.SHARED_A, 8, 2)])
def test_bruteforce_mod_q(fmt, N, k):
    d1, d2, d3, log_delta = N * k, 10, 7, 20
    ps = ctgen.primes(2)
    q = ps[0] * ps[1]
    ct = ctgen.encrypt(fmt, N, d1, d2, 1, log_delta, ps)
    U = ctgen.U_matrix(1, d2, d3, 8)
    outs = [_cpmm_oracle(ct, U, l) for l in range(2)]
    # brute force in Z_q: lift the ciphertext matrices to Z_q by CRT, multiply exactly
    A0, B0 = outs[0][0], outs[0][1]
    A1, B1 = outs[1][0], outs[1][1]
    Aq = np.array([[oracle.crt_centred([A0[r, c], A1[r, c]], ps) % q for c in range(d2)] for r in range(A0.shape[0])],
                  dtype=object)
    Bq = np.array([[oracle.crt_centred([B0[r, c], B1[r, c]], ps) % q for c in range(d2)] for r in range(d1)],
                  dtype=object)
    AUq = Aq.dot(U.astype(object)) % q
    BUq = Bq.dot(U.astype(object)) % q
    for l, p in enumerate(ps):
        assert (outs[l][2].T.astype(object) == AUq % p).all()
        assert (outs[l][3].T.astype(object) == BUq % p).all()


@pytest.mark.parametrize("fmt,N,k", [(ctgen.RLWE, 64, 1), (ctgen.SHARED_S, 16, 4), (ctgen.SHARED_A, 16, 4)])
def test_decryption_identity_and_bound(fmt, N, k):
    d1, d2, d3, log_delta = N * k, 64, 9, 20
    ps = ctgen.primes(1)
    p = ps[0]
    ct = ctgen.encrypt(fmt, N, d1, d2, 2, log_delta, ps)
    U = ctgen.U_matrix(2, d2, d3, 4)
    _, _, AU, BU = _cpmm_oracle(ct, U, 0)
    nk = k if fmt == ctgen.SHARED_A else 1
    sks = [ctgen.sk(2, t, N) for t in range(nk)]
    P = ctgen.plain_matrix(2, N, d1, range(d1), range(d2), log_delta)
    PU = P.astype(object).dot(U.astype(object))  # exact integers
    M = ctgen.msg_matrix(2, d1, range(d1), range(d2))
    MU = M.dot(U.astype(np.float64))
    bound = np.abs(U).max() * d2 * (20 + 0.5)
    for j in range(d3):
        dec = oracle.decrypt_col(fmt, N, d1, sks, AU[j], BU[j], p)
        assert (dec.astype(object) == PU[:, j] % p).all()  # exact identity mod p
        cen = [oracle.crt_centred([v], [p]) for v in dec]
        assert cen == list(PU[:, j])  # |P·U| < p/2 here: the centred residue is the integer
        err = np.abs(np.array(cen, dtype=np.float64) - MU[:, j] * 2.0 ** log_delta)
        assert err.max() <= bound


def test_config1_end_to_end():
    c = ctgen.CONFIGS["c1"]
    ps = ctgen.primes(c.L)
    ct = ctgen.encrypt(c.fmt, c.N, c.d1, c.d2, c.seed, c.log_delta, ps)
    U = ctgen.U_matrix(c.seed, c.d2, c.d3, c.u_bound)
    _, _, AU, BU = _cpmm_oracle(ct, U, 0)
    sks = [ctgen.sk(c.seed, 0, c.N)]
    M = ctgen.msg_matrix(c.seed, c.d1, range(c.d1), range(c.d2))
    MU = M.dot(U.astype(np.float64))
    dec = np.stack([oracle.decrypt_col(c.fmt, c.N, c.d1, sks, AU[j], BU[j], ps[0]) for j in range(c.d3)], axis=1)
    cen = np.array([[oracle.crt_centred([v], ps) for v in row] for row in dec], dtype=np.float64)
    approx = oracle.decode(cen, c.log_delta)
    rel = np.abs(approx - MU).max() / np.abs(MU).max()
    # reading Q15: 1e-6 is unattainable at Δ=2^20, d2=64; the exact bound of Q16 holds instead
    assert np.abs(approx - MU).max() <= np.abs(U).max() * c.d2 * 20.5 / 2 ** c.log_delta
    assert rel < 1e-4
    assert oracle.precision_bits(MU, approx) > 12
