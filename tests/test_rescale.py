"""RNS Rescale (Alg. 6 / Alg. 7 step 2), -m "not gpu".

Rescale(A', B') = (⌊A'/Δ⌉, ⌊B'/Δ⌉) with Δ replaced by a divisor q_1 of q:
here q_1 is the last RNS prime.  Pins for the oracle's plain definition (CRT → exact integer →
round → reduce) against the defining property of nearest rounding, hand-computed edge values,
the generator's exact encoding of a real U at a non-power-of-two scale, and Algorithm 6 with
step 2 end to end (decryption error within the Rescale bound).
"""
from fractions import Fraction

import numpy as np
import pytest

import ctgen
import oracle


def test_round_div_is_round_half_up():
    rng = np.random.default_rng(0)
    for _ in range(2000):
        x = int(rng.integers(-10 ** 12, 10 ** 12))
        d = int(rng.integers(1, 10 ** 6))
        f = Fraction(x, d) + Fraction(1, 2)
        assert oracle.round_div(x, d) == f.numerator // f.denominator
    assert oracle.round_div(5, 2) == 3 and oracle.round_div(-5, 2) == -2  # ⌊x⌉ = ⌊x + ½⌋
    assert oracle.round_div(7, 7) == 1 and oracle.round_div(3, 7) == 0 and oracle.round_div(4, 7) == 1


def _res(x, ps):
    return np.array([[int(x) % int(p)] for p in ps], dtype=np.uint32)


def test_rescale_edge_values():
    ps = ctgen.primes(3)
    q1 = ps[-1]
    h = (q1 - 1) // 2
    q_out = ps[0] * ps[1]
    for x, want in [(0, 0), (h, 0), (h + 1, 1), (-h, 0), (-h - 1, -1), (5 * q1, 5), (5 * q1 + h, 5),
                    (5 * q1 + h + 1, 6), (-7 * q1 - h - 1, -8), (123456789 * q1 + 17, 123456789)]:
        y = oracle.rescale_last(_res(x, ps), ps)
        assert oracle.crt_centred([int(y[0, 0]), int(y[1, 0])], ps[:2]) == want, x
        assert (int(y[0, 0]) - want) % ps[0] == 0 and int(y[1, 0]) == want % ps[1]
    assert q_out > 2 ** 61


def test_rescale_nearest_property_random():
    """|y·q_1 − x| ≤ (q_1 − 1)/2 for the exact integer x, any x ∈ (−q/2, q/2]."""
    ps = ctgen.primes(4)
    q = 1
    for p in ps:
        q *= p
    rng = np.random.default_rng(5)
    xs = [int.from_bytes(rng.bytes(16), "little") % q - q // 2 for _ in range(300)]
    res = np.array([[x % p for x in xs] for p in ps], dtype=np.uint32)
    out = oracle.rescale_last(res, ps)
    for i, x in enumerate(xs):
        y = oracle.crt_centred([int(out[l, i]) for l in range(3)], ps[:3])
        assert abs(y * ps[-1] - x) <= (ps[-1] - 1) // 2


def test_generator_encodes_real_U_exactly():
    """U0 = ⌊scale·U⌉ with scale = a 31-bit prime (not a power of two), ties up."""
    p = ctgen.primes(1)[0]
    real, enc = ctgen.U_real(3, 20, 30, p)
    assert real.min() >= -1.0 and real.max() < 1.0
    for k in range(20):
        for j in range(30):
            f = Fraction(p) * Fraction(real[k, j]) + Fraction(1, 2)
            assert enc[k, j] == f.numerator // f.denominator
            assert real[k, j] == ctgen.u_real(3, 30, k, j)


@pytest.mark.parametrize("fmt", [ctgen.SHARED_S, ctgen.RLWE, ctgen.SHARED_A])
def test_algorithm6_with_rescale_small(fmt):
    """(A', B') = (A·U0, B·U0) mod each p, Rescale by q_1 = p_{L−1}; the result decrypts under
    the same S to ⌊ΔM⌉·U0/q_1 + (S·ε_A + ε_B) over Z_{q/q_1}, |ε| ≤ ½, and with
    Δ_U = q_1 it decodes to M·U at scale Δ."""
    N, k = 16, (1 if fmt == ctgen.RLWE else 2)
    d1, d2, d3, L, log_delta, seed = N * k, 24, 5, 3, 20, 2
    ps = ctgen.primes(L)
    q1 = ps[-1]
    ct = ctgen.encrypt(fmt, N, d1, d2, seed, log_delta, ps)
    Ur, U0 = ctgen.U_real(seed, d2, d3, q1)
    prods = []
    for l, p in enumerate(ps):
        A, B = oracle.format_matrices(fmt, N, d1, ct.a_polys[l], ct.b_polys[l])
        AU = oracle.modmatmul(np.ascontiguousarray(A.T), U0, p)  # [d3][rows_A]
        BU = oracle.modmatmul(np.ascontiguousarray(B.T), U0, p)
        prods.append(np.concatenate([AU, BU], axis=1))  # [d3][R]
    X = np.stack([pr.reshape(-1) for pr in prods])  # [L][d3·R]
    Y = oracle.rescale_last(X, ps).reshape(L - 1, d3, -1)
    ra = oracle.rows_A(fmt, N, d1)
    nk = k if fmt == ctgen.SHARED_A else 1
    sks = [ctgen.sk(seed, t, N) for t in range(nk)]
    h = max(int(np.abs(s).sum()) for s in sks)  # every row of S holds ±(one key's coefficients)
    P = ctgen.plain_matrix(seed, N, d1, range(d1), range(d2), log_delta)
    M = np.array([[ctgen.msg(seed, d1, i, j) for j in range(d2)] for i in range(d1)])
    PU = P.astype(object).dot(U0.astype(object))
    worst = 0.0
    for j in range(d3):
        decs = [oracle.decrypt_col(fmt, N, d1, sks, Y[l, j, :ra], Y[l, j, ra:], ps[l]) for l in range(L - 1)]
        cen = oracle.crt_centred_array(np.stack(decs), ps[:2])
        for i in range(d1):
            err = Fraction(cen[i]) - Fraction(PU[i, j], q1)
            assert abs(err) <= Fraction(h + 1, 2), (i, j, float(err))
        mu = M.dot(Ur[:, j])
        worst = max(worst, np.abs(np.array(cen, dtype=np.float64) / 2.0 ** log_delta - mu).max())
    # encoding error of U0 and of ⌊ΔM⌉+E plus the Rescale error, all divided by Δ
    assert worst <= (d2 * 0.5 / q1 + d2 * 20.5 / 2 ** log_delta + (h + 1) / 2 / 2 ** log_delta) * 1.01
