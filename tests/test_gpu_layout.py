"""GPU parity of the format layout (ctpt_layout): the stacked K-major
X = [A; B] the library writes must equal the oracle's format matrices (P:45–71, P:1071,
reading Q18) entry by entry, zero padded to d2p columns — through the 16-byte kernel
(k_layout_v4, rows_A and d1 multiples of 4) and the 4-byte kernel k_layout (every shape whose
4-row chunks would straddle A and B: rows_A or d1 not a multiple of 4)."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(__file__))

import ctgen  # noqa: E402
import oracle  # noqa: E402

pytestmark = pytest.mark.gpu

R, S, A, SA = ctgen.RLWE, ctgen.SHARED_S, ctgen.SHARED_A, ctgen.STRUCT_A

SHAPES = [
    # fmt, N, k, d2, L — ragged tiles in r (64) and k (64), d2 not a multiple of 16, N < 4
    (R, 64, 1, 64, 1),
    (S, 16, 3, 200, 2),
    (A, 256, 2, 130, 3),
    (SA, 64, 3, 77, 2),
    (A, 8, 4, 33, 1),
    (R, 2, 1, 5, 1),    # rows_A = 2: 4-row chunks straddle A and B -> 4-byte kernel
    (S, 2, 3, 70, 2),
    (R, 1024, 1, 1000, 2),
]


def _expected(fmt, N, d1, d2, ct, L, d2p):
    out = []
    for l in range(L):
        Am, Bm = oracle.format_matrices(fmt, N, d1, ct.a_polys[l], ct.b_polys[l])
        X = np.zeros((Am.shape[0] + Bm.shape[0], d2p), np.uint32)
        X[:Am.shape[0], :d2] = Am
        X[Am.shape[0]:, :d2] = Bm
        out.append(X)
    return np.stack(out)


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "f%d_N%d_k%d_d2%d_L%d" % s)
def test_layout_matches_oracle(shape):
    import torch

    from paper_2503_16080_b200 import ctpt
    from paper_2503_16080_b200.engine import CpmmEngine

    fmt, N, k, d2, L = shape
    d1 = N * k
    ps = ctgen.primes(L)
    ct = ctgen.encrypt(fmt, N, d1, d2, 3, 20, ps)
    eng = CpmmEngine(ctpt.Spec(fmt, N, d1, d2, 4, ps), "cuda")
    eng.ctmat = torch.full((eng.sizes.ctmat_bytes,), 0xAB, dtype=torch.uint8, device="cuda")  # poison
    eng.layout(ct.a_polys, ct.b_polys, validate=True)
    torch.cuda.synchronize()
    got = eng.ctmat[256:].cpu().numpy().view(np.uint32).reshape(L, eng.sizes.R, eng.sizes.d2p)
    want = _expected(fmt, N, d1, d2, ct, L, eng.sizes.d2p)
    assert np.array_equal(got, want), np.argwhere(got != want)[:5]


@pytest.mark.parametrize("N", [64, 2])  # 16-byte kernel; 4-byte kernel (rows_A = 2)
def test_layout_validate_flags_out_of_range(N):
    """validate = 1: a residue ≥ its prime anywhere (A part, B part, last prime) → ERR_RANGE."""
    from paper_2503_16080_b200 import ctpt
    from paper_2503_16080_b200.engine import CpmmEngine

    fmt, k, d2, L = A, 2, 100, 2
    ps = ctgen.primes(L)
    for where in ("a", "b"):
        ct = ctgen.encrypt(fmt, N, N * k, d2, 0, 20, ps)
        arr = ct.a_polys if where == "a" else ct.b_polys
        arr[L - 1].reshape(-1)[-1] = ps[L - 1]  # == p: out of range
        eng = CpmmEngine(ctpt.Spec(fmt, N, N * k, d2, 4, ps), "cuda")
        with pytest.raises(ctpt.CtptError, match="ERR_RANGE"):
            eng.layout(ct.a_polys, ct.b_polys, validate=True)
