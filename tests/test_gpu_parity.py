"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit-exact residues.

Bar: residues are integers, so every compared entry must be
identical.  Small shapes and configs c1/c2 are compared element by element; the
large configs on sampled entries, tile-boundary rows/columns, Freivalds and the
decryption identity (tests/test_gpu_configs.py).
"""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(__file__))

import ctgen  # noqa: E402
import oracle  # noqa: E402
from gpu_helpers import NTHREADS, U_residues, oracle_outputs, run_gpu  # noqa: E402

pytestmark = pytest.mark.gpu

R, S, A, SA = ctgen.RLWE, ctgen.SHARED_S, ctgen.SHARED_A, ctgen.STRUCT_A
AUTO, SPLIT_GEMM, FUSED, MV_K = 0, 1, 2, 3  # ctpt_problem.kernel (include/ctpt.h ctpt_kernel)

SHAPES = [
    # fmt, N, k, d2, d3, L  — several tiles + ragged tails in every dimension
    (R, 16, 1, 16, 1, 1),
    (R, 64, 1, 64, 64, 1),
    (S, 16, 2, 48, 7, 2),
    (A, 16, 4, 200, 129, 3),
    (S, 64, 2, 64, 300, 1),
    (A, 256, 2, 4112, 64, 1),
    (R, 256, 1, 129, 130, 2),
    (A, 8, 4, 33, 5, 1),
    (S, 4, 8, 128, 128, 1),
    (A, 1024, 3, 1000, 257, 2),
    (SA, 64, 3, 300, 260, 2),    # structured-A shared-a (Algorithm 7): only B·U
    (SA, 16, 5, 130, 100, 1),
    (S, 16, 2, 48, 300, 8),      # L = 8 primes (config c5's basis) on a small shape
]


def _check(fmt, N, k, d2, d3, L, seed=0, u_bound=8, simt=False, col_begin=0, col_end=0, unsigned="auto",
           U=None, split_overlap=0, kernel=AUTO, raster_group=0, max_ctas=0):
    d1 = N * k
    ps = ctgen.primes(L)
    ct = ctgen.encrypt(fmt, N, d1, d2, seed, 20, ps, nthreads=NTHREADS)
    if U is None:
        U = ctgen.U_matrix(seed, d2, d3, u_bound)
    (AU, BU), eng = run_gpu(fmt, N, d1, d2, d3, ps, ct.a_polys, ct.b_polys, U=U, simt=simt, col_begin=col_begin,
                            col_end=col_end, unsigned=unsigned, split_overlap=split_overlap, kernel=kernel,
                            raster_group=raster_group, max_ctas=max_ctas)
    c1 = col_end or d3
    cols = np.arange(col_begin, c1)
    for l, p in enumerate(ps):
        wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[l], ct.b_polys[l], U, p, cols=cols)
        assert np.array_equal(AU[l], wa), f"A·U mismatch prime {l}: {np.argwhere(AU[l] != wa)[:5]}"
        assert np.array_equal(BU[l], wb), f"B·U mismatch prime {l}: {np.argwhere(BU[l] != wb)[:5]}"


@pytest.fixture(params=["split_gemm", "auto"])
def gemm_kernel(request):
    """ctpt_problem.kernel: force the limb split + the tcgen05 GEMM k_gemm_tc, or leave
    ctpt_matmul's automatic choice (the raw-byte kernel at d3_loc <= 32, the fused skinny kernel
    at d3_loc <= 256 when kU = 1 and u_offset = 0, else split + GEMM)."""
    return SPLIT_GEMM if request.param == "split_gemm" else AUTO


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "f%d_N%d_k%d_d2%d_d3%d_L%d" % s)
def test_shapes_tcgen05(shape, gemm_kernel):
    _check(*shape, unsigned="never", kernel=gemm_kernel)


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "f%d_N%d_k%d_d2%d_d3%d_L%d" % s)
def test_shapes_unsigned_U(shape, gemm_kernel):
    """The unsigned-U plane (U + u_offset as u8, u8 × u8 MMAs, row-sum correction in the
    epilogue); with u_offset != 0 the automatic choice is always split + GEMM."""
    _check(*shape, unsigned="always", kernel=gemm_kernel)


@pytest.mark.parametrize("lo,hi", [(-128, 127), (0, 255), (3, 200), (-1, 0), (0, 0)])
def test_unsigned_U_ranges(lo, hi):
    """u_offset = max(0, −min U) for every admissible span, incl. offset 0 (no correction; the
    fused skinny kernel then runs u8 × u8) and U = 0."""
    rng = np.random.default_rng(hi - lo)
    for d3 in (100, 300):
        U = rng.integers(lo, hi + 1, (260, d3)).astype(np.int64)
        _check(A, 64, 3, 260, d3, 2, U=U, unsigned="always")


def test_unsigned_U_refusals():
    from paper_2503_16080_b200 import ctpt

    fmt, N, d2 = R, 16, 64
    ps = ctgen.primes(1)
    ct = ctgen.encrypt(fmt, N, N, d2, 0, 20, ps)
    with pytest.raises(ctpt.CtptError, match="ERR_RANGE"):
        run_gpu(fmt, N, N, d2, 4, ps, ct.a_polys, ct.b_polys, U=np.full((d2, 4), 256, np.int64), unsigned="always")
    with pytest.raises(ctpt.CtptError, match="ERR_RANGE"):
        U = np.zeros((d2, 4), np.int64)
        U[0, 0], U[1, 1] = -100, 200
        run_gpu(fmt, N, N, d2, 4, ps, ct.a_polys, ct.b_polys, U=U, unsigned="always")
    # "auto" falls back to balanced digits and stays exact
    U = np.zeros((d2, 300), np.int64)
    U[0, 0], U[1, 1] = -100, 200
    (AU, BU), eng = run_gpu(fmt, N, N, d2, 300, ps, ct.a_polys, ct.b_polys, U=U)
    assert eng.spec.u_unsigned == 0
    wa, wb = oracle_outputs(fmt, N, N, ct.a_polys[0], ct.b_polys[0], U, ps[0])
    assert np.array_equal(AU[0], wa) and np.array_equal(BU[0], wb)


def test_unsigned_U_max_d2_bound():
    """d2 = 33025 (the u8·u8 exactness limit) with every limb at 255 and U' at 255."""
    fmt, N, d2, d3 = R, 16, 33025, 300
    ps = ctgen.primes(1)
    p = ps[0]
    a = np.full((1, d2, N), (64 << 24) | 0xFFFFFF, np.uint32)
    b = np.full((1, d2, N), p - 1, np.uint32)
    U = np.full((d2, d3), 127, np.int64)
    U[:, ::2] = -128
    (AU, BU), eng = run_gpu(fmt, N, N, d2, d3, ps, a, b, U=U, unsigned="always")
    assert eng.spec.u_unsigned == 1 and eng.spec.u_offset == 128
    wa, wb = oracle_outputs(fmt, N, N, a[0], b[0], U, p)
    assert np.array_equal(AU[0], wa) and np.array_equal(BU[0], wb)


def test_column_shard_both_kernels(gemm_kernel):
    _check(S, 128, 2, 160, 600, 1, col_begin=37, col_end=591, kernel=gemm_kernel)
    _check(A, 64, 3, 300, 600, 2, col_begin=300, col_end=555, kernel=gemm_kernel)  # d3_loc = 255: fused when auto


# ------------------------------------------------------------------ skinny regime (§8(f) row 1)
SKINNY = [
    # fmt, N, k, d2, d3, L — d3 across the fused kernel's shapes: 1 (CP-Mv), < 128, = 128 (64-row
    # tiles, 4 limb stages), 129..160 (3 stages), 161..192 (2 stages), 193..224 (2 half-K-block
    # stages), 225..256 (32-row tiles);
    # ragged R and d2 (not multiples of 64 / 128), long K so the 2- and 3-stage rings wrap
    (S, 64, 3, 1000, 1, 2),
    (R, 512, 1, 130, 2, 1),
    (A, 128, 4, 520, 64, 1),
    (S, 32, 5, 384, 128, 1),
    (A, 16, 3, 77, 129, 2),
    (R, 1024, 1, 520, 144, 2),
    (S, 64, 3, 1000, 160, 1),
    (A, 32, 5, 300, 176, 1),
    (A, 128, 2, 3000, 192, 1),
    (R, 1024, 1, 2056, 200, 1),
    (S, 32, 5, 1000, 224, 1),
    (A, 64, 3, 900, 240, 1),
    (S, 128, 2, 640, 256, 1),
    (A, 8, 2, 16, 256, 1),       # R = 24 rows < one tile
    (SA, 256, 2, 700, 1, 2),     # Algorithm 7 CP-Mv: the output is a shared-s vector
]


@pytest.mark.parametrize("shape", SKINNY, ids=lambda s: "f%d_N%d_k%d_d2%d_d3%d_L%d" % s)
def test_skinny_fused(shape):
    """The fused kernel forced (kernel = FUSED) on every skinny width, d3 <= 32 included (which the
    automatic choice gives to the raw-byte kernel), and the automatic choice on the same shapes."""
    _check(*shape, kernel=FUSED)
    _check(*shape, seed=1)


@pytest.mark.parametrize("cols", [(0, 129), (20, 220), (44, 300), (171, 300)])
def test_skinny_column_shards(cols):
    """k_gemm_fused_t on column blocks [c0, c1) of a wider U (129 columns: 64-row tiles with 3 limb
    stages; 200: 64-row tiles with half-K-block stages; 256: 32-row tiles; U^T rows j_off .. j_off + N partly past the block and, for
    (171, 300), past d3), with ragged R (not a multiple of the tile) and more CTAs than tiles."""
    _check(A, 64, 3, 333, 300, 2, col_begin=cols[0], col_end=cols[1], seed=5, kernel=FUSED)
    _check(S, 512, 9, 300, 300, 1, col_begin=cols[0], col_end=cols[1], seed=6, kernel=FUSED)  # R = 9216: 144 tiles


MV = [
    # fmt, N, k, d2, d3, L — the raw-byte kernel (d3 <= 32): every padded width NC = 16/32/64/128,
    # ragged R and d2, K split into several units per tile (exact int32 partials + tickets)
    (S, 64, 3, 1000, 1, 2),
    (R, 512, 1, 130, 2, 1),
    (A, 128, 4, 520, 4, 1),
    (S, 32, 5, 384, 5, 2),
    (A, 16, 3, 77, 8, 1),
    (R, 1024, 1, 2056, 16, 1),
    (S, 128, 2, 640, 17, 1),
    (A, 8, 2, 16, 31, 1),        # R = 24 rows < one tile, one K block
    (SA, 256, 3, 4112, 32, 2),   # structured-A, long K
    (S, 1024, 4, 8200, 3, 1),    # R = 8192: 64 tiles, several K splits each
]


@pytest.mark.parametrize("shape", MV, ids=lambda s: "f%d_N%d_k%d_d2%d_d3%d_L%d" % s)
def test_mv_raw_bytes(shape):
    _check(*shape, kernel=MV_K)
    _check(*shape, seed=1)  # the tickets were left at zero for the next launch


def test_mv_column_shard_and_entry_point():
    """A 1..32-column block [col_begin, col_end) of a wider U through ctpt_gemm_mv, per prime."""
    import torch

    from paper_2503_16080_b200 import ctpt
    from paper_2503_16080_b200.engine import CpmmEngine

    fmt, N, k, d2, d3, L = A, 64, 4, 700, 300, 2
    d1 = N * k
    ps = ctgen.primes(L)
    ct = ctgen.encrypt(fmt, N, d1, d2, 13, 20, ps)
    U = ctgen.U_matrix(13, d2, d3, 8)
    for c0, c1 in [(0, 1), (77, 78), (250, 282), (5, 21)]:
        eng = CpmmEngine(ctpt.Spec(fmt, N, d1, d2, d3, ps, c0, c1), "cuda")
        eng.layout(ct.a_polys, ct.b_polys)
        eng.precompute(U)
        AU, BU = eng.alloc_outputs()
        ra, n = eng.sizes.rows_A, c1 - c0
        for l in range(L):
            ctpt.gemm_mv(eng.spec, l, eng.ctmat, eng.plain, AU[l * n * ra:], BU[l * n * d1:], eng.ws)
        torch.cuda.synchronize()
        AUn, BUn = eng.outputs_numpy(AU, BU)
        for l, p in enumerate(ps):
            wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[l], ct.b_polys[l], U, p, cols=np.arange(c0, c1))
            assert np.array_equal(AUn[l], wa) and np.array_equal(BUn[l], wb), (c0, c1, l)


def test_skinny_long_k_ring_wraparound():
    """Long K (33–65 k-blocks per tile) wraps the raw-X and limb rings many times; a premature
    release of a raw tile once corrupted whole output rows intermittently — run it repeatedly."""
    for rep in range(5):
        _check(A, 256, 2, 4112, 64, 1, seed=rep)
        _check(S, 128, 3, 8200, 100, 1, seed=rep)
        _check(R, 512, 1, 4096, 256, 1, seed=rep)
        _check(S, 256, 4, 8200, 200, 1, seed=rep)


def test_skinny_fused_direct_entry_point():
    """ctpt_gemm_fused per prime (the stage entry point) == the oracle; and it refuses
    d3_loc > 256 with ERR_UNSUPPORTED."""
    import torch

    from paper_2503_16080_b200 import ctpt
    from paper_2503_16080_b200.engine import CpmmEngine

    fmt, N, k, d2, d3, L = S, 64, 2, 300, 100, 2
    d1 = N * k
    ps = ctgen.primes(L)
    ct = ctgen.encrypt(fmt, N, d1, d2, 11, 20, ps)
    U = ctgen.U_matrix(11, d2, d3, 8)
    eng = CpmmEngine(ctpt.Spec(fmt, N, d1, d2, d3, ps), "cuda")
    eng.layout(ct.a_polys, ct.b_polys)
    eng.precompute(U)
    AU, BU = eng.alloc_outputs()
    ra = eng.sizes.rows_A
    for l in range(L):
        ctpt.gemm_fused(eng.spec, l, eng.ctmat, eng.plain, AU[l * d3 * ra:], BU[l * d3 * d1:])
    torch.cuda.synchronize()
    AUn, BUn = eng.outputs_numpy(AU, BU)
    for l, p in enumerate(ps):
        wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[l], ct.b_polys[l], U, p)
        assert np.array_equal(AUn[l], wa) and np.array_equal(BUn[l], wb)
    big = ctpt.Spec(fmt, N, d1, d2, 300, ps)
    with pytest.raises(ctpt.CtptError, match="ERR_UNSUPPORTED"):
        ctpt.gemm_fused(big, 0, eng.ctmat, eng.plain, AU, BU)


@pytest.mark.parametrize("d3", [130, 20])
def test_skinny_adversarial_residues(d3):
    """The fused split (d3 = 130) and the raw-byte kernel (d3 = 20, K split into exact partials)
    on residues 0, 1, (p±1)/2, p−1, p−2 with U digits at −128 / 127 and d2 = 65536 (the int32
    exactness limit) — C_ℓ reaches ±d2·255·128."""
    fmt, N, d2 = R, 64, 65536
    ps = ctgen.primes(1)
    p = ps[0]
    rng = np.random.default_rng(3)
    special = np.array([0, 1, (p - 1) // 2, (p + 1) // 2, p - 1, p - 2, (64 << 24) | 0xFFFFFF], dtype=np.uint32)
    a = special[rng.integers(0, len(special), (1, d2, N))]
    b = special[rng.integers(0, len(special), (1, d2, N))]
    a[0, :, 0] = (64 << 24) | 0xFFFFFF
    U = rng.choice(np.array([-128, 127, -1, 0, 1], dtype=np.int64), size=(d2, d3))
    U[:, 0] = -128
    U[:, d3 - 1] = 127
    (AU, BU), eng = run_gpu(fmt, N, N, d2, d3, ps, a, b, U=U)
    assert eng.spec.kU == 1
    wa, wb = oracle_outputs(fmt, N, N, a[0], b[0], U, p)
    assert np.array_equal(AU[0], wa) and np.array_equal(BU[0], wb)


def test_multi_digit_U_two_digits():
    fmt, N, k, d2, d3 = A, 64, 2, 256, 300
    d1 = N * k
    ps = ctgen.primes(1)
    ct = ctgen.encrypt(fmt, N, d1, d2, 9, 20, ps)
    U = ctgen.U_matrix(9, d2, d3, 3000)
    (AU, BU), eng = run_gpu(fmt, N, d1, d2, d3, ps, ct.a_polys, ct.b_polys, U=U)
    assert eng.spec.kU == 2
    wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[0], ct.b_polys[0], U, ps[0])
    assert np.array_equal(AU[0], wa) and np.array_equal(BU[0], wb)


@pytest.mark.parametrize("shape", SHAPES[:6], ids=lambda s: "f%d_N%d_k%d_d2%d_d3%d_L%d" % s)
def test_shapes_simt_diagnostic(shape):
    _check(*shape, simt=True)


def test_column_shard():
    _check(A, 64, 2, 96, 300, 2, col_begin=70, col_end=211)


def test_empty_U_columns_zero():
    # U = 0 → outputs are 0 (degenerate case); U = I → outputs are A and B themselves
    fmt, N, k, d2 = S, 32, 2, 64
    d1 = N * k
    ps = ctgen.primes(1)
    ct = ctgen.encrypt(fmt, N, d1, d2, 3, 20, ps)
    (AU, BU), _ = run_gpu(fmt, N, d1, d2, 5, ps, ct.a_polys, ct.b_polys, U=np.zeros((d2, 5), np.int64))
    assert (AU == 0).all() and (BU == 0).all()
    (AU, BU), _ = run_gpu(fmt, N, d1, d2, d2, ps, ct.a_polys, ct.b_polys, U=np.eye(d2, dtype=np.int64))
    A_, B_ = oracle.format_matrices(fmt, N, d1, ct.a_polys[0], ct.b_polys[0])
    assert np.array_equal(AU[0], A_.T) and np.array_equal(BU[0], B_.T)


def test_adversarial_residues_and_digits():
    """Residues 0, 1, (p±1)/2, p−1 and U at the int8 digit extremes −128 / 127."""
    fmt, N, k, d2, d3 = A, 64, 2, 384, 96
    d1 = N * k
    ps = ctgen.primes(2)
    rng = np.random.default_rng(0)
    a = np.empty((2, d2, N), np.uint32)
    b = np.empty((2, d2 * k, N), np.uint32)
    for l, p in enumerate(ps):
        special = np.array([0, 1, (p - 1) // 2, (p + 1) // 2, p - 1, p - 2], dtype=np.uint32)
        a[l] = special[rng.integers(0, 6, a[l].shape)]
        b[l] = special[rng.integers(0, 6, b[l].shape)]
        a[l, :, 0] = p - 1
    U = rng.choice(np.array([-128, 127, -1, 0, 1], dtype=np.int64), size=(d2, d3))
    U[:, 0] = -128
    U[:, 1] = 127
    (AU, BU), eng = run_gpu(fmt, N, d1, d2, d3, ps, a, b, U=U)
    assert eng.spec.kU == 1
    for l, p in enumerate(ps):
        wa, wb = oracle_outputs(fmt, N, d1, a[l], b[l], U, p)
        assert np.array_equal(AU[l], wa) and np.array_equal(BU[l], wb)


def test_max_d2_int32_bound():
    """d2 = 65536 (the exactness limit d2·255·128 < 2^31) with every limb and digit at its
    extreme: C_ℓ reaches −d2·255·128 and must not wrap."""
    fmt, N, d2, d3 = R, 16, 65536, 16
    ps = ctgen.primes(1)
    p = ps[0]
    a = np.full((1, d2, N), 0xFF_FF_FF & 0, np.uint32)
    # residues whose bytes are all 255 in limbs 0..2 (p > 2^30, so 2^24·64 + 0xFFFFFF < p)
    a[:] = (64 << 24) | 0xFFFFFF
    b = np.full((1, d2, N), p - 1, np.uint32)
    U = np.full((d2, d3), -128, np.int64)
    U[:, 1::2] = 127
    (AU, BU), _ = run_gpu(fmt, N, N, d2, d3, ps, a, b, U=U)
    wa, wb = oracle_outputs(fmt, N, N, a[0], b[0], U, p)
    assert np.array_equal(AU[0], wa) and np.array_equal(BU[0], wb)


def test_multi_digit_U():
    """|U| up to 30000 → k_U = 2 balanced digits; the second pass accumulates 2^8·(X·U_1) mod p."""
    fmt, N, k, d2, d3 = S, 32, 2, 160, 40
    d1 = N * k
    ps = ctgen.primes(2)
    ct = ctgen.encrypt(fmt, N, d1, d2, 5, 20, ps)
    U = ctgen.U_matrix(5, d2, d3, 30000)
    (AU, BU), eng = run_gpu(fmt, N, d1, d2, d3, ps, ct.a_polys, ct.b_polys, U=U)
    assert eng.spec.kU == 2
    for l, p in enumerate(ps):
        wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[l], ct.b_polys[l], U, p)
        assert np.array_equal(AU[l], wa) and np.array_equal(BU[l], wb)


def test_general_U_residues_rns():
    """U ∈ Z_q given by residues (ctpt_plain_precompute_rns, k_U = 4 per prime)."""
    fmt, N, k, d2, d3 = A, 32, 3, 130, 70
    d1 = N * k
    ps = ctgen.primes(3)
    ct = ctgen.encrypt(fmt, N, d1, d2, 6, 20, ps)
    rng = np.random.default_rng(6)
    Ub = rng.integers(-(2 ** 62), 2 ** 62, (d2, d3), dtype=np.int64)  # |U| ≫ p: a genuine element of Z_q
    Ures = U_residues(Ub, ps)
    (AU, BU), eng = run_gpu(fmt, N, d1, d2, d3, ps, ct.a_polys, ct.b_polys, Ures=Ures)
    assert eng.spec.kU == 4 and eng.spec.plain_per_prime == 1
    for l, p in enumerate(ps):
        wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[l], ct.b_polys[l], Ub, p)
        assert np.array_equal(AU[l], wa) and np.array_equal(BU[l], wb)


@pytest.mark.parametrize("fmt,N,k,d2,d3,L,u_bound,chunk,cols", [
    (A, 64, 3, 200, 130, 2, 8, 64, (0, 0)),         # many chunks, A/B boundary inside a chunk
    (S, 32, 4, 96, 300, 1, 8, 0, (17, 250)),        # default chunking, column shard
    (R, 256, 1, 130, 64, 3, 30000, 192, (0, 0)),    # k_U = 2 through the host path
    (A, 16, 2, 40, 7, 1, 8, 4096, (0, 0)),          # one chunk larger than R
    (S, 64, 3, 300, 256, 2, 8, 128, (0, 0)),        # fused skinny kernel on each chunk
    (R, 512, 1, 200, 600, 1, 8, 320, (100, 101)),   # d3_loc = 1 (CP-Mv) column shard
    (A, 64, 4, 300, 520, 2, 8, 192, (0, 0)),        # unsigned-U plane: row sums per chunk
    (S, 2048, 2, 130, 300, 2, 8, 0, (0, 0)),        # default chunks of >= 1024 rows: graded first / last chunk
    (A, 2048, 4, 72, 64, 1, 8, 0, (0, 0)),          # the same through the fused skinny kernel, A / B parts
])
def test_matmul_host_pipeline(fmt, N, k, d2, d3, L, u_bound, chunk, cols):
    """ctpt_matmul_host (host buffers, chunked 3-stream pipeline) == the oracle."""
    import torch

    from paper_2503_16080_b200 import ctpt
    from paper_2503_16080_b200.engine import CpmmEngine

    d1 = N * k
    ps = ctgen.primes(L)
    ct = ctgen.encrypt(fmt, N, d1, d2, 4, 20, ps)
    U = ctgen.U_matrix(4, d2, d3, u_bound)
    eng = CpmmEngine(ctpt.Spec(fmt, N, d1, d2, d3, ps, cols[0], cols[1]), "cuda")
    eng.precompute(U)
    a_h = torch.from_numpy(ct.a_polys.view(np.int32)).pin_memory()
    b_h = torch.from_numpy(ct.b_polys.view(np.int32)).pin_memory()
    AU_h = torch.zeros(eng.sizes.out_AU_bytes // 4, dtype=torch.int32).pin_memory()
    BU_h = torch.zeros(eng.sizes.out_BU_bytes // 4, dtype=torch.int32).pin_memory()
    ws = torch.empty(ctpt.host_workspace_bytes(eng.spec, chunk), dtype=torch.uint8, device="cuda")
    ctpt.matmul_host(eng.spec, a_h, b_h, eng.plain, AU_h, BU_h, ws, chunk_rows=chunk)
    torch.cuda.synchronize()
    d3l = eng.sizes.d3_loc
    AU = AU_h.numpy().view(np.uint32).reshape(L, d3l, -1)
    BU = BU_h.numpy().view(np.uint32).reshape(L, d3l, d1)
    c1 = cols[1] or d3
    for l, p in enumerate(ps):
        wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[l], ct.b_polys[l], U, p, cols=np.arange(cols[0], c1))
        assert np.array_equal(AU[l], wa) and np.array_equal(BU[l], wb)


@pytest.mark.parametrize("chunk", [0, 64, 192])
def test_matmul_host_units_one_pipeline(chunk):
    """ctpt_matmul_host_units: the units of a 3-rank plan's rank (one prime each, column blocks of
    different widths, so the skinny fused kernel, the raw-byte kernel and split + GEMM alternate
    along one pipeline, staging buffers sized for the largest unit) == the oracle, unit by unit."""
    import torch

    from paper_2503_16080_b200 import ctpt
    from paper_2503_16080_b200.engine import CpmmEngine

    fmt, N, k, d2, d3, L = A, 64, 3, 200, 600, 3
    d1 = N * k
    ps = ctgen.primes(L)
    ct = ctgen.encrypt(fmt, N, d1, d2, 6, 20, ps)
    U = ctgen.U_matrix(6, d2, d3, 8)
    units = [(0, 0, 600), (1, 0, 300), (1, 300, 301), (2, 17, 250), (0, 599, 600), (2, 250, 600)]
    specs, plains, a_h, b_h, outs = [], [], [], [], []
    for l, c0, c1 in units:
        eng = CpmmEngine(ctpt.Spec(fmt, N, d1, d2, d3, [ps[l]], c0, c1), "cuda")
        eng.precompute(U)
        specs.append(eng.spec)
        plains.append(eng.plain)
        a_h.append(torch.from_numpy(np.ascontiguousarray(ct.a_polys[l]).view(np.int32)).pin_memory())
        b_h.append(torch.from_numpy(np.ascontiguousarray(ct.b_polys[l]).view(np.int32)).pin_memory())
        outs.append((torch.zeros(eng.sizes.out_AU_bytes // 4, dtype=torch.int32).pin_memory(),
                     torch.zeros(eng.sizes.out_BU_bytes // 4, dtype=torch.int32).pin_memory()))
    ws_bytes = ctpt.host_workspace_bytes_units(specs, chunk)
    assert ws_bytes >= max(ctpt.host_workspace_bytes(sp, chunk) for sp in specs)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    ctpt.matmul_host_units(specs, a_h, b_h, plains, [o[0] for o in outs], [o[1] for o in outs], ws, chunk_rows=chunk)
    torch.cuda.synchronize()
    for (l, c0, c1), (au, bu) in zip(units, outs):
        wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[l], ct.b_polys[l], U, ps[l], cols=np.arange(c0, c1))
        assert np.array_equal(au.numpy().view(np.uint32).reshape(c1 - c0, N), wa), (l, c0, c1)
        assert np.array_equal(bu.numpy().view(np.uint32).reshape(c1 - c0, d1), wb), (l, c0, c1)


def test_shard_units_on_one_gpu():
    """Every unit of a 4-rank plan (L = 3 primes: column-split units) computed through
    shard.gpu_compute_fn on this GPU and placed as rank 0's gather would place it == the oracle."""
    import torch

    from paper_2503_16080_b200.shard import gpu_compute_fn, plan_units

    fmt, N, k, d2, d3, L = A, 64, 2, 130, 300, 3
    d1 = N * k
    ps = ctgen.primes(L)
    ct = ctgen.encrypt(fmt, N, d1, d2, 8, 20, ps)
    U = ctgen.U_matrix(8, d2, d3, 8)
    compute = gpu_compute_fn(fmt, N, d1, d2, d3, ps, lambda l: (ct.a_polys[l], ct.b_polys[l]), U, "cuda")
    full_AU = np.zeros((L, d3, N), np.uint32)
    full_BU = np.zeros((L, d3, d1), np.uint32)
    for units in plan_units(L, d3, 4):
        for u in units:
            au, bu = compute(u)
            torch.cuda.synchronize()
            full_AU[u.l, u.c0:u.c1] = au.cpu().numpy().view(np.uint32)
            full_BU[u.l, u.c0:u.c1] = bu.cpu().numpy().view(np.uint32)
    for l, p in enumerate(ps):
        wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[l], ct.b_polys[l], U, p)
        assert np.array_equal(full_AU[l], wa) and np.array_equal(full_BU[l], wb)


def test_validate_flags_out_of_range():
    from paper_2503_16080_b200 import ctpt

    fmt, N, d2 = R, 16, 32
    ps = ctgen.primes(1)
    ct = ctgen.encrypt(fmt, N, N, d2, 0, 20, ps)
    ct.b_polys[0, 3, 5] = ps[0]  # = p: not a canonical residue
    with pytest.raises(ctpt.CtptError, match="ERR_RANGE"):
        run_gpu(fmt, N, N, d2, 4, ps, ct.a_polys, ct.b_polys, U=np.ones((d2, 4), np.int64), validate=True)


def test_config1_full_and_decrypt():
    c = ctgen.CONFIGS["c1"]
    ps = ctgen.primes(c.L)
    ct = ctgen.encrypt(c.fmt, c.N, c.d1, c.d2, c.seed, c.log_delta, ps)
    U = ctgen.U_matrix(c.seed, c.d2, c.d3, c.u_bound)
    (AU, BU), _ = run_gpu(c.fmt, c.N, c.d1, c.d2, c.d3, ps, ct.a_polys, ct.b_polys, U=U)
    wa, wb = oracle_outputs(c.fmt, c.N, c.d1, ct.a_polys[0], ct.b_polys[0], U, ps[0])
    assert np.array_equal(AU[0], wa) and np.array_equal(BU[0], wb)
    # decryption identity and decode (readings Q15, Q16)
    sk = [ctgen.sk(c.seed, 0, c.N)]
    P = ctgen.plain_block(c.seed, c.N, c.d1, c.log_delta, 0, c.d1, 0, c.d2)
    PU = P.astype(object).dot(U.astype(object))
    M = ctgen.msg_block(c.seed, c.d1, 0, c.d1, 0, c.d2)
    MU = M.dot(U.astype(np.float64))
    dec = np.stack([oracle.decrypt_col(c.fmt, c.N, c.d1, sk, AU[0, j], BU[0, j], ps[0]) for j in range(c.d3)], 1)
    cen = np.array([[oracle.crt_centred([v], ps) for v in row] for row in dec], dtype=object)
    assert (cen == PU).all()
    approx = cen.astype(np.float64) / 2.0 ** c.log_delta
    assert np.abs(approx - MU).max() <= np.abs(U).max() * c.d2 * 20.5 / 2.0 ** c.log_delta


@pytest.mark.parametrize("split_overlap", [0, 1])
def test_config2_full(split_overlap):
    """Config c2 (RLWE, N = d = 4096, two primes): every output entry vs the oracle, plus the
    decryption identity and the 1e-6 decode bound on sampled columns.  split_overlap = 1 is the
    launch configuration bench.py times for c2 (d3 <= 8192): prime 1 is split inside prime 0's
    k_gemm_tc."""
    c = ctgen.CONFIGS["c2"]
    ps = ctgen.primes(c.L)
    ct = ctgen.encrypt(c.fmt, c.N, c.d1, c.d2, c.seed, c.log_delta, ps, nthreads=NTHREADS)
    U = ctgen.U_matrix(c.seed, c.d2, c.d3, c.u_bound, nthreads=NTHREADS)
    (AU, BU), _ = run_gpu(c.fmt, c.N, c.d1, c.d2, c.d3, ps, ct.a_polys, ct.b_polys, U=U, split_overlap=split_overlap)
    for l, p in enumerate(ps):
        wa, wb = oracle_outputs(c.fmt, c.N, c.d1, ct.a_polys[l], ct.b_polys[l], U, p)
        assert np.array_equal(AU[l], wa), "A·U mismatch"
        assert np.array_equal(BU[l], wb), "B·U mismatch"
    _decrypt_check(c, ps, AU, BU, U, cols=[0, 1, 127, 128, 2049, c.d3 - 1])


def _decrypt_check(c, ps, AU, BU, U, cols):
    """S·A' + B' ≡ (⌊ΔM⌉+E)·U (mod q) exactly on `cols`, and the decoded value is within 1e-6
    relative of M·U in float64 (readings Q15, Q16)."""
    nk = c.k if c.fmt == A else 1
    sks = [ctgen.sk(c.seed, t, c.N) for t in range(nk)]
    P = ctgen.plain_block(c.seed, c.N, c.d1, c.log_delta, 0, c.d1, 0, c.d2, nthreads=NTHREADS)
    M = ctgen.msg_block(c.seed, c.d1, 0, c.d1, 0, c.d2, nthreads=NTHREADS)
    Uc = U[:, cols]
    PU = P.astype(object).dot(Uc.astype(object)) if c.log_delta > 48 else P.dot(Uc).astype(object)
    MU = M.dot(Uc.astype(np.float64))
    worst = 0.0
    for ci, j in enumerate(cols):
        decs = np.stack([oracle.decrypt_col(c.fmt, c.N, c.d1, sks, AU[l, j], BU[l, j], p, nthreads=NTHREADS)
                         for l, p in enumerate(ps)])
        cen = oracle.crt_centred_array(decs, ps)
        assert cen == list(PU[:, ci]), f"decryption identity fails in column {j}"
        approx = np.array([float(v) for v in cen]) / 2.0 ** c.log_delta
        worst = max(worst, np.abs(approx - MU[:, ci]).max() / np.abs(MU).max())
    assert worst <= 1e-6, worst


def test_struct_a_algorithm7_decrypts():
    """Algorithm 7 end to end on the GPU: B' = B·U from ctpt_matmul; then Ã·(S·U) + B' ≡
    (⌊ΔM⌉+E)·U (mod p) for every output column and prime."""
    fmt, N, k, d2, d3, L = SA, 32, 3, 96, 20, 2
    d1 = N * k
    ps = ctgen.primes(L)
    ct = ctgen.encrypt(fmt, N, d1, d2, 12, 20, ps)
    U = ctgen.U_matrix(12, d2, d3, 8)
    (AU, BU), eng = run_gpu(fmt, N, d1, d2, d3, ps, ct.a_polys, ct.b_polys, U=U)
    assert AU.shape == (L, d3, 0) and eng.sizes.out_AU_bytes == 0
    sks = [ctgen.sk(12, j, N) for j in range(d2)]
    P = ctgen.plain_matrix(12, N, d1, range(d1), range(d2), 20)
    PU = P.astype(object).dot(U.astype(object))
    for l, p in enumerate(ps):
        wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[l], ct.b_polys[l], U, p)
        assert np.array_equal(BU[l], wb)
        for j in range(d3):
            dec = oracle.decrypt_col(fmt, N, d1, [oracle.su_column(sks, U, j)], ct.a_polys[l], BU[l, j], p)
            assert [int(x) for x in dec] == [int(v) % p for v in PU[:, j]]


# ------------------------------------------------------------------ RNS Rescale (§8(f) row 3)
RESCALE = [
    # fmt, N, k, d2, d3, L, U: "real" (U0 = ⌊q_1·U⌉ as residues, kU = 4) or "int" (|U| ≤ 8, kU = 1)
    (S, 64, 2, 300, 200, 3, "real"),
    (A, 32, 3, 130, 70, 2, "real"),
    (R, 128, 1, 96, 40, 4, "int"),      # kU = 1 → fused skinny kernel + Rescale epilogue
    (SA, 16, 3, 77, 300, 3, "int"),     # structured-A (Algorithm 7 step 2), split + GEMM path
    (A, 8, 3, 50, 33, 2, "real"),       # R = 32: one partial tile
    (S, 32, 2, 100, 20, 3, "int"),      # d3 <= 32: raw-byte kernel + Rescale (K-split partials)
]


def _rescale_check(fmt, N, k, d2, d3, L, ukind, seed=21):
    d1 = N * k
    ps = ctgen.primes(L)
    ct = ctgen.encrypt(fmt, N, d1, d2, seed, 20, ps, nthreads=NTHREADS)
    if ukind == "real":
        _, U0 = ctgen.U_real(seed, d2, d3, ps[-1])
        (AU, BU), eng = run_gpu(fmt, N, d1, d2, d3, ps, ct.a_polys, ct.b_polys, Ures=U_residues(U0, ps), rescale=1)
        assert eng.spec.kU == 4
    else:
        U0 = ctgen.U_matrix(seed, d2, d3, 8)
        (AU, BU), eng = run_gpu(fmt, N, d1, d2, d3, ps, ct.a_polys, ct.b_polys, U=U0, rescale=1)
        assert eng.spec.kU == 1
    assert AU.shape[0] == L - 1 and BU.shape[0] == L - 1
    ra = eng.sizes.rows_A
    prods = []
    for l, p in enumerate(ps):
        wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[l], ct.b_polys[l], U0, p)
        prods.append(np.concatenate([wa, wb], axis=1).reshape(-1))
    want = oracle.rescale_last(np.stack(prods), ps).reshape(L - 1, d3, ra + d1)
    got = np.concatenate([AU, BU], axis=2)
    bad = np.argwhere(got != want)
    assert bad.size == 0, f"{len(bad)} rescaled residues differ, first {bad[:5]}"


@pytest.mark.parametrize("case", RESCALE, ids=lambda s: "f%d_N%d_k%d_d2%d_d3%d_L%d_%s" % s)
def test_rescale_fused_epilogue(case):
    _rescale_check(*case)


# ------------------------------------------------------------------ Mod-PP-MM entry point (§8(f) row 4)
@pytest.mark.parametrize("M,K,Nc,L", [(100, 77, 50, 1), (300, 1000, 257, 2), (64, 16, 1, 3), (1000, 2049, 300, 2),
                                      (33, 4112, 129, 1)])
def test_modmatmul_full_residues(M, K, Nc, L):
    """Z = X·Y mod p with X and Y full residues on both sides (the Mod-PP-MM stage of Alg. 8/9)."""
    import torch

    from paper_2503_16080_b200 import ctpt

    ps = ctgen.primes(L)
    ldx, plain_bytes, ws_bytes = ctpt.modmatmul_sizes(ps, M, K, Nc)
    rng = np.random.default_rng(M + K + Nc)
    X = np.zeros((L, M, ldx), np.uint32)
    Y = np.empty((L, K, Nc), np.uint32)
    for l, p in enumerate(ps):
        X[l, :, :K] = rng.integers(0, p, (M, K))
        Y[l] = rng.integers(0, p, (K, Nc))
        X[l, 0, :K] = p - 1  # extreme residues
        Y[l, :, 0] = p - 1
    Xd = torch.from_numpy(X.view(np.int32)).cuda()
    Yd = torch.from_numpy(Y.view(np.int32)).cuda()
    plain = torch.empty(plain_bytes, dtype=torch.uint8, device="cuda")
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device="cuda")
    ZT = torch.empty(L * Nc * M, dtype=torch.int32, device="cuda")
    ctpt.modmatmul_precompute(ps, M, K, Nc, Yd, plain)
    ctpt.modmatmul(ps, M, K, Nc, Xd, ldx, plain, ZT, ws)
    torch.cuda.synchronize()
    got = ZT.cpu().numpy().view(np.uint32).reshape(L, Nc, M)
    for l, p in enumerate(ps):
        want = oracle.modmatmul(np.ascontiguousarray(X[l, :, :K].T), Y[l].astype(np.int64), p, nthreads=NTHREADS)
        assert np.array_equal(got[l], want), f"prime {l}: {np.count_nonzero(got[l] != want)} entries differ"


# ------------------------------------------------------------------ CUDA graph capture
@pytest.mark.parametrize("shape", [(R, 64, 1, 64, 64, 1), (A, 64, 3, 300, 20, 2), (S, 32, 2, 200, 300, 2)],
                         ids=["c1_fused", "mv", "split_gemm"])
def test_matmul_is_graph_capturable(shape):
    """ctpt_matmul never synchronises or allocates, so a CUDA graph can capture it (every kernel
    path: fused, raw-byte with its memset + U expansion, split + GEMM) and replay it: the replayed
    outputs equal the oracle, and a replay after changing the inputs in place recomputes them."""
    import torch

    from paper_2503_16080_b200 import ctpt
    from paper_2503_16080_b200.engine import CpmmEngine

    fmt, N, k, d2, d3, L = shape
    d1 = N * k
    ps = ctgen.primes(L)
    eng = CpmmEngine(ctpt.Spec(fmt, N, d1, d2, d3, ps), "cuda")
    U = ctgen.U_matrix(3, d2, d3, 8)
    AU, BU = eng.alloc_outputs()
    s = torch.cuda.Stream()
    for seed in (3, 4):
        ct = ctgen.encrypt(fmt, N, d1, d2, seed, 20, ps)
        eng.layout(ct.a_polys, ct.b_polys)
        if seed == 3:
            eng.precompute(U)
            with torch.cuda.stream(s):
                ctpt.matmul(eng.spec, eng.ctmat, eng.plain, AU, BU, eng.ws, stream=s)  # warm-up
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                ctpt.matmul(eng.spec, eng.ctmat, eng.plain, AU, BU, eng.ws, stream=s)
        AU.zero_()
        BU.zero_()
        g.replay()
        torch.cuda.synchronize()
        AUn, BUn = eng.outputs_numpy(AU, BU)
        for l, p in enumerate(ps):
            wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[l], ct.b_polys[l], U, p)
            assert np.array_equal(AUn[l], wa) and np.array_equal(BUn[l], wb), (seed, l)


def test_rescale_standalone_matches_oracle():
    """ctpt_rescale on residue arrays (incl. the values around ±q_1/2 and 0) == the oracle's
    plain ⌊x/q_1⌉ (CRT, exact division)."""
    import torch

    from paper_2503_16080_b200 import ctpt

    ps = ctgen.primes(3)
    q = ps[0] * ps[1] * ps[2]
    rng = np.random.default_rng(8)
    xs = [int.from_bytes(rng.bytes(16), "little") % q for _ in range(3000)]
    h = (ps[2] - 1) // 2
    xs += [0, 1, q - 1, h, h + 1, q - h, q - h - 1, 5 * ps[2] + h, 5 * ps[2] + h + 1]
    res = np.array([[x % p for x in xs] for p in ps], dtype=np.uint32)
    out = torch.empty((2, len(xs)), dtype=torch.int32, device="cuda")
    ctpt.rescale(ps, len(xs), torch.from_numpy(res.view(np.int32)).cuda(), out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().view(np.uint32), oracle.rescale_last(res, ps))


def test_struct_a_algorithm7_with_rescale():
    """Algorithm 7 with its step 2: B'' = Rescale(B·U) from ctpt_matmul(rescale=1) and
    Ã'' = Rescale(Ã) from ctpt_rescale on the a-polynomials; (Ã'', B'') decrypts under (S·U)_j over
    the remaining primes to (P·U)/q_1 within (‖(S·U)_j‖₁ + 1)/2 (exact rational check)."""
    from fractions import Fraction

    import torch

    from paper_2503_16080_b200 import ctpt

    fmt, N, k, d2, d3, L, seed = SA, 16, 3, 40, 6, 3, 14
    d1 = N * k
    ps = ctgen.primes(L)
    q1 = ps[-1]
    ct = ctgen.encrypt(fmt, N, d1, d2, seed, 20, ps)
    U = ctgen.U_matrix(seed, d2, d3, 8)
    (AU, BU), eng = run_gpu(fmt, N, d1, d2, d3, ps, ct.a_polys, ct.b_polys, U=U, rescale=1)
    a_in = torch.from_numpy(ct.a_polys.reshape(L, -1).view(np.int32)).cuda()
    a_out = torch.empty((L - 1, a_in.shape[1]), dtype=torch.int32, device="cuda")
    ctpt.rescale(ps, a_in.shape[1], a_in, a_out)
    torch.cuda.synchronize()
    a2 = a_out.cpu().numpy().view(np.uint32).reshape(L - 1, k, N)
    assert np.array_equal(a2.reshape(L - 1, -1), oracle.rescale_last(ct.a_polys.reshape(L, -1), ps))
    sks = [ctgen.sk(seed, j, N) for j in range(d2)]
    P = ctgen.plain_matrix(seed, N, d1, range(d1), range(d2), 20)
    PU = P.astype(object).dot(U.astype(object))
    for j in range(d3):
        w = oracle.su_column(sks, U, j)
        decs = np.stack([oracle.decrypt_col(fmt, N, d1, [w], a2[l], BU[l, j], ps[l]) for l in range(L - 1)])
        cen = oracle.crt_centred_array(decs, ps[:2])
        bound = Fraction(int(np.abs(w).sum()) + 1, 2)
        for i in range(d1):
            assert abs(Fraction(cen[i]) - Fraction(int(PU[i, j]), q1)) <= bound, (j, i)


# ------------------------------------------------------------------ split of prime l+1 inside GEMM l
@pytest.mark.parametrize("unsigned", ["never", "always"])
def test_split_overlap_matmul(unsigned):
    """ctpt_problem.split_overlap = 1: ctpt_matmul splits prime 0 on its own and every further
    prime inside the previous prime's GEMM (warps 2–3 of k_gemm_tc), alternating two limb buffers
    — L = 3 and 4 primes, the u8 plane with its row correction and the s8 plane, multi-digit U
    (side split in pass 0 only)."""
    import torch

    from paper_2503_16080_b200 import ctpt
    from paper_2503_16080_b200.engine import CpmmEngine

    for (fmt, N, k, d2, d3, L, ub) in [(A, 64, 3, 300, 260, 3, 8), (S, 32, 4, 129, 300, 4, 8),
                                        (R, 256, 1, 200, 140, 2, 300)]:
        d1 = N * k
        ps = ctgen.primes(L)
        ct = ctgen.encrypt(fmt, N, d1, d2, 21, 20, ps)
        U = ctgen.U_matrix(21, d2, d3, ub)
        eng = CpmmEngine(ctpt.Spec(fmt, N, d1, d2, d3, ps, split_overlap=1, kernel=SPLIT_GEMM), "cuda")
        eng.layout(ct.a_polys, ct.b_polys)
        eng.precompute(U, unsigned=unsigned if ub <= 127 else "never")
        AU, BU = eng.matmul()
        torch.cuda.synchronize()
        AUn, BUn = eng.outputs_numpy(AU, BU)
        for l, p in enumerate(ps):
            wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[l], ct.b_polys[l], U, p)
            assert np.array_equal(AUn[l], wa) and np.array_equal(BUn[l], wb), (fmt, l)


def test_split_overlap_stage_entry_points():
    """The per-stage form a benchmark times: ctpt_split(0), then ctpt_gemm_next(l) per prime;
    ctpt_gemm_next refuses a problem without split_overlap."""
    import torch

    from paper_2503_16080_b200 import ctpt
    from paper_2503_16080_b200.engine import CpmmEngine

    fmt, N, k, d2, d3, L = A, 128, 2, 520, 400, 3
    d1 = N * k
    ps = ctgen.primes(L)
    ct = ctgen.encrypt(fmt, N, d1, d2, 22, 20, ps)
    U = ctgen.U_matrix(22, d2, d3, 8)
    eng = CpmmEngine(ctpt.Spec(fmt, N, d1, d2, d3, ps, split_overlap=1), "cuda")
    eng.layout(ct.a_polys, ct.b_polys)
    eng.precompute(U)
    AU, BU = eng.alloc_outputs()
    ra = eng.sizes.rows_A
    for rep in range(2):  # the second step reuses both limb buffers
        ctpt.split(eng.spec, 0, eng.ctmat, eng.ws)
        for l in range(L):
            ctpt.gemm_next(eng.spec, l, eng.ctmat, eng.ws, eng.plain, AU[l * d3 * ra:], BU[l * d3 * d1:])
    torch.cuda.synchronize()
    AUn, BUn = eng.outputs_numpy(AU, BU)
    for l, p in enumerate(ps):
        wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[l], ct.b_polys[l], U, p)
        assert np.array_equal(AUn[l], wa) and np.array_equal(BUn[l], wb), l
    plain = ctpt.Spec(fmt, N, d1, d2, d3, ps, kU=eng.spec.kU, u_unsigned=eng.spec.u_unsigned,
                      u_offset=eng.spec.u_offset)
    with pytest.raises(ctpt.CtptError, match="ERR_ARG"):
        ctpt.gemm_next(plain, 0, eng.ctmat, eng.ws, eng.plain, AU, BU)


# ------------------------------------------------------------------ seeded random shapes (fuzz)
def _fuzz_cases(n=48, seed=2025):
    rng = np.random.default_rng(seed)
    cases = []
    for i in range(n):
        fmt = int(rng.choice([R, S, A, SA]))
        N = int(rng.choice([2, 4, 8, 16, 32, 64, 128, 256]))
        k = 1 if fmt == R else int(rng.integers(1, 5))
        d2 = int(rng.integers(1, 700))
        d3 = int(rng.choice([1, 2, 5, 16, 31, 33, 64, 100, 128, 129, 200, 256, 257, 300, 520]))
        L = int(rng.integers(1, 4))
        ub = int(rng.choice([1, 8, 127, 128, 300, 40000]))
        c0 = int(rng.integers(0, d3)) if rng.random() < 0.3 else 0
        c1 = int(rng.integers(c0 + 1, d3 + 1)) if c0 or rng.random() < 0.2 else 0
        cases.append((fmt, N, k, d2, d3, L, ub, c0, c1, i))
    return cases


@pytest.mark.parametrize("case", _fuzz_cases(), ids=lambda c: "f%d_N%d_k%d_d2%d_d3%d_L%d_u%d_c%d-%d_%d" % c)
def test_fuzz_shapes_against_oracle(case):
    """Seeded random problems across every dimension regime the library dispatches on (d3_loc ≤ 32
    raw-byte kernel, ≤ 256 fused kernel, else split + GEMM; k_U = 1..3 digits; s8 or u8 U
    planes; column shards; d2 from 1; N from 2; every other case with split_overlap = 1; every
    third case with split + GEMM forced) — each output entry against the oracle."""
    fmt, N, k, d2, d3, L, ub, c0, c1, i = case
    _check(fmt, N, k, d2, d3, L, seed=100 + i, u_bound=ub, col_begin=c0, col_end=c1, split_overlap=i % 2,
           kernel=SPLIT_GEMM if i % 3 == 0 else AUTO)


@pytest.mark.parametrize("raster_group,max_ctas", [(1, 0), (3, 0), (1000, 0), (0, 1), (0, 7), (5, 3)])
def test_raster_group_and_grid_cap_keep_results_exact(raster_group, max_ctas):
    """ctpt_problem.raster_group (k_gemm_tc's tile order) and max_ctas (the persistent grids' CTA
    cap, for SMs left to a concurrent NCCL kernel) change the schedule, never a residue — in the
    split + GEMM, fused and raw-byte regimes, with the next prime's split inside the GEMM."""
    _check(A, 64, 3, 700, 300, 2, seed=51, raster_group=raster_group, max_ctas=max_ctas, split_overlap=1)
    _check(S, 32, 4, 520, 100, 1, seed=52, raster_group=raster_group, max_ctas=max_ctas)
    _check(S, 256, 4, 4112, 8, 1, seed=53, raster_group=raster_group, max_ctas=max_ctas)


def test_forced_kernel_refusals():
    """A forced kernel that does not apply is refused (ERR_UNSUPPORTED), never silently replaced."""
    from paper_2503_16080_b200 import ctpt

    fmt, N, d2 = R, 64, 100
    ps = ctgen.primes(1)
    ct = ctgen.encrypt(fmt, N, N, d2, 0, 20, ps)
    U = ctgen.U_matrix(0, d2, 300, 8)
    with pytest.raises(ctpt.CtptError, match="ERR_UNSUPPORTED"):
        run_gpu(fmt, N, N, d2, 300, ps, ct.a_polys, ct.b_polys, U=U, kernel=FUSED)
    with pytest.raises(ctpt.CtptError, match="ERR_UNSUPPORTED"):
        run_gpu(fmt, N, N, d2, 40, ps, ct.a_polys, ct.b_polys, U=U[:, :40], kernel=MV_K)


@pytest.mark.parametrize("shape,max_ctas", [
    ((S, 64, 3, 1000, 1, 2), 0),      # CP-Mv through the TMEM kernel with u_offset
    ((A, 128, 4, 520, 64, 1), 0),
    ((S, 32, 5, 384, 128, 2), 1),     # one CTA loops over every tile: the row-sum buffers wrap
    ((A, 16, 3, 77, 129, 2), 0),      # 32-row tiles (d3 > 128), one K-block: a converter group with no K-block
    ((R, 1024, 1, 2056, 160, 1), 3),
    ((S, 128, 2, 100, 192, 1), 1),    # num_kb = 1 with 32-row tiles, several tiles per CTA
], ids=lambda s: str(s))
def test_skinny_unsigned_plane_row_sums(shape, max_ctas):
    """The limbs-in-TMEM skinny kernel with the u8 plane U' = U + u_offset: the converters form
    Σ_k X[r][k] (IDP4A byte sums of the limbs) while they split X, the epilogue subtracts
    u_offset·Σ_k X[r][k] mod p (X·U = X·U' − u_offset·rowsum) — against the oracle, forced and
    automatic kernel choice, several tiles per CTA."""
    _check(*shape, unsigned="always", kernel=FUSED, max_ctas=max_ctas)
    _check(*shape, unsigned="always", max_ctas=max_ctas, seed=3)
