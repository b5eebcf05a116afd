"""The C-ABI library loads, exports every symbol include/ctpt.h declares, and validates
arguments on the host (no GPU needed: validation and size queries touch no device)."""
import ctypes
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ctpt():
    import __graft_entry__

    __graft_entry__.build_ctpt()
    from paper_2503_16080_b200 import ctpt as m

    return m


def test_exports_every_header_symbol(ctpt):
    syms = ctpt.header_symbols()
    assert "ctpt_matmul" in syms and "ctpt_layout" in syms and "ctpt_plain_precompute" in syms
    lib = ctypes.CDLL(ctpt.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), f"libctpt.so does not export {s}"


def test_version(ctpt):
    assert "sm_100a" in ctpt.version()


def _spec(ctpt, **kw):
    base = dict(fmt=ctpt.SHARED_A, N=16, d1=64, d2=48, d3=20, primes=[2147352577])
    base.update(kw)
    return ctpt.Spec(**base)


def test_sizes(ctpt):
    s = ctpt.query_sizes(_spec(ctpt))
    assert s.rows_A == 16 and s.R == 80 and s.d2p == 48 and s.d3_loc == 20
    assert s.ctmat_bytes == 256 + 80 * 48 * 4
    # d3 = 20 ≤ 32: the limb planes, then the raw-byte kernel's U_exp (NC = 4·32 rows × 4·d2p bytes)
    assert s.workspace_bytes >= 4 * 80 * 48 + 128 * 4 * 48
    # byte limbs in 32-KB tiles: rows padded to 64, K to 128 (kernels.cuh limb_tile_off)
    assert ctpt.query_sizes(_spec(ctpt, d3=40)).workspace_bytes == 4 * 128 * 128
    assert s.out_AU_bytes == 20 * 16 * 4 and s.out_BU_bytes == 20 * 64 * 4
    s2 = ctpt.query_sizes(_spec(ctpt, fmt=ctpt.SHARED_S, d2=50, col_begin=3, col_end=11))
    assert s2.rows_A == 64 and s2.R == 128 and s2.d2p == 64 and s2.d3_loc == 8
    s3 = ctpt.query_sizes(_spec(ctpt, fmt=ctpt.RLWE, d1=16, primes=[2147352577, 2146959361]))
    assert s3.out_BU_bytes == 2 * 20 * 16 * 4


@pytest.mark.parametrize("kw,status", [
    (dict(fmt=0, N=16, d1=32), "ERR_SHAPE"),
    (dict(N=12, d1=24), "ERR_SHAPE"),
    (dict(d1=40), "ERR_SHAPE"),
    (dict(d2=0), "ERR_SHAPE"),
    (dict(col_begin=5, col_end=5), "ERR_SHAPE"),
    (dict(col_end=21), "ERR_SHAPE"),
    (dict(primes=[2147352577, 2147352577]), "ERR_MODULUS"),
    (dict(primes=[2 ** 31 + 11]), "ERR_MODULUS"),
    (dict(primes=[1024]), "ERR_MODULUS"),
    (dict(primes=[2147352577, 2147352577 - 2]), "ERR_MODULUS"),  # odd composite (divisible by 5)
    (dict(primes=[2147352577, 1 << 30 | 1]), "ERR_MODULUS"),      # 2^30 + 1 = 5^2 · 13 · 41 · 61 · 1321
    (dict(d2=70000), "ERR_OVERFLOW"),
    (dict(fmt=7), "ERR_UNSUPPORTED"),
])
def test_validation(ctpt, kw, status):
    with pytest.raises(ctpt.CtptError) as ei:
        ctpt.query_sizes(_spec(ctpt, **kw))
    assert str(ei.value).startswith(status)


def test_null_pointers_rejected_without_gpu(ctpt):
    # argument validation happens before any CUDA call
    lib = ctpt.raw_lib()
    pb = _spec(ctpt).cstruct()
    assert lib.ctpt_layout(ctypes.byref(pb), None, None, None, 0, None) == 1
    assert lib.ctpt_matmul(ctypes.byref(pb), None, None, None, None, None, 0, None) == 1
    assert b"null" in lib.ctpt_last_error()


def test_fused_refuses_wide_or_multidigit_U_without_gpu(ctpt):
    # the skinny kernel's eligibility (d3_loc <= 256, kU = 1) is checked before any CUDA call
    lib = ctpt.raw_lib()
    fake = ctypes.c_void_p(256)  # never dereferenced
    pb = _spec(ctpt, d3=300).cstruct()
    assert lib.ctpt_gemm_fused(ctypes.byref(pb), 0, fake, fake, fake, fake, None) == 6
    pb = _spec(ctpt, d3=300, col_begin=10, col_end=266, kU=2).cstruct()
    assert lib.ctpt_gemm_fused(ctypes.byref(pb), 0, fake, fake, fake, fake, None) == 6
    pb = _spec(ctpt, d3=20).cstruct()
    assert lib.ctpt_gemm_fused(ctypes.byref(pb), 1, fake, fake, fake, fake, None) == 1  # prime index


def test_modmatmul_sizes_and_ldx_check_without_gpu(ctpt):
    """Mod-PP-MM entry points validate on the host: ldx = K rounded up to 16, d2 overflow."""
    ps = [2147352577, 2146959361]
    ldx, plain, ws = ctpt.modmatmul_sizes(ps, 100, 77, 50)
    assert ldx == 80 and plain == 256 + 2 * 4 * 50 * 80 and ws == 4 * 128 * 128  # limbs in 32-KB tiles
    lib = ctpt.raw_lib()
    arr = (ctypes.c_uint32 * 2)(*ps)
    fake = ctypes.c_void_p(256)
    assert lib.ctpt_modmatmul(2, ctypes.cast(arr, ctypes.c_void_p), 100, 77, 50, fake, 77, fake, fake, fake,
                              1 << 20, None) == 2  # ERR_SHAPE: ldx must be 80
    with pytest.raises(ctpt.CtptError, match="ERR_OVERFLOW"):
        ctpt.modmatmul_sizes(ps, 10, 70000, 10)


def test_split_overlap_workspace_and_validation(ctpt):
    """split_overlap = 1 adds a second limb buffer (+ row-sum buffer) to the workspace when the
    problem has ≥ 2 primes and no Rescale; any other value than 0 / 1 is refused."""
    ps = [2147352577, 2146959361]
    base = ctpt.query_sizes(_spec(ctpt, d3=300, primes=ps))
    ovl = ctpt.query_sizes(_spec(ctpt, d3=300, primes=ps, split_overlap=1))
    limbs = 4 * base.R * base.d2p
    assert ovl.workspace_bytes >= base.workspace_bytes + limbs
    one = ctpt.query_sizes(_spec(ctpt, d3=300, primes=ps[:1], split_overlap=1))  # one prime: nothing to overlap
    assert one.workspace_bytes == ctpt.query_sizes(_spec(ctpt, d3=300, primes=ps[:1])).workspace_bytes
    resc = ctpt.query_sizes(_spec(ctpt, d3=300, primes=ps, split_overlap=1, rescale=1))
    assert resc.workspace_bytes == ctpt.query_sizes(_spec(ctpt, d3=300, primes=ps, rescale=1)).workspace_bytes
    with pytest.raises(ctpt.CtptError, match="ERR_ARG"):
        ctpt.query_sizes(_spec(ctpt, primes=ps, split_overlap=2))
