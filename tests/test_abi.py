"""The C-ABI library loads, exports every symbol include/ctpt.h declares, and validates
arguments on the host (no GPU needed: validation and size queries touch no device)."""
import ctypes
import os
import types

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


def test_schedule_fields_validated_without_gpu(ctpt):
    """ctpt_problem.kernel / raster_group / max_ctas: out-of-range values are refused on the host;
    a forced kernel that does not apply to the problem is refused by ctpt_matmul before any CUDA
    call (ERR_UNSUPPORTED), never replaced by another path."""
    for kw in (dict(kernel=4), dict(kernel=-1), dict(raster_group=-1), dict(max_ctas=-2)):
        with pytest.raises(ctpt.CtptError, match="ERR_ARG"):
            ctpt.query_sizes(_spec(ctpt, **kw))
    ctpt.query_sizes(_spec(ctpt, kernel=ctpt.KERNEL_FUSED, raster_group=3, max_ctas=7))
    lib = ctpt.raw_lib()
    fake = ctypes.c_void_p(256)  # never dereferenced
    ws = 1 << 30
    pb = _spec(ctpt, d3=300, kernel=ctpt.KERNEL_FUSED).cstruct()        # d3_loc > 256
    assert lib.ctpt_matmul(ctypes.byref(pb), fake, fake, fake, fake, fake, ws, None) == 6
    pb = _spec(ctpt, d3=40, kernel=ctpt.KERNEL_MV).cstruct()            # d3_loc > 32
    assert lib.ctpt_matmul(ctypes.byref(pb), fake, fake, fake, fake, fake, ws, None) == 6
    pb = _spec(ctpt, d3=20, kU=2, kernel=ctpt.KERNEL_MV).cstruct()      # kU > 1
    assert lib.ctpt_matmul(ctypes.byref(pb), fake, fake, fake, fake, fake, ws, None) == 6
    assert b"needs" in lib.ctpt_last_error()


def test_version_names_the_source_hash(ctpt):
    """ctpt_version() carries src=<sha256 prefix of csrc/ + include/>, the hash build() compiles in."""
    import __graft_entry__

    assert ctpt.source_hash() == __graft_entry__.source_hash()


def test_ipc_and_peer_entry_points_validate_without_gpu(ctpt):
    """The multi-GPU gather plumbing refuses null arguments on the host (CTPT_ERR_ARG)."""
    lib = ctpt.raw_lib()
    h = (ctypes.c_char * ctpt.IPC_HANDLE_BYTES)()
    off = ctypes.c_uint64(0)
    base, ptr = ctypes.c_void_p(), ctypes.c_void_p()
    assert lib.ctpt_ipc_export(None, ctypes.cast(h, ctypes.c_void_p), ctypes.byref(off)) == 1
    assert lib.ctpt_ipc_export(ctypes.c_void_p(256), None, ctypes.byref(off)) == 1
    assert lib.ctpt_ipc_open(None, 0, ctypes.byref(base), ctypes.byref(ptr)) == 1
    assert lib.ctpt_ipc_open(ctypes.cast(h, ctypes.c_void_p), 0, None, ctypes.byref(ptr)) == 1
    assert lib.ctpt_ipc_close(None) == 1
    assert lib.ctpt_peer_access(0, 0, None) == 1
    can = ctypes.c_int32(0)
    assert lib.ctpt_peer_access(3, 3, ctypes.byref(can)) == 0 and can.value == 1  # a device reaches itself


def test_host_units_workspace_and_validation_without_gpu(ctpt):
    """ctpt_host_workspace_bytes_units: n = 1 is ctpt_host_workspace_bytes; a batch is sized for its
    largest unit in every staging region; n < 1, a Rescale unit, or a bad unit anywhere in the
    batch is refused before anything is enqueued (no device pointer is touched)."""
    a = _spec(ctpt, d3=300)
    b = _spec(ctpt, d3=40, col_begin=10, col_end=30)
    one = ctpt.host_workspace_bytes_units([a], 64)
    assert one == ctpt.host_workspace_bytes(a, 64)
    both = ctpt.host_workspace_bytes_units([a, b], 64)
    assert both >= max(one, ctpt.host_workspace_bytes(b, 64))
    assert ctpt.host_workspace_bytes_units([b, a], 64) == both
    lib = ctpt.raw_lib()
    n = ctypes.c_size_t(0)
    assert lib.ctpt_host_workspace_bytes_units(0, ctypes.cast(ctpt._problems([a]), ctpt._PP), 64, ctypes.byref(n)) == 1
    with pytest.raises(ctpt.CtptError, match="ERR_UNSUPPORTED"):
        ctpt.host_workspace_bytes_units([a, _spec(ctpt, d3=300, rescale=1, primes=[2147352577, 2146959361])], 0)
    with pytest.raises(ctpt.CtptError, match="ERR_ARG"):
        ctpt.host_workspace_bytes_units([a, _spec(ctpt, kernel=4)], 0)
    fake = 256  # never dereferenced: the null host pointer of unit 1 is refused first
    ws_t = types.SimpleNamespace(data_ptr=lambda: 256, numel=lambda: both, element_size=lambda: 1)
    with pytest.raises(ctpt.CtptError, match="ERR_ARG"):
        ctpt.matmul_host_units([a, b], [fake, fake], [fake, None], [fake, fake], [fake, fake], [fake, fake], ws_t,
                               chunk_rows=64, stream=0)
    with pytest.raises(ctpt.CtptError, match="workspace too small"):
        ctpt.matmul_host_units([a, b], [fake] * 2, [fake] * 2, [fake] * 2, [fake] * 2, [fake] * 2,
                               types.SimpleNamespace(data_ptr=lambda: 256, numel=lambda: one - 1,
                                                     element_size=lambda: 1), chunk_rows=64, stream=0)
