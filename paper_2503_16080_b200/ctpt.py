"""Thin ctypes binding of libctpt.so (include/ctpt.h) — argument marshalling only.

Every step of the CP-MM path runs in the library's CUDA kernels; this module only
turns torch tensors into device pointers and the current CUDA stream into the
``void* stream`` argument.  There is no CPU fallback: importing this module on a
machine without the built library raises, and every call that returns a non-OK
status raises :class:`CtptError`.
"""
from __future__ import annotations

import ctypes
import os
import re
from dataclasses import dataclass

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CTPT_LIB") or os.path.join(_HERE, "libctpt.so")  # CTPT_LIB: A/B of two builds
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "ctpt.h")

RLWE, SHARED_S, SHARED_A, STRUCT_A = 0, 1, 2, 3
KERNEL_AUTO, KERNEL_SPLIT_GEMM, KERNEL_FUSED, KERNEL_MV = 0, 1, 2, 3  # ctpt_kernel
STATUS = {0: "OK", 1: "ERR_ARG", 2: "ERR_SHAPE", 3: "ERR_MODULUS", 4: "ERR_OVERFLOW", 5: "ERR_RANGE",
          6: "ERR_UNSUPPORTED", 7: "ERR_CUDA"}


class CtptError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


if not os.path.exists(LIB_PATH):
    raise ImportError(f"libctpt.so not built at {LIB_PATH}; run __graft_entry__.build() (no CPU fallback exists)")

_lib = ctypes.CDLL(LIB_PATH)


class Problem(ctypes.Structure):
    _fields_ = [("fmt", ctypes.c_int32), ("L", ctypes.c_int32), ("N", ctypes.c_int64), ("d1", ctypes.c_int64),
                ("d2", ctypes.c_int64), ("d3", ctypes.c_int64), ("primes", ctypes.POINTER(ctypes.c_uint32)),
                ("col_begin", ctypes.c_int64), ("col_end", ctypes.c_int64), ("kU", ctypes.c_int32),
                ("plain_per_prime", ctypes.c_int32), ("rescale", ctypes.c_int32),
                ("u_unsigned", ctypes.c_int32), ("u_offset", ctypes.c_int32), ("split_overlap", ctypes.c_int32),
                ("kernel", ctypes.c_int32), ("raster_group", ctypes.c_int32), ("max_ctas", ctypes.c_int32)]


class Sizes(ctypes.Structure):
    _fields_ = [("ctmat_bytes", ctypes.c_size_t), ("plain_bytes", ctypes.c_size_t),
                ("plain_rns_bytes", ctypes.c_size_t), ("workspace_bytes", ctypes.c_size_t),
                ("out_AU_bytes", ctypes.c_size_t), ("out_BU_bytes", ctypes.c_size_t), ("rows_A", ctypes.c_int64),
                ("R", ctypes.c_int64), ("d2p", ctypes.c_int64), ("d3_loc", ctypes.c_int64)]


_P = ctypes.c_void_p
_PP = ctypes.POINTER(Problem)
_sig = {
    "ctpt_last_error": (ctypes.c_char_p, []),
    "ctpt_version": (ctypes.c_char_p, []),
    "ctpt_query_sizes": (ctypes.c_int, [_PP, ctypes.POINTER(Sizes)]),
    "ctpt_layout": (ctypes.c_int, [_PP, _P, _P, _P, ctypes.c_int, _P]),
    "ctpt_plain_precompute": (ctypes.c_int, [_PP, _P, _P, ctypes.POINTER(ctypes.c_int32), _P]),
    "ctpt_plain_precompute_rns": (ctypes.c_int, [_PP, _P, _P, ctypes.POINTER(ctypes.c_int32), _P]),
    "ctpt_plain_precompute_unsigned": (ctypes.c_int, [_PP, _P, _P, ctypes.POINTER(ctypes.c_int32), _P]),
    "ctpt_matmul": (ctypes.c_int, [_PP, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "ctpt_split": (ctypes.c_int, [_PP, ctypes.c_int32, _P, _P, ctypes.c_size_t, _P]),
    "ctpt_gemm": (ctypes.c_int, [_PP, ctypes.c_int32, _P, ctypes.c_size_t, _P, _P, _P, _P]),
    "ctpt_gemm_simt": (ctypes.c_int, [_PP, ctypes.c_int32, _P, ctypes.c_size_t, _P, _P, _P, _P]),
    "ctpt_gemm_next": (ctypes.c_int, [_PP, ctypes.c_int32, _P, _P, ctypes.c_size_t, _P, _P, _P, _P]),
    "ctpt_gemm_fused": (ctypes.c_int, [_PP, ctypes.c_int32, _P, _P, _P, _P, _P]),
    "ctpt_gemm_mv": (ctypes.c_int, [_PP, ctypes.c_int32, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "ctpt_rescale": (ctypes.c_int, [ctypes.c_int32, _P, ctypes.c_int64, _P, _P, _P]),
    "ctpt_modmatmul_sizes": (ctypes.c_int, [ctypes.c_int32, _P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                            ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_size_t),
                                            ctypes.POINTER(ctypes.c_size_t)]),
    "ctpt_modmatmul_precompute": (ctypes.c_int, [ctypes.c_int32, _P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                                 _P, _P, _P]),
    "ctpt_modmatmul": (ctypes.c_int, [ctypes.c_int32, _P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _P,
                                      ctypes.c_int64, _P, _P, _P, ctypes.c_size_t, _P]),
    "ctpt_host_workspace_bytes": (ctypes.c_int, [_PP, ctypes.c_int64, ctypes.POINTER(ctypes.c_size_t)]),
    "ctpt_matmul_host": (ctypes.c_int, [_PP, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, ctypes.c_int64, _P]),
    "ctpt_host_workspace_bytes_units": (ctypes.c_int, [ctypes.c_int32, _PP, ctypes.c_int64,
                                                       ctypes.POINTER(ctypes.c_size_t)]),
    "ctpt_matmul_host_units": (ctypes.c_int, [ctypes.c_int32, _PP, _P, _P, _P, _P, _P, _P, ctypes.c_size_t,
                                              ctypes.c_int64, _P]),
    "ctpt_ipc_export": (ctypes.c_int, [_P, _P, ctypes.POINTER(ctypes.c_uint64)]),
    "ctpt_ipc_open": (ctypes.c_int, [_P, ctypes.c_uint64, ctypes.POINTER(_P), ctypes.POINTER(_P)]),
    "ctpt_ipc_close": (ctypes.c_int, [_P]),
    "ctpt_peer_access": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def header_symbols() -> list[str]:
    """Every function name include/ctpt.h declares."""
    txt = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"\b(ctpt_[a-z0-9_]+)\s*\(", txt)))


def _check(status: int):
    if status != 0:
        raise CtptError(status, _lib.ctpt_last_error().decode())


def version() -> str:
    return _lib.ctpt_version().decode()


def source_hash() -> str:
    """The src=<hash> the loaded library was built with (see __graft_entry__.source_hash)."""
    v = version()
    return v.split("src=", 1)[1].split()[0] if "src=" in v else "unknown"


@dataclass
class Spec:
    """A CP-MM problem (or shard): format, ring degree, dims, primes, U column block."""
    fmt: int
    N: int
    d1: int
    d2: int
    d3: int
    primes: list
    col_begin: int = 0
    col_end: int = 0
    kU: int = 1
    plain_per_prime: int = 0
    rescale: int = 0
    u_unsigned: int = 0
    u_offset: int = 0
    split_overlap: int = 0
    kernel: int = KERNEL_AUTO
    raster_group: int = 0
    max_ctas: int = 0

    def cstruct(self) -> Problem:
        arr = (ctypes.c_uint32 * len(self.primes))(*[int(p) for p in self.primes])
        pb = Problem(self.fmt, len(self.primes), self.N, self.d1, self.d2, self.d3, arr, self.col_begin,
                     self.col_end, self.kU, self.plain_per_prime, self.rescale, self.u_unsigned,
                     self.u_offset, self.split_overlap, self.kernel, self.raster_group, self.max_ctas)
        pb._keep = arr  # keep the host prime array alive with the struct
        return pb


def _ptr(t) -> ctypes.c_void_p:
    if t is None:
        return ctypes.c_void_p(0)
    if isinstance(t, int):
        return ctypes.c_void_p(t)
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream) -> ctypes.c_void_p:
    if stream is None:
        import torch

        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def query_sizes(spec: Spec) -> Sizes:
    s = Sizes()
    pb = spec.cstruct()
    _check(_lib.ctpt_query_sizes(ctypes.byref(pb), ctypes.byref(s)))
    return s


def layout(spec: Spec, a_polys, b_polys, ctmat, validate: bool = False, stream=None):
    pb = spec.cstruct()
    _check(_lib.ctpt_layout(ctypes.byref(pb), _ptr(a_polys), _ptr(b_polys), _ptr(ctmat), int(validate),
                            _stream(stream)))


def plain_precompute(spec: Spec, U, plain, stream=None) -> int:
    pb = spec.cstruct()
    kU = ctypes.c_int32(0)
    _check(_lib.ctpt_plain_precompute(ctypes.byref(pb), _ptr(U), _ptr(plain), ctypes.byref(kU), _stream(stream)))
    return kU.value


def plain_precompute_unsigned(spec: Spec, U, plain, stream=None) -> int:
    """One u8 plane U + u_offset (returns u_offset); raises CtptError(ERR_RANGE) when U spans > 255."""
    pb = spec.cstruct()
    off = ctypes.c_int32(0)
    _check(_lib.ctpt_plain_precompute_unsigned(ctypes.byref(pb), _ptr(U), _ptr(plain), ctypes.byref(off),
                                               _stream(stream)))
    return off.value


def plain_precompute_rns(spec: Spec, Ures, plain, stream=None) -> int:
    pb = spec.cstruct()
    kU = ctypes.c_int32(0)
    _check(_lib.ctpt_plain_precompute_rns(ctypes.byref(pb), _ptr(Ures), _ptr(plain), ctypes.byref(kU),
                                          _stream(stream)))
    return kU.value


def matmul(spec: Spec, ctmat, plain, AU, BU, ws, stream=None):
    pb = spec.cstruct()
    nbytes = ws.numel() * ws.element_size()
    _check(_lib.ctpt_matmul(ctypes.byref(pb), _ptr(ctmat), _ptr(plain), _ptr(AU), _ptr(BU), _ptr(ws), nbytes,
                            _stream(stream)))


def split(spec: Spec, l: int, ctmat, ws, stream=None):
    pb = spec.cstruct()
    _check(_lib.ctpt_split(ctypes.byref(pb), l, _ptr(ctmat), _ptr(ws), ws.numel() * ws.element_size(),
                           _stream(stream)))


def gemm(spec: Spec, l: int, ws, plain, AU_l, BU_l, stream=None, simt: bool = False):
    pb = spec.cstruct()
    f = _lib.ctpt_gemm_simt if simt else _lib.ctpt_gemm
    _check(f(ctypes.byref(pb), l, _ptr(ws), ws.numel() * ws.element_size(), _ptr(plain), _ptr(AU_l), _ptr(BU_l),
             _stream(stream)))


def gemm_next(spec: Spec, l: int, ctmat, ws, plain, AU_l, BU_l, stream=None):
    """ctpt_gemm of prime l with prime l+1's limb split inside the same kernel (spec.split_overlap = 1)."""
    pb = spec.cstruct()
    _check(_lib.ctpt_gemm_next(ctypes.byref(pb), l, _ptr(ctmat), _ptr(ws), ws.numel() * ws.element_size(), _ptr(plain),
                               _ptr(AU_l), _ptr(BU_l), _stream(stream)))


def gemm_fused(spec: Spec, l: int, ctmat, plain, AU_l, BU_l, stream=None):
    """Skinny-U kernel (d3_loc <= 256, kU = 1): split fused into the GEMM's load path."""
    pb = spec.cstruct()
    _check(_lib.ctpt_gemm_fused(ctypes.byref(pb), l, _ptr(ctmat), _ptr(plain), _ptr(AU_l), _ptr(BU_l),
                                _stream(stream)))


def gemm_mv(spec: Spec, l: int, ctmat, plain, AU_l, BU_l, ws, stream=None):
    """Very-skinny kernel (d3_loc <= 32, kU = 1): raw residue bytes against an expanded U."""
    pb = spec.cstruct()
    _check(_lib.ctpt_gemm_mv(ctypes.byref(pb), l, _ptr(ctmat), _ptr(plain), _ptr(AU_l), _ptr(BU_l), _ptr(ws),
                             ws.numel() * ws.element_size(), _stream(stream)))


def _primes_arr(primes):
    return (ctypes.c_uint32 * len(primes))(*[int(p) for p in primes])


def rescale(primes, n: int, x_in, x_out, stream=None):
    """x_out [L-1][n] = round(x / primes[-1]) mod primes[l] for x_in [L][n] residues (device tensors)."""
    arr = _primes_arr(primes)
    _check(_lib.ctpt_rescale(len(primes), ctypes.cast(arr, _P), n, _ptr(x_in), _ptr(x_out), _stream(stream)))


def modmatmul_sizes(primes, M: int, K: int, Nc: int):
    """(ldx, plain_bytes, ws_bytes) for Mod-PP-MM_{M,K,Nc} over `primes`."""
    arr = _primes_arr(primes)
    ldx, pb_, ws = ctypes.c_int64(0), ctypes.c_size_t(0), ctypes.c_size_t(0)
    _check(_lib.ctpt_modmatmul_sizes(len(primes), ctypes.cast(arr, _P), M, K, Nc, ctypes.byref(ldx),
                                     ctypes.byref(pb_), ctypes.byref(ws)))
    return ldx.value, pb_.value, ws.value


def modmatmul_precompute(primes, M: int, K: int, Nc: int, Y, plain, stream=None):
    arr = _primes_arr(primes)
    _check(_lib.ctpt_modmatmul_precompute(len(primes), ctypes.cast(arr, _P), M, K, Nc, _ptr(Y), _ptr(plain),
                                          _stream(stream)))


def modmatmul(primes, M: int, K: int, Nc: int, X, ldx: int, plain, ZT, ws, stream=None):
    """Z^T = (X·Y mod p)^T per prime: X [L][M][ldx], Z^T [L][Nc][M] device tensors."""
    arr = _primes_arr(primes)
    _check(_lib.ctpt_modmatmul(len(primes), ctypes.cast(arr, _P), M, K, Nc, _ptr(X), ldx, _ptr(plain), _ptr(ZT),
                               _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))


def host_workspace_bytes(spec: Spec, chunk_rows: int = 0) -> int:
    pb = spec.cstruct()
    n = ctypes.c_size_t(0)
    _check(_lib.ctpt_host_workspace_bytes(ctypes.byref(pb), chunk_rows, ctypes.byref(n)))
    return n.value


def matmul_host(spec: Spec, a_polys_h, b_polys_h, plain, AU_h, BU_h, ws, chunk_rows: int = 0, stream=None):
    """a_polys_h / b_polys_h / AU_h / BU_h: pinned host tensors (or raw host addresses)."""
    pb = spec.cstruct()
    _check(_lib.ctpt_matmul_host(ctypes.byref(pb), _ptr(a_polys_h), _ptr(b_polys_h), _ptr(plain), _ptr(AU_h),
                                 _ptr(BU_h), _ptr(ws), ws.numel() * ws.element_size(), chunk_rows, _stream(stream)))


def _problems(specs) -> ctypes.Array:
    """A C array of ctpt_problem (the prime arrays kept alive on the array object)."""
    structs = [sp.cstruct() for sp in specs]
    arr = (Problem * len(structs))(*structs)
    arr._keep = [pb._keep for pb in structs]
    return arr


def _ptrs(ts) -> ctypes.Array:
    return (ctypes.c_void_p * len(ts))(*[_ptr(t).value for t in ts])


def host_workspace_bytes_units(specs, chunk_rows: int = 0) -> int:
    arr = _problems(specs)
    n = ctypes.c_size_t(0)
    _check(_lib.ctpt_host_workspace_bytes_units(len(specs), ctypes.cast(arr, _PP), chunk_rows, ctypes.byref(n)))
    return n.value


def matmul_host_units(specs, a_polys_h, b_polys_h, plains, AU_h, BU_h, ws, chunk_rows: int = 0, stream=None):
    """ctpt_matmul_host_units: unit u = (specs[u], a_polys_h[u], b_polys_h[u], plains[u], AU_h[u], BU_h[u]),
    all units in one copy / compute pipeline (host tensors pinned)."""
    arr = _problems(specs)
    lists = [_ptrs(x) for x in (a_polys_h, b_polys_h, plains, AU_h, BU_h)]
    _check(_lib.ctpt_matmul_host_units(len(specs), ctypes.cast(arr, _PP), *[ctypes.cast(x, _P) for x in lists],
                                       _ptr(ws), ws.numel() * ws.element_size(), chunk_rows, _stream(stream)))


IPC_HANDLE_BYTES = 64  # CTPT_IPC_HANDLE_BYTES


def ipc_export(t) -> tuple[bytes, int]:
    """(handle bytes, byte offset) of device tensor / address t's allocation (ctpt_ipc_export)."""
    h = (ctypes.c_char * IPC_HANDLE_BYTES)()
    off = ctypes.c_uint64(0)
    _check(_lib.ctpt_ipc_export(_ptr(t), ctypes.cast(h, _P), ctypes.byref(off)))
    return bytes(h.raw), off.value


def ipc_open(handle: bytes, offset: int) -> tuple[int, int]:
    """Map another process's allocation into the CURRENT device (peer access enabled as needed);
    returns (base, address) — base for ipc_close, address = base + offset."""
    h = (ctypes.c_char * IPC_HANDLE_BYTES).from_buffer_copy(handle)
    base, ptr = _P(), _P()
    _check(_lib.ctpt_ipc_open(ctypes.cast(h, _P), offset, ctypes.byref(base), ctypes.byref(ptr)))
    return base.value, ptr.value


def ipc_close(base: int):
    _check(_lib.ctpt_ipc_close(_P(base)))


def peer_access(device: int, peer: int) -> bool:
    can = ctypes.c_int32(0)
    _check(_lib.ctpt_peer_access(device, peer, ctypes.byref(can)))
    return bool(can.value)


def raw_lib():
    return _lib
