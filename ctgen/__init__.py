"""Seeded synthetic-input generator (its own module; see ctgen.c's header).

Serves both the CUDA product path (bench.py) and the CPU oracle (tests/).  It
holds none of the method's arithmetic: it only draws random numbers and builds
the RLWE ciphertexts that are the INPUT of Algorithm 6.
The recipe (primes, samplers, streams) is documented in DESIGN.md §Inputs.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libctgen.so")

RLWE, SHARED_S, SHARED_A, STRUCT_A = 0, 1, 2, 3
FORMAT_NAMES = {RLWE: "rlwe", SHARED_S: "shared-s", SHARED_A: "shared-a", STRUCT_A: "struct-a shared-a"}


def n_a_polys(fmt: int, N: int, d1: int, ncols: int) -> int:
    """Number of a-polynomials a format stores for `ncols` columns: one per (column, chunk) for
    shared-s, one per column for RLWE / shared-a, one per ROW BLOCK (d1/N, independent of the
    columns) for structured-A shared-a."""
    k = d1 // N
    if fmt == SHARED_S:
        return ncols * k
    if fmt == STRUCT_A:
        return k
    return ncols


def rows_A_of(fmt: int, N: int, d1: int) -> int:
    """Rows of the matrix A the CP-MM multiplies: d1 (shared-s), N (RLWE, shared-a), 0 for
    structured-A shared-a, whose Ã is not multiplied (Algorithm 7 step 1)."""
    return d1 if fmt == SHARED_S else (0 if fmt == STRUCT_A else N)

_lib = None


def build(force: bool = False) -> str:
    import subprocess

    src = os.path.join(_HERE, "ctgen.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(
            ["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC", "-std=c11",
             "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        u64, i64, u32, i32 = ctypes.c_uint64, ctypes.c_int64, ctypes.c_uint32, ctypes.c_int32
        P = ctypes.c_void_p
        L.ctgen_draw64.restype = u64
        L.ctgen_draw64.argtypes = [u64, u64, u64]
        L.ctgen_primes.restype = ctypes.c_int
        L.ctgen_primes.argtypes = [ctypes.c_int, P]
        L.ctgen_is_prime.restype = ctypes.c_int
        L.ctgen_is_prime.argtypes = [u64]
        L.ctgen_err.restype = i32
        L.ctgen_err.argtypes = [u64, u64, u64]
        L.ctgen_sk_coeff.restype = i32
        L.ctgen_sk_coeff.argtypes = [u64, u64, u64]
        L.ctgen_sk.restype = None
        L.ctgen_sk.argtypes = [u64, u64, i64, P]
        L.ctgen_a_coeff.restype = u32
        L.ctgen_a_coeff.argtypes = [u64, u32, u64, u64]
        L.ctgen_msg.restype = ctypes.c_double
        L.ctgen_msg.argtypes = [u64, i64, i64, i64]
        L.ctgen_encoded.restype = i64
        L.ctgen_encoded.argtypes = [u64, i64, i64, i64, ctypes.c_int]
        L.ctgen_plain.restype = i64
        L.ctgen_plain.argtypes = [u64, i64, i64, i64, i64, ctypes.c_int]
        L.ctgen_u.restype = i64
        L.ctgen_u.argtypes = [u64, i64, i64, i64, i64]
        L.ctgen_U.restype = None
        L.ctgen_U.argtypes = [u64, i64, i64, i64, P, ctypes.c_int]
        L.ctgen_U_real.restype = None
        L.ctgen_U_real.argtypes = [u64, i64, i64, u64, P, P, ctypes.c_int]
        L.ctgen_u_real.restype = ctypes.c_double
        L.ctgen_u_real.argtypes = [u64, i64, i64, i64]
        L.ctgen_uniform.restype = u64
        L.ctgen_uniform.argtypes = [u64, u64, u64, u64]
        L.ctgen_negacyclic_ntt.restype = ctypes.c_int
        L.ctgen_negacyclic_ntt.argtypes = [P, P, i64, u32, P]
        L.ctgen_encrypt.restype = ctypes.c_int
        L.ctgen_encrypt.argtypes = [ctypes.c_int, i64, i64, i64, u64, ctypes.c_int, ctypes.c_int, P,
                                    i64, i64, P, P, ctypes.c_int]
        L.ctgen_msg_block.restype = None
        L.ctgen_msg_block.argtypes = [u64, i64, i64, i64, i64, i64, P, ctypes.c_int]
        L.ctgen_plain_block.restype = None
        L.ctgen_plain_block.argtypes = [u64, i64, i64, ctypes.c_int, i64, i64, i64, i64, P, ctypes.c_int]
        L.ctgen_uniform_residues.restype = None
        L.ctgen_uniform_residues.argtypes = [u64, u32, i64, P, ctypes.c_int]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return ctypes.c_void_p(a.ctypes.data)


def primes(L: int) -> list[int]:
    """The L largest primes p < 2^31 with p ≡ 1 (mod 2^16), descending (reading Q5)."""
    out = np.zeros(L, dtype=np.uint32)
    n = lib().ctgen_primes(L, _ptr(out))
    assert n == L
    return [int(x) for x in out]


def draw64(seed: int, tag: int, idx: int) -> int:
    return int(lib().ctgen_draw64(seed, tag, idx))


def sk(seed: int, t: int, N: int) -> np.ndarray:
    out = np.zeros(N, dtype=np.int8)
    lib().ctgen_sk(seed, t, N, _ptr(out))
    return out


def err(seed: int, poly: int, coeffs) -> np.ndarray:
    L = lib()
    return np.array([L.ctgen_err(seed, poly, int(c)) for c in coeffs], dtype=np.int64)


def msg(seed: int, d1: int, i: int, j: int) -> float:
    return float(lib().ctgen_msg(seed, d1, i, j))


def msg_matrix(seed: int, d1: int, rows, cols) -> np.ndarray:
    """M[i][j] for i in rows, j in cols (float64; small sizes)."""
    L = lib()
    return np.array([[L.ctgen_msg(seed, d1, int(i), int(j)) for j in cols] for i in rows], dtype=np.float64)


def err_matrix(seed: int, N: int, d1: int, rows, cols) -> np.ndarray:
    """E[i][j]: the encryption error added to entry (i, j): b-poly j*k + i//N, coefficient i%N."""
    L = lib()
    k = d1 // N
    return np.array([[L.ctgen_err(seed, int(j) * k + int(i) // N, int(i) % N) for j in cols] for i in rows],
                    dtype=np.int64)


def plain_matrix(seed: int, N: int, d1: int, rows, cols, log_delta: int) -> np.ndarray:
    """P[i][j] = ⌊Δ M_ij⌉ + E_ij as exact int64 (generator's own integer encoder)."""
    L = lib()
    return np.array([[L.ctgen_plain(seed, N, d1, int(i), int(j), log_delta) for j in cols] for i in rows],
                    dtype=np.int64)


def msg_block(seed: int, d1: int, r0: int, nrows: int, c0: int, ncols: int, nthreads: int = 0) -> np.ndarray:
    out = np.empty((nrows, ncols), dtype=np.float64)
    lib().ctgen_msg_block(seed, d1, r0, nrows, c0, ncols, _ptr(out), nthreads)
    return out


def plain_block(seed: int, N: int, d1: int, log_delta: int, r0: int, nrows: int, c0: int, ncols: int,
                nthreads: int = 0) -> np.ndarray:
    out = np.empty((nrows, ncols), dtype=np.int64)
    lib().ctgen_plain_block(seed, N, d1, log_delta, r0, nrows, c0, ncols, _ptr(out), nthreads)
    return out


def U_matrix(seed: int, d2: int, d3: int, bound: int, nthreads: int = 0) -> np.ndarray:
    """U ∈ Z^{d2×d3}, uniform integers in {-bound..bound} (reading Q11), row-major int64."""
    out = np.empty((d2, d3), dtype=np.int64)
    lib().ctgen_U(seed, d2, d3, bound, _ptr(out), nthreads)
    return out


def U_real(seed: int, d2: int, d3: int, scale: int, nthreads: int = 0):
    """Real U ∈ [-1,1)^{d2×d3} (53-bit grid) and its encoding U0 = ⌊scale·U⌉ (Alg. 6 REQUIRE,
    P:1697) as exact int64 — the input of the Rescale workloads (scale = Δ_U)."""
    real = np.empty((d2, d3), dtype=np.float64)
    enc = np.empty((d2, d3), dtype=np.int64)
    lib().ctgen_U_real(seed, d2, d3, int(scale), _ptr(real), _ptr(enc), nthreads)
    return real, enc


def u_real(seed: int, d3: int, k: int, j: int) -> float:
    return lib().ctgen_u_real(seed, d3, k, j)


def uniform(seed: int, stream: int, n: int, mod: int) -> np.ndarray:
    L = lib()
    return np.array([L.ctgen_uniform(seed, stream, i, mod) for i in range(n)], dtype=np.uint64)


def negacyclic_ntt(a: np.ndarray, s: np.ndarray, p: int) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint32)
    s = np.ascontiguousarray(s, dtype=np.int8)
    out = np.zeros_like(a)
    rc = lib().ctgen_negacyclic_ntt(_ptr(a), _ptr(s), a.shape[0], p, _ptr(out))
    assert rc == 0, rc
    return out


@dataclass
class Ciphertexts:
    """Per-column ciphertexts of a structured-S matrix encryption."""

    fmt: int
    N: int
    d1: int
    d2: int
    primes: list
    col_begin: int
    col_end: int
    a_polys: np.ndarray  # uint32 [L][n_a][N]
    b_polys: np.ndarray  # uint32 [L][ncols*k][N]

    @property
    def k(self) -> int:
        return self.d1 // self.N

    @property
    def rows_A(self) -> int:
        return rows_A_of(self.fmt, self.N, self.d1)


def encrypt(fmt: int, N: int, d1: int, d2: int, seed: int, log_delta: int, prime_list, col_begin: int = 0,
            col_end: int | None = None, nthreads: int = 0, out_a: np.ndarray | None = None,
            out_b: np.ndarray | None = None) -> Ciphertexts:
    """Encrypt columns [col_begin, col_end) of the seeded M in format `fmt` under each prime."""
    if col_end is None:
        col_end = d2
    k = d1 // N
    ncols = col_end - col_begin
    L = len(prime_list)
    n_a = n_a_polys(fmt, N, d1, ncols)
    a = out_a if out_a is not None else np.empty((L, n_a, N), dtype=np.uint32)
    b = out_b if out_b is not None else np.empty((L, ncols * k, N), dtype=np.uint32)
    assert a.dtype == np.uint32 and a.size == L * n_a * N and a.flags["C_CONTIGUOUS"]
    assert b.dtype == np.uint32 and b.size == L * ncols * k * N and b.flags["C_CONTIGUOUS"]
    pr = np.array(prime_list, dtype=np.uint32)
    rc = lib().ctgen_encrypt(fmt, N, d1, d2, seed, log_delta, L, _ptr(pr), col_begin, col_end, _ptr(a), _ptr(b),
                             nthreads)
    if rc != 0:
        raise ValueError(f"ctgen_encrypt failed: {rc}")
    return Ciphertexts(fmt, N, d1, d2, list(prime_list), col_begin, col_end, a, b)


def uniform_residues(seed: int, p: int, n: int, nthreads: int = 0, out: np.ndarray | None = None) -> np.ndarray:
    o = out if out is not None else np.empty(n, dtype=np.uint32)
    lib().ctgen_uniform_residues(seed, p, n, _ptr(o), nthreads)
    return o


# --------------------------------------------------------------------------------------
# The five BASELINE.json configurations, made concrete
# --------------------------------------------------------------------------------------
@dataclass(frozen=True)
class Config:
    name: str
    fmt: int
    N: int
    d1: int
    d2: int
    d3: int
    L: int
    log_delta: int
    u_bound: int
    seed: int = 0

    @property
    def k(self) -> int:
        return self.d1 // self.N

    @property
    def rows_A(self) -> int:
        return rows_A_of(self.fmt, self.N, self.d1)

    @property
    def R(self) -> int:
        return self.rows_A + self.d1

    @property
    def residue_macs(self) -> int:
        return self.L * self.R * self.d2 * self.d3


CONFIGS = {
    "c1": Config("c1", RLWE, 64, 64, 64, 64, 1, 20, 4),
    "c2": Config("c2", RLWE, 4096, 4096, 4096, 4096, 2, 40, 8),
    "c3": Config("c3", SHARED_A, 4096, 16384, 16384, 16384, 3, 45, 8),
    "c4": Config("c4", SHARED_S, 8192, 32768, 32768, 4096, 4, 50, 8),
    "c5": Config("c5", SHARED_S, 16384, 32768, 32768, 32768, 8, 60, 8),
    # Algorithm 7 (CP-MM with precomputation) on c3's shapes in the
    # structured-A shared-a format — only B·U is computed (R = d1 = 16384 instead of 20480).
    "c3a": Config("c3a", STRUCT_A, 4096, 16384, 16384, 16384, 3, 45, 8),
}
