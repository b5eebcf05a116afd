"""Shared helpers for the -m gpu parity tests: generate seeded inputs (ctgen), run the
CUDA path through the C ABI, and compute the oracle's answer on the same inputs."""
from __future__ import annotations

import os

import numpy as np

import ctgen
import oracle

NTHREADS = os.cpu_count() or 8


def run_gpu(fmt, N, d1, d2, d3, primes, a_polys, b_polys, U=None, Ures=None, col_begin=0, col_end=0, simt=False,
            validate=True, rescale=0, unsigned="auto", split_overlap=0, kernel=0, raster_group=0, max_ctas=0):
    import torch

    from paper_2503_16080_b200 import ctpt
    from paper_2503_16080_b200.engine import CpmmEngine

    eng = CpmmEngine(ctpt.Spec(fmt, N, d1, d2, d3, list(primes), col_begin, col_end, rescale=rescale,
                               split_overlap=split_overlap, kernel=kernel, raster_group=raster_group,
                               max_ctas=max_ctas), "cuda")
    eng.layout(a_polys, b_polys, validate=validate)
    if Ures is not None:
        eng.precompute_rns(Ures)
    else:
        eng.precompute(U, unsigned=unsigned)
    if simt:
        AU, BU = eng.alloc_outputs()
        L = len(primes)
        d3l, ra = eng.sizes.d3_loc, eng.sizes.rows_A
        for l in range(L):
            ctpt.split(eng.spec, l, eng.ctmat, eng.ws)
            ctpt.gemm(eng.spec, l, eng.ws, eng.plain, AU[l * d3l * ra:], BU[l * d3l * d1:], simt=True)
    else:
        AU, BU = eng.matmul()
    torch.cuda.synchronize()
    return eng.outputs_numpy(AU, BU), eng


def oracle_outputs(fmt, N, d1, a_polys_l, b_polys_l, U, p, cols=None):
    """(A·U mod p, B·U mod p) per output column [ncols][rows] by the schoolbook oracle."""
    d2 = U.shape[0]
    if N * d2 <= 1 << 16:
        A, B = oracle.format_matrices(fmt, N, d1, a_polys_l, b_polys_l)
        Ac, Bc = np.ascontiguousarray(A.T), np.ascontiguousarray(B.T)
    else:  # the same matrices without the copy (test_gpu_parity checks the equivalence)
        Ac, Bc = colmajor_views(fmt, N, d1, d2, a_polys_l, b_polys_l)
    AU = oracle.modmatmul(Ac, U, p, cols=cols, nthreads=NTHREADS)
    BU = oracle.modmatmul(Bc, U, p, cols=cols, nthreads=NTHREADS)
    return AU, BU


def colmajor_views(fmt, N, d1, d2, a_polys_l, b_polys_l):
    """Column-major A [d2][rows_A] and B [d2][d1] views of one prime's per-column ciphertexts
    (no copy: poly j*k+t of column j is contiguous)."""
    ra = oracle.rows_A(fmt, N, d1)
    A = np.empty((d2, 0), np.uint32) if ra == 0 else a_polys_l.reshape(d2, ra)  # structured-A: no A·U
    return A, b_polys_l.reshape(d2, d1)


def U_residues(U: np.ndarray, primes) -> np.ndarray:
    return np.stack([(U % int(p)).astype(np.uint32) for p in primes])
