#!/usr/bin/env python
"""Small cases of every kernel path, each checked against the oracle, for checked builds.

compute-sanitizer is closed on this GPU pool (runs under it left GPUs needing a reset), so the
substitute is (a) a debug build of the library with device-side bounds / invariant checks that
trap with the failing site, and mbarrier waits that trap with the barrier after 4 s instead of
hanging (`python tools/ab_build.py /tmp/dbg.so -DCTPT_DEBUG_CHECKS`, loaded with CTPT_LIB), and
(b) stress repetitions that change the schedule (grid caps 1 … 148 CTAs, so each CTA loops over a
different number of tiles and the rings wrap at different points) and compare every output with
the oracle each time — a race that corrupts data shows up as a mismatch.

    CTPT_LIB=/tmp/dbg.so python tools/sanitize_cases.py [--cases a,b,...] [--stress 5]

Cases (kept small: the sanitizers slow kernels down 10–100×):
  gemm          limb split + k_gemm_tc, 3 primes, ragged R / d2 / d3 (several tiles, 2 raster groups)
  gemm_side     the same with split_overlap = 1 (prime l+1 split by warps 2–3 inside GEMM l)
  gemm_u8       the unsigned-U plane (row-sum correction in the epilogue), k_U = 2 (accumulating passes)
  fused_wrap    the skinny kernel k_gemm_fused_t with long K (65 k-blocks: the rings wrap many times),
                64-row tiles with 4 / 3 / 2 limb stages (d3 ≤ 128 / 160 / 192), 2 half-K-block stages
                (≤ 224) and 32-row tiles (≤ 256), the u8 plane's in-kernel row sums, and one CTA
                looping over 4–8 tiles
  mv_tickets    k_gemm_mv with the K loop split into units that meet on an atomic ticket
  layout        k_layout_v4 (16-byte) and k_layout (4-byte) with validate = 1
  host          ctpt_matmul_host (three streams, double-buffered staging), split + GEMM and fused chunks
  rescale       ctpt_matmul with the fused RNS Rescale epilogue
  ipc           two processes on one GPU: rank 1's GEMM epilogues store into rank 0's buffer through
                a CUDA IPC mapping (tests/test_gpu_fused_gather.py's path)
Prints one line per case; exits 1 on any mismatch.
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import ctgen  # noqa: E402
from gpu_helpers import oracle_outputs, run_gpu  # noqa: E402

R, S, A = ctgen.RLWE, ctgen.SHARED_S, ctgen.SHARED_A


STRESS = [0]  # grid caps cycled through by --stress


def check(name, fmt, N, k, d2, d3, L, seed=0, u_bound=8, **kw):
    bad = 0
    for i, cap in enumerate(STRESS):
        kw2 = dict(kw)
        if cap and "max_ctas" not in kw:
            kw2["max_ctas"] = cap
        bad += _check1(name, fmt, N, k, d2, d3, L, seed + i, u_bound, **kw2)
    return bad


def _check1(name, fmt, N, k, d2, d3, L, seed=0, u_bound=8, **kw):
    d1 = N * k
    ps = ctgen.primes(L)
    ct = ctgen.encrypt(fmt, N, d1, d2, seed, 20, ps)
    U = ctgen.U_matrix(seed, d2, d3, u_bound)
    (AU, BU), eng = run_gpu(fmt, N, d1, d2, d3, ps, ct.a_polys, ct.b_polys, U=U, **kw)
    bad = 0
    for l, p in enumerate(ps):
        wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[l], ct.b_polys[l], U, p)
        bad += int(np.count_nonzero(AU[l] != wa)) + int(np.count_nonzero(BU[l] != wb))
    print(f"{name}: fmt={fmt} N={N} k={k} d2={d2} d3={d3} L={L} kU={eng.spec.kU} u8={eng.spec.u_unsigned} "
          f"max_ctas={kw.get('max_ctas', 0)} mismatches={bad}", flush=True)
    return bad


def case_host():
    import torch

    from paper_2503_16080_b200 import ctpt
    from paper_2503_16080_b200.engine import CpmmEngine

    bad = 0
    for fmt, N, k, d2, d3, L in [(A, 64, 3, 300, 300, 2), (S, 32, 4, 200, 100, 1)]:
        d1 = N * k
        ps = ctgen.primes(L)
        ct = ctgen.encrypt(fmt, N, d1, d2, 4, 20, ps)
        U = ctgen.U_matrix(4, d2, d3, 8)
        eng = CpmmEngine(ctpt.Spec(fmt, N, d1, d2, d3, ps), "cuda")
        eng.precompute(U)
        a_h = torch.from_numpy(ct.a_polys.view(np.int32)).pin_memory()
        b_h = torch.from_numpy(ct.b_polys.view(np.int32)).pin_memory()
        AU = torch.empty(eng.sizes.out_AU_bytes // 4, dtype=torch.int32).pin_memory()
        BU = torch.empty(eng.sizes.out_BU_bytes // 4, dtype=torch.int32).pin_memory()
        chunk = 64
        ws = torch.empty(ctpt.host_workspace_bytes(eng.spec, chunk), dtype=torch.uint8, device="cuda")
        ctpt.matmul_host(eng.spec, a_h, b_h, eng.plain, AU, BU, ws, chunk_rows=chunk)
        torch.cuda.synchronize()
        AUn = AU.numpy().view(np.uint32).reshape(L, d3, -1)
        BUn = BU.numpy().view(np.uint32).reshape(L, d3, d1)
        for l, p in enumerate(ps):
            wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[l], ct.b_polys[l], U, p)
            bad += int(np.count_nonzero(AUn[l] != wa)) + int(np.count_nonzero(BUn[l] != wb))
        print(f"host: fmt={fmt} d3={d3} chunk_rows={chunk} mismatches={bad}", flush=True)
    return bad


def case_rescale():
    import oracle
    from paper_2503_16080_b200 import ctpt  # noqa: F401

    fmt, N, k, d2, d3, L = S, 32, 2, 150, 300, 3
    d1 = N * k
    ps = ctgen.primes(L)
    ct = ctgen.encrypt(fmt, N, d1, d2, 8, 20, ps)
    rng = np.random.default_rng(8)
    U0 = rng.integers(-(1 << 20), 1 << 20, (d2, d3)).astype(np.int64)
    Ures = np.stack([(U0 % int(p)).astype(np.uint32) for p in ps])
    (AU, BU), _ = run_gpu(fmt, N, d1, d2, d3, ps, ct.a_polys, ct.b_polys, Ures=Ures, rescale=1)
    prods = []
    for l, p in enumerate(ps):
        wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[l], ct.b_polys[l], U0, p)
        prods.append(np.concatenate([wa, wb], axis=1))
    want = oracle.rescale_last(np.stack(prods).reshape(L, -1), ps).reshape(L - 1, d3, -1)
    got = np.concatenate([AU, BU], axis=2)
    bad = int(np.count_nonzero(got != want))
    print(f"rescale: mismatches={bad}", flush=True)
    return bad


def case_layout():
    import torch

    import oracle
    from paper_2503_16080_b200 import ctpt
    from paper_2503_16080_b200.engine import CpmmEngine

    bad = 0
    for fmt, N, k, d2, L in [(A, 256, 2, 130, 2), (R, 2, 1, 70, 2)]:  # 16-byte kernel; 4-byte kernel
        d1 = N * k
        ps = ctgen.primes(L)
        ct = ctgen.encrypt(fmt, N, d1, d2, 3, 20, ps)
        eng = CpmmEngine(ctpt.Spec(fmt, N, d1, d2, 4, ps), "cuda")
        eng.layout(ct.a_polys, ct.b_polys, validate=True)
        torch.cuda.synchronize()
        got = eng.ctmat[256:].cpu().numpy().view(np.uint32).reshape(L, eng.sizes.R, eng.sizes.d2p)
        for l in range(L):
            Am, Bm = oracle.format_matrices(fmt, N, d1, ct.a_polys[l], ct.b_polys[l])
            bad += int(np.count_nonzero(got[l, :Am.shape[0], :d2] != Am))
            bad += int(np.count_nonzero(got[l, Am.shape[0]:, :d2] != Bm))
        print(f"layout: fmt={fmt} N={N} mismatches={bad}", flush=True)
    return bad


def case_ipc():
    import tempfile

    import pytest

    import test_gpu_fused_gather as t

    with tempfile.TemporaryDirectory() as d:
        from pathlib import Path

        cfg = (2, 64, 2, 300, 600, 3)
        t.test_fused_gather_two_processes_one_gpu(cfg, Path(d))
    print("ipc: two processes, rank 1 stores into rank 0's buffer through ctpt_ipc_open: ok", flush=True)
    del pytest
    return 0


CASES = {
    "gemm": lambda: check("gemm", A, 64, 3, 300, 300, 3, kernel=1, unsigned="never", raster_group=2),
    "gemm_side": lambda: check("gemm_side", S, 32, 4, 200, 260, 3, kernel=1, split_overlap=1),
    "gemm_u8": lambda: check("gemm_u8", R, 256, 1, 200, 140, 2, u_bound=300, kernel=1) +
                       check("gemm_u8", A, 64, 2, 129, 300, 1, kernel=1, unsigned="always"),
    "fused_wrap": lambda: check("fused_wrap", A, 64, 2, 8200, 100, 1, kernel=2) +
                          check("fused_wrap", S, 32, 3, 8200, 200, 1, kernel=2) +
                          check("fused_wrap", A, 64, 2, 8200, 150, 1, kernel=2) +
                          check("fused_wrap", S, 32, 3, 8200, 190, 1, kernel=2) +
                          check("fused_wrap", A, 64, 2, 8200, 250, 1, kernel=2) +
                          check("fused_multi", S, 32, 4, 520, 100, 1, kernel=2, max_ctas=1) +
                          check("fused_multi", S, 32, 4, 520, 200, 1, kernel=2, max_ctas=1) +
                          check("fused_multi", S, 32, 4, 520, 180, 1, kernel=2, max_ctas=1) +
                          check("fused_u8", S, 32, 4, 520, 100, 1, kernel=2, unsigned="always", max_ctas=1) +
                          check("fused_u8", A, 64, 2, 8200, 200, 1, kernel=2, unsigned="always"),
    "mv_tickets": lambda: check("mv_tickets", S, 512, 2, 8200, 3, 1, kernel=3) +
                          check("mv_tickets", A, 64, 3, 4112, 20, 2, kernel=3),
    "layout": case_layout,
    "host": case_host,
    "rescale": case_rescale,
    "ipc": case_ipc,
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default=",".join(CASES))
    ap.add_argument("--stress", type=int, default=1, help="repetitions per case with grid caps 0, 1, 3, 7, 37, ...")
    args = ap.parse_args()
    caps = [0, 1, 3, 7, 37, 148, 2, 5, 19, 64]
    STRESS[:] = [caps[i % len(caps)] for i in range(max(1, args.stress))]
    bad = 0
    for name in args.cases.split(","):
        bad += CASES[name]()
    print("ALL OK" if bad == 0 else f"MISMATCHES: {bad}", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
