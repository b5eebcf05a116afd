#!/usr/bin/env python
"""Probe: can the kernels move the e2e data over PCIe themselves (zero-copy), instead of DMA
copies + staging?  c3's ciphertexts in pinned host memory:

  1. ctpt_layout reading the per-column ciphertexts straight from pinned host memory (UVA) and
     writing the laid-out X in HBM — a fused "H2D + layout";
  2. ctpt_matmul whose epilogues store the output residues straight into pinned host memory — a
     fused "GEMM + D2H";
  3. the DMA baselines (cudaMemcpy of the same bytes, each direction).

Prints one JSON line per measurement (GB/s over the PCIe-crossing bytes).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps=3):
    import torch

    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best


def main():
    import torch

    import ctgen
    from paper_2503_16080_b200 import ctpt
    from paper_2503_16080_b200.engine import CpmmEngine

    c = ctgen.CONFIGS["c3"]
    ps = ctgen.primes(c.L)
    cores = os.cpu_count() or 1
    ct = ctgen.encrypt(c.fmt, c.N, c.d1, c.d2, c.seed, c.log_delta, ps, nthreads=cores)
    U = ctgen.U_matrix(c.seed, c.d2, c.d3, c.u_bound, nthreads=cores)
    a_h = torch.from_numpy(ct.a_polys.view(np.int32)).pin_memory()
    b_h = torch.from_numpy(ct.b_polys.view(np.int32)).pin_memory()
    in_bytes = (a_h.numel() + b_h.numel()) * 4
    eng = CpmmEngine(ctpt.Spec(c.fmt, c.N, c.d1, c.d2, c.d3, ps), "cuda")
    eng.ctmat = torch.empty(eng.sizes.ctmat_bytes, dtype=torch.uint8, device="cuda")
    eng.precompute(U)
    AU_h = torch.empty(eng.sizes.out_AU_bytes // 4, dtype=torch.int32).pin_memory()
    BU_h = torch.empty(eng.sizes.out_BU_bytes // 4, dtype=torch.int32).pin_memory()
    out_bytes = eng.sizes.out_AU_bytes + eng.sizes.out_BU_bytes
    a_d = torch.empty_like(a_h, device="cuda")
    b_d = torch.empty_like(b_h, device="cuda")
    AU_d, BU_d = eng.alloc_outputs()

    res = []
    t = timed(lambda: (a_d.copy_(a_h, non_blocking=True), b_d.copy_(b_h, non_blocking=True)))
    res.append({"probe": "dma_h2d", "bytes": in_bytes, "s": t, "gbs": in_bytes / t / 1e9})
    t = timed(lambda: ctpt.layout(eng.spec, a_d, b_d, eng.ctmat))
    res.append({"probe": "layout_device_to_device", "bytes": in_bytes, "s": t, "gbs": in_bytes / t / 1e9})
    t = timed(lambda: ctpt.layout(eng.spec, a_h, b_h, eng.ctmat))
    res.append({"probe": "layout_reading_pinned_host (fused h2d+layout)", "bytes": in_bytes, "s": t,
                "gbs": in_bytes / t / 1e9})
    t = timed(lambda: (AU_h.copy_(AU_d, non_blocking=True), BU_h.copy_(BU_d, non_blocking=True)))
    res.append({"probe": "dma_d2h", "bytes": out_bytes, "s": t, "gbs": out_bytes / t / 1e9})
    t = timed(lambda: ctpt.matmul(eng.spec, eng.ctmat, eng.plain, AU_d, BU_d, eng.ws))
    res.append({"probe": "matmul_device_outputs", "s": t})
    t = timed(lambda: ctpt.matmul(eng.spec, eng.ctmat, eng.plain, AU_h, BU_h, eng.ws))
    res.append({"probe": "matmul_writing_pinned_host (fused gemm+d2h)", "bytes": out_bytes, "s": t,
                "gbs": out_bytes / t / 1e9})
    # correctness of the zero-copy results against the device-resident path
    ctpt.matmul(eng.spec, eng.ctmat, eng.plain, AU_d, BU_d, eng.ws)
    torch.cuda.synchronize()
    same = bool(torch.equal(AU_d.cpu(), AU_h) and torch.equal(BU_d.cpu(), BU_h))
    res.append({"probe": "zero_copy_outputs_equal_device_outputs", "ok": same})
    for r in res:
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
