#!/usr/bin/env python
"""Does the operand data change how fast k_gemm_tc runs under the 1000 W power cap?

c3's GEMM shape (R = 20480, d2 = d3 = 16384, one prime per launch) run back to back for
~`--seconds` per case with different operand distributions; reports sustained int8 TOP/s, the
median SM clock and the power draw (nvidia-smi sampled every 100 ms).  Experiment only: the
bench's inputs are always the real ciphertexts.

    python tools/power_operands.py [--seconds 4]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=4.0)
    ap.add_argument("--cases", default="")
    args = ap.parse_args()
    import torch

    import ctgen
    from bench import ClockSampler
    from paper_2503_16080_b200 import ctpt
    from paper_2503_16080_b200.engine import CpmmEngine

    c = ctgen.CONFIGS["c3"]
    p = ctgen.primes(1)[0]
    spec = ctpt.Spec(c.fmt, c.N, c.d1, c.d2, c.d3, [p])
    eng = CpmmEngine(spec, "cuda")
    eng.ctmat = torch.zeros(eng.sizes.ctmat_bytes, dtype=torch.uint8, device="cuda")
    X = eng.ctmat[256:].view(torch.int32).view(c.R, eng.sizes.d2p)
    AU, BU = eng.alloc_outputs()
    g = torch.Generator(device="cuda").manual_seed(0)

    def setX(kind):
        if kind == "uniform":
            X.copy_(torch.randint(0, p, X.shape, device="cuda", generator=g, dtype=torch.int64).to(torch.int32))
        elif kind == "zero":
            X.zero_()
        elif kind == "small":  # residues < 2^8: limbs 1..3 are zero
            X.copy_(torch.randint(0, 256, X.shape, device="cuda", generator=g, dtype=torch.int32))
        elif kind == "bytes16":  # every limb byte uniform in [0, 16]: X carries U's entropy per byte
            b = torch.randint(0, 17, X.shape + (4,), device="cuda", generator=g, dtype=torch.int32)
            X.copy_(b[..., 0] | (b[..., 1] << 8) | (b[..., 2] << 16) | (b[..., 3] << 24))
        elif kind == "bytes8":  # every limb byte uniform in [0, 8]
            b = torch.randint(0, 9, X.shape + (4,), device="cuda", generator=g, dtype=torch.int32)
            X.copy_(b[..., 0] | (b[..., 1] << 8) | (b[..., 2] << 16) | (b[..., 3] << 24))

    def setU(lo, hi):
        U = torch.randint(lo, hi + 1, (c.d2, c.d3), device="cuda", generator=g, dtype=torch.int64)
        kU = eng.precompute(U)
        assert kU == 1

    # the last four swap the entropies of the two MMA operands (A = U^T tile, 4 KB per MMA; B = the
    # four X limb tiles, 8 KB per MMA): what a kernel with X as the A operand would see
    cases = [("uniform", (-8, 8)), ("uniform", (0, 16)), ("uniform", (0, 0)), ("zero", (-8, 8)),
             ("uniform", (-128, 127)), ("uniform", (-1, 1)), ("small", (-8, 8)), ("uniform", (-8, 8)),
             ("bytes16", (0, 255)), ("uniform", (0, 16)), ("bytes16", (0, 16)), ("bytes8", (0, 255))]
    if args.cases:
        keep = set(args.cases.split(";"))
        cases = [cs for cs in cases if f"{cs[0]}:{cs[1][0]},{cs[1][1]}" in keep]
    stream = torch.cuda.current_stream()
    limb_macs = 4 * c.R * c.d2 * c.d3
    for xk, (lo, hi) in cases:
        setX(xk)
        setU(lo, hi)
        ctpt.split(eng.spec, 0, eng.ctmat, eng.ws, stream=stream)
        for _ in range(3):
            ctpt.gemm(eng.spec, 0, eng.ws, eng.plain, AU, BU, stream=stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = max(1, int(args.seconds / 0.016))
        clk = ClockSampler(0)
        time.sleep(0.3)
        e0.record(stream)
        for _ in range(n):
            ctpt.gemm(eng.spec, 0, eng.ws, eng.plain, AU, BU, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        cl = clk.stop()
        s = e0.elapsed_time(e1) / 1e3 / n
        print(json.dumps({"X": xk, "U": [lo, hi], "launches": n, "ms_per_launch": s * 1e3,
                          "tops": 2 * limb_macs / s / 1e12, "sm_mhz_median": cl.get("sm_mhz"),
                          "power_w_max": cl.get("power_w_max"), "reasons": cl.get("reasons")}), flush=True)
        time.sleep(2.0)  # let the power manager settle between cases


if __name__ == "__main__":
    main()
