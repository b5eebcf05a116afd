#!/usr/bin/env python
"""Mod-PP-MM with full residues on both sides (the stage CC-MM, Alg. 8,
and the RGSW product, Alg. 9, reduce to) through ctpt_modmatmul.

Z = X·Y mod p for L primes, X ∈ Z_p^{M×K}, Y ∈ Z_p^{K×Nc} uniform residues; Y's precompute
(4 balanced digits per residue) is outside the timed region, as for a reused operand.  One JSON
line: residue-MAC/s and limb-MAC/s (16 limb MACs per residue MAC) against the INT8 datasheet.

    python tools/bench_modmm.py [--M 16384 --K 16384 --N 16384 --L 3 --steps 5 --warmup 2]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=16384)
    ap.add_argument("--K", type=int, default=16384)
    ap.add_argument("--N", type=int, default=16384)
    ap.add_argument("--L", type=int, default=3)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    import torch

    import ctgen
    from paper_2503_16080_b200 import ctpt

    ps = ctgen.primes(args.L)
    M, K, Nc = args.M, args.K, args.N
    ldx, plain_bytes, ws_bytes = ctpt.modmatmul_sizes(ps, M, K, Nc)
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.zeros((args.L, M, ldx), dtype=torch.int32, device="cuda")
    Y = torch.empty((args.L, K, Nc), dtype=torch.int32, device="cuda")
    for l, p in enumerate(ps):
        X[l, :, :K] = torch.randint(0, p, (M, K), generator=g, device="cuda", dtype=torch.int64).to(torch.int32)
        Y[l] = torch.randint(0, p, (K, Nc), generator=g, device="cuda", dtype=torch.int64).to(torch.int32)
    plain = torch.empty(plain_bytes, dtype=torch.uint8, device="cuda")
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    ZT = torch.empty((args.L, Nc, M), dtype=torch.int32, device="cuda")
    ctpt.modmatmul_precompute(ps, M, K, Nc, Y, plain)
    for _ in range(args.warmup):
        ctpt.modmatmul(ps, M, K, Nc, X, ldx, plain, ZT, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        ctpt.modmatmul(ps, M, K, Nc, X, ldx, plain, ZT, ws)
    e1.record()
    torch.cuda.synchronize()
    s = e0.elapsed_time(e1) / 1e3 / args.steps
    macs = args.L * M * K * Nc
    print(json.dumps({"bench": "modmatmul", "M": M, "K": K, "N": Nc, "L": args.L, "ms_per_call": s * 1e3,
                      "residue_macs_per_s": macs / s, "limb_macs_per_s": 16 * macs / s,
                      "pct_int8_datasheet": 100 * 16 * macs / s / 2.25e15}))


if __name__ == "__main__":
    main()
