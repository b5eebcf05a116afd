#!/usr/bin/env python
"""Launch-bound small CP-MMs: eager ctpt_matmul calls vs one CUDA graph replay per call.

ctpt_matmul never synchronises or allocates, so a caller can capture it once (TMA descriptors
are kernel parameters, baked into the graph) and replay it for new ciphertexts written in place.
For config c1-sized problems the per-call host work (validation, descriptor encoding, launches)
dominates; the graph removes it.  One JSON line per (config, mode): µs per call.

    python tools/bench_graph.py [--configs c1,c2] [--iters 200]
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
    ap.add_argument("--configs", default="c1,c2")
    ap.add_argument("--iters", type=int, default=200)
    args = ap.parse_args()
    import torch

    import ctgen
    from paper_2503_16080_b200 import ctpt
    from paper_2503_16080_b200.engine import CpmmEngine

    for name in args.configs.split(","):
        c = ctgen.CONFIGS[name]
        ps = ctgen.primes(c.L)
        ct = ctgen.encrypt(c.fmt, c.N, c.d1, c.d2, c.seed, c.log_delta, ps, nthreads=os.cpu_count() or 1)
        U = ctgen.U_matrix(c.seed, c.d2, c.d3, c.u_bound)
        eng = CpmmEngine(ctpt.Spec(c.fmt, c.N, c.d1, c.d2, c.d3, ps), "cuda")
        eng.layout(ct.a_polys, ct.b_polys)
        eng.precompute(U)
        AU, BU = eng.alloc_outputs()
        s = torch.cuda.Stream()

        def call():
            ctpt.matmul(eng.spec, eng.ctmat, eng.plain, AU, BU, eng.ws, stream=s)

        with torch.cuda.stream(s):
            for _ in range(10):
                call()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            call()
        for mode in ("eager", "graph"):
            fn = call if mode == "eager" else g.replay
            with torch.cuda.stream(s):
                for _ in range(10):
                    fn()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(args.iters):
                    fn()
                e1.record(s)
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / args.iters
            print(json.dumps({"config": name, "mode": mode, "us_per_call": us,
                              "residue_macs_per_s": c.residue_macs / (us / 1e6)}), flush=True)


if __name__ == "__main__":
    main()
