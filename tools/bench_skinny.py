#!/usr/bin/env python
"""Skinny-U sweep (SURVEY.md §8(d) "supplementary skinny sweep", §8(f) row 1).

Config c4's ciphertexts (shared-s, N = 8192, d1 = d2 = 32768, R = 65536 stacked rows, L primes)
times a U with d3 ∈ {1, 64, 128, 256} — Table 4's d3 values and CP-Mv (d3 = 1).
Below the ridge (≈ d3 limb MACs per byte of X) the step is HBM-bound, so each line reports the
achieved algorithmic GB/s of the dominant kernel against MEASURED_PEAKS.json's copy bandwidth:

    algorithmic bytes per launch (one prime) = 4·R·d2 (X, int32) + d3·d2 (U digits) + 4·R·d3 (out)

Two paths per d3: "fused" (ctpt_gemm_fused: split inside the GEMM's load path, X read once) and
"split+gemm" (ctpt_split + ctpt_gemm, the square-regime kernels).  One JSON line per (d3, path).

    python tools/bench_skinny.py [--L 4] [--steps 10] [--warmup 3] [--d3 1,64,128,256]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=4)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--d3", default="1,16,32,64,128,256")
    ap.add_argument("--u-shift", type=int, default=0,
                    help="add this to U (e.g. 8: U in [0, 16], so the u8 plane needs no row correction)")
    ap.add_argument("--plane", default="auto", choices=["auto", "always", "never"],
                    help="the U plane mode (engine.precompute's `unsigned`): always = u8, never = s8 digits")
    ap.add_argument("--paths", default="auto,fused,split+gemm",
                    help="auto = ctpt_matmul's choice per prime (mv for d3 <= 32, else fused); fused = the "
                         "converter kernel (ctpt_gemm_fused); mv = ctpt_gemm_mv; split+gemm")
    args = ap.parse_args()

    import torch

    import bench
    import ctgen
    from paper_2503_16080_b200 import ctpt
    from paper_2503_16080_b200.engine import CpmmEngine

    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        hbm_peak = float(json.load(f)["hbm_gbs"])
    c = ctgen.CONFIGS["c4"]
    ps = ctgen.primes(c.L)[:args.L]
    cores = os.cpu_count() or 1
    d3s = [int(x) for x in args.d3.split(",")]
    d3max = max(d3s)
    ct = ctgen.encrypt(c.fmt, c.N, c.d1, c.d2, c.seed, c.log_delta, ps, nthreads=cores)
    U = ctgen.U_matrix(c.seed, c.d2, d3max, c.u_bound, nthreads=cores)
    eng = CpmmEngine(ctpt.Spec(c.fmt, c.N, c.d1, c.d2, d3max, ps), "cuda")
    eng.layout(ct.a_polys, ct.b_polys)
    del ct
    U = U + args.u_shift
    kU = eng.precompute(U, unsigned=args.plane)
    assert kU == 1
    stream = torch.cuda.current_stream()
    R, d2 = c.R, c.d2
    import dataclasses

    ws_need = max(ctpt.query_sizes(dataclasses.replace(eng.spec, col_begin=0, col_end=x)).workspace_bytes for x in d3s)
    if eng.ws.numel() < ws_need:
        eng.ws = torch.empty(ws_need, dtype=torch.uint8, device="cuda")
    for d3 in d3s:
        import dataclasses

        sp = dataclasses.replace(eng.spec, col_begin=0, col_end=d3)
        sz = ctpt.query_sizes(sp)
        AU = torch.empty(sz.out_AU_bytes // 4, dtype=torch.int32, device="cuda")
        BU = torch.empty(sz.out_BU_bytes // 4, dtype=torch.int32, device="cuda")
        ra = sz.rows_A
        for path in args.paths.split(","):

            def step(evs=None):
                for l in range(len(ps)):
                    au, bu = AU[l * d3 * ra:], BU[l * d3 * c.d1:]
                    if path == "mv" or (path == "auto" and bench.kernel_path(d3, 1, 0, 0, R) == "mv"):
                        if evs is not None:
                            evs[l][0].record(stream)
                        ctpt.gemm_mv(sp, l, eng.ctmat, eng.plain, au, bu, eng.ws, stream=stream)
                    elif path.startswith("fused") or path == "auto":
                        if evs is not None:
                            evs[l][0].record(stream)
                        ctpt.gemm_fused(sp, l, eng.ctmat, eng.plain, au, bu, stream=stream)
                    else:
                        ctpt.split(sp, l, eng.ctmat, eng.ws, stream=stream)
                        if evs is not None:
                            evs[l][0].record(stream)
                        ctpt.gemm(sp, l, eng.ws, eng.plain, au, bu, stream=stream)
                    if evs is not None:
                        evs[l][1].record(stream)

            for _ in range(args.warmup):
                step()
            torch.cuda.synchronize()
            clk = bench.ClockSampler(torch.device("cuda", torch.cuda.current_device()))
            evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in ps]
                   for _ in range(args.steps)]
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            for s in range(args.steps):
                step(evs[s])
            t1.record(stream)
            torch.cuda.synchronize()
            clocks = clk.stop()
            ms_step = t0.elapsed_time(t1) / args.steps
            k_ms = statistics.mean(a.elapsed_time(b) for row in evs for (a, b) in row)
            alg_bytes = 4 * R * d2 + d3 * d2 + 4 * R * d3
            macs = len(ps) * R * d2 * d3
            gbs = alg_bytes / (k_ms / 1e3) / 1e9
            print(json.dumps({
                "sweep": "skinny", "path": path, "d3": d3, "u_plane": "u8" if eng.spec.u_unsigned else "s8",
                "u_offset": eng.spec.u_offset, "L": len(ps), "R": R, "d2": d2,
                "ms_per_step": ms_step, "residue_macs_per_s": macs / (ms_step / 1e3),
                "kernel": ("k_gemm_mv" if path == "mv" or (path == "auto" and bench.kernel_path(d3, 1, 0, 0, R) == "mv") else
                           "k_gemm_fused_t" if path.startswith("fused") or path == "auto"
                           else "k_gemm_tc (after k_split)"),
                "avg_launch_ms": k_ms,
                "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s",
                             "frac": gbs / hbm_peak, "per_launch_bytes": alg_bytes},
                "step_gbs_algorithmic": len(ps) * alg_bytes / (ms_step / 1e3) / 1e9,
                "clocks": clocks,
            }), flush=True)
        del AU, BU


if __name__ == "__main__":
    main()
