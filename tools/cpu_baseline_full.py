#!/usr/bin/env python
"""Full CPU-oracle runs of configs c1, c2 (median of 3) and c3 (one run, every prime), as
SURVEY.md §8(d) asks for the CPU baseline, on all host cores of the GPU box — and, since the
oracle then holds every output entry, every entry of the GPU's outputs for the same inputs is
compared with them (c3: all three primes, 1.65e13 residue MACs; SURVEY.md §8(c) c5 "every entry
if the host's oracle time allows").

    python tools/cpu_baseline_full.py [--configs c1,c2,c3] [--reps 3] > profiles/r02/cpu_baseline_full.jsonl

One JSON line per config: oracle seconds per run (all primes, A·U and B·U), residue-MAC/s, the
host (lscpu), the GPU step time of the same problem through ctpt_matmul, and the parity verdict.
The paper's own timing is single-threaded and the mean of 10 runs; the single-thread
rate is reported on a slab (one output column block) next to it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def lscpu() -> dict:
    try:
        txt = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
    except (OSError, subprocess.SubprocessError):
        return {}
    kv = {}
    for line in txt.splitlines():
        if ":" in line:
            k, v = line.split(":", 1)
            kv[k.strip()] = v.strip()
    keep = ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core", "CPU(s)", "CPU max MHz", "L3 cache")
    return {k: kv[k] for k in keep if k in kv}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3")
    ap.add_argument("--reps", type=int, default=3, help="oracle runs for c1/c2 (median); c3 runs once")
    args = ap.parse_args()

    import torch

    import ctgen
    import oracle
    from gpu_helpers import colmajor_views, run_gpu

    cores = os.cpu_count() or 1
    host = lscpu()
    for name in args.configs.split(","):
        c = ctgen.CONFIGS[name]
        ps = ctgen.primes(c.L)
        t0 = time.perf_counter()
        ct = ctgen.encrypt(c.fmt, c.N, c.d1, c.d2, c.seed, c.log_delta, ps, nthreads=cores)
        U = ctgen.U_matrix(c.seed, c.d2, c.d3, c.u_bound, nthreads=cores)
        gen_s = time.perf_counter() - t0
        # GPU: the bench's ctpt_matmul on the same inputs (outputs kept on the host for the comparison)
        (AU, BU), eng = run_gpu(c.fmt, c.N, c.d1, c.d2, c.d3, ps, ct.a_polys, ct.b_polys, U=U)
        del eng
        torch.cuda.empty_cache()
        reps = args.reps if name in ("c1", "c2") else 1
        times, bad = [], 0
        for rep in range(reps):
            t1 = time.perf_counter()
            outs = []
            for l, p in enumerate(ps):
                Ac, Bc = colmajor_views(c.fmt, c.N, c.d1, c.d2, ct.a_polys[l], ct.b_polys[l])
                wa = oracle.modmatmul(Ac, U, p, nthreads=cores) if c.rows_A else None
                wb = oracle.modmatmul(Bc, U, p, nthreads=cores)
                outs.append((wa, wb))
            times.append(time.perf_counter() - t1)
            if rep == 0:
                for l, (wa, wb) in enumerate(outs):
                    if wa is not None:
                        bad += int(np.count_nonzero(AU[l] != wa))
                    bad += int(np.count_nonzero(BU[l] != wb))
            del outs
        # single-thread rate on a slab: 8 output columns of B·U for prime 0 (the paper's setting)
        Ac, Bc = colmajor_views(c.fmt, c.N, c.d1, c.d2, ct.a_polys[0], ct.b_polys[0])
        ncol = min(8, c.d3)
        t1 = time.perf_counter()
        oracle.modmatmul(Bc, U, ps[0], cols=np.arange(ncol), nthreads=1)
        st = c.d1 * c.d2 * ncol / (time.perf_counter() - t1)
        med = statistics.median(times)
        print(json.dumps({
            "config": name, "residue_macs": c.residue_macs, "oracle_runs": reps, "oracle_s": times,
            "oracle_s_median": med, "oracle_residue_macs_per_s": c.residue_macs / med, "threads": cores,
            "host": host, "single_thread_residue_macs_per_s": st,
            "single_thread_sample": f"prime 0, {ncol} columns of B·U x {c.d1} rows x d2={c.d2}",
            "gpu_vs_oracle": {"entries": int(sum((AU[l].size if c.rows_A else 0) + BU[l].size for l in range(c.L))),
                              "mismatches": bad, "verdict": "bit-exact" if bad == 0 else "MISMATCH"},
            "input_generation_s": gen_s,
            "kind": "oracle (schoolbook, unsigned __int128 accumulation, one % p per output; OpenMP over outputs)",
        }), flush=True)
        del ct, AU, BU


if __name__ == "__main__":
    main()
