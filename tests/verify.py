#!/usr/bin/env python
"""Command-line parity check of the CUDA path against the CPU oracle on a BASELINE config
(SURVEY.md §5 "config / flags", SPEC's exit-code convention S:671: 0 = verified,
3 = a mismatch).  It lives under tests/ because it runs the oracle (test infrastructure).

    python tests/verify.py --config c2 [--seed 0] [--verify full|freivalds|sample] [--threads N]

  full       every output entry of every prime by the schoolbook oracle (c1, c2; c3 takes long)
  freivalds  two Freivalds trials per prime and output matrix (probability of a missed error
             ≤ p^-2) + boundary rows/columns + random entries (c3–c5)
  sample     boundary rows/columns + random entries only
Also checks the decryption identity on two output columns for every prime.
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--verify", default=None, choices=["full", "freivalds", "sample"])
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()

    import dataclasses

    import ctgen
    import oracle
    from gpu_helpers import colmajor_views, run_gpu

    c = ctgen.CONFIGS[args.config]
    if args.seed is not None:
        c = dataclasses.replace(c, seed=args.seed)
    mode = args.verify or ("full" if c.residue_macs < 1e12 else "freivalds")
    ps = ctgen.primes(c.L)
    U = ctgen.U_matrix(c.seed, c.d2, c.d3, c.u_bound, nthreads=args.threads)
    rng = np.random.default_rng(c.seed + 17)
    bad = 0
    for l, p in enumerate(ps):  # one prime at a time keeps c5 within host and device memory
        ct = ctgen.encrypt(c.fmt, c.N, c.d1, c.d2, c.seed, c.log_delta, [p], nthreads=args.threads)
        (AU, BU), _ = run_gpu(c.fmt, c.N, c.d1, c.d2, c.d3, [p], ct.a_polys, ct.b_polys, U=U)
        Ac, Bc = colmajor_views(c.fmt, c.N, c.d1, c.d2, ct.a_polys[0], ct.b_polys[0])
        for name, Xc, C in (("A·U", Ac, AU[0]), ("B·U", Bc, BU[0])):
            rows = Xc.shape[1]
            if rows == 0:
                continue
            if mode == "full":
                want = oracle.modmatmul(Xc, U, p, nthreads=args.threads)
                n = int(np.count_nonzero(C != want))
            else:
                n = 0
                if mode == "freivalds":
                    for _ in range(2):
                        v = rng.integers(0, p, c.d3, dtype=np.uint64)
                        n += oracle.freivalds(Xc, U, C, p, v, nthreads=args.threads)
                r_idx = np.concatenate([[0, rows - 1, min(63, rows - 1), min(64, rows - 1)],
                                        rng.integers(0, rows, 4096)])
                j_idx = np.concatenate([[0, c.d3 - 1, min(127, c.d3 - 1), min(128, c.d3 - 1)],
                                        rng.integers(0, c.d3, 4096)])
                want = oracle.modmatmul_entries(Xc, U, p, r_idx, j_idx, nthreads=args.threads)
                n += int(np.count_nonzero(C[j_idx, r_idx] != want))
            print(f"prime {l} {name}: {'ok' if n == 0 else f'{n} MISMATCHES'} ({mode})", flush=True)
            bad += n
        # decryption identity S·A' + B' ≡ (⌊ΔM⌉+E)·U (mod p) on two output columns
        nk = c.k if c.fmt == ctgen.SHARED_A else 1
        if c.fmt != ctgen.STRUCT_A:
            sks = [ctgen.sk(c.seed, t, c.N) for t in range(nk)]
            for j in (0, c.d3 - 1):
                dec = oracle.decrypt_col(c.fmt, c.N, c.d1, sks, AU[0][j], BU[0][j], p, nthreads=args.threads)
                pu = np.zeros(c.d1, dtype=np.uint64)
                for k0 in range(0, c.d2, 2048):
                    kb = min(2048, c.d2 - k0)
                    P = ctgen.plain_block(c.seed, c.N, c.d1, c.log_delta, 0, c.d1, k0, kb, nthreads=args.threads)
                    part = oracle.modmatmul(np.ascontiguousarray((P.T % p).astype(np.uint32)), U[k0:k0 + kb, j:j + 1],
                                            p, nthreads=args.threads)[0]
                    pu = (pu + part) % p
                n = int(np.count_nonzero(dec.astype(np.uint64) != pu))
                print(f"prime {l} decryption identity, column {j}: {'ok' if n == 0 else 'MISMATCH'}", flush=True)
                bad += n
    print("VERIFIED" if bad == 0 else f"FAILED: {bad} mismatches")
    return 0 if bad == 0 else 3


if __name__ == "__main__":
    sys.exit(main())
