"""Debug: where does k_gemm_fused (TMA raw ring) differ from the oracle?"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import ctgen
from gpu_helpers import run_gpu, oracle_outputs

for load in ["tma", "regs"]:
    os.environ["CTPT_FUSED_LOAD"] = load
    for (fmt, N, k, d2, d3) in [(2, 256, 2, 4112, 64), (2, 256, 2, 4096, 64), (2, 256, 2, 1024, 64), (2, 64, 2, 640, 64),
                                (2, 256, 2, 4112, 200)]:
        d1 = N * k
        ps = ctgen.primes(1)
        ct = ctgen.encrypt(fmt, N, d1, d2, 0, 20, ps)
        U = ctgen.U_matrix(0, d2, d3, 8)
        (AU, BU), eng = run_gpu(fmt, N, d1, d2, d3, ps, ct.a_polys, ct.b_polys, U=U)
        wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[0], ct.b_polys[0], U, ps[0])
        got = np.concatenate([AU[0], BU[0]], 1)
        want = np.concatenate([wa, wb], 1)
        bad = np.argwhere(got != want)
        rows = np.unique(bad[:, 1]) if len(bad) else []
        print(load, (fmt, N, k, d2, d3), "bad", len(bad), "of", got.size, "rows", len(rows), list(rows[:40]),
              "cols", list(np.unique(bad[:, 0])[:10]) if len(bad) else [], flush=True)
