"""Debug: which shapes make the k_gemm_mv launch fail?"""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import ctgen
from gpu_helpers import run_gpu, oracle_outputs
from paper_2503_16080_b200 import ctpt

for (N, d2, d3) in [(64, 16384, 20), (64, 32768, 20), (64, 49152, 20), (64, 65536, 20), (64, 65536, 4), (256, 65536, 20),
                    (64, 40000, 20), (64, 33000, 20), (64, 32768 + 16, 20)]:
    ps = ctgen.primes(1)
    ct = ctgen.encrypt(0, N, N, d2, 1, 20, ps)
    U = ctgen.U_matrix(1, d2, d3, 8)
    try:
        (AU, BU), eng = run_gpu(0, N, N, d2, d3, ps, ct.a_polys, ct.b_polys, U=U)
        wa, wb = oracle_outputs(0, N, N, ct.a_polys[0], ct.b_polys[0], U, ps[0])
        print(N, d2, d3, "ok" if np.array_equal(AU[0], wa) and np.array_equal(BU[0], wb) else "MISMATCH", flush=True)
    except ctpt.CtptError as e:
        print(N, d2, d3, "ERR", e, flush=True)
