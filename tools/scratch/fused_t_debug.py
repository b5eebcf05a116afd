import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import ctgen
from gpu_helpers import run_gpu, oracle_outputs
S, A = ctgen.SHARED_S, ctgen.SHARED_A
for (fmt, N, k, d2, d3, L, mc) in [(S, 32, 4, 520, 100, 1, 1), (S, 32, 4, 520, 100, 1, 2), (S, 32, 4, 512, 100, 1, 1),
                                   (S, 32, 4, 520, 128, 1, 1), (S, 32, 4, 520, 200, 1, 1), (S, 32, 4, 128, 100, 1, 1),
                                   (S, 32, 4, 520, 100, 1, 0)]:
    d1 = N * k
    ps = ctgen.primes(L)
    ct = ctgen.encrypt(fmt, N, d1, d2, 52, 20, ps)
    U = ctgen.U_matrix(52, d2, d3, 8)
    (AU, BU), eng = run_gpu(fmt, N, d1, d2, d3, ps, ct.a_polys, ct.b_polys, U=U, kernel=2, max_ctas=mc)
    wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[0], ct.b_polys[0], U, ps[0])
    got = np.concatenate([AU[0], BU[0]], axis=1); want = np.concatenate([wa, wb], axis=1)
    bad = np.argwhere(got != want)
    print(f"d2={d2} d3={d3} max_ctas={mc}: {len(bad)} bad of {got.size}")
    if len(bad):
        rows = bad[:, 1]; cols = bad[:, 0]
        print("  tiles", sorted(set((rows // 32).tolist()))[:20], "row%32", sorted(set((rows % 32).tolist())))
        print("  cols", sorted(set(cols.tolist()))[:40], "col%4", sorted(set((cols % 4).tolist())))
