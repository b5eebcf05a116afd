import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import ctgen
from gpu_helpers import run_gpu, oracle_outputs
S, A = ctgen.SHARED_S, ctgen.SHARED_A
cases = [(S, 32, 4, 520, 100, 1, 1), (S, 32, 4, 520, 128, 1, 1), (S, 32, 4, 520, 200, 1, 1), (S, 32, 4, 128, 100, 1, 1),
         (S, 32, 4, 520, 100, 1, 0), (S, 64, 8, 4112, 64, 1, 3), (S, 64, 8, 4112, 256, 1, 5)]
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
  for (fmt, N, k, d2, d3, L, mc) in cases:
    d1 = N * k
    ps = ctgen.primes(L)
    ct = ctgen.encrypt(fmt, N, d1, d2, 52 + rep, 20, ps)
    U = ctgen.U_matrix(52 + rep, d2, d3, 8)
    (AU, BU), eng = run_gpu(fmt, N, d1, d2, d3, ps, ct.a_polys, ct.b_polys, U=U, kernel=2, max_ctas=mc)
    wa, wb = oracle_outputs(fmt, N, d1, ct.a_polys[0], ct.b_polys[0], U, ps[0])
    got = np.concatenate([AU[0], BU[0]], axis=1); want = np.concatenate([wa, wb], axis=1)
    bad = np.argwhere(got != want)
    print(f"rep {rep} d2={d2} d3={d3} R={got.shape[1]} max_ctas={mc}: {len(bad)} bad of {got.size}", flush=True)
    if len(bad):
        rows = bad[:, 1]; cols = bad[:, 0]
        print("  tiles", sorted(set((rows // 32).tolist()))[:20], "row%32", sorted(set((rows % 32).tolist())))
        print("  cols", sorted(set(cols.tolist()))[:20], "col%4", sorted(set((cols % 4).tolist())), flush=True)
