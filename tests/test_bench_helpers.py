"""bench.py's host-side arithmetic (no GPU): roofline bytes, launch counts, peak choice."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import ctgen  # noqa: E402


def test_roofline_fused_bytes_and_fraction():
    c = ctgen.CONFIGS["c4"]
    mp = {"hbm_gbs": 6556.2}
    r = bench.roofline_fused(c, 128, 1e-3, 0.9, mp, "measured")
    alg = 4 * c.R * c.d2 + 128 * c.d2 + 4 * c.R * 128
    assert r["bound"] == "hbm" and abs(r["achieved"] - alg / 1e-3 / 1e9) < 1e-6
    assert abs(r["frac"] - r["achieved"] / 6556.2) < 1e-12


def test_host_launch_count_matches_library_chunking():
    c = ctgen.CONFIGS["c3"]
    chunk = ((c.R + 5) // 6 + 63) // 64 * 64  # ctpt.cu host_plan default
    n_chunks = -(-c.R // chunk)
    assert bench.host_launches(c, 3, 1, True) == 3 * n_chunks * 3   # layout + split + GEMM per chunk
    assert bench.host_launches(c, 2, 1, False) == 2 * n_chunks * 2  # layout + fused


def test_cublaslt_ratio_uses_burst_for_short_runs():
    with open(os.path.join(ROOT, "profiles", "r01", "int8_cublaslt_probe.json")) as f:
        pr = json.load(f)
    r = bench.cublaslt_ratio(1e15, 500.0)
    assert r["which"] == "burst_tops" and abs(r["ratio"] - 2e15 / 1e12 / pr["burst_tops"]) < 1e-12
    assert bench.cublaslt_ratio(1e15, 5000.0)["which"] == "sustained_tops"


def test_workload_desc_names_the_config():
    d = bench.workload_desc(ctgen.CONFIGS["c3"])
    assert d["workload"].startswith("c3: shared-a") and d["rows_stacked_R"] == 20480
    d = bench.workload_desc(ctgen.CONFIGS["c3a"])
    assert d["rows_stacked_R"] == 16384 and "struct-a" in d["workload"]


def _oracle_outputs_tensor(c, ps, ct, U):
    import numpy as np
    import torch

    import oracle

    AU, BU = [], []
    for l, p in enumerate(ps):
        Ac = ct.a_polys[l].reshape(c.d2, c.rows_A)
        Bc = ct.b_polys[l].reshape(c.d2, c.d1)
        AU.append(oracle.modmatmul(Ac, U, p, nthreads=2))
        BU.append(oracle.modmatmul(Bc, U, p, nthreads=2))
    to_t = lambda a: torch.from_numpy(np.stack(a).view(np.int32))  # noqa: E731
    return to_t(AU), to_t(BU)


def test_precision_on_sample_decodes_oracle_outputs():
    """bench.precision_on_sample decrypts + CRT-decodes sampled output columns: on the oracle's
    exact (A·U, B·U) of c1 (RLWE, Δ = 2^20, d2 = 64) and of a 2-prime shared-a case it reports the
    precision the error bound allows (reading Q16: |err| ≤ ‖U‖∞·d2·(B_e + ½)/Δ), and a single
    corrupted residue collapses it."""
    import numpy as np

    for name, c in [("c1", ctgen.CONFIGS["c1"]),
                    ("sa", ctgen.Config("sa", ctgen.SHARED_A, 64, 128, 96, 40, 2, 30, 8))]:
        ps = ctgen.primes(c.L)
        ct = ctgen.encrypt(c.fmt, c.N, c.d1, c.d2, c.seed, c.log_delta, ps)
        U = ctgen.U_matrix(c.seed, c.d2, c.d3, c.u_bound)
        AU, BU = _oracle_outputs_tensor(c, ps, ct, U)
        r = bench.precision_on_sample(c, ps, AU, BU, U, [0, c.d3 - 1], 2)
        bound = c.u_bound * c.d2 * 20.5 / 2.0 ** c.log_delta
        assert r["precision_bits"] > 5 and r["rel_err_inf"] < 1.0, (name, r)
        mu_scale = 1.0  # ‖M·U‖∞ ≥ 1 for these sizes (sums of d2 products of uniform[-1,1) and integers)
        assert r["rel_err_inf"] * mu_scale <= bound, (name, r, bound)
        BU[0, 0, 3] = (int(BU[0, 0, 3]) + 12345) % int(ps[0])
        bad = bench.precision_on_sample(c, ps, AU, BU, U, [0], 2)
        assert bad["precision_bits"] < r["precision_bits"] - 5, (name, bad, r)
