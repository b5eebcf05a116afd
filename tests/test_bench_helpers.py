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


def test_kernel_path_mirrors_the_library_choice():
    """bench.kernel_path = ctpt.cu choose_path under CTPT_KERNEL_AUTO (launch counting, roofline)."""
    assert bench.kernel_path(16384, 1, 1, 8) == "split_gemm"   # c3: u8 plane with offset
    assert bench.kernel_path(256, 1, 0, 0) == "fused"
    assert bench.kernel_path(256, 1, 1, 8) == "fused"          # the fused kernel forms the row sums itself
    assert bench.kernel_path(257, 1, 1, 8) == "split_gemm"
    assert bench.kernel_path(32, 1, 1, 8, R=8192) == "fused"    # raw-byte kernel: no row correction
    assert bench.kernel_path(32, 1, 0, 0, R=8192) == "mv"       # 128 tiles of 64 rows < 148 SMs
    assert bench.kernel_path(32, 1, 0, 0, R=65536) == "fused"   # enough rows: limbs-in-TMEM kernel
    assert bench.kernel_path(100, 2, 0, 0) == "split_gemm"     # kU > 1


def test_both_arms_report_the_same_config():
    """The reference (oracle) arm and our arm build `config` with the same function."""
    import argparse

    c = ctgen.CONFIGS["c3"]
    for world in (1, 2, 8):
        for mode in ("auto", "strong", "weak"):
            args = argparse.Namespace(mode=mode)
            m = bench.arm_mode(args, world)
            assert bench.config_for(c, world, m) == bench.config_for(c, world, "weak" if mode == "weak" else "strong")
    assert "strong" in bench.config_for(c, 8, "strong")["parallelism"]


def test_gpus_flag_relaunches_under_torchrun_and_refuses_a_mismatch(tmp_path):
    """`bench.py --gpus 2` outside torchrun re-runs itself as 2 ranks (here the reference arm on
    c1, which needs no GPU: rank 0 prints one JSON line with n_gpus = 2, the other rank exits 0);
    under a launcher whose WORLD_SIZE differs from --gpus it refuses to run (exit 2)."""
    import subprocess

    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--config", "c1", "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env,
                       timeout=600, cwd=str(tmp_path))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference", r.stdout
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference"],
                       capture_output=True, text=True, env=dict(env, WORLD_SIZE="1"), timeout=120)
    assert r.returncode == 2 and "refusing" in r.stderr


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
