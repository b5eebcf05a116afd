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
