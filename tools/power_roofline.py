#!/usr/bin/env python
"""Power roofline: how close are the power-capped kernels to what 1000 W allows?

The skinny kernel near d3 = 256 and k_gemm_tc both run at the B200's 1000 W cap
(`sw_power_cap`), where neither the HBM roofline nor the tensor roofline is the binding limit:
the energy of the bytes moved plus the energy of the MACs issued is.  This tool measures the two
energies on this box and gives each kernel's energy-additive bound (DESIGN.md §6 "Power roofline"):

  P_0   : board power with the GPU idle between cases (median of nvidia-smi samples);
  e_B   : J per algorithmic byte of the HBM stream = (P_stream − P_0) / BW_stream, from the skinny
          kernel at d3 = 1 (X read once, ≈ no tensor work) run back to back;
  e_op  : J per int8 op of the MMA with k_gemm_tc's operand statistics = (P_mma − P_0) / TOPS_mma,
          from tools/mma_ceiling (operands resident in shared memory, at the cap);
  bound : t* = max(bytes / BW, ops / TOPS_uncapped, (e_B·bytes + e_op·ops) / (P_cap − P_0)).

For each kernel run back to back for `--seconds`: the measured launch time t, `frac_power` = t* / t,
the HBM-only fraction for comparison, and the model's predicted mean power (P_0 + (e_B·bytes +
e_op·ops)/t) beside the measured median — the self-check of the additive model.  The model is an
upper estimate of the bound's time: e_op is taken at the clock the MMA-only run settles at (≈ 1.7
GHz), while the kernels below run at lower clocks and voltage, where an op costs less.

Inputs are uniform residues mod p (statistically what RLWE ciphertexts are) and U ∈ [−8, 8], the
shapes of c4 (skinny: R = 65536, d2 = 32768) and c3 (GEMM: R = 20480, d2 = d3 = 16384); the
bench's own inputs are always real ciphertexts.  Experiment only.

    python tools/power_roofline.py [--seconds 3] [--d3 1,64,128,160,192,224,256]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

P_CAP = 1000.0           # W, the board's power limit on this pool (power_w_max of the capped runs)
TOPS_UNCAPPED = 4610.0   # int8 TOP/s of the MMA with zero operands at 1965 MHz, no cap (profiles/r01/int8_mma_ceiling.jsonl)


def idle_power(dev, seconds: float = 2.0) -> float:
    from bench import ClockSampler

    clk = ClockSampler(dev)
    time.sleep(seconds)
    return clk.stop().get("power_w_median")


def sustained(fn, per_call_s: float, seconds: float, dev):
    """Run fn() back to back for ~seconds; returns (s per call from CUDA events, clocks dict)."""
    import torch

    from bench import ClockSampler

    n = max(3, int(seconds / max(per_call_s, 1e-5)))
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(dev)
    time.sleep(0.3)
    e0.record(stream)
    for _ in range(n):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    cl = clk.stop()
    return e0.elapsed_time(e1) / 1e3 / n, cl


def calib(fn):
    import torch

    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / 3


def fill_uniform(eng, R, primes, g):
    import torch

    d2p = eng.sizes.d2p
    for l, p in enumerate(primes):
        off = 256 + l * R * d2p * 4
        X = eng.ctmat[off:off + R * d2p * 4].view(torch.int32).view(R, d2p)
        for r0 in range(0, R, 8192):
            X[r0:r0 + 8192].copy_(torch.randint(0, p, X[r0:r0 + 8192].shape, device="cuda", generator=g,
                                                dtype=torch.int64).to(torch.int32))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=3.0)
    ap.add_argument("--d3", default="1,64,128,160,192,224,256")
    ap.add_argument("--no-gemm", action="store_true")
    ap.add_argument("--dram-gb-c3", type=float, default=11.9,
                    help="k_gemm_tc's DRAM bytes per c3 launch (ncu; profiles/r02/serp_group/)")
    args = ap.parse_args()
    import dataclasses

    import torch

    import ctgen
    import mma_ceiling
    from paper_2503_16080_b200 import ctpt
    from paper_2503_16080_b200.engine import CpmmEngine

    dev = torch.device("cuda", 0)
    torch.cuda.init()
    g = torch.Generator(device="cuda").manual_seed(0)
    out = []

    def emit(d):
        print(json.dumps(d), flush=True)
        out.append(d)

    P0 = idle_power(dev)
    emit({"case": "idle", "power_w_median": P0})

    # --- e_op: the MMA alone, k_gemm_tc's operand statistics (tools/mma_ceiling.py) -------------
    lib = ctypes.CDLL(mma_ceiling.build())
    lib.mma_ceiling_run.restype = ctypes.c_int
    lib.mma_ceiling_run.argtypes = [ctypes.c_int, ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_uint,
                                    ctypes.POINTER(ctypes.c_float), ctypes.c_void_p]
    blocks = torch.cuda.get_device_properties(0).multi_processor_count
    ms = ctypes.c_float()
    assert lib.mma_ceiling_run(blocks, 20000, 0, 0, 1, ctypes.byref(ms), None) == 0
    iters = int(20000 * args.seconds * 1e3 / max(ms.value, 1e-3))
    from bench import ClockSampler

    clk = ClockSampler(dev)
    time.sleep(0.3)
    assert lib.mma_ceiling_run(blocks, iters, 16, 255, 7, ctypes.byref(ms), None) == 0
    cl = clk.stop()
    tops_mma = 2 * blocks * iters * (4 * 128 * 256 * 32) / (ms.value / 1e3) / 1e12
    P_mma = cl.get("power_w_median")
    e_op = (P_mma - P0) / (tops_mma * 1e12)
    emit({"case": "mma only (A in [0,16], B uniform)", "tops": tops_mma, "power_w_median": P_mma,
          "sm_mhz": cl.get("sm_mhz"), "reasons": cl.get("reasons"), "e_op_pj": e_op * 1e12})
    time.sleep(2.0)

    # --- the skinny kernel on c4-shaped uniform residues --------------------------------------
    c = ctgen.CONFIGS["c4"]
    L = 4
    ps = ctgen.primes(c.L)[:L]
    d3s = [int(x) for x in args.d3.split(",")]
    d3max = max(d3s)
    eng = CpmmEngine(ctpt.Spec(c.fmt, c.N, c.d1, c.d2, d3max, ps), "cuda")
    eng.ctmat = torch.zeros(eng.sizes.ctmat_bytes, dtype=torch.uint8, device="cuda")
    fill_uniform(eng, c.R, ps, g)
    U = torch.randint(-c.u_bound, c.u_bound + 1, (c.d2, d3max), device="cuda", generator=g, dtype=torch.int64)
    assert eng.precompute(U) == 1
    R, d2 = c.R, c.d2
    e_B = None
    BW_stream = None
    for d3 in d3s:
        sp = dataclasses.replace(eng.spec, col_begin=0, col_end=d3)
        sz = ctpt.query_sizes(sp)
        AU = torch.empty(sz.out_AU_bytes // 4, dtype=torch.int32, device="cuda")
        BU = torch.empty(sz.out_BU_bytes // 4, dtype=torch.int32, device="cuda")
        ra = sz.rows_A

        def step():
            for l in range(L):
                ctpt.gemm_fused(sp, l, eng.ctmat, eng.plain, AU[l * d3 * ra:], BU[l * d3 * c.d1:])

        t, cl = sustained(step, calib(step), args.seconds, dev)
        t /= L  # per launch (one prime)
        nbytes = 4 * R * d2 + d3 * d2 + 4 * R * d3
        ops = 2 * 4 * R * d2 * d3  # 4 limb MACs per residue MAC, 2 ops per MAC
        P = cl.get("power_w_median")
        rec = {"case": "skinny", "kernel": "k_gemm_fused_t", "d3": d3, "ms_per_launch": t * 1e3,
               "gbs": nbytes / t / 1e9, "tops": ops / t / 1e12, "power_w_median": P, "sm_mhz": cl.get("sm_mhz"),
               "reasons": cl.get("reasons")}
        if e_B is None:  # d3 = 1 (the first case) calibrates the stream energy
            e_op_part = e_op * ops / t
            e_B = (P - P0 - e_op_part) / (nbytes / t)
            BW_stream = nbytes / t
            rec["e_B_pj_per_byte"] = e_B * 1e12
        bound = max(nbytes / BW_stream, ops / (TOPS_UNCAPPED * 1e12), (e_B * nbytes + e_op * ops) / (P_CAP - P0))
        rec.update({"t_hbm_ms": nbytes / BW_stream * 1e3, "t_power_ms": (e_B * nbytes + e_op * ops) / (P_CAP - P0) * 1e3,
                    "frac_hbm": (nbytes / BW_stream) / t, "frac_power": bound / t,
                    "power_pred_w": P0 + (e_B * nbytes + e_op * ops) / t})
        emit(rec)
        del AU, BU
        time.sleep(2.0)
    del eng
    torch.cuda.empty_cache()

    # --- k_gemm_tc on c3's GEMM shape ---------------------------------------------------------
    if not args.no_gemm:
        c = ctgen.CONFIGS["c3"]
        p = ctgen.primes(1)[0]
        eng = CpmmEngine(ctpt.Spec(c.fmt, c.N, c.d1, c.d2, c.d3, [p]), "cuda")
        eng.ctmat = torch.zeros(eng.sizes.ctmat_bytes, dtype=torch.uint8, device="cuda")
        fill_uniform(eng, c.R, [p], g)
        U = torch.randint(-c.u_bound, c.u_bound + 1, (c.d2, c.d3), device="cuda", generator=g, dtype=torch.int64)
        assert eng.precompute(U) == 1
        AU, BU = eng.alloc_outputs()
        ctpt.split(eng.spec, 0, eng.ctmat, eng.ws)

        def gemm():
            ctpt.gemm(eng.spec, 0, eng.ws, eng.plain, AU, BU)

        t, cl = sustained(gemm, calib(gemm), max(args.seconds, 4.0), dev)
        ops = 2 * 4 * c.R * c.d2 * c.d3
        dram = args.dram_gb_c3 * 1e9
        P = cl.get("power_w_median")
        t_pow = (e_B * dram + e_op * ops) / (P_CAP - P0)
        bound = max(dram / BW_stream, ops / (TOPS_UNCAPPED * 1e12), t_pow)
        emit({"case": "gemm", "kernel": "k_gemm_tc", "config": "c3 (one prime)", "ms_per_launch": t * 1e3,
              "tops": ops / t / 1e12, "dram_gb_per_launch": args.dram_gb_c3, "power_w_median": P,
              "sm_mhz": cl.get("sm_mhz"), "reasons": cl.get("reasons"), "t_tensor_at_cap_ms": ops / (tops_mma * 1e12) * 1e3,
              "t_power_ms": t_pow * 1e3, "frac_power": bound / t, "frac_mma_ceiling": (ops / t / 1e12) / tops_mma,
              "power_pred_w": P0 + (e_B * dram + e_op * ops) / t})
    summary = {"case": "summary", "P0_w": P0, "P_cap_w": P_CAP, "e_op_pj": e_op * 1e12,
               "e_B_pj_per_byte": e_B * 1e12 if e_B is not None else None, "bw_stream_gbs": (BW_stream or 0) / 1e9,
               "tops_mma_at_cap": tops_mma}
    emit(summary)


if __name__ == "__main__":
    main()
