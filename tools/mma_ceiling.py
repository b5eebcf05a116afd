#!/usr/bin/env python
"""Measured INT8 tensor-pipe ceiling for k_gemm_tc's MMA shape (tools/mma_ceiling/mma_ceiling.cu).

Every SM issues tcgen05.mma.kind::i8 (M = 128, N = 256, K = 32) back to back on operands resident
in shared memory — no TMA, no epilogue, no DRAM — for ~`--seconds`, with operand bytes drawn like
the real GEMM's (A = U + 8 ∈ [0, 16], B = uniform X-limb bytes) and, for reference, all-zero and
all-uniform operands.  One JSON line per case: TOP/s (2 ops per MAC), median SM clock, power,
throttle reasons.  Divide k_gemm_tc's achieved TOP/s by the "gemm-like" line for the fraction of
the power-limited tensor ceiling it reaches.

    python tools/mma_ceiling.py [--seconds 4]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SRC = os.path.join(ROOT, "tools", "mma_ceiling", "mma_ceiling.cu")
LIB = os.path.join(ROOT, "tools", "mma_ceiling", "libmma_ceiling.so")


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        import __graft_entry__ as g

        r = subprocess.run([g._nvcc()] + g.NVCC_FLAGS + ["-o", LIB, SRC], capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed for libmma_ceiling.so")
    return LIB


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=4.0)
    ap.add_argument("--mainloop", action="store_true",
                    help="also run k_gemm_tc's TMA + MMA main loop without its epilogue on c3-shaped operands: "
                         "real coordinates (mode 0, DRAM + L2 traffic) and always the same L2-resident "
                         "k-block (mode 1, no DRAM)")
    ap.add_argument("--launches", type=int, default=250)
    ap.add_argument("--skip-ceiling", action="store_true")
    ap.add_argument("--reuse", action="store_true", help="A-operand collector reuse probe")
    args = ap.parse_args()
    import torch

    from bench import ClockSampler

    lib = ctypes.CDLL(build())
    lib.mma_ceiling_run.restype = ctypes.c_int
    lib.mma_ceiling_run.argtypes = [ctypes.c_int, ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_uint,
                                    ctypes.POINTER(ctypes.c_float), ctypes.c_void_p]
    torch.cuda.init()
    blocks = torch.cuda.get_device_properties(0).multi_processor_count
    macs_per_iter = 4 * 128 * 256 * 32
    cases = [("gemm-like: A in [0,16], B uniform", 16, 255), ("zero operands", 0, 0),
             ("uniform operands", 255, 255), ("gemm-like (repeat)", 16, 255)]
    ms = ctypes.c_float()
    # calibrate iterations for ~args.seconds at the zero-operand (uncapped) rate
    rc = lib.mma_ceiling_run(blocks, 2000, 0, 0, 1, ctypes.byref(ms), None)
    assert rc == 0, rc
    rc = lib.mma_ceiling_run(blocks, 20000, 0, 0, 1, ctypes.byref(ms), None)
    assert rc == 0, rc
    iters = int(20000 * args.seconds * 1e3 / max(ms.value, 1e-3))
    for name, a, b in ([] if args.skip_ceiling else cases):
        clk = ClockSampler(0)
        time.sleep(0.3)
        rc = lib.mma_ceiling_run(blocks, iters, a, b, 7, ctypes.byref(ms), None)
        cl = clk.stop()
        assert rc == 0, rc
        s = ms.value / 1e3
        tops = 2 * blocks * iters * macs_per_iter / s / 1e12
        print(json.dumps({"case": name, "a_max": a, "b_max": b, "blocks": blocks, "iters": iters, "seconds": s,
                          "tops": tops, "pct_of_4500": 100 * tops / 4500.0, "sm_mhz": cl.get("sm_mhz"),
                          "power_w_max": cl.get("power_w_max"), "reasons": cl.get("reasons"),
                          "per_clock_pct": (100 * tops * 1e12 / (2 * blocks * 8192 * cl["sm_mhz"] * 1e6)
                                            if cl.get("sm_mhz") else None)}), flush=True)
        time.sleep(2.0)
    if args.mainloop:
        mainloop(lib, args.launches)
    if args.reuse:
        reuse_probe(lib, blocks, iters // 2)


def reuse_probe(lib, blocks: int, iters: int):
    """Two MMAs per K slice sharing A, with / without .collector::a::fill / ::lastuse."""
    from bench import ClockSampler

    lib.mma_reuse_run.restype = ctypes.c_int
    lib.mma_reuse_run.argtypes = [ctypes.c_int, ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_uint,
                                  ctypes.c_int, ctypes.POINTER(ctypes.c_float), ctypes.c_void_p]
    ms = ctypes.c_float()
    macs = 8 * 128 * 256 * 32
    for reuse in (0, 1, 0, 1):
        clk = ClockSampler(0)
        time.sleep(0.3)
        rc = lib.mma_reuse_run(blocks, iters, 16, 255, 7, reuse, ctypes.byref(ms), None)
        cl = clk.stop()
        assert rc == 0, rc
        tops = 2 * blocks * iters * macs / (ms.value / 1e3) / 1e12
        print(json.dumps({"case": "A shared by 2 MMAs, collector reuse" if reuse else "A shared by 2 MMAs, no hint",
                          "tops": tops, "sm_mhz": cl.get("sm_mhz"), "power_w_max": cl.get("power_w_max"),
                          "per_clock_pct": (100 * tops * 1e12 / (2 * blocks * 8192 * cl["sm_mhz"] * 1e6)
                                            if cl.get("sm_mhz") else None)}), flush=True)
        time.sleep(2.0)


def mainloop(lib, launches: int):
    import torch

    from bench import ClockSampler

    lib.mainloop_probe_run.restype = ctypes.c_int
    lib.mainloop_probe_run.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_longlong,
                                       ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_float), ctypes.c_void_p]
    R, K, d3 = 20480, 16384, 16384  # c3: one prime's stacked rows, d2, d3
    g = torch.Generator(device="cuda").manual_seed(0)
    u = torch.randint(0, 17, (d3, K), dtype=torch.uint8, device="cuda", generator=g)
    x = torch.randint(0, 256, (4, R, K), dtype=torch.uint8, device="cuda", generator=g)
    x[3] >>= 1  # the top limb of a 31-bit residue has 7 bits
    ms = ctypes.c_float()
    stream = torch.cuda.current_stream().cuda_stream
    macs = 4 * R * K * d3
    for mode, name in [(0, "main loop, real coordinates (DRAM + L2), no epilogue"),
                       (1, "main loop, one L2-resident k-block (no DRAM), no epilogue"),
                       (2, "main loop, real coordinates, X in 32-KB tile-contiguous blocks"),
                       (6, "main loop, X and U^T both tile-contiguous"),
                       (2, "main loop, tile-contiguous X (repeat)"),
                       (6, "main loop, X and U^T tile-contiguous (repeat)")]:
        rc = lib.mainloop_probe_run(u.data_ptr(), x.data_ptr(), R, K, d3, 16, mode, 3, ctypes.byref(ms), stream)
        assert rc == 0, rc
        clk = ClockSampler(0)
        time.sleep(0.3)
        rc = lib.mainloop_probe_run(u.data_ptr(), x.data_ptr(), R, K, d3, 16, mode, launches, ctypes.byref(ms), stream)
        cl = clk.stop()
        assert rc == 0, rc
        tops = 2 * macs / (ms.value / 1e3) / 1e12
        print(json.dumps({"case": name, "mode": mode, "launches": launches, "ms_per_launch": ms.value, "tops": tops,
                          "sm_mhz": cl.get("sm_mhz"), "power_w_max": cl.get("power_w_max"),
                          "reasons": cl.get("reasons"),
                          "per_clock_pct": (100 * tops * 1e12 / (2 * 148 * 8192 * cl["sm_mhz"] * 1e6)
                                            if cl.get("sm_mhz") else None)}), flush=True)
        time.sleep(2.0)


if __name__ == "__main__":
    main()
