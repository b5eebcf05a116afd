#!/usr/bin/env python
"""What does a plain HBM stream cost in board power, next to the skinny kernel at d3 = 1?

tools/power_roofline.py found the skinny kernel drawing ≈ 995 W at d3 = 1 (X read once at the copy
bandwidth, almost no tensor work).  Is that the price of streaming HBM at full rate on this board,
or of this kernel's SM-side path (TMA → shared memory → LDS → PRMT → tcgen05.st)?  This probe runs,
back to back for `--seconds` each with nvidia-smi sampling (bench.ClockSampler): a device-to-device
copy (read + write), a read-only reduction (torch.sum over int32), and a fill (write-only), on 8-GiB
buffers (≫ L2).  Experiment only; torch's own kernels, not the product path.

    python tools/power_stream_probe.py [--seconds 3]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=3.0)
    args = ap.parse_args()
    import torch

    from bench import ClockSampler

    dev = torch.device("cuda", 0)
    n = 2 << 30  # int32 elements = 8 GiB
    a = torch.randint(0, 1 << 31, (n,), device=dev, dtype=torch.int32)
    b = torch.empty_like(a)

    def run(name, fn, nbytes):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        per = e0.elapsed_time(e1) / 1e3
        reps = max(3, int(args.seconds / per))
        clk = ClockSampler(dev)
        time.sleep(0.3)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        cl = clk.stop()
        t = e0.elapsed_time(e1) / 1e3 / reps
        print(json.dumps({"case": name, "gbs": nbytes / t / 1e9, "ms": t * 1e3, "power_w_median": cl.get("power_w_median"),
                          "power_w_max": cl.get("power_w_max"), "sm_mhz": cl.get("sm_mhz"), "reasons": cl.get("reasons")}),
              flush=True)
        time.sleep(2.0)

    clk = ClockSampler(dev)
    time.sleep(2.0)
    print(json.dumps({"case": "idle", "power_w_median": clk.stop().get("power_w_median")}), flush=True)
    run("copy (read + write)", lambda: b.copy_(a), 2 * 4 * n)
    run("read-only sum", lambda: a.sum(dtype=torch.int64), 4 * n)
    run("write-only fill", lambda: b.fill_(7), 4 * n)


if __name__ == "__main__":
    main()
