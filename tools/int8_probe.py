"""Measured INT8 tensor-core ceiling on this GPU: cuBLASLt int8 GEMM via torch._int_mm
(16384^3, burst = best of 10, sustained = back to back for 4 s), as MEASURED_PEAKS.json
does for bf16.  Context for the roofline of k_gemm_tc."""
import json
import time

import torch


def main(n=16384):
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    try:
        torch._int_mm(a, b)
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"int8_probe": "unavailable", "why": str(e)[:200]}))
        return
    torch.cuda.synchronize()
    ops = 2.0 * n ** 3
    best = 1e9
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch._int_mm(a, b)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    t0 = time.time()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    k = 0
    while time.time() - t0 < 4.0:
        for _ in range(8):
            torch._int_mm(a, b)
        k += 8
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    sus = s.elapsed_time(e) / 1e3 / k
    print(json.dumps({"int8_probe": "torch._int_mm (cuBLASLt) int8->int32", "n": n,
                      "burst_tops": ops / best / 1e12, "sustained_tops": ops / sus / 1e12}))


if __name__ == "__main__":
    main()
