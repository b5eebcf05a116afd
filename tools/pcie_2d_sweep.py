#!/usr/bin/env python
"""Probe: PCIe rate of the host executor's strided (2-D) copies vs chunk width and vs the number of
concurrent copy streams per direction.

ctpt_matmul_host copies, per chunk of `rows` rows, the chunk's rows of every ciphertext column
(cudaMemcpy2DAsync, height = d2 segments of rows·4 bytes at the host pitch) and back the chunk's
rows of every output column.  The e2e chunk sweep (profiles/r02/e2e_chunks/) found narrower chunks
SLOWER end to end (c3: 1728-row chunks 117 ms vs 3456-row 90 ms per step) although the pipeline
model says the fill / drain shrinks with the chunk.  This times, for c3's shapes, per width:
one 2-D copy per direction alone and both directions at once, and the same bytes split over
k = 2 / 4 streams per direction (row bands of the 2-D copy: several copy engines in flight).
One JSON line per (rows, k).
"""
from __future__ import annotations

import json

import torch
from cuda.bindings import runtime as rt


def check(err):
    e = err[0] if isinstance(err, tuple) else err
    if e != rt.cudaError_t.cudaSuccess:
        raise RuntimeError(str(e))


def main():
    d2, total_rows = 16384, 20480  # c3: d2 = 16384, R = 20480 stacked rows (host pitch 80 KB)
    pitch = total_rows * 4
    max_rows = 5120
    host = torch.empty(d2 * total_rows, dtype=torch.int32).pin_memory()
    host2 = torch.empty(d2 * total_rows, dtype=torch.int32).pin_memory()
    dev = torch.empty(d2 * max_rows, dtype=torch.int32, device="cuda")
    dev2 = torch.empty(d2 * max_rows, dtype=torch.int32, device="cuda")
    H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost
    streams = [torch.cuda.Stream() for _ in range(8)]

    def run(rows, k, dirs, reps=4):
        width = rows * 4
        nbytes = width * d2
        band = d2 // k
        best = None
        for _ in range(reps):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream())
            ends = []
            for di, kind in enumerate(dirs):
                for i in range(k):
                    st = streams[di * 4 + i]
                    st.wait_event(e0)
                    h0 = i * band
                    if kind == "h2d":
                        check(rt.cudaMemcpy2DAsync(dev.data_ptr() + h0 * width, width, host.data_ptr() + h0 * pitch,
                                                   pitch, width, band, H2D, st.cuda_stream))
                    else:
                        check(rt.cudaMemcpy2DAsync(host2.data_ptr() + h0 * pitch, pitch, dev2.data_ptr() + h0 * width,
                                                   width, width, band, D2H, st.cuda_stream))
                    e = torch.cuda.Event(enable_timing=True)
                    e.record(st)
                    ends.append((kind, e))
            torch.cuda.synchronize()
            t = {}
            for kind, e in ends:
                t[kind] = max(t.get(kind, 0.0), e0.elapsed_time(e) / 1e3)
            best = t if best is None else {x: min(best[x], t[x]) for x in t}
        return {x: nbytes / best[x] / 1e9 for x in best}

    for rows in (640, 1024, 1280, 1728, 2048, 2560, 3456, 5120):
        for k in (1, 2, 4):
            out = {"rows": rows, "width_B": rows * 4, "streams_per_dir": k,
                   "h2d_alone": run(rows, k, ["h2d"])["h2d"], "d2h_alone": run(rows, k, ["d2h"])["d2h"]}
            both = run(rows, k, ["h2d", "d2h"])
            out["h2d_both"], out["d2h_both"] = both["h2d"], both["d2h"]
            print(json.dumps(out), flush=True)
    # contiguous reference (same bytes as the 3456-row chunk)
    nb = 3456 * 4 * d2
    for k in (1,):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(streams[0])
        check(rt.cudaMemcpyAsync(dev.data_ptr(), host.data_ptr(), nb, H2D, streams[0].cuda_stream))
        e1.record(streams[0])
        torch.cuda.synchronize()
        print(json.dumps({"contiguous_h2d_gbs": nb / (e0.elapsed_time(e1) / 1e3) / 1e9}))


if __name__ == "__main__":
    main()
