#!/usr/bin/env python
"""Probe: is the e2e executor's strided (2-D) copy pattern slower than contiguous copies?

The host executor (ctpt_matmul_host) copies, per chunk, the chunk's rows of every ciphertext
column: cudaMemcpy2DAsync with `height` = d2 column segments of `width` bytes.  This measures,
for c3's chunk shape, H2D and D2H of the same bytes as one contiguous copy, as one 2-D copy, and
both directions at once.  Uses cuda-python's runtime bindings directly.
"""
from __future__ import annotations

import json

import torch
from cuda.bindings import runtime as rt


def check(err):
    e = err[0] if isinstance(err, tuple) else err
    if e != rt.cudaError_t.cudaSuccess:
        raise RuntimeError(str(e))
    return err[1:] if isinstance(err, tuple) and len(err) > 1 else None


def main():
    d2, chunk_rows, total_rows = 16384, 3456, 20480  # c3: R = 20480, R/6 rows per chunk
    width = chunk_rows * 4
    pitch = total_rows * 4
    host = torch.empty(d2 * total_rows, dtype=torch.int32).pin_memory()
    host2 = torch.empty(d2 * total_rows, dtype=torch.int32).pin_memory()
    dev = torch.empty(d2 * chunk_rows, dtype=torch.int32, device="cuda")
    dev2 = torch.empty(d2 * chunk_rows, dtype=torch.int32, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    nbytes = width * d2
    H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost

    def timed(fns, reps=5):
        best = None
        for _ in range(reps):
            torch.cuda.synchronize()
            evs = []
            for stream, fn in fns:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                fn(stream)
                e1.record(stream)
                evs.append((e0, e1))
            torch.cuda.synchronize()
            t = [a.elapsed_time(b) / 1e3 for a, b in evs]
            best = t if best is None else [min(x, y) for x, y in zip(best, t)]
        return best

    def h2d_contig(st):
        check(rt.cudaMemcpyAsync(dev.data_ptr(), host.data_ptr(), nbytes, H2D, st.cuda_stream))

    def h2d_2d(st):
        check(rt.cudaMemcpy2DAsync(dev.data_ptr(), width, host.data_ptr(), pitch, width, d2, H2D, st.cuda_stream))

    def d2h_contig(st):
        check(rt.cudaMemcpyAsync(host2.data_ptr(), dev2.data_ptr(), nbytes, D2H, st.cuda_stream))

    def d2h_2d(st):
        check(rt.cudaMemcpy2DAsync(host2.data_ptr(), pitch, dev2.data_ptr(), width, width, d2, D2H, st.cuda_stream))

    out = {"chunk_bytes": nbytes, "width": width, "height": d2}
    for name, fns in [("h2d_contig", [(s1, h2d_contig)]), ("h2d_2d", [(s1, h2d_2d)]),
                      ("d2h_contig", [(s2, d2h_contig)]), ("d2h_2d", [(s2, d2h_2d)]),
                      ("both_contig", [(s1, h2d_contig), (s2, d2h_contig)]),
                      ("both_2d", [(s1, h2d_2d), (s2, d2h_2d)])]:
        t = timed(fns)
        out[name] = [nbytes / x / 1e9 for x in t]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
