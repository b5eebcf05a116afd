#!/bin/bash
# The bench's multi-rank strong-scaling path on ONE B200 (code-path check, not a scaling number):
# `bench.py --gpus 2` relaunches itself under torchrun; CTPT_BENCH_ONE_DEVICE=1 puts both ranks on
# cuda:0 and CTPT_DIST_BACKEND=gloo replaces NCCL (which refuses two ranks on one device).  The
# gather is the fused IPC one: rank 1's GEMM epilogues store into rank 0's buffers through a
# ctpt_ipc_open mapping (same device here; no kernel waits on another rank's).  Then c5 at N = 1
# (8 primes streamed as per-prime units).
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build_mr.log 2>&1
CTPT_BENCH_ONE_DEVICE=1 CTPT_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 3 --warmup 1 \
  --e2e-steps 1 > gpurun_out/r02/mr_c3_gpus2.json 2> gpurun_out/r02/mr_c3_gpus2.err; echo "rc=$?" >> gpurun_out/r02/mr_c3_gpus2.err
CTPT_BENCH_ONE_DEVICE=1 CTPT_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 3 --config c2 --steps 3 --warmup 1 \
  --e2e-steps 1 > gpurun_out/r02/mr_c2_gpus3.json 2> gpurun_out/r02/mr_c2_gpus3.err; echo "rc=$?" >> gpurun_out/r02/mr_c2_gpus3.err
timeout 1500 python bench.py --config c5 --steps 2 --warmup 1 --e2e-steps 1 > gpurun_out/r02/bench_c5_n1.json \
  2> gpurun_out/r02/bench_c5_n1.err; echo "rc=$?" >> gpurun_out/r02/bench_c5_n1.err
for f in mr_c3_gpus2 mr_c2_gpus3 bench_c5_n1; do echo "== $f"; tail -3 gpurun_out/r02/$f.err; head -c 1500 gpurun_out/r02/$f.json; echo; done
