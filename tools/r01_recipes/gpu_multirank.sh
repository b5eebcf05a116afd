#!/bin/bash
# The bench's multi-rank code path (barriers, max-over-ranks, e2e aggregation, rank-0 print) with
# 2 ranks on ONE B200 over gloo — a code-path check, not a scaling measurement.
set -u
O=gpurun_out
export CTPT_BENCH_ONE_DEVICE=1 CTPT_DIST_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 5 --warmup 3 --e2e-steps 2 > $O/mr_weak.json 2> $O/mr_weak.err
echo "weak rc=$?" >> $O/mr.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --gpus 2 --config c3 --shard --gather ipc --steps 2 --warmup 2 > $O/mr_ipc.json 2> $O/mr_ipc.err
echo "ipc rc=$?" >> $O/mr.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 \
  bench.py --gpus 2 --impl reference --steps 2 --warmup 1 > $O/mr_ref.json 2> $O/mr_ref.err
echo "ref rc=$?" >> $O/mr.log
