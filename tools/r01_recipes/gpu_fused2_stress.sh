#!/bin/bash
# Stress the CTA-pair fused kernel (CTPT_FUSED2=pair): repeated sweeps per converter-group setting.
set -u
O=gpurun_out
for rep in 1 2 3 4 5 6 7 8; do
  for g in 2 1; do
    CTPT_FUSED2=pair CTPT_F2_GROUPS=$g timeout 300 python tools/bench_skinny.py --L 2 --steps 30 --warmup 3 --d3 129,256 --paths fused > $O/stress_g${g}_r$rep.jsonl 2> $O/stress_g${g}_r$rep.err
    echo "g=$g rep=$rep rc=$?" >> $O/stress.log
  done
done
CTPT_FUSED2=off timeout 300 python tools/bench_skinny.py --L 2 --steps 30 --warmup 3 --d3 129,256 --paths fused > $O/stress_single.jsonl 2> $O/stress_single.err
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "skinny" >> $O/stress.log 2>&1
echo done >> $O/stress.log
