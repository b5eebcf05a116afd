#!/bin/bash
# Two converter groups in the single-CTA fused kernel (CTPT_FUSED_LOAD=tma2): parity, C client, then
# the skinny sweep interleaved against the one-group TMA ring.
set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_c_client.py -m gpu -x -q -k "skinny or c_client" > $O/tma2_tests.log 2>&1
echo "rc=$?" >> $O/tma2_tests.log
for rep in 1 2; do
  CTPT_FUSED_LOAD=tma2 timeout 600 python tools/bench_skinny.py --d3 64,128,192,256 --paths fused > $O/sw_tma2_r$rep.jsonl 2>> $O/tma2.err
  timeout 600 python tools/bench_skinny.py --d3 64,128,192,256 --paths fused > $O/sw_tma_r$rep.jsonl 2>> $O/tma2.err
done
echo done
