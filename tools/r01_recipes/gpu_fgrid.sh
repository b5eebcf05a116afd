#!/bin/bash
set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "skinny" > $O/fg_tests.log 2>&1
echo "rc=$?" >> $O/fg_tests.log
for rep in 1 2; do
  timeout 600 python tools/table4.py --rows 2-8 > $O/fg_new_r$rep.jsonl 2>> $O/fg.err
  CTPT_FUSED_GRID=sms timeout 600 python tools/table4.py --rows 2-8 > $O/fg_old_r$rep.jsonl 2>> $O/fg.err
done
timeout 900 python tools/bench_skinny.py --d3 64,128,256 --paths auto > $O/fg_sweep.jsonl 2>> $O/fg.err
