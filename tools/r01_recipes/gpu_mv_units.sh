#!/bin/bash
set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "mv" > $O/mvu_tests.log 2>&1
echo "rc=$?" >> $O/mvu_tests.log
timeout 900 python tools/table4.py --rows 1-8 > $O/mvu_table4.jsonl 2> $O/mvu.err
timeout 900 python tools/bench_skinny.py --d3 1,16,32 --paths auto > $O/mvu_sweep.jsonl 2>> $O/mvu.err
