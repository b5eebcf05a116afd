#!/bin/bash
# CTA-pair fused kernel (k_gemm_fused2, 128 < d3 <= 256): parity, then the skinny sweep A/B.
set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "skinny" > $O/fused2_tests.log 2>&1
echo "rc=$?" >> $O/fused2_tests.log
tail -3 $O/fused2_tests.log
for rep in 1 2; do
  timeout 600 python tools/bench_skinny.py --d3 129,192,256 --paths fused > $O/sweep_pair_g2_r$rep.jsonl 2>> $O/fused2.err
  CTPT_F2_GROUPS=1 timeout 600 python tools/bench_skinny.py --d3 129,192,256 --paths fused > $O/sweep_pair_g1_r$rep.jsonl 2>> $O/fused2.err
  CTPT_FUSED2=off timeout 600 python tools/bench_skinny.py --d3 129,192,256 --paths fused > $O/sweep_single_r$rep.jsonl 2>> $O/fused2.err
done
echo done
