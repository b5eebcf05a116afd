#!/bin/bash
set -u
O=gpurun_out
CTPT_GEMM_EP32=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "(shapes_tcgen05 and 1cta) or (unsigned and 1cta) or split_overlap or rescale" > $O/ep32_tests.log 2>&1
echo "rc=$?" >> $O/ep32_tests.log
B="python bench.py --no-cpu-baseline --e2e-steps 0 --steps 20 --warmup 5"
for r in 1 2 3; do
  CTPT_GEMM_EP32=1 timeout 300 $B > $O/ep32_on_r$r.json 2>> $O/ep32.err
  timeout 300 $B > $O/ep32_off_r$r.json 2>> $O/ep32.err
done
echo done
