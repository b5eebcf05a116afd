#!/bin/bash
set -u
O=gpurun_out
CTPT_GEMM_CS=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "(shapes_tcgen05 and 1cta) or (unsigned and 1cta) or rescale" > $O/cs_tests.log 2>&1
echo "rc=$?" >> $O/cs_tests.log
B="python bench.py --no-cpu-baseline --e2e-steps 0 --steps 20 --warmup 5"
for r in 1 2 3; do
  CTPT_GEMM_CS=1 timeout 300 $B > $O/cs_on_r$r.json 2>> $O/cs.err
  timeout 300 $B > $O/cs_off_r$r.json 2>> $O/cs.err
done
CTPT_GEMM_CS=1 timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --config c4 --steps 10 --warmup 3 > $O/cs_on_c4.json 2>> $O/cs.err
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --config c4 --steps 10 --warmup 3 > $O/cs_off_c4.json 2>> $O/cs.err
echo done
