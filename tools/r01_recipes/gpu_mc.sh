#!/bin/bash
# Multicast-cluster GEMM (k_gemm_tc_mc): parity, then interleaved A/B against k_gemm_tc on c3 / c4.
set -u
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "shapes_tcgen05 or unsigned or column_shard or split_overlap or multi_digit" > $O/mc_tests.log 2>&1
echo "rc=$?" >> $O/mc_tests.log
B="python bench.py --no-cpu-baseline --e2e-steps 0"
for rep in 1 2; do
  CTPT_GEMM=mc timeout 300 $B --steps 20 --warmup 5 > $O/mc_c3_r$rep.json 2>> $O/mc.err
  timeout 300 $B --steps 20 --warmup 5 > $O/tc_c3_r$rep.json 2>> $O/mc.err
done
CTPT_GEMM=mc timeout 300 $B --steps 100 --warmup 5 > $O/mc_c3_100.json 2>> $O/mc.err
timeout 300 $B --steps 100 --warmup 5 > $O/tc_c3_100.json 2>> $O/mc.err
CTPT_GEMM=mc timeout 300 $B --config c4 --steps 10 --warmup 3 > $O/mc_c4.json 2>> $O/mc.err
timeout 300 $B --config c4 --steps 10 --warmup 3 > $O/tc_c4.json 2>> $O/mc.err
echo done
