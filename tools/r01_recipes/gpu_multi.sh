#!/bin/bash
# All k_U digits in one GEMM launch (k_gemm_tc<true>): parity, then A/B on the Rescale workload and Mod-PP-MM.
set -u
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q \
  -k "multi_digit or general_U or rescale or modmatmul or fuzz or split_overlap or k_split or struct_a" > $O/multi_tests.log 2>&1
echo "rc=$?" >> $O/multi_tests.log
for rep in 1 2; do
  timeout 600 python bench.py --rescale --steps 5 --warmup 3 --no-cpu-baseline > $O/mu_on_resc_r$rep.json 2>> $O/mu.err
  CTPT_GEMM_MULTI=off timeout 600 python bench.py --rescale --steps 5 --warmup 3 --no-cpu-baseline > $O/mu_off_resc_r$rep.json 2>> $O/mu.err
done
timeout 600 python tools/bench_modmm.py > $O/mu_on_modmm.json 2>> $O/mu.err
CTPT_GEMM_MULTI=off timeout 600 python tools/bench_modmm.py > $O/mu_off_modmm.json 2>> $O/mu.err
echo done
