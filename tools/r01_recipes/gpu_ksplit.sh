#!/bin/bash
# K split of the limb GEMM (CTPT_GEMM_KSPLIT): parity with 2 and 3 chunks, then interleaved A/B on c3 / c4.
set -u
O=gpurun_out
for ks in 2 3; do
  CTPT_GEMM_KSPLIT=$ks timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q \
    -k "(shapes_tcgen05 and 1cta) or (unsigned and 1cta) or rescale or multi_digit or split_overlap or max_d2 or adversarial or modmatmul or general_U" > $O/ks_tests_$ks.log 2>&1
  echo "ks=$ks rc=$?" >> $O/ks.log
done
B="python bench.py --no-cpu-baseline --e2e-steps 0"
for rep in 1 2; do
  for ks in 1 2 3; do
    CTPT_GEMM_KSPLIT=$ks timeout 300 $B --steps 20 --warmup 5 > $O/ks_c3_${ks}_r$rep.json 2>> $O/ks.err
  done
done
for ks in 1 2 4; do
  CTPT_GEMM_KSPLIT=$ks timeout 300 $B --config c4 --steps 10 --warmup 3 > $O/ks_c4_${ks}.json 2>> $O/ks.err
done
echo done
