#!/bin/bash
# CTA-pair GEMM vs single-CTA, interleaved on one box with the final code (c3, c4).
set -u
O=gpurun_out
B="python bench.py --no-cpu-baseline --e2e-steps 0"
for rep in 1 2; do
  CTPT_GEMM=2cta timeout 300 $B --steps 20 --warmup 5 > $O/re2_2cta_c3_r$rep.json 2>> $O/re2.err
  timeout 300 $B --steps 20 --warmup 5 > $O/re2_1cta_c3_r$rep.json 2>> $O/re2.err
done
CTPT_GEMM=2cta timeout 300 $B --steps 100 --warmup 5 > $O/re2_2cta_c3_100.json 2>> $O/re2.err
timeout 300 $B --steps 100 --warmup 5 > $O/re2_1cta_c3_100.json 2>> $O/re2.err
CTPT_GEMM=2cta timeout 300 $B --config c4 --steps 10 --warmup 3 > $O/re2_2cta_c4.json 2>> $O/re2.err
timeout 300 $B --config c4 --steps 10 --warmup 3 > $O/re2_1cta_c4.json 2>> $O/re2.err
echo done
