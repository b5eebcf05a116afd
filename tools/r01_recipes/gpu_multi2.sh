#!/bin/bash
set -u
O=gpurun_out
for rep in 1 2; do
  timeout 600 python bench.py --rescale --steps 5 --warmup 3 --no-cpu-baseline > $O/mu2_on_resc_r$rep.json 2>> $O/mu2.err
  CTPT_GEMM_MULTI=off timeout 600 python bench.py --rescale --steps 5 --warmup 3 --no-cpu-baseline > $O/mu2_off_resc_r$rep.json 2>> $O/mu2.err
done
timeout 600 python tools/bench_modmm.py > $O/mu2_on_modmm.json 2>> $O/mu2.err
CTPT_GEMM_MULTI=off timeout 600 python tools/bench_modmm.py > $O/mu2_off_modmm.json 2>> $O/mu2.err
echo done
