#!/bin/bash
# X-panel L2 prefetch by one CTA per group (CTPT_GEMM_PFX = k-blocks ahead), interleaved on one box.
set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "shapes_tcgen05 and 1cta" > $O/pfx_tests.log 2>&1
CTPT_GEMM_PFX=8 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "shapes_tcgen05 and 1cta" >> $O/pfx_tests.log 2>&1
B="python bench.py --no-cpu-baseline --e2e-steps 0 --steps 20 --warmup 5"
for rep in 1 2; do
  for pf in 0 4 8 16; do
    CTPT_GEMM_PFX=$pf timeout 300 $B > $O/pfx_${pf}_r$rep.json 2>> $O/pfx.err
  done
done
for pf in 0 8; do
  CTPT_GEMM_PFX=$pf timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 100 --warmup 5 > $O/pfx_${pf}_100.json 2>> $O/pfx.err
done
echo done
