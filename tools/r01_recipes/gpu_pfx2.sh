#!/bin/bash
# X-tile L2 prefetch by the group's leading CTA (CTPT_GEMM_PFX) re-measured with the limbs in 32-KB tiles.
set -u
O=gpurun_out
B="python bench.py --no-cpu-baseline --e2e-steps 0 --steps 20 --warmup 5"
for rep in 1 2; do
  for pf in 0 2 4 8; do
    CTPT_GEMM_PFX=$pf timeout 300 $B > $O/pfx2_${pf}_r$rep.json 2>> $O/pfx2.err
  done
done
echo done
