#!/bin/bash
# Raster group re-sweep with the limb tiles (c4: 8 / 16 / 32, c3: 12 / 16 / 24), interleaved.
set -u
O=gpurun_out
B="python bench.py --no-cpu-baseline --e2e-steps 0"
for rep in 1 2; do
  for g in 8 16 32; do
    CTPT_GROUP_J=$g timeout 300 $B --config c4 --steps 10 --warmup 3 > $O/g2_c4_${g}_r$rep.json 2>> $O/g2.err
  done
  for g in 12 16 24; do
    CTPT_GROUP_J=$g timeout 300 $B --steps 20 --warmup 5 > $O/g2_c3_${g}_r$rep.json 2>> $O/g2.err
  done
done
echo done
