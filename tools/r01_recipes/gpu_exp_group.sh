#!/bin/bash
# Raster-group re-measurement (interleaved on one box) + the bench's c1 graph mode and setup-stage rates.
set -u
O=gpurun_out
B="python bench.py --no-cpu-baseline --e2e-steps 0"
timeout 300 python bench.py --config c1 --steps 200 --warmup 20 --no-cpu-baseline > $O/c1_graph.json 2> $O/c1_graph.err
timeout 300 $B --config c1 --graph off --steps 200 --warmup 20 > $O/c1_eager.json 2> $O/c1_eager.err
for rep in 1 2; do
  for g in 16 24 32; do
    CTPT_GROUP_J=$g timeout 300 $B --steps 20 --warmup 5 > $O/c3_g${g}_r${rep}.json 2>> $O/group.err
  done
done
for rep in 1 2; do
  for g in 16 32; do
    CTPT_GROUP_J=$g timeout 300 $B --config c4 --steps 10 --warmup 3 > $O/c4_g${g}_r${rep}.json 2>> $O/group.err
  done
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/c3_setup.json 2> $O/c3_setup.err
echo done
