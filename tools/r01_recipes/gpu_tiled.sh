#!/bin/bash
# Limbs in 32-KB tiles: GPU parity (GEMM paths), then interleaved A/B against the flat-layout build.
set -u
O=gpurun_out

B="python bench.py --no-cpu-baseline --e2e-steps 0"
for rep in 1 2; do
  timeout 300 $B --steps 20 --warmup 5 > $O/tl_new_c3_r$rep.json 2>> $O/tl.err
  CTPT_LIB=$PWD/tools/ab/libctpt_flat.so timeout 300 $B --steps 20 --warmup 5 > $O/tl_old_c3_r$rep.json 2>> $O/tl.err
done
timeout 300 $B --steps 100 --warmup 5 > $O/tl_new_c3_100.json 2>> $O/tl.err
CTPT_LIB=$PWD/tools/ab/libctpt_flat.so timeout 300 $B --steps 100 --warmup 5 > $O/tl_old_c3_100.json 2>> $O/tl.err
timeout 300 $B --config c4 --steps 10 --warmup 3 > $O/tl_new_c4.json 2>> $O/tl.err
CTPT_LIB=$PWD/tools/ab/libctpt_flat.so timeout 300 $B --config c4 --steps 10 --warmup 3 > $O/tl_old_c4.json 2>> $O/tl.err
timeout 300 $B --config c2 --steps 200 --warmup 10 > $O/tl_new_c2.json 2>> $O/tl.err
CTPT_LIB=$PWD/tools/ab/libctpt_flat.so timeout 300 $B --config c2 --steps 200 --warmup 10 > $O/tl_old_c2.json 2>> $O/tl.err
echo done
