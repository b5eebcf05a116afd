#!/bin/bash
# ncu --set full of the final k_gemm_tc (limb tiles): c3 (no side split, the bench default) and c4
# (with the side split), each after the same command exited 0 without ncu.
set -u
O=gpurun_out
S3="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 600 $S3 > $O/nf_plain_c3.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 3 -c 1 -o $O/prof_gemm_tc_c3_tiles -f $S3 > $O/nf_c3.log 2>&1
echo "c3 rc=$?" >> $O/nf.log
S4="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 600 $S4 > $O/nf_plain_c4.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 4 -c 1 -o $O/prof_gemm_tc_c4_tiles -f $S4 > $O/nf_c4.log 2>&1
echo "c4 rc=$?" >> $O/nf.log
