#!/bin/bash
# ncu --set full of k_gemm_tc on c3 as bench.py runs it (prime 0's GEMM with prime 1's split inside),
# plus the launch list of the default short bench — each after the command exits 0 without ncu.
set -u
O=gpurun_out
SHORT="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 $SHORT > $O/c3_plain_short.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c3.csv $SHORT > $O/ncu_launches_c3.log 2>&1
echo "launches rc=$?" >> $O/ncu_c3.log
S1="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 600 $S1 > $O/c3_plain_s1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 3 -c 1 \
    -o $O/prof_gemm_tc_c3_sidesplit -f $S1 > $O/ncu_gemm_c3.log 2>&1
echo "full rc=$?" >> $O/ncu_c3.log
