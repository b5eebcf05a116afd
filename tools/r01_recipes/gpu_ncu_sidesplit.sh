#!/bin/bash
# ncu --set full of k_gemm_tc with the next prime's split inside (bench default for d3 <= 8192): c2, c4.
set -u
O=gpurun_out
for cfg in c2 c4; do
  S1="python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
  timeout 600 $S1 > $O/ss_plain_$cfg.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 4 -c 1 \
      -o $O/prof_gemm_tc_${cfg}_sidesplit -f $S1 > $O/ncu_ss_$cfg.log 2>&1
  echo "$cfg rc=$?" >> $O/ncu_ss.log
done
