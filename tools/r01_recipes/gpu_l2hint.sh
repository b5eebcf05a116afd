#!/bin/bash
# TMA L2 eviction hints in k_gemm_tc: U evict_last only (hint 2) x raster group, interleaved on one box.
set -u
O=gpurun_out
B="python bench.py --no-cpu-baseline --e2e-steps 0 --steps 20 --warmup 5"
for rep in 1 2; do
  timeout 300 $B > $O/l2h2_off_g16_r$rep.json 2>> $O/l2h2.err
  for g in 16 32 64 128; do
    CTPT_GROUP_J=$g CTPT_GEMM_L2HINT=2 timeout 300 $B > $O/l2h2_on_g${g}_r$rep.json 2>> $O/l2h2.err
  done
done
S1="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
for g in 16 32 64; do
  CTPT_GROUP_J=$g CTPT_GEMM_L2HINT=2 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_gemm_tc -s 3 -c 1 --csv $S1 > $O/l2h2_ncu_g$g.csv 2>> $O/l2h2.err
done
echo done
