#!/bin/bash
# One `ncu --set full` capture of k_gemm_tc per GEMM-regime config (c2, c4, c3a), and of the
# layout and split kernels on c3 — each after its command exits 0 without ncu.
set -u
O=gpurun_out
for cfg in c2 c4 c3a; do
  SHORT="python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
  timeout 600 $SHORT > $O/ncu_plain_$cfg.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 2 -c 1 \
      -o $O/prof_gemm_tc_$cfg -f $SHORT > $O/ncu_gemm_$cfg.log 2>&1
  echo "$cfg rc=$?" >> $O/ncu_configs.log
done
SHORT="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 600 $SHORT > $O/ncu_plain_c3.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_layout_v4|k_split_rows" -c 2 \
    -o $O/prof_layout_split_c3 -f $SHORT > $O/ncu_layout_split.log 2>&1
echo "layout/split rc=$?" >> $O/ncu_configs.log
