#!/bin/bash
# One measurement pass on a B200 (run under gpurun): build, GPU parity, the skinny sweep,
# the default bench line, the ncu launch list of a short bench command, and one
# `ncu --set full` capture of each hot kernel (k_gemm_tc on c3, k_gemm_fused on c4 d3=128).
set -u
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $O/gpu_parity.log 2>&1; echo "rc=$?" >> $O/gpu_parity.log
timeout 600 python tools/bench_skinny.py > $O/skinny.jsonl 2> $O/skinny.err
timeout 400 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
SHORT="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$SHORT > $O/plain_short.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $SHORT > $O/ncu_launches.log 2>&1
$SHORT > $O/plain_short2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 3 -c 1 -o $O/prof_gemm_tc -f $SHORT > $O/ncu_gemm.log 2>&1
SK="python tools/bench_skinny.py --L 1 --d3 128 --paths fused --steps 1 --warmup 1"
$SK > $O/plain_sk.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_gemm_fused -s 1 -c 1 -o $O/prof_fused -f $SK > $O/ncu_fused.log 2>&1
echo done
