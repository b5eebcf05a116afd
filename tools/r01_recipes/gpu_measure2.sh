#!/bin/bash
# GPU parity (all parity tests) + skinny sweep + rescale/c3a bench lines + ncu of k_gemm_fused at d3=256.
set -u
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q > $O/gpu_parity.log 2>&1; echo "rc=$?" >> $O/gpu_parity.log
timeout 600 python tools/bench_skinny.py --paths fused,split+gemm > $O/skinny.jsonl 2> $O/skinny.err
timeout 400 python bench.py --steps 5 --warmup 3 --rescale --no-cpu-baseline > $O/bench_rescale.json 2> $O/bench_rescale.err
timeout 400 python bench.py --steps 10 --warmup 3 --config c3a --no-cpu-baseline > $O/bench_c3a.json 2> $O/bench_c3a.err
SK="python tools/bench_skinny.py --L 1 --d3 256 --paths fused --steps 1 --warmup 1"
$SK > $O/plain_sk.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_gemm_fused -s 1 -c 1 -o $O/prof_fused256 -f $SK > $O/ncu_fused256.log 2>&1
echo done
