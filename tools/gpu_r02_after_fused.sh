#!/bin/bash
# After the skinny-kernel consolidation: the skinny sweep first (fresh box), then parity, the
# checked build over every path, and stress repetitions.
mkdir -p gpurun_out/r02/after_fused
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/after_fused/build.log 2>&1
python tools/ab_build.py /tmp/libctpt_checked.so -DCTPT_DEBUG_CHECKS >> gpurun_out/r02/after_fused/build.log 2>&1
timeout 900 python tools/bench_skinny.py --L 4 --d3 1,16,32,64,96,128,160,192,224,256 --paths auto --steps 10 \
  > gpurun_out/r02/after_fused/sweep_L4.jsonl 2> gpurun_out/r02/after_fused/sweep.err
python - <<'PY'
import json
for l in open('gpurun_out/r02/after_fused/sweep_L4.jsonl'):
    d = json.loads(l)
    print('sweep', d['d3'], d['kernel'], d['u_plane'], '%.3f' % d['roofline']['frac'], '%.3f ms' % d['avg_launch_ms'])
PY
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused_gather.py tests/test_gpu_layout.py tests/test_c_client.py \
  tests/test_gpu_bench_multirank.py -q -x > gpurun_out/r02/after_fused/tests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/r02/after_fused/tests.log
tail -2 gpurun_out/r02/after_fused/tests.log
CTPT_LIB=/tmp/libctpt_checked.so timeout 1200 python tools/sanitize_cases.py --stress 3 > gpurun_out/r02/after_fused/checked_build.log 2>&1
echo "rc=$?" >> gpurun_out/r02/after_fused/checked_build.log; tail -3 gpurun_out/r02/after_fused/checked_build.log
timeout 1200 python tools/sanitize_cases.py --stress 10 --cases gemm,gemm_side,gemm_u8,fused_wrap,mv_tickets,rescale \
  > gpurun_out/r02/after_fused/stress_release.log 2>&1; echo "rc=$?" >> gpurun_out/r02/after_fused/stress_release.log
grep -c "mismatches=0" gpurun_out/r02/after_fused/stress_release.log; tail -2 gpurun_out/r02/after_fused/stress_release.log
