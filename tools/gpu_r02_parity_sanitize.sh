#!/bin/bash
# parity suites of the small shapes, then one compute-sanitizer tool ($1: racecheck | synccheck | memcheck)
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build_ps.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke_ps.log 2>&1; tail -1 gpurun_out/r02/smoke_ps.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused_gather.py tests/test_gpu_layout.py tests/test_c_client.py \
  -q -x > gpurun_out/r02/parity_ps.log 2>&1; echo "tests_rc=$?" >> gpurun_out/r02/parity_ps.log; tail -2 gpurun_out/r02/parity_ps.log
if [ -n "$1" ]; then bash tools/gpu_r02_sanitize_$1.sh; fi
