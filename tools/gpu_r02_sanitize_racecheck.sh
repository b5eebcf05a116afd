#!/bin/bash
# compute-sanitizer --tool racecheck over every kernel path's small cases (tools/sanitize_cases.py),
# one tool per gpurun call (B200_PROFILING.md).  Log -> gpurun_out/r02/sanitize_racecheck.log
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build_racecheck.log 2>&1
timeout 3000 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 50 \
  --target-processes all python tools/sanitize_cases.py > gpurun_out/r02/sanitize_racecheck.log 2>&1
echo "sanitizer_rc=$?" >> gpurun_out/r02/sanitize_racecheck.log
tail -25 gpurun_out/r02/sanitize_racecheck.log
