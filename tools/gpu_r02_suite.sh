#!/bin/bash
# Round 2: the whole -m gpu suite (incl. the slow full-prime c3 check), smoke(), the default bench
# line, each to its own log under gpurun_out/r02/.
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/r02/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/r02/gpu_tests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/r02/gpu_tests.log
python bench.py > gpurun_out/r02/bench_c3.json 2> gpurun_out/r02/bench_c3.err; echo "bench_rc=$?" >> gpurun_out/r02/bench_c3.err
tail -3 gpurun_out/r02/gpu_tests.log; tail -1 gpurun_out/r02/smoke.log; head -c 600 gpurun_out/r02/bench_c3.json
