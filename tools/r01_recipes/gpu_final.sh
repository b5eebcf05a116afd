#!/bin/bash
# Round-end style verification on one B200: build, smoke, the whole -m gpu suite, the default
# bench line, and the ncu launch list of a short bench command.
set -u
O=gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > $O/gpu_all.log 2>&1; echo "rc=$?" >> $O/gpu_all.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
SHORT="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$SHORT > $O/plain_short.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $SHORT > $O/ncu_launches.log 2>&1
echo done
