#!/bin/bash
# Round 2, final: the default -m gpu suite must fit the round-end driver's 1200-s step (the three
# longest full-size cases run their reduced form by default, tests/test_gpu_configs.py), then the
# bench lines, the reference arm, smoke, the default bench's launch list, and last the full forms
# of the reduced cases (CTPT_SLOW=1).
O=gpurun_out/r02/final6; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
S=$(date +%s)
timeout 1200 python -m pytest tests -m gpu -q -x --durations=15 > $O/gpu_tests_default.log 2>&1; echo "tests_rc=$? wall_s=$(( $(date +%s) - S ))" >> $O/gpu_tests_default.log
tail -3 $O/gpu_tests_default.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke_rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench_rc=$?" >> $O/bench_c3.err
for cfg in c2 c3a c4; do
  timeout 900 python bench.py --config $cfg > $O/bench_$cfg.json 2> $O/bench_$cfg.err
done
timeout 1200 python bench.py --config c5 --steps 3 --warmup 1 --e2e-steps 1 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/reference_c3.json 2> $O/reference_c3.err
CMD="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
$CMD > $O/bench_short.json 2> $O/bench_short.err && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/c3_launches.csv $CMD > $O/ncu.log 2>&1
echo "ncu_rc=$?" >> $O/ncu.log
for f in $O/bench_*.json $O/reference_c3.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', '%.4e'%d['value'], d.get('pct_int8_datasheet'), d.get('roofline',{}).get('frac'), (d.get('e2e') or {}).get('value'), d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'))" 2>/dev/null; done
S=$(date +%s)
CTPT_SLOW=1 timeout 2400 python -m pytest tests/test_gpu_configs.py -m gpu -q -x --durations=10 \
  -k "all_primes or all_of_BU or test_config4_full_size" > $O/gpu_tests_slow.log 2>&1; echo "tests_rc=$? wall_s=$(( $(date +%s) - S ))" >> $O/gpu_tests_slow.log
tail -3 $O/gpu_tests_slow.log
