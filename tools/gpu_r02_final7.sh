#!/bin/bash
# Round 2, last check of HEAD (source hash 99bf561e, two host-pipeline parity cases added since
# final6): the default -m gpu suite inside the driver's 1200-s step, smoke, the default bench line.
O=gpurun_out/r02/final7; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
S=$(date +%s)
timeout 1200 python -m pytest tests -m gpu -q -x --durations=10 > $O/gpu_tests_default.log 2>&1; echo "tests_rc=$? wall_s=$(( $(date +%s) - S ))" >> $O/gpu_tests_default.log
tail -3 $O/gpu_tests_default.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke_rc=$?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench_rc=$?" >> $O/bench_c3.err
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_c3_driver_flags.json 2> $O/bench_c3_driver_flags.err
python -c "
import json
for f in ('bench_c3','bench_c3_driver_flags'):
    d=json.loads(open('$O/'+f+'.json').read().strip().splitlines()[-1])
    print(f, '%.4e'%d['value'], d.get('pct_int8_datasheet'), d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
