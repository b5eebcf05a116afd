#!/bin/bash
# 64-row tiles (two sub-tiles per U^T stage) for 128 < d3 <= 192 with 3 / 2 limb stages in TMEM
# (default build) vs 32-row tiles above 128 (build -DCTPT_FT_SUB2_MAX=128): parity, then the
# sweep at d3 = 144 .. 192 (+ 128, 224 as controls), interleaved, fresh box first.
O=gpurun_out/r02/sub2wide; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/ab_build.py /tmp/libctpt_old.so -DCTPT_FT_SUB2_MAX=128 >> $O/build.log 2>&1
for rep in 1 2 3; do
  timeout 600 python tools/bench_skinny.py --L 4 --d3 128,144,160,176,192,224 --paths fused > $O/new_$rep.jsonl 2>>$O/err.log
  CTPT_LIB=/tmp/libctpt_old.so timeout 600 python tools/bench_skinny.py --L 4 --d3 144,160,176,192 --paths fused > $O/old_$rep.jsonl 2>>$O/err.log
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "skinny or column_shard or fuzz or unsigned" \
  > $O/tests.log 2>&1; echo "tests_rc=$?" >> $O/tests.log; tail -2 $O/tests.log
python tools/ab_build.py /tmp/libctpt_dbg.so -DCTPT_DEBUG_CHECKS >> $O/build.log 2>&1
CTPT_LIB=/tmp/libctpt_dbg.so timeout 600 python tools/sanitize_cases.py --cases fused_wrap --stress 3 > $O/checked.log 2>&1; tail -1 $O/checked.log
timeout 600 python tools/sanitize_cases.py --cases fused_wrap --stress 10 > $O/stress.log 2>&1; tail -1 $O/stress.log
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r02/sub2wide/*.jsonl')):
    for l in open(f):
        d = json.loads(l)
        print(f.split('/')[-1], d['d3'], d['kernel'], '%.3f' % d['roofline']['frac'], '%.3f ms' % d['avg_launch_ms'], d.get('clocks', {}).get('sm_mhz'))
PY
