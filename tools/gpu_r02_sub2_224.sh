#!/bin/bash
# 64-row tiles at 193 <= d3 <= 224 with two half-K-block limb stages (default build) vs 32-row tiles
# (-DCTPT_FT_SUB2_MAX=192); and half-K-block stages from NPMAX = 160 up (-DCTPT_FT_AW_FROM=160:
# 6 / 4 half stages at 160 / 192 instead of 3 / 2 whole ones). Parity + checked build + stress first.
O=gpurun_out/r02/sub2_224; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/ab_build.py /tmp/libctpt_old.so -DCTPT_FT_SUB2_MAX=192 >> $O/build.log 2>&1
python tools/ab_build.py /tmp/libctpt_aw.so -DCTPT_FT_AW_FROM=160 >> $O/build.log 2>&1
python tools/ab_build.py /tmp/libctpt_dbg.so -DCTPT_DEBUG_CHECKS >> $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "skinny_fused" > $O/tests_quick.log 2>&1
rc=$?; echo "tests_rc=$rc" >> $O/tests_quick.log; tail -2 $O/tests_quick.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "skinny or column_shard or fuzz or unsigned or grid_cap" \
  > $O/tests.log 2>&1; echo "tests_rc=$?" >> $O/tests.log; tail -2 $O/tests.log
CTPT_LIB=/tmp/libctpt_aw.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "skinny or column_shard" \
  > $O/tests_aw.log 2>&1; echo "tests_rc=$?" >> $O/tests_aw.log; tail -2 $O/tests_aw.log
CTPT_LIB=/tmp/libctpt_dbg.so timeout 600 python tools/sanitize_cases.py --cases fused_wrap --stress 3 > $O/checked.log 2>&1; tail -1 $O/checked.log
timeout 600 python tools/sanitize_cases.py --cases fused_wrap --stress 10 > $O/stress.log 2>&1; tail -1 $O/stress.log
for rep in 1 2 3; do
  timeout 600 python tools/bench_skinny.py --L 4 --d3 160,192,208,224,256 --paths fused > $O/new_$rep.jsonl 2>>$O/err.log
  CTPT_LIB=/tmp/libctpt_old.so timeout 600 python tools/bench_skinny.py --L 4 --d3 208,224 --paths fused > $O/old_$rep.jsonl 2>>$O/err.log
  CTPT_LIB=/tmp/libctpt_aw.so timeout 600 python tools/bench_skinny.py --L 4 --d3 160,192 --paths fused > $O/aw_$rep.jsonl 2>>$O/err.log
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r02/sub2_224/*.jsonl')):
    for l in open(f):
        d = json.loads(l)
        print(f.split('/')[-1], d['d3'], '%.3f' % d['roofline']['frac'], '%.3f ms' % d['avg_launch_ms'], d.get('clocks', {}).get('sm_mhz'))
PY
