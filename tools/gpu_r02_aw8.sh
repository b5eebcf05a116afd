#!/bin/bash
# Quarter-K-block limb stages (AW = 8, 4 stages of 16 TMEM columns) vs half-K-block stages (AW = 16,
# 2 stages of 32 columns) for the 64-row skinny tiles at 193 <= d3 <= 224: the same TMEM, but a
# stage can be refilled while three others wait for the MMA.  Parity with the variant first.
O=gpurun_out/r02/aw8; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/ab_build.py /tmp/aw8.so -DCTPT_FT_AW8_FROM=224 >> $O/build.log 2>&1
CTPT_LIB=/tmp/aw8.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "skinny" > $O/tests_aw8.log 2>&1
echo "tests_rc=$?" >> $O/tests_aw8.log; tail -2 $O/tests_aw8.log
CTPT_LIB=/tmp/aw8.so timeout 900 python tools/sanitize_cases.py --cases fused_wrap,host --stress 3 > $O/stress_aw8.log 2>&1
echo "stress_rc=$?" >> $O/stress_aw8.log; tail -1 $O/stress_aw8.log
for rep in 1 2 3; do
  for v in aw16 aw8; do
    if [ $v = aw8 ]; then export CTPT_LIB=/tmp/aw8.so; else unset CTPT_LIB; fi
    timeout 600 python tools/bench_skinny.py --L 4 --d3 200,208,224 --paths fused --steps 10 > $O/${v}_$rep.jsonl 2>> $O/err.log
  done
done
unset CTPT_LIB
python - <<'PY'
import json, glob, collections
res = collections.defaultdict(list)
for f in sorted(glob.glob('gpurun_out/r02/aw8/*.jsonl')):
    v = f.split('/')[-1].split('_')[0]
    for l in open(f):
        d = json.loads(l)
        res[(d['d3'], v)].append(d['roofline']['frac'])
for k in sorted(res):
    print(k, ' '.join('%.3f' % x for x in res[k]))
PY
