#!/bin/bash
# (Measured in round 2; 4 U^T + 6 raw stages won and the A/B macros were removed.)
# 32-row tiles (193 <= d3 <= 256): U^T stages vs raw stages in shared memory. Default 4 U^T + 6 raw
# (96 KB of X in flight) vs 3 + 8 (128 KB) vs 2 + 10 (160 KB); interleaved on one box.
O=gpurun_out/r02/wide_stages; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/ab_build.py /tmp/u3r8.so -DCTPT_FT_US_WIDE=3 -DCTPT_FT_RAW_WIDE=8 >> $O/build.log 2>&1
python tools/ab_build.py /tmp/u2r10.so -DCTPT_FT_US_WIDE=2 -DCTPT_FT_RAW_WIDE=10 >> $O/build.log 2>&1
for rep in 1 2 3; do
  timeout 600 python tools/bench_skinny.py --L 4 --d3 208,224,256 --paths fused > $O/u4r6_$rep.jsonl 2>>$O/err.log
  CTPT_LIB=/tmp/u3r8.so timeout 600 python tools/bench_skinny.py --L 4 --d3 208,224,256 --paths fused > $O/u3r8_$rep.jsonl 2>>$O/err.log
  CTPT_LIB=/tmp/u2r10.so timeout 600 python tools/bench_skinny.py --L 4 --d3 208,224,256 --paths fused > $O/u2r10_$rep.jsonl 2>>$O/err.log
done
for v in u3r8 u2r10; do
  CTPT_LIB=/tmp/$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "skinny or column_shard" > $O/tests_$v.log 2>&1
  echo "tests_rc=$?" >> $O/tests_$v.log; tail -2 $O/tests_$v.log
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r02/wide_stages/*.jsonl')):
    for l in open(f):
        d = json.loads(l)
        print(f.split('/')[-1], d['d3'], '%.3f' % d['roofline']['frac'], '%.3f ms' % d['avg_launch_ms'], d.get('clocks', {}).get('sm_mhz'))
PY
