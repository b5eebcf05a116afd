#!/bin/bash
# Serpentine K order only above the L2 footprint threshold (c4, c5 on; c3 off): c5 A/B, c3 / c4 check.
O=gpurun_out/r02/serpentine2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/ab_build.py /tmp/noserp.so -DCTPT_TC_NO_SERPENTINE >> $O/build.log 2>&1
for rep in 1 2; do
  for v in auto asc; do
    if [ $v = asc ]; then export CTPT_LIB=/tmp/noserp.so; else unset CTPT_LIB; fi
    timeout 1200 python bench.py --config c5 --steps 3 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $O/c5_${v}_$rep.json 2>> $O/err.log
    timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/c4_${v}_$rep.json 2>> $O/err.log
    timeout 600 python bench.py --config c3 --e2e-steps 0 --no-cpu-baseline > $O/c3_${v}_$rep.json 2>> $O/err.log
  done
done
unset CTPT_LIB
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r02/serpentine2/c*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    r = d['roofline']
    print(f.split('/')[-1], '%.4e' % d['value'], '%.3f ms' % r['avg_launch_ms'], d['clocks'].get('sm_mhz'))
PY
