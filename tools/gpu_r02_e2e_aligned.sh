#!/bin/bash
# Host executor chunks cut separately within A's and B's rows (default now) vs fixed R/6-row chunks
# that straddle the A / B boundary (CTPT_E2E_CHUNK = the old size), c3 and c2, interleaved.
O=gpurun_out/r02/e2e_aligned; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "host" > $O/tests.log 2>&1; echo "tests_rc=$?" >> $O/tests.log; tail -2 $O/tests.log
for rep in 1 2 3; do
  CTPT_E2E_CHUNK=0 timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --e2e-steps 5 --no-cpu-baseline > $O/c3_aligned_$rep.json 2>> $O/err.log
  CTPT_E2E_CHUNK=3456 timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --e2e-steps 5 --no-cpu-baseline > $O/c3_fixed_$rep.json 2>> $O/err.log
  CTPT_E2E_CHUNK=0 timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --e2e-steps 10 --no-cpu-baseline > $O/c2_aligned_$rep.json 2>> $O/err.log
  CTPT_E2E_CHUNK=1408 timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --e2e-steps 10 --no-cpu-baseline > $O/c2_fixed_$rep.json 2>> $O/err.log
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r02/e2e_aligned/c*.json')):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    e = d['e2e']
    print(f.split('/')[-1], '%.4e' % e['value'], '%.2f ms' % e['ms_per_step'], 'floor %.3f' % e['pcie']['frac_of_floor'])
PY
