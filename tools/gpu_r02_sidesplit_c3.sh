#!/bin/bash
# c3: the next prime's limb split inside the GEMM (--split-overlap on) vs standalone splits (auto = off
# for d3 > 8192), interleaved, with the current kernels.
O=gpurun_out/r02/sidesplit_c3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for rep in 1 2 3 4; do
  for v in off on; do
    timeout 600 python bench.py --config c3 --split-overlap $v --e2e-steps 0 --no-cpu-baseline > $O/c3_${v}_$rep.json 2>> $O/err.log
  done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r02/sidesplit_c3/c*.json')):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f.split('/')[-1], '%.4e' % d['value'], '%.3f ms' % d['roofline']['avg_launch_ms'], '%.2f ms/step' % d['ms_per_step'], d['clocks'].get('sm_mhz'))
PY
