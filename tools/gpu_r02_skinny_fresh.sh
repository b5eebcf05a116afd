#!/bin/bash
# The skinny sweep first thing on a fresh box (clocks sampled per point): L = 4 and L = 2 on c4's ciphertexts.
mkdir -p gpurun_out/r02/skinny_fresh
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/skinny_fresh/build.log 2>&1
timeout 900 python tools/bench_skinny.py --L 4 --d3 1,16,32,64,96,128,160,192,224,256 --paths auto --steps 10 \
  > gpurun_out/r02/skinny_fresh/sweep_L4.jsonl 2> gpurun_out/r02/skinny_fresh/err.log
timeout 900 python tools/bench_skinny.py --L 2 --d3 64,128,160,192,256 --paths auto --steps 10 \
  > gpurun_out/r02/skinny_fresh/sweep_L2.jsonl 2>> gpurun_out/r02/skinny_fresh/err.log
python - <<'PY'
import json
for f in ('sweep_L4', 'sweep_L2'):
    for l in open(f'gpurun_out/r02/skinny_fresh/{f}.jsonl'):
        d = json.loads(l)
        print(f, d['d3'], d['kernel'], '%.3f' % d['roofline']['frac'], '%.3f ms' % d['avg_launch_ms'], d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))
PY
