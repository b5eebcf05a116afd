#!/bin/bash
# Operand-energy probe for the power-bound skinny regime: the same fused kernels with the current s8
# digit plane (U in [-8, 8]) vs a u8 plane (U + 8 in [0, 16], u_offset 0): what a row-sum
# correction in the fused kernels would buy at d3 = 128..256.  Interleaved.
mkdir -p gpurun_out/r02/u8_skinny
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/u8_skinny/build.log 2>&1
for rep in 1 2; do
  timeout 600 python tools/bench_skinny.py --L 4 --d3 128,160,192,224,256 --paths fused --plane never \
    > gpurun_out/r02/u8_skinny/s8_$rep.jsonl 2>>gpurun_out/r02/u8_skinny/err.log
  timeout 600 python tools/bench_skinny.py --L 4 --d3 128,160,192,224,256 --paths fused --plane always --u-shift 8 \
    > gpurun_out/r02/u8_skinny/u8_$rep.jsonl 2>>gpurun_out/r02/u8_skinny/err.log
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r02/u8_skinny/*.jsonl')):
    for l in open(f):
        d = json.loads(l)
        print(f.split('/')[-1], d['u_plane'], d['d3'], '%.3f' % d['roofline']['frac'], '%.3f ms' % d['avg_launch_ms'], d['clocks'].get('sm_mhz'))
PY
