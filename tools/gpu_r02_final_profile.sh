#!/bin/bash
# Final measurements of round 2 on one box: every config's bench line, the skinny sweep, the c3
# launch list, and one ncu --set full capture of k_gemm_tc on c3 and on c4 (with the next prime's
# split inside it, the bench's launch configuration for d3 <= 8192).
set -x
mkdir -p gpurun_out/r02/final
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/final/build.log 2>&1
for cfg in c3 c1 c2 c3a c4; do
  python bench.py --config $cfg > gpurun_out/r02/final/bench_$cfg.json 2> gpurun_out/r02/final/bench_$cfg.err
done
python bench.py --config c3 --rescale --e2e-steps 0 > gpurun_out/r02/final/bench_c3_rescale.json 2> gpurun_out/r02/final/bench_c3_rescale.err
python bench.py --config modmm > gpurun_out/r02/final/bench_modmm.json 2> gpurun_out/r02/final/bench_modmm.err
python bench.py --config c5 --steps 3 --warmup 1 --e2e-steps 1 > gpurun_out/r02/final/bench_c5.json 2> gpurun_out/r02/final/bench_c5.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02/final/reference_c3.json 2> gpurun_out/r02/final/reference_c3.err
timeout 900 python tools/bench_skinny.py --L 4 --d3 1,16,32,64,96,128,160,192,224,256 --paths auto --steps 10 \
  > gpurun_out/r02/final/skinny_sweep.jsonl 2> gpurun_out/r02/final/skinny_sweep.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02/final/plain_c3_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/final/c3_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02/final/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 3 -c 1 -o gpurun_out/r02/final/prof_c3 \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02/final/ncu_c3.log 2>&1
python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02/final/plain_c4_short.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 4 -c 1 -o gpurun_out/r02/final/prof_c4 \
  python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02/final/ncu_c4.log 2>&1
for f in gpurun_out/r02/final/bench_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', '%.4e'%d['value'], d.get('pct_int8_datasheet'), d.get('roofline',{}).get('frac'), d.get('clocks',{}).get('sm_mhz'))" 2>/dev/null; done
