#!/bin/bash
# k_gemm_tc with a serpentine K order (odd waves walk K backwards, so the U^T panel lines the last
# wave touched are the next wave's first reads) vs K always ascending (-DCTPT_TC_NO_SERPENTINE).
# Parity first (small shapes with CTAs looping over several tiles, stress over grid caps, c4 full
# size), then c3 / c4 interleaved, then the DRAM bytes of one c4 GEMM launch for each build.
O=gpurun_out/r02/serpentine; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/ab_build.py /tmp/noserp.so -DCTPT_TC_NO_SERPENTINE >> $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tcgen05 or column_shard or unsigned or config2" > $O/tests.log 2>&1
echo "tests_rc=$?" >> $O/tests.log; tail -2 $O/tests.log
timeout 900 python tools/sanitize_cases.py --cases gemm,gemm_side,gemm_u8,host --stress 3 > $O/stress.log 2>&1
echo "stress_rc=$?" >> $O/stress.log; tail -2 $O/stress.log
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -k "config4_full_size" > $O/tests_c4.log 2>&1
echo "tests_rc=$?" >> $O/tests_c4.log; tail -2 $O/tests_c4.log
for rep in 1 2 3; do
  for v in serp asc; do
    if [ $v = asc ]; then export CTPT_LIB=/tmp/noserp.so; else unset CTPT_LIB; fi
    timeout 600 python bench.py --config c3 --e2e-steps 0 --no-cpu-baseline > $O/c3_${v}_$rep.json 2>> $O/err.log
    timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/c4_${v}_$rep.json 2>> $O/err.log
  done
done
unset CTPT_LIB
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r02/serpentine/c*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    r = d['roofline']
    print(f.split('/')[-1], '%.4e' % d['value'], '%.3f ms' % r['avg_launch_ms'], d['clocks'].get('sm_mhz'))
PY
# DRAM bytes per c4 GEMM launch (one prime, no side split), both builds
CMD="python bench.py --config c4 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --split-overlap off"
$CMD > $O/plain_ncu.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_gemm_tc -s 2 -c 1 \
  --csv --log-file $O/c4_dram_serp.csv $CMD > $O/ncu_serp.log 2>&1
CTPT_LIB=/tmp/noserp.so ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_gemm_tc -s 2 -c 1 \
  --csv --log-file $O/c4_dram_asc.csv $CMD > $O/ncu_asc.log 2>&1
grep -h dram__bytes $O/c4_dram_*.csv | cut -d, -f5,13-15
