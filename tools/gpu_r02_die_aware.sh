#!/bin/bash
# EXPERIMENT: die-aware raster for k_gemm_tc (tools/ab/gemm_tc_die_aware.cuh) against the default, c3 and
# c4 interleaved on one box; sampled parity from the bench's oracle leg; DRAM bytes per launch (ncu).
O=gpurun_out/r02/die_aware3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
rm -rf /tmp/absrc /tmp/include && mkdir -p /tmp/absrc && cp -r paper_2503_16080_b200/csrc /tmp/absrc/ && cp -r include /tmp/include && \
  cp tools/ab/gemm_tc_die_aware.cuh /tmp/absrc/csrc/gemm_tc.cuh
python tools/ab_build.py /tmp/die.so --src=/tmp/absrc/csrc >> $O/build.log 2>&1
ls -la /tmp/die.so >> $O/build.log
# parity first: the bench's oracle leg compares ~15 M outputs of the last timed step
CTPT_LIB=/tmp/die.so timeout 600 python bench.py --e2e-steps 0 > $O/c3_die_parity.json 2> $O/c3_die_parity.err
echo "rc=$?" >> $O/c3_die_parity.err
CTPT_LIB=/tmp/die.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "tcgen05 or config2" > $O/tests_die.log 2>&1; echo "tests_rc=$?" >> $O/tests_die.log
tail -2 $O/tests_die.log
for rep in 1 2 3; do
  for v in default die; do
    if [ $v = die ]; then export CTPT_LIB=/tmp/die.so; else unset CTPT_LIB; fi
    timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 > $O/c3_${v}_$rep.json 2>> $O/err.log
  done
done
for rep in 1; do
  for v in default die; do
    if [ $v = die ]; then export CTPT_LIB=/tmp/die.so; else unset CTPT_LIB; fi
    timeout 600 python bench.py --config c4 --no-cpu-baseline --e2e-steps 0 > $O/c4_${v}_$rep.json 2>> $O/err.log
  done
done
for v in default die; do
  if [ $v = die ]; then export CTPT_LIB=/tmp/die.so; else unset CTPT_LIB; fi
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_gemm_tc --launch-skip 6 -c 3 --csv --log-file $O/c3_dram_$v.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/ncu_$v.log 2>&1
done
unset CTPT_LIB
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r02/die_aware3/c*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    r = d['roofline']
    print(f.split('/')[-1], '%.4e' % d['value'], '%.3f ms' % r['avg_launch_ms'], d['clocks'].get('sm_mhz'), (d.get('cpu_baseline') or {}).get('parity_on_sample'))
PY
grep -h "die-aware\|die probe" $O/*.err $O/*.log $O/*.json 2>/dev/null | sort -u | head -12
grep -h "dram__bytes" $O/c3_dram_*.csv | cut -d, -f5,13- | head -12
