#!/bin/bash
# Serpentine K order by wave (mode 1) or by r-tile (mode 2: CTAs of an r-tile straddling two waves walk
# K the same way) against larger raster groups on c3: with U^T kept resident across waves, a group of
# 24 / 32 j-tiles streams X 5.3 / 4 times per prime instead of 8.  DRAM bytes per launch by ncu.
O=gpurun_out/r02/serp_group; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/ab_build.py /tmp/s1.so -DCTPT_TC_SERPENTINE_MODE=1 >> $O/build.log 2>&1
python tools/ab_build.py /tmp/s2.so -DCTPT_TC_SERPENTINE_MODE=2 >> $O/build.log 2>&1
CTPT_LIB=/tmp/s2.so timeout 900 python tools/sanitize_cases.py --cases gemm,gemm_side,gemm_u8 --stress 3 > $O/stress_s2.log 2>&1
echo "stress_rc=$?" >> $O/stress_s2.log; tail -1 $O/stress_s2.log
for rep in 1 2; do
  for G in 16 24 32; do
    for v in s0 s1 s2; do
      if [ $v = s0 ]; then unset CTPT_LIB; else export CTPT_LIB=/tmp/$v.so; fi
      timeout 600 python bench.py --config c3 --raster-group $G --e2e-steps 0 --no-cpu-baseline > $O/c3_g${G}_${v}_$rep.json 2>> $O/err.log
    done
  done
  for v in s0 s2; do
    if [ $v = s0 ]; then unset CTPT_LIB; else export CTPT_LIB=/tmp/$v.so; fi
    timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/c4_g16_${v}_$rep.json 2>> $O/err.log
  done
done
unset CTPT_LIB
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r02/serp_group/c*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    r = d['roofline']
    print(f.split('/')[-1], '%.4e' % d['value'], '%.3f ms' % r['avg_launch_ms'], d['clocks'].get('sm_mhz'))
PY
M="dram__bytes_read.sum,gpu__time_duration.sum"
for v in "s0 16" "s0 32" "s2 32" "s2 16"; do
  set -- $v
  if [ $1 = s0 ]; then unset CTPT_LIB; else export CTPT_LIB=/tmp/$1.so; fi
  CMD="python bench.py --config c3 --raster-group $2 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
  $CMD > $O/plain_$1_$2.log 2>&1 && ncu --metrics $M --clock-control none -k regex:k_gemm_tc -s 2 -c 1 --csv \
    --log-file $O/dram_c3_$1_g$2.csv $CMD > $O/ncu_$1_$2.log 2>&1
  python - "$O/dram_c3_$1_g$2.csv" <<'PY'
import csv, io, sys
txt = open(sys.argv[1]).read(); txt = txt[txt.index('"ID"'):]
print(sys.argv[1].split('/')[-1], [(r['Metric Name'], r['Metric Value']) for r in csv.DictReader(io.StringIO(txt))])
PY
done
