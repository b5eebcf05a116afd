#!/bin/bash
# k_gemm_tc with separate U^T / X TMA rings: X 5 stages ahead (U^T 3, one staging buffer per epilogue
# warp; or U^T 2, two buffers) vs the default 4 + 4 and vs the single 48-KB-stage ring it replaced
# (tools/ab/gemm_tc_single_ring.cuh): parity + stress per build, then c3 / c4 interleaved on one box.
# Then the power roofline (tools/power_roofline.py).
# (The first run of this recipe, profiles/r02/rings/, found the two-ring producer recomputing the tile
# coordinates with integer divisions every k-block: 2.75e14 on c3; fixed before this run -> rings2/.)
O=gpurun_out/r02/rings2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
rm -rf /tmp/oldsrc /tmp/include && mkdir -p /tmp/oldsrc && cp -r paper_2503_16080_b200/csrc /tmp/oldsrc/ && cp -r include /tmp/include && \
  cp tools/ab/gemm_tc_single_ring.cuh /tmp/oldsrc/csrc/gemm_tc.cuh
python tools/ab_build.py /tmp/old.so --src=/tmp/oldsrc/csrc >> $O/build.log 2>&1
python tools/ab_build.py /tmp/r531.so -DCTPT_TC_XS=5 -DCTPT_TC_US=3 -DCTPT_TC_OUT_HALVES=1 >> $O/build.log 2>&1
ls -la /tmp/*.so >> $O/build.log
lib_of() { case $1 in old) echo /tmp/old.so;; r531) echo /tmp/r531.so;; r522) echo /tmp/r522.so;; *) echo "";; esac; }
for v in new r531; do
  L=$(lib_of $v); if [ -n "$L" ]; then export CTPT_LIB=$L; else unset CTPT_LIB; fi
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_c_client.py -q -x > $O/tests_$v.log 2>&1
  echo "tests_rc=$?" >> $O/tests_$v.log
  timeout 600 python tools/sanitize_cases.py --cases gemm,gemm_side,gemm_u8,host,rescale --stress 4 > $O/stress_$v.log 2>&1
  echo "stress_rc=$?" >> $O/stress_$v.log
  echo "$v: $(tail -2 $O/tests_$v.log | tr '\n' ' ') $(tail -1 $O/stress_$v.log)"
done
for rep in 1 2 3; do
  for v in old new r531; do
    L=$(lib_of $v); if [ -n "$L" ]; then export CTPT_LIB=$L; else unset CTPT_LIB; fi
    timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 > $O/c3_${v}_$rep.json 2>> $O/err.log
  done
done
for rep in 1 2; do
  for v in old new r531; do
    L=$(lib_of $v); if [ -n "$L" ]; then export CTPT_LIB=$L; else unset CTPT_LIB; fi
    timeout 600 python bench.py --config c4 --no-cpu-baseline --e2e-steps 0 > $O/c4_${v}_$rep.json 2>> $O/err.log
  done
done
unset CTPT_LIB
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r02/rings2/c*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    r = d['roofline']
    print(f.split('/')[-1], '%.4e' % d['value'], '%.3f ms' % r['avg_launch_ms'], r.get('frac'), d['clocks'].get('sm_mhz'))
PY
P=gpurun_out/r02/power; mkdir -p $P
timeout 900 python tools/power_roofline.py --seconds 3 --d3 1,128,192,256 > $P/power_roofline.jsonl 2> $P/power_roofline.err
echo "rc=$?" >> $P/power_roofline.err
tail -3 $P/power_roofline.err; cat $P/power_roofline.jsonl
