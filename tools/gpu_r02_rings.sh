#!/bin/bash
# k_gemm_tc: the single 48-KB-stage TMA ring (the default) against a variant with separate U^T / X
# rings of their own depths (tools/ab/gemm_tc_two_rings.cuh: 4 + 4 stages, or X 5 ahead with U^T 3 and
# one staging buffer per epilogue warp): parity + stress per build, then c3 / c4 interleaved on one
# box; then the power roofline (tools/power_roofline.py).
# History: this recipe first ran with the two-ring kernel as the default ("new") and the single ring
# as "old" (profiles/r02/rings/: the two-ring producer recomputed tile coordinates every k-block,
# 2.75e14 on c3; profiles/r02/rings2/ after that fix: old 3.80-3.81e14 / new 3.57-3.58 / 5+3 2.79-2.80
# on c3, 3.51 / 3.43 / 2.74 on c4) -> the single ring stayed.  Below: the same commands with the roles
# as they are now ("two" = the variant).
O=gpurun_out/r02/rings3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
rm -rf /tmp/absrc /tmp/include && mkdir -p /tmp/absrc && cp -r paper_2503_16080_b200/csrc /tmp/absrc/ && cp -r include /tmp/include && \
  cp tools/ab/gemm_tc_two_rings.cuh /tmp/absrc/csrc/gemm_tc.cuh
python tools/ab_build.py /tmp/two.so --src=/tmp/absrc/csrc >> $O/build.log 2>&1
python tools/ab_build.py /tmp/r531.so --src=/tmp/absrc/csrc -DCTPT_TC_XS=5 -DCTPT_TC_US=3 -DCTPT_TC_OUT_HALVES=1 >> $O/build.log 2>&1
ls -la /tmp/*.so >> $O/build.log
lib_of() { case $1 in two) echo /tmp/two.so;; r531) echo /tmp/r531.so;; *) echo "";; esac; }
for v in two r531; do
  L=$(lib_of $v); if [ -n "$L" ]; then export CTPT_LIB=$L; else unset CTPT_LIB; fi
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_c_client.py -q -x > $O/tests_$v.log 2>&1
  echo "tests_rc=$?" >> $O/tests_$v.log
  timeout 600 python tools/sanitize_cases.py --cases gemm,gemm_side,gemm_u8,host,rescale --stress 4 > $O/stress_$v.log 2>&1
  echo "stress_rc=$?" >> $O/stress_$v.log
  echo "$v: $(tail -2 $O/tests_$v.log | tr '\n' ' ') $(tail -1 $O/stress_$v.log)"
done
for rep in 1 2 3; do
  for v in default two r531; do
    L=$(lib_of $v); if [ -n "$L" ]; then export CTPT_LIB=$L; else unset CTPT_LIB; fi
    timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 > $O/c3_${v}_$rep.json 2>> $O/err.log
  done
done
for rep in 1 2; do
  for v in default two r531; do
    L=$(lib_of $v); if [ -n "$L" ]; then export CTPT_LIB=$L; else unset CTPT_LIB; fi
    timeout 600 python bench.py --config c4 --no-cpu-baseline --e2e-steps 0 > $O/c4_${v}_$rep.json 2>> $O/err.log
  done
done
unset CTPT_LIB
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r02/rings3/c*.json')):
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
