#!/bin/bash
# Host executor: graded ends (the call's first and last chunk cut into a quarter + the rest, so the
# pipeline's fill and drain shrink; -DCTPT_HOST_GRADED=1) against uniform chunks (=0): host-path
# parity per build, then the e2e leg of c3 / c2 (3 interleaved reps) and c5 (1 rep) on one box.
O=gpurun_out/r02/graded; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
# the variant lives in tools/ab/host_graded.patch (not kept: c3 93.5 vs 92.7 ms, c2 6.66 vs 6.75 ms, c5 tie)
rm -rf /tmp/absrc /tmp/include && mkdir -p /tmp/absrc && cp -r paper_2503_16080_b200/csrc /tmp/absrc/ && cp -r include /tmp/include && \
  patch -d /tmp/absrc -p2 < tools/ab/host_graded.patch >> $O/build.log 2>&1
python tools/ab_build.py /tmp/g0.so >> $O/build.log 2>&1
python tools/ab_build.py /tmp/g1.so --src=/tmp/absrc/csrc -DCTPT_HOST_GRADED=1 >> $O/build.log 2>&1
ls -la /tmp/g0.so /tmp/g1.so >> $O/build.log
for v in g0 g1; do
  CTPT_LIB=/tmp/$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "host" > $O/tests_$v.log 2>&1
  echo "tests_rc=$?" >> $O/tests_$v.log
  CTPT_LIB=/tmp/$v.so timeout 600 python tools/sanitize_cases.py --cases host --stress 3 > $O/stress_$v.log 2>&1
  echo "stress_rc=$?" >> $O/stress_$v.log
  echo "$v: $(tail -2 $O/tests_$v.log | tr '\n' ' ') $(tail -1 $O/stress_$v.log)"
done
for rep in 1 2 3; do
  for v in g0 g1; do
    CTPT_LIB=/tmp/$v.so timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 8 --no-cpu-baseline > $O/c3_${v}_$rep.json 2>> $O/err.log
    CTPT_LIB=/tmp/$v.so timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --e2e-steps 20 --no-cpu-baseline > $O/c2_${v}_$rep.json 2>> $O/err.log
  done
done
for v in g0 g1; do
  CTPT_LIB=/tmp/$v.so timeout 1200 python bench.py --config c5 --steps 2 --warmup 1 --e2e-steps 2 --no-cpu-baseline > $O/c5_${v}_1.json 2>> $O/err.log
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r02/graded/c*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    e = d.get('e2e') or {}
    print(f.split('/')[-1], 'e2e %.4e' % e.get('value', 0), '%.2f ms' % e.get('ms_per_step', 0), (e.get('pcie') or {}).get('frac_of_floor'))
PY
