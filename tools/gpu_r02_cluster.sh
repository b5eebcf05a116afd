#!/bin/bash
# (Measured in round 2; the cluster variant lost and was removed, so -DCTPT_FT_CLUSTER no longer exists.)
# k_gemm_fused_t in 2-CTA clusters sharing each U^T stage by TMA multicast (default build) vs one CTA
# per U^T stream (-DCTPT_FT_CLUSTER=1): parity + checked build + stress first, then the skinny sweep
# interleaved.
O=gpurun_out/r02/cluster; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/ab_build.py /tmp/libctpt_cl1.so -DCTPT_FT_CLUSTER=1 >> $O/build.log 2>&1
python tools/ab_build.py /tmp/libctpt_dbg.so -DCTPT_DEBUG_CHECKS >> $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "skinny_fused" > $O/tests_quick.log 2>&1
rc=$?; echo "tests_rc=$rc" >> $O/tests_quick.log; tail -2 $O/tests_quick.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "skinny or column_shard or fuzz or unsigned or grid_cap" \
  > $O/tests.log 2>&1; echo "tests_rc=$?" >> $O/tests.log; tail -2 $O/tests.log
CTPT_LIB=/tmp/libctpt_dbg.so timeout 600 python tools/sanitize_cases.py --cases fused_wrap --stress 4 > $O/checked.log 2>&1; tail -1 $O/checked.log
timeout 600 python tools/sanitize_cases.py --cases fused_wrap --stress 10 > $O/stress.log 2>&1; tail -1 $O/stress.log
for rep in 1 2 3; do
  timeout 600 python tools/bench_skinny.py --L 4 --d3 16,64,128,160,192,224,256 --paths fused > $O/cl2_$rep.jsonl 2>>$O/err.log
  CTPT_LIB=/tmp/libctpt_cl1.so timeout 600 python tools/bench_skinny.py --L 4 --d3 16,64,128,160,192,224,256 --paths fused > $O/cl1_$rep.jsonl 2>>$O/err.log
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r02/cluster/*.jsonl')):
    for l in open(f):
        d = json.loads(l)
        print(f.split('/')[-1], d['d3'], '%.3f' % d['roofline']['frac'], '%.3f ms' % d['avg_launch_ms'], d.get('clocks', {}).get('sm_mhz'))
PY
