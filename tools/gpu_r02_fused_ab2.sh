#!/bin/bash
# (1) d3 <= 32: the raw-byte kernel k_gemm_mv vs the limbs-in-TMEM kernel; (2) 128 < d3 <= 256: the
# limbs-in-shared-memory kernel (default) vs 32-row limbs-in-TMEM tiles (-DCTPT_FUSED_T256).
mkdir -p gpurun_out/r02/fused_ab2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/fused_ab2/build.log 2>&1
python tools/ab_build.py /tmp/libctpt_t256.so -DCTPT_FUSED_T256 >> gpurun_out/r02/fused_ab2/build.log 2>&1
CTPT_LIB=/tmp/libctpt_t256.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "skinny or fuzz or column_shard or raster" \
  > gpurun_out/r02/fused_ab2/tests_t256.log 2>&1; echo "tests_rc=$?" >> gpurun_out/r02/fused_ab2/tests_t256.log
tail -2 gpurun_out/r02/fused_ab2/tests_t256.log
for rep in 1 2; do
  timeout 600 python tools/bench_skinny.py --L 2 --d3 1,8,16,32 --paths mv,fused --steps 10 > gpurun_out/r02/fused_ab2/small_$rep.jsonl 2>>gpurun_out/r02/fused_ab2/err.log
  for v in smem t256; do
    if [ $v = t256 ]; then export CTPT_LIB=/tmp/libctpt_t256.so; else unset CTPT_LIB; fi
    timeout 600 python tools/bench_skinny.py --L 2 --d3 160,192,224,256 --paths fused --steps 10 \
      > gpurun_out/r02/fused_ab2/big_${v}_$rep.jsonl 2>> gpurun_out/r02/fused_ab2/err.log
  done
  unset CTPT_LIB
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r02/fused_ab2/*.jsonl')):
    for l in open(f):
        d = json.loads(l); print(f.split('/')[-1], d['path'], 'd3=%d frac=%.3f ms=%.3f' % (d['d3'], d['roofline']['frac'], d['avg_launch_ms']))
PY
