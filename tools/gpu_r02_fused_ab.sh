#!/bin/bash
# Limbs-in-TMEM skinny kernel (k_gemm_fused_t) vs the limbs-in-shared-memory kernel (k_gemm_fused,
# build flag -DCTPT_FUSED_SMEM_LIMBS): parity first, then the c4-ciphertext skinny sweep interleaved.
mkdir -p gpurun_out/r02/fused_ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/fused_ab/build.log 2>&1
python tools/ab_build.py /tmp/libctpt_smemlimbs.so -DCTPT_FUSED_SMEM_LIMBS >> gpurun_out/r02/fused_ab/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "skinny or fuzz or graph or column_shard or raster or mv_column" \
  > gpurun_out/r02/fused_ab/tests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/r02/fused_ab/tests.log
tail -3 gpurun_out/r02/fused_ab/tests.log
if grep -q "tests_rc=0" gpurun_out/r02/fused_ab/tests.log; then
  for rep in 1 2; do
    for v in tmem smem; do
      if [ $v = smem ]; then export CTPT_LIB=/tmp/libctpt_smemlimbs.so; else unset CTPT_LIB; fi
      timeout 600 python tools/bench_skinny.py --L 2 --d3 32,64,96,128,192,256 --paths fused --steps 10 \
        > gpurun_out/r02/fused_ab/sweep_${v}_$rep.jsonl 2>> gpurun_out/r02/fused_ab/err.log
      python - <<PY
import json
for l in open('gpurun_out/r02/fused_ab/sweep_${v}_$rep.jsonl'):
    d=json.loads(l); print('$v $rep d3=%d frac=%.3f ms=%.3f' % (d['d3'], d['roofline']['frac'], d['avg_launch_ms']))
PY
    done
  done
fi
