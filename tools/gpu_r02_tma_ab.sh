#!/bin/bash
# TMA-store epilogue: parity (GPU parity/gather/layout/C-client tests), then the c3/c4 bench
# interleaved against a build with the 16-byte STG epilogue (-DCTPT_NO_TMA_STORE), then the
# multi-rank code path (tools/gpu_r02_multirank.sh).
mkdir -p gpurun_out/r02/tma_ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/tma_ab/build.log 2>&1
python tools/ab_build.py /tmp/libctpt_stg.so -DCTPT_NO_TMA_STORE >> gpurun_out/r02/tma_ab/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused_gather.py tests/test_gpu_layout.py \
  tests/test_c_client.py -q -x > gpurun_out/r02/tma_ab/tests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/r02/tma_ab/tests.log
tail -2 gpurun_out/r02/tma_ab/tests.log
for rep in 1 2 3; do
  for v in tma stg; do
    if [ $v = stg ]; then export CTPT_LIB=/tmp/libctpt_stg.so; else unset CTPT_LIB; fi
    python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02/tma_ab/c3_${v}_$rep.json 2>>gpurun_out/r02/tma_ab/err.log
    python -c "import json;d=json.load(open('gpurun_out/r02/tma_ab/c3_${v}_$rep.json'));print('c3 $v $rep',d['value'],d['roofline']['frac'],d['clocks']['sm_mhz'])"
  done
done
for rep in 1 2; do
  for v in tma stg; do
    if [ $v = stg ]; then export CTPT_LIB=/tmp/libctpt_stg.so; else unset CTPT_LIB; fi
    python bench.py --config c4 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02/tma_ab/c4_${v}_$rep.json 2>>gpurun_out/r02/tma_ab/err.log
    python -c "import json;d=json.load(open('gpurun_out/r02/tma_ab/c4_${v}_$rep.json'));print('c4 $v $rep',d['value'],d['roofline']['frac'],d['clocks']['sm_mhz'])"
  done
done
unset CTPT_LIB
bash tools/gpu_r02_multirank.sh
