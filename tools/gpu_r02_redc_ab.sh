#!/bin/bash
# Montgomery recombination in the epilogues (u8 limbs × u8 U plane) vs Barrett (-DCTPT_NO_REDC):
# parity, then c3 / c4 bench lines interleaved on one box.
mkdir -p gpurun_out/r02/redc_ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/redc_ab/build.log 2>&1
python tools/ab_build.py /tmp/libctpt_barrett.so -DCTPT_NO_REDC >> gpurun_out/r02/redc_ab/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused_gather.py tests/test_c_client.py -q -x \
  > gpurun_out/r02/redc_ab/tests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/r02/redc_ab/tests.log; tail -2 gpurun_out/r02/redc_ab/tests.log
for rep in 1 2 3; do
  for v in redc barrett; do
    if [ $v = barrett ]; then export CTPT_LIB=/tmp/libctpt_barrett.so; else unset CTPT_LIB; fi
    python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02/redc_ab/c3_${v}_$rep.json 2>>gpurun_out/r02/redc_ab/err.log
    python -c "import json;d=json.load(open('gpurun_out/r02/redc_ab/c3_${v}_$rep.json'));print('c3 $v $rep',d['value'],d['roofline']['frac'],d['clocks']['sm_mhz'],d['roofline']['avg_launch_ms'])"
  done
done
for rep in 1 2; do
  for v in redc barrett; do
    if [ $v = barrett ]; then export CTPT_LIB=/tmp/libctpt_barrett.so; else unset CTPT_LIB; fi
    python bench.py --config c4 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02/redc_ab/c4_${v}_$rep.json 2>>gpurun_out/r02/redc_ab/err.log
    python -c "import json;d=json.load(open('gpurun_out/r02/redc_ab/c4_${v}_$rep.json'));print('c4 $v $rep',d['value'],d['roofline']['frac'],d['clocks']['sm_mhz'],d['roofline']['avg_launch_ms'])"
  done
done
