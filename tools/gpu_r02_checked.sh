#!/bin/bash
# compute-sanitizer substitute (it is closed on this pool): the small cases of every kernel path
# under the checked debug build (device bounds / invariant checks, trapping mbarrier timeouts),
# then stress repetitions with changing grid caps on the release build; every output vs the oracle.
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build_checked.log 2>&1
python tools/ab_build.py /tmp/libctpt_checked.so -DCTPT_DEBUG_CHECKS >> gpurun_out/r02/build_checked.log 2>&1
CTPT_LIB=/tmp/libctpt_checked.so timeout 1200 python tools/sanitize_cases.py --stress 3 > gpurun_out/r02/checked_build.log 2>&1
echo "rc=$?" >> gpurun_out/r02/checked_build.log; tail -4 gpurun_out/r02/checked_build.log
timeout 1200 python tools/sanitize_cases.py --stress 10 --cases gemm,gemm_side,gemm_u8,fused_wrap,mv_tickets,rescale > gpurun_out/r02/stress_release.log 2>&1
echo "rc=$?" >> gpurun_out/r02/stress_release.log; tail -4 gpurun_out/r02/stress_release.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused_gather.py tests/test_gpu_layout.py tests/test_c_client.py \
  -q -x > gpurun_out/r02/parity_ps.log 2>&1; echo "tests_rc=$?" >> gpurun_out/r02/parity_ps.log; tail -2 gpurun_out/r02/parity_ps.log
