#!/bin/bash
# k_layout_v4 (16-byte) vs k_layout (4-byte): parity tests, then the bench's setup_stages and e2e.
set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_layout.py tests/test_gpu_parity.py -m gpu -x -q \
  -k "layout or shapes_tcgen05 or matmul_host or validate or config1 or config2 or graph" > $O/layout_tests.log 2>&1
echo "rc=$?" >> $O/layout_tests.log
for rep in 1 2; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > $O/layout_v4_r$rep.json 2>> $O/layout_ab.err
  CTPT_LAYOUT=scalar timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > $O/layout_scalar_r$rep.json 2>> $O/layout_ab.err
done
echo done
