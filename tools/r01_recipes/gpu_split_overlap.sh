#!/bin/bash
# Split of prime l+1 inside GEMM l (ctpt_gemm_next): parity, then interleaved A/B on c2, c3, c4.
set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "split_overlap or shapes_tcgen05 or unsigned or graph" > $O/ovl_tests.log 2>&1
echo "rc=$?" >> $O/ovl_tests.log
B="python bench.py --no-cpu-baseline --e2e-steps 0"
for rep in 1 2; do
  for cfg in c3 c4 c2; do
    st=20; [ $cfg = c4 ] && st=10; [ $cfg = c2 ] && st=200
    timeout 300 $B --config $cfg --steps $st --warmup 5 --split-overlap on > $O/ovl_on_${cfg}_r$rep.json 2>> $O/ovl.err
    timeout 300 $B --config $cfg --steps $st --warmup 5 --split-overlap off > $O/ovl_off_${cfg}_r$rep.json 2>> $O/ovl.err
  done
done
echo done
