#!/bin/bash
# ncu --set full of the limbs-in-TMEM skinny kernel in its 64-row variants (d3 = 192: 2 whole-K-block
# limb stages; 224: 2 half-K-block stages) on c4's ciphertexts, one prime.
O=gpurun_out/r02/ncu_skinny; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for d3 in 192 224; do
  CMD="python tools/bench_skinny.py --L 1 --d3 $d3 --paths fused --steps 1 --warmup 1"
  $CMD > $O/plain_$d3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_gemm_fused -c 1 -o $O/fused_$d3 $CMD > $O/ncu_$d3.log 2>&1
  echo "d3=$d3 ncu_rc=$?"
  ncu -i $O/fused_$d3.ncu-rep --page details > $O/fused_${d3}_details.txt 2>&1
done
