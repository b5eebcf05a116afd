#!/bin/bash
# (1) ncu --set full of the two skinny kernels at d3 = 256 on c4's ciphertexts (one prime): the
#     limbs-in-TMEM kernel (build -DCTPT_FUSED_TMEM_MAXD3=256) and the limbs-in-SMEM kernel (default);
# (2) the full CPU-oracle baseline of c1, c2, c3 with every GPU output compared (tools/cpu_baseline_full.py).
mkdir -p gpurun_out/r02/ncu256
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/ncu256/build.log 2>&1
python tools/ab_build.py /tmp/libctpt_t256.so -DCTPT_FUSED_TMEM_MAXD3=256 >> gpurun_out/r02/ncu256/build.log 2>&1
CMD="python tools/bench_skinny.py --L 1 --d3 256 --paths fused --steps 1 --warmup 1"
CTPT_LIB=/tmp/libctpt_t256.so $CMD > gpurun_out/r02/ncu256/plain_tmem.log 2>&1 && \
CTPT_LIB=/tmp/libctpt_t256.so ncu --set full --clock-control none --import-source on -k regex:k_gemm_fused -c 1 \
  -o gpurun_out/r02/ncu256/tmem $CMD > gpurun_out/r02/ncu256/ncu_tmem.log 2>&1
$CMD > gpurun_out/r02/ncu256/plain_smem.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemm_fused -c 1 \
  -o gpurun_out/r02/ncu256/smem $CMD > gpurun_out/r02/ncu256/ncu_smem.log 2>&1
echo "ncu done"
timeout 2400 python tools/cpu_baseline_full.py > gpurun_out/r02/cpu_baseline_full.jsonl 2> gpurun_out/r02/cpu_baseline_full.err
echo "cpu_rc=$?"; cat gpurun_out/r02/cpu_baseline_full.jsonl | cut -c1-400
