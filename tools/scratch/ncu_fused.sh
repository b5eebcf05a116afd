python -c "import __graft_entry__ as g; g.build_ctpt()" > gpurun_out/ncu_build.log 2>&1
mkdir -p gpurun_out/r02/ncu_fused
python tools/bench_skinny.py --L 1 --d3 64,128 --paths fused --steps 2 --warmup 1 > gpurun_out/r02/ncu_fused/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemm_fused -c 2 -o gpurun_out/r02/ncu_fused/prof \
  python tools/bench_skinny.py --L 1 --d3 64,128 --paths fused --steps 1 --warmup 0 > gpurun_out/r02/ncu_fused/ncu.log 2>&1
echo "ncu_rc=$?"; tail -3 gpurun_out/r02/ncu_fused/ncu.log
