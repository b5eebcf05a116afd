#!/bin/bash
# k_gemm_tc raster group re-measured with round 2's code (TMA-store epilogue): c4 and c3, interleaved.
mkdir -p gpurun_out/r02/raster
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/raster/build.log 2>&1
for rep in 1 2; do
  for g in 16 8 12 20 24; do
    python bench.py --config c4 --raster-group $g --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02/raster/c4_g${g}_$rep.json 2>>gpurun_out/r02/raster/err.log
    python -c "import json;d=json.load(open('gpurun_out/r02/raster/c4_g${g}_$rep.json'));print('c4 g=$g $rep','%.4e'%d['value'],d['roofline']['avg_launch_ms'],d['clocks']['sm_mhz'])"
  done
done
for rep in 1 2; do
  for g in 16 12 20; do
    python bench.py --config c3 --raster-group $g --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02/raster/c3_g${g}_$rep.json 2>>gpurun_out/r02/raster/err.log
    python -c "import json;d=json.load(open('gpurun_out/r02/raster/c3_g${g}_$rep.json'));print('c3 g=$g $rep','%.4e'%d['value'],d['roofline']['avg_launch_ms'],d['clocks']['sm_mhz'])"
  done
done
