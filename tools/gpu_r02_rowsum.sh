#!/bin/bash
# The limbs-in-TMEM skinny kernel with the u8 plane and in-kernel row sums: parity, then
# (a) the skinny sweep with the new default planes, (b) d3 = 224 / 256: TMEM kernel + u8 plane
# (build -DCTPT_FUSED_TMEM_MAXD3=256) vs the shared-memory kernel + s8 digits (default build).
mkdir -p gpurun_out/r02/rowsum
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/rowsum/build.log 2>&1
python tools/ab_build.py /tmp/libctpt_t256.so -DCTPT_FUSED_TMEM_MAXD3=256 >> gpurun_out/r02/rowsum/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused_gather.py tests/test_c_client.py -q -x \
  > gpurun_out/r02/rowsum/tests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/r02/rowsum/tests.log; tail -2 gpurun_out/r02/rowsum/tests.log
CTPT_LIB=/tmp/libctpt_t256.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "skinny or column_shard or fuzz" \
  > gpurun_out/r02/rowsum/tests_t256.log 2>&1; echo "tests_rc=$?" >> gpurun_out/r02/rowsum/tests_t256.log; tail -2 gpurun_out/r02/rowsum/tests_t256.log
for rep in 1 2; do
  timeout 600 python tools/bench_skinny.py --L 4 --d3 64,128,160,192 --paths auto > gpurun_out/r02/rowsum/auto_$rep.jsonl 2>>gpurun_out/r02/rowsum/err.log
  timeout 600 python tools/bench_skinny.py --L 4 --d3 224,256 --paths fused --plane never > gpurun_out/r02/rowsum/big_smem_s8_$rep.jsonl 2>>gpurun_out/r02/rowsum/err.log
  CTPT_LIB=/tmp/libctpt_t256.so timeout 600 python tools/bench_skinny.py --L 4 --d3 224,256 --paths fused --plane always \
    > gpurun_out/r02/rowsum/big_tmem_u8_$rep.jsonl 2>>gpurun_out/r02/rowsum/err.log
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r02/rowsum/*.jsonl')):
    for l in open(f):
        d = json.loads(l)
        print(f.split('/')[-1], d['u_plane'], d['u_offset'], d['d3'], d['kernel'], '%.3f' % d['roofline']['frac'], '%.3f ms' % d['avg_launch_ms'])
PY
