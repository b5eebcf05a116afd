#!/bin/bash
# End-to-end leg (ctpt_matmul_host: pinned host buffers, chunked H2D || layout + split + GEMM || D2H)
# vs the pipeline's chunk size, on c3 and c2 (the two configs below 0.9 of the PCIe floor).
# Model: T = sum of the copies + max over chunks of (H2D + compute of one chunk), so smaller chunks
# should approach the floor until per-chunk costs (2-D copy efficiency, GEMM tails) take over.
O=gpurun_out/r02/e2e_chunks; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for rep in 1 2; do
  for ch in 0 640 1024 1280 1728 2560; do
    CTPT_E2E_CHUNK=$ch timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --e2e-steps 5 --no-cpu-baseline \
      > $O/c3_ch${ch}_$rep.json 2>>$O/err.log
  done
  for ch in 0 256 512 768 1024 2048; do
    CTPT_E2E_CHUNK=$ch timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --e2e-steps 10 --no-cpu-baseline \
      > $O/c2_ch${ch}_$rep.json 2>>$O/err.log
  done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r02/e2e_chunks/*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    e = d['e2e']
    print(f.split('/')[-1], '%.4e' % e['value'], '%.2f ms' % e['ms_per_step'], 'floor %.3f' % e['pcie']['frac_of_floor'])
PY
