#!/bin/bash
# The batched host executor (ctpt_matmul_host_units) + the PCIe 2-D copy sweep.
O=gpurun_out/r02/units; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python tools/pcie_2d_sweep.py > $O/pcie_2d_sweep.jsonl 2> $O/pcie.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_multirank.py tests/test_abi.py -q -x \
  -k "host or multirank or units or abi" > $O/tests.log 2>&1; echo "tests_rc=$?" >> $O/tests.log
tail -3 $O/tests.log
timeout 1200 python bench.py --config c5 --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
python - <<'PY'
import json
for l in open('gpurun_out/r02/units/pcie_2d_sweep.jsonl'):
    print(l.strip())
d = json.loads(open('gpurun_out/r02/units/bench_c5.json').read().strip().splitlines()[-1])
print('c5', d['value'], d['ms_per_step'], d['e2e'])
PY
