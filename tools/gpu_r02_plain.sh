#!/bin/bash
# k_plain with 16-byte stores: parity (every GPU test goes through the precompute) + setup_stages.
O=gpurun_out/r02/plain; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_c_client.py -q -x > $O/tests.log 2>&1; echo "tests_rc=$?" >> $O/tests.log
tail -2 $O/tests.log
for cfg in c3 c4; do
  timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/bench_$cfg.json 2>> $O/err.log
  python -c "import json;d=json.loads(open('$O/bench_$cfg.json').read().strip().splitlines()[-1]);print('$cfg', d['value'], d['setup_stages'])"
done
