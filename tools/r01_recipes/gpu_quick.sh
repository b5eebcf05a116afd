#!/bin/bash
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "mv or skinny or shapes_tcgen05 or rescale or host_pipeline or struct" > $O/gpu_parity_q.log 2>&1; echo "rc=$?" >> $O/gpu_parity_q.log
timeout 900 python tools/bench_skinny.py --paths auto,fused > $O/skinny_q.jsonl 2> $O/skinny_q.err
