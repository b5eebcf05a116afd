#!/bin/bash
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "skinny or modmatmul or rescale" > $O/gpu_parity_q.log 2>&1; echo "rc=$?" >> $O/gpu_parity_q.log
CTPT_FUSED_PF=8 CTPT_FUSED_LOAD=regs timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "skinny_fused" > $O/gpu_parity_q2.log 2>&1; echo "rc=$?" >> $O/gpu_parity_q2.log
timeout 900 python tools/bench_skinny.py --paths fused,fused-regs,fused-regs-pf4,fused-regs-pf8,fused-regs-pf16 > $O/skinny_q.jsonl 2> $O/skinny_q.err
