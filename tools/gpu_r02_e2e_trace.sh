#!/bin/bash
# Timeline of the host executor's pipeline (trace build: events around every chunk's H2D, compute,
# D2H) on c3 at three chunk sizes, to see where narrower chunks lose (profiles/r02/e2e_chunks/).
O=gpurun_out/r02/e2e_trace; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/ab_build.py /tmp/trace.so -DCTPT_HOST_TRACE >> $O/build.log 2>&1
for ch in 0 1728 1024; do
  CTPT_LIB=/tmp/trace.so CTPT_E2E_CHUNK=$ch timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --e2e-steps 1 \
    --no-cpu-baseline > $O/c3_ch$ch.json 2> $O/c3_ch$ch.trace
  grep -c "^trace" $O/c3_ch$ch.trace
done
