#!/bin/bash
# Board power of plain HBM streams (copy / read-only / write-only) next to the skinny kernel at d3 = 1.
O=gpurun_out/r02/stream_power; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python tools/power_stream_probe.py --seconds 3 > $O/stream_power.jsonl 2> $O/stream_power.err; echo "rc=$?" >> $O/stream_power.err
timeout 600 python tools/power_roofline.py --seconds 3 --d3 1,256 --no-gemm > $O/power_roofline.jsonl 2>> $O/stream_power.err
cat $O/stream_power.jsonl $O/power_roofline.jsonl; tail -2 $O/stream_power.err
