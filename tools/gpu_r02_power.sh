#!/bin/bash
# Round 2: power roofline of the power-capped kernels (tools/power_roofline.py).
O=gpurun_out/r02/power; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python tools/power_roofline.py --seconds 3 > $O/power_roofline.jsonl 2> $O/power_roofline.err
echo "rc=$?" >> $O/power_roofline.err
tail -3 $O/power_roofline.err; cat $O/power_roofline.jsonl
