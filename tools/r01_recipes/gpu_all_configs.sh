#!/bin/bash
# Every BASELINE config and the extra workloads on ONE box with the final code (bench defaults).
set -u
O=gpurun_out/final_cfgs
mkdir -p $O
for cfg in c1 c2 c3 c4 c3a; do
  timeout 900 python bench.py --config $cfg > $O/bench_$cfg.json 2> $O/bench_$cfg.err
  echo "$cfg rc=$?" >> $O/status.log
done
timeout 900 python bench.py --rescale --steps 5 --warmup 3 > $O/bench_c3_rescale.json 2> $O/bench_c3_rescale.err
echo "rescale rc=$?" >> $O/status.log
timeout 1500 python bench.py --config c5 --shard --gather ipc --steps 3 --warmup 3 > $O/bench_c5_ipc.json 2> $O/bench_c5_ipc.err
echo "c5 rc=$?" >> $O/status.log
timeout 900 python tools/bench_skinny.py > $O/skinny_sweep.jsonl 2> $O/skinny.err
echo "skinny rc=$?" >> $O/status.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
echo "reference rc=$?" >> $O/status.log
