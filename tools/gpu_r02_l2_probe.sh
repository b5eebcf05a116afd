#!/bin/bash
# L2 capacity for data shared by every SM vs private to one SM (tools/l2_probe/l2_probe.cu).
O=gpurun_out/r02/l2_probe; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2_probe tools/l2_probe/l2_probe.cu > $O/build.log 2>&1
timeout 600 /tmp/l2_probe > $O/l2_probe.jsonl 2> $O/l2_probe.err; echo "rc=$?" >> $O/l2_probe.err
cat $O/l2_probe.jsonl; tail -1 $O/l2_probe.err
