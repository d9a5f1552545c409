#!/bin/bash
out=gpurun_out/prof; mkdir -p $out
for t in peer peer-push nccl; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29000 + RANDOM % 900)) \
    tools/probes/step_profile.py 4 s1 $t > $out/prof_n4_$t.json 2> $out/prof_n4_$t.err; echo "prof $t rc=$?"
done
