#!/bin/bash
out=gpurun_out/prof; mkdir -p $out
for n in 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2990$n \
    tools/probes/step_profile.py $n s1 > $out/prof_n$n.json 2> $out/prof_n$n.err; echo "prof n$n rc=$?"
done
