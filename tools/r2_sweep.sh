#!/bin/bash
# 4-GPU measurements (gpurun --gpus 4): the extended selector sweep on both transports and the
# model-level steps with the baseline schedule beside S1.  Outputs under gpurun_out/sw/.
set -u
out=gpurun_out/sw; mkdir -p $out
export NCCL_DEBUG_FILE=/dev/stderr
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29721 tools/selector_sweep.py --grid extended --transport both --out $out/selector_p4.csv \
  > $out/selector_p4.log 2>&1; echo "sweep rc=$?"
for m in bert gpt2; do
  for cfg in "s1 peer" "s1 nccl" "s2 peer" "baseline nccl"; do
    set -- $cfg
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port 29731 tools/model_step.py --model $m --gpus 4 --schedule $1 --transport $2 \
      >> $out/model_steps_n4.jsonl 2>> $out/model_steps.err; echo "model $m $1 $2 rc=$?"
  done
  python tools/model_step.py --model $m >> $out/model_steps_n1.jsonl 2>> $out/model_steps.err; echo "model $m n1 rc=$?"
  python tools/model_step.py --model $m --moe torch >> $out/model_steps_n1.jsonl 2>> $out/model_steps.err; echo "model $m torch rc=$?"
done
grep SUMMARY $out/selector_p4.log | cut -c1-400
