#!/bin/bash
# Model-level steps (BERT-large-MoE, GPT-2-MoE) at 1 and 4 GPUs with the baseline schedule beside S1/S2.
set -u
out=gpurun_out/models; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
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
