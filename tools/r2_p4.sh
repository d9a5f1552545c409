#!/bin/bash
# Round-2 4-GPU evidence (gpurun --gpus 4): NVLink counters of the fused peer kernels (ncu, one
# process driving all GPUs), NCCL bus bandwidth, then the extended selector sweep and the
# model-level steps (tools/r2_sweep.sh).  Outputs under gpurun_out/p4/ and gpurun_out/sw/.
set -u
out=gpurun_out/p4; mkdir -p $out
M=gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum
for g in 2 4; do
  devs=$(seq -s, 0 $((g-1)))
  CUDA_VISIBLE_DEVICES=$devs timeout 300 python tools/probes/nvlink_probe.py > $out/nvlink_probe_p$g.json 2> $out/nvlink_probe_p$g.err
  echo "probe p$g rc=$?"
  CUDA_VISIBLE_DEVICES=$devs timeout 600 ncu --metrics $M --clock-control none --csv \
    -k regex:"route_dispatch|moe_gemm_pair|combine_fwd|dispatch_bwd" -c 40 \
    --log-file $out/ncu_nvlink_p$g.csv python tools/probes/nvlink_probe.py > $out/ncu_nvlink_p$g.log 2>&1
  echo "ncu nvlink p$g rc=$?"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29741 tools/nccl_busbw.py > $out/nccl_busbw_p4.jsonl 2> $out/nccl_busbw_p4.err; echo "busbw rc=$?"
bash tools/r2_sweep.sh
