#!/bin/bash
# NVLink evidence refresh (peer-view bulk rings): probe timings + ncu nvltx/nvlrx bytes at P=2/4
set -u
out=gpurun_out/nvl; mkdir -p $out
M=gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum
for g in 2 4; do
  devs=$(seq -s, 0 $((g-1)))
  CUDA_VISIBLE_DEVICES=$devs timeout 300 python tools/probes/nvlink_probe.py > $out/nvlink_probe_p$g.json 2>&1; echo "probe p$g rc=$?"
  CUDA_VISIBLE_DEVICES=$devs timeout 900 ncu --metrics $M --clock-control none --csv \
    -k regex:"route_dispatch|moe_gemm_pair|combine_fwd|dispatch_bwd" -c 200 \
    --log-file $out/ncu_nvlink_p$g.csv python tools/probes/nvlink_probe.py > $out/ncu_nvlink_p$g.log 2>&1; echo "ncu nvlink p$g rc=$?"
done
