#!/bin/bash
# Round-2 multi-GPU + profile pass (gpurun --gpus 4): dist parity tests, bench lines N=1/2/4 and the
# reference arm, ncu NVLink counters of the peer kernels at P=2/4, the N=1 launch list and one
# ncu --set full capture of the fused GEMM launches.  Outputs under gpurun_out/mg/.
set -u
out=gpurun_out/mg; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests/test_gpu_dist.py -v -p no:cacheprovider > $out/pytest_dist.log 2>&1; echo "dist rc=$?"; tail -2 $out/pytest_dist.log
timeout 600 python bench.py > $out/bench_n1.json 2> $out/bench_n1.err; echo "n1 rc=$?"
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2980$n bench.py --gpus $n > $out/bench_n$n.json 2> $out/bench_n$n.err; echo "n$n rc=$?"
done
timeout 600 python bench.py --impl reference > $out/bench_reference.json 2> $out/bench_reference.err; echo "ref rc=$?"
M=gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum
for g in 2 4; do
  devs=$(seq -s, 0 $((g-1)))
  CUDA_VISIBLE_DEVICES=$devs timeout 300 python tools/probes/nvlink_probe.py > $out/nvlink_probe_p$g.json 2>&1; echo "probe p$g rc=$?"
  CUDA_VISIBLE_DEVICES=$devs timeout 900 ncu --metrics $M --clock-control none --csv \
    -k regex:"route_dispatch|moe_gemm_pair|combine_fwd|dispatch_bwd" -c 200 \
    --log-file $out/ncu_nvlink_p$g.csv python tools/probes/nvlink_probe.py > $out/ncu_nvlink_p$g.log 2>&1; echo "ncu nvlink p$g rc=$?"
done
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_n1.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_launch.log 2>&1; echo "ncu list rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"moe_gemm_pair" -c 2 -o $out/gemm_full \
  python tools/step_once.py 1 > $out/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gate_fwd|route_dispatch|combine|dispatch_bwd|gate_wgrad|sum_partials" -c 7 -o $out/tok_full \
  python tools/step_once.py 1 > $out/ncu_tok.log 2>&1; echo "ncu tok rc=$?"
for f in $out/bench_n1.json $out/bench_n2.json $out/bench_n4.json; do python -c "
import json,sys; d=json.load(open('$f')); r=d['roofline']
print('$f', d['ms_per_step'], d['value'], r['frac'], r['avg_launch_ms'], d.get('speedup_vs_baseline_schedule'), d.get('speedup_vs_baseline_schedule_same_transport'), d['e2e']['value'])"; done
