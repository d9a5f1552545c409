#!/bin/bash
# Round-end measurement on a 4-GPU box (gpurun --gpus 4): bench lines N=1/2/4, the reference
# arm, the N=1 ncu launch list and one ncu --set full capture of the grouped GEMMs.
#   /usr/local/graft/bin/gpurun --gpus 4 --timeout 1500 -- bash tools/final_measure.sh
set -u
out=gpurun_out/final
mkdir -p $out
python bench.py > $out/bench_n1.json 2> $out/bench_n1.err; echo "n1 rc=$?"
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2960$n bench.py --gpus $n > $out/bench_n$n.json 2> $out/bench_n$n.err; echo "n$n rc=$?"
done
python bench.py --impl reference > $out/bench_reference.json 2> $out/bench_reference.err; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_n1.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_launch.log 2>&1; echo "ncu list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:moe_gemm_pair -c 6 -o $out/gemm_full \
  python tools/step_once.py 1 > $out/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -c 400 $out/bench_n1.json
