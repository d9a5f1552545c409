#!/bin/bash
# 4-GPU checks (gpurun --gpus 4): the multi-GPU parity tests, bench lines at N=2 and N=4,
# and a short selector sweep.  Outputs under gpurun_out/mg/.
set -u
out=gpurun_out/mg; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_dist.py -v -p no:cacheprovider > $out/pytest_dist.log 2>&1; echo "dist rc=$?"
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2970$n bench.py --gpus $n > $out/bench_n$n.json 2> $out/bench_n$n.err; echo "bench n$n rc=$?"
done
if [ "${SWEEP_LIMIT:-0}" != "0" ]; then
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29711 tools/selector_sweep.py --limit $SWEEP_LIMIT --out $out/sweep_smoke.csv > $out/sweep_smoke.log 2>&1
  echo "sweep rc=$?"
fi
tail -3 $out/pytest_dist.log
