#!/bin/bash
# token-side kernels after an arithmetic change: GPU parity (all), per-kernel warm/cold timings, launch list
out=gpurun_out/tok; mkdir -p $out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_module.py -m gpu -x -q > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest.log
timeout 600 python tools/probes/kbench.py > $out/kbench.log 2>&1; echo "kbench rc=$?"; cat $out/kbench.log | grep warm
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_n1.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_launch.log 2>&1; echo "ncu list rc=$?"
