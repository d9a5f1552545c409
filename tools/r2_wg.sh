#!/bin/bash
# gate_wgrad with the partial sum in the same launch: parity, launch list
out=gpurun_out/wg; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wgrad or layer or module or fused or golden" > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest.log
timeout 600 python tools/probes/kbench.py > $out/kbench.log 2>&1; echo "kbench rc=$?"; grep -i "wgrad\|sum" $out/kbench.log | head
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_n1.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_launch.log 2>&1; echo "ncu list rc=$?"
