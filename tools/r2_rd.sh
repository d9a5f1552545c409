#!/bin/bash
# route_dispatch with batched pick fetches: parity (all GPU parity tests), bit identity vs the previous build, timings
out=gpurun_out/rd; mkdir -p $out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_module.py -m gpu -x -q > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest.log
timeout 600 python tools/probes/bitident.py tools/probes/variants/prev.so > $out/bitident.log 2>&1; echo "bitident rc=$?"; tail -5 $out/bitident.log
timeout 600 python tools/probes/kbench.py > $out/kbench.log 2>&1; echo "kbench rc=$?"; grep warm $out/kbench.log
