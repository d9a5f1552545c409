mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "fused or layer_fwd_bwd" > gpurun_out/ab/pytest_k.log 2>&1; echo "pytest -k rc=$?"; tail -2 gpurun_out/ab/pytest_k.log
set -u
out=gpurun_out/ab; mkdir -p $out
nvidia-smi --query-gpu=clocks.sm,power.draw,power.limit --format=csv
timeout 300 python tools/probes/step_ab.py 30 tools/probes/variants/nodeps_static.so > $out/step_ab.txt 2>&1; echo "step_ab rc=$?"; cat $out/step_ab.txt
