set -u
out=gpurun_out/ab; mkdir -p $out
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "gate" > $out/pytest_k.log 2>&1; echo "pytest -k rc=$?"; tail -2 $out/pytest_k.log
timeout 300 python tools/probes/gate_trace.py tools/probes/variants/gtrace.so > $out/gate_trace.txt 2>&1; echo "trace rc=$?"; cat $out/gate_trace.txt
timeout 300 python tools/probes/kbench.py > $out/kbench.txt 2>&1; echo "kbench rc=$?"; head -1 $out/kbench.txt
