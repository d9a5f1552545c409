#!/bin/bash
# One-GPU iteration check: build, gate error probe, targeted then full GPU tests, the N=1 bench
# line and the per-kernel in-step times.  Outputs under gpurun_out/it/.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- bash tools/r2_iter.sh [pytest -k expr]
set -u
out=gpurun_out/it; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1; echo "build rc=$?"
timeout 120 tools/probes/gate_err_probe > $out/gate_err_probe.json 2>&1; echo "gate probe rc=$?"; cat $out/gate_err_probe.json
if [ -n "${1:-}" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$1" > $out/pytest_k.log 2>&1; echo "pytest -k rc=$?"
  tail -15 $out/pytest_k.log
fi
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 $out/pytest_gpu.log
timeout 600 python bench.py > $out/bench_n1.json 2> $out/bench_n1.err; echo "bench rc=$?"
timeout 300 python tools/profile_step.py > $out/profile_step.txt 2>&1; echo "profile rc=$?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/it/bench_n1.json"))
r = d["roofline"]
print("ms", d["ms_per_step"], "tok/s", d["value"], "gemm avg ms", r["avg_launch_ms"], "frac", r["frac"], "e2e", d["e2e"]["value"])
PY
head -40 $out/profile_step.txt
