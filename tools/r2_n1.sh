#!/bin/bash
# One-GPU check: GPU tests, smoke, the N=1 bench line + reference arm, the ncu launch list of the
# bench command, ncu --set full of the fused GEMM launches and of the token-side kernels.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- bash tools/r2_n1.sh
set -u
out=gpurun_out/n1; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $out/bench_n1.json 2> $out/bench_n1.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $out/bench_reference.json 2> $out/bench_reference.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_n1.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_launch.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:moe_gemm_pair -c 2 -o $out/gemm_full \
  python tools/step_once.py 1 > $out/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gate_fwd|route_dispatch|combine|dispatch_bwd|gate_wgrad|sum_partials" -c 7 -o $out/tok_full \
  python tools/step_once.py 1 > $out/ncu_tok.log 2>&1; echo "ncu tok rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/n1/bench_n1.json").read().strip().splitlines()[-1])
r = d["roofline"]
print("ms", d["ms_per_step"], "tok/s", d["value"], "frac", r["frac"], "gemm ms/launch", r["avg_launch_ms"],
      "e2e", d["e2e"]["value"], "clocks", d["clocks"])
PY
