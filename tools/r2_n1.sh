#!/bin/bash
# One-GPU round-2 check: GPU tests, smoke, the N=1 bench line, the ncu launch list of the same
# bench command, and one ncu --set full capture of the token-side kernels of an eager step.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- bash tools/r2_n1.sh
set -u
out=gpurun_out/n1; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $out/bench_n1.json 2> $out/bench_n1.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_n1.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_launch.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^(?!moe_gemm)' -c 12 -o $out/small_full \
  python tools/step_once.py 1 > $out/ncu_small.log 2>&1; echo "ncu small rc=$?"
tail -c 600 $out/bench_n1.json
