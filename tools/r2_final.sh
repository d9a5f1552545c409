#!/bin/bash
# Final pass on the committed build: build, every GPU test (1 GPU) + smoke + N=1 bench and reference
# arm; with 4 GPUs visible also the dist parity tests and the N=2/4 bench lines.
set -u
out=gpurun_out/final; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1; echo "build rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest(1 GPU) rc=$?"; tail -1 $out/pytest_gpu.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > $out/bench_n1.json 2> $out/bench_n1.err; echo "bench n1 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference > $out/bench_reference.json 2> $out/bench_reference.err; echo "ref rc=$?"
ng=$(nvidia-smi -L | wc -l)
if [ "$ng" -ge 4 ]; then
  timeout 1200 python -m pytest tests/test_gpu_dist.py -q -p no:cacheprovider > $out/pytest_dist.log 2>&1; echo "dist rc=$?"; tail -1 $out/pytest_dist.log
  for n in 2 4; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 2985$n bench.py --gpus $n > $out/bench_n$n.json 2> $out/bench_n$n.err; echo "n$n rc=$?"
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 2986$n bench.py --impl reference --gpus $n > $out/bench_ref_n$n.json 2> $out/bench_ref_n$n.err; echo "ref n$n rc=$?"
  done
fi
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/final/bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d.get("ms_per_step"), d.get("value"), (d.get("e2e") or {}).get("value"), (d.get("roofline") or {}).get("frac"))
    except Exception as e:
        print(f, "ERR", e)
PY
