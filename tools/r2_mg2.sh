#!/bin/bash
# 4-GPU check of the peer-view bulk-copy rings: dist parity tests, A/B of the step (this build vs
# tools/probes/variants/prev.so, register kernels for peer views) at N=2 and N=4, bench lines N=2/4
set -u
out=gpurun_out/mg2; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_dist.py -v -p no:cacheprovider > $out/pytest_dist.log 2>&1; echo "dist rc=$?"; tail -2 $out/pytest_dist.log
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2980$n bench.py --gpus $n > $out/bench_n$n.json 2> $out/bench_n$n.err; echo "n$n rc=$?"
  cp paper_2407_00599_b200/libparm_b200.so /tmp/cur.so; cp tools/probes/variants/prev.so paper_2407_00599_b200/libparm_b200.so
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2981$n bench.py --gpus $n > $out/bench_n${n}_prev.json 2> $out/bench_n${n}_prev.err; echo "n$n prev rc=$?"
  cp /tmp/cur.so paper_2407_00599_b200/libparm_b200.so
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2982$n bench.py --gpus $n > $out/bench_n${n}_b.json 2> $out/bench_n${n}_b.err; echo "n$n again rc=$?"
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/mg2/bench_n*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], d.get("schedules_ms"), d["roofline"]["frac"])
    except Exception as e:
        print(f, "ERR", e)
PY
