#!/bin/bash
# N=2/4 step A/B of this build vs tools/probes/variants/prev.so (swapped in place), alternating, then dist parity
set -u
out=gpurun_out/ab4; mkdir -p $out
cp paper_2407_00599_b200/libparm_b200.so /tmp/cur.so
for rep in 1 2; do
for n in 2 4; do
  for v in cur prev; do
    if [ $v = prev ]; then cp tools/probes/variants/prev.so paper_2407_00599_b200/libparm_b200.so; else cp /tmp/cur.so paper_2407_00599_b200/libparm_b200.so; fi
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 29$((RANDOM % 90 + 10))$n bench.py --gpus $n --no-compare > $out/b_n${n}_${v}_$rep.json 2> $out/b_n${n}_${v}_$rep.err; echo "n$n $v $rep rc=$?"
  done
done
done
cp /tmp/cur.so paper_2407_00599_b200/libparm_b200.so
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -p no:cacheprovider > $out/pytest_dist.log 2>&1; echo "dist rc=$?"; tail -2 $out/pytest_dist.log
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/ab4/b_n*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d["ms_per_step"], 4))
    except Exception as e:
        print(f, "ERR", e)
PY
