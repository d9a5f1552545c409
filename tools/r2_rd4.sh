#!/bin/bash
# route_dispatch warps/stages at N=4: step A/B (in-tree 8x10 vs 12x6 vs 16x6), swapped libraries, alternating
set -u
out=gpurun_out/rd4; mkdir -p $out
cp paper_2407_00599_b200/libparm_b200.so /tmp/cur.so
for rep in 1 2; do
  for v in cur rd12 rd16; do
    if [ $v = cur ]; then cp /tmp/cur.so paper_2407_00599_b200/libparm_b200.so; else cp tools/probes/variants/$v.so paper_2407_00599_b200/libparm_b200.so; fi
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port $((29000 + RANDOM % 900)) bench.py --gpus 4 --no-compare > $out/b_${v}_$rep.json 2> $out/b_${v}_$rep.err; echo "$v $rep rc=$?"
  done
done
cp /tmp/cur.so paper_2407_00599_b200/libparm_b200.so
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/rd4/b_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d["ms_per_step"], 4))
    except Exception as e:
        print(f, "ERR", e)
PY
