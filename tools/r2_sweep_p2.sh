#!/bin/bash
# The extended selector sweep on 2 GPUs (gpurun --gpus 2), both transports; CSV + log in gpurun_out/sw/.
set -u
out=gpurun_out/sw; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
timeout 3300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29722 tools/selector_sweep.py --grid extended --transport both --out $out/selector_p2.csv \
  > $out/selector_p2.log 2>&1; echo "sweep rc=$?"
grep SUMMARY $out/selector_p2.log | cut -c1-600
