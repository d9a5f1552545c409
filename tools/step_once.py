"""A few eager fwd+bwd steps of the bench workload on one GPU (a short target for ncu)."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2407_00599_b200.config import MoEConfig  # noqa: E402
from paper_2407_00599_b200.runtime import MoELayer  # noqa: E402
from paper_2407_00599_b200.world import LocalWorld  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = torch.device("cuda", 0)
cfg = MoEConfig(**bench.C2)
layout = bench.layout_for(1)
layer = MoELayer(cfg, layout, LocalWorld(layout, dev))
layer.init_random(0)
x = torch.randn(cfg.tokens_per_rank, cfg.embed_dim, device=dev).to(torch.bfloat16)
d = torch.randn(cfg.tokens_per_rank, cfg.embed_dim, device=dev).to(torch.bfloat16)
for _ in range(steps):
    layer.forward("s1", {0: x})
    layer.backward({0: d})
torch.cuda.synchronize()
print("ok")
