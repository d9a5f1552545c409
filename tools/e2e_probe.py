"""Repeatability of bench.py's end-to-end (host-buffer) measurement at N=1."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2407_00599_b200.config import MoEConfig  # noqa: E402
from paper_2407_00599_b200.runtime import MoELayer  # noqa: E402
from paper_2407_00599_b200.world import LocalWorld  # noqa: E402

dev = torch.device("cuda", 0)
cfg = MoEConfig(**bench.C2)
layout = bench.layout_for(1)
layer = MoELayer(cfg, layout, LocalWorld(layout, dev))
layer.init_random(0)
x = torch.randn(cfg.tokens_per_rank, cfg.embed_dim, device=dev).to(torch.bfloat16)
d = torch.randn(cfg.tokens_per_rank, cfg.embed_dim, device=dev).to(torch.bfloat16)
print("device step ms", bench.time_steps(layer, "s1", {0: x}, {0: d}, 30, 5, None, dev, True))
hx, hd = x.cpu().pin_memory(), d.cpu().pin_memory()
print("h2d GB/s", bench.h2d_bandwidth(hx, dev))
for i in range(6):
    ms, _, _ = bench.time_e2e(layer, "s1", hx, hd, 30, 5, None, dev, True)
    print(f"e2e run {i}: {ms:.3f} ms/step", flush=True)
