"""Where the end-to-end (host-buffer) step loses time against the device step at N=1."""
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
for i in range(3):
    ms, _, _ = bench.time_e2e(layer, "s1", hx, hd, 30, 5, None, dev, True)
    print(f"e2e: {ms:.3f} ms/step, copy engine {bench.time_e2e.h2d_ms:.3f} ms", flush=True)
# the replay loop alone (same double-buffered graphs, no H2D)
bufs = [(x.clone(), d.clone()) for _ in range(2)]            # the graphs read these: keep them alive
g = [layer.capture_step("s1", {0: bx}, {0: bd}) for bx, bd in bufs]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
metric = torch.empty(8, dtype=torch.int32).pin_memory()
for mode in ("replay", "replay+d2h"):
    torch.cuda.synchronize()
    e0.record()
    for i in range(30):
        g[i % 2].replay()
        if mode == "replay+d2h":
            metric.copy_(layer.routing(0).fill, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    print(mode, e0.elapsed_time(e1) / 30)
