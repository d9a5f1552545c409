"""Whole-step A/B at the bench shape (N=1): the layer with the expert FFN as multi-problem GEMM
launches (fused_ffn=True) vs one launch per GEMM, CUDA-graph replays interleaved over several
rounds (boost clocks drift with power), median per round.

    python tools/probes/step_ab.py [rounds] [variant.so ...]   (each variant: fused, timed like the others)
"""
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2407_00599_b200 import _lib  # noqa: E402
from paper_2407_00599_b200.config import MoEConfig  # noqa: E402
from paper_2407_00599_b200.runtime import MoELayer  # noqa: E402
from paper_2407_00599_b200.world import LocalWorld  # noqa: E402


def main():
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    variants = sys.argv[2:]
    dev = torch.device("cuda", 0)
    cfg = MoEConfig(**bench.C2)
    layout = bench.layout_for(1)
    x = torch.randn(cfg.tokens_per_rank, cfg.embed_dim, device=dev).to(torch.bfloat16)
    d = torch.randn(cfg.tokens_per_rank, cfg.embed_dim, device=dev).to(torch.bfloat16)
    base = _lib.load()
    graphs = {}
    for name, lib, fused in [("fused", None, True), ("unfused", None, False)] + [(Path(v).stem, v, True)
                                                                                 for v in variants]:
        _lib._lib = _lib.load(lib) if lib else base
        layer = MoELayer(cfg, layout, LocalWorld(layout, dev), fused_ffn=fused)
        layer.init_random(0)
        graphs[name] = (layer, layer.capture_step("s1", {0: x}, {0: d}))
    _lib._lib = base
    res = {k: [] for k in graphs}
    for _ in range(rounds):
        for name, (_, g) in graphs.items():
            g.replay()
            torch.cuda.synchronize()
            ts = []
            for _ in range(10):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[name].append(statistics.median(ts))
    for name, v in res.items():
        print(f"{name:12s} median {statistics.median(v):.4f} ms; per round: " + " ".join(f"{t:.3f}" for t in v))
    ref = res["unfused"]
    for name, v in res.items():
        if name != "unfused":
            print(f"{name} faster than unfused in {sum(a < b for a, b in zip(v, ref))} of {rounds} rounds")


if __name__ == "__main__":
    main()
