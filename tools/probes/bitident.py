"""Bit-identity of the layer step across two library builds (same inputs, same weights): the
forward output, dx and every weight gradient compared with torch.equal.

    python tools/probes/bitident.py other.so
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2407_00599_b200 import _lib  # noqa: E402
from paper_2407_00599_b200.config import MoEConfig, ParallelLayout  # noqa: E402
from paper_2407_00599_b200.runtime import MoELayer  # noqa: E402
from paper_2407_00599_b200.world import LocalWorld, PeerLocalWorld  # noqa: E402


CASES = [("bench N=1 s1", None, "s1", False), ("P=4 (2,2,2) peer s1", (2, 2, 2, 4), "s1", True),
         ("P=4 (2,2,2) peer s2", (2, 2, 2, 4), "s2", True), ("P=4 (2,2,2) baseline", (2, 2, 2, 4), "baseline", False)]


def run(lib, lay, schedule, peer):
    _lib._lib = lib
    dev = torch.device("cuda", 0)
    if lay is None:
        cfg = MoEConfig(**bench.C2)
        layout = bench.layout_for(1)
        W = LocalWorld(layout, dev)
    else:
        cfg = MoEConfig(2, 512, 1024, 2048, 8, 2, 1.2)
        layout = ParallelLayout(*lay)
        W = PeerLocalWorld(layout) if peer else LocalWorld(layout)
    layer = MoELayer(cfg, layout, W)
    layer.init_random(0)
    g = torch.Generator(device=dev).manual_seed(0)
    G = layout.world_size // layout.mp_size
    xs = [torch.randn(cfg.tokens_per_rank, cfg.embed_dim, device=dev, generator=g).to(torch.bfloat16) for _ in range(G)]
    ds = [torch.randn(cfg.tokens_per_rank, cfg.embed_dim, device=dev, generator=g).to(torch.bfloat16) for _ in range(G)]
    outs = layer.forward(schedule, {r: xs[r // layout.mp_size] for r in layer.ranks})
    dxs = layer.backward({r: ds[r // layout.mp_size] for r in layer.ranks})
    res = {}
    for r in layer.ranks:
        res[f"out{r}"] = outs[r].clone()
        res[f"dx{r}"] = dxs[r].clone()
        for k, v in layer.shard_grads(r).items():
            res[f"{k}{r}"] = v.clone()
    torch.cuda.synchronize()
    return res


def main():
    base = _lib.load()
    other = _lib.load(sys.argv[1])
    allok = True
    for name, lay, sch, peer in CASES:
        a = run(base, lay, sch, peer)
        b = run(other, lay, sch, peer)
        bad = [k for k in a if not torch.equal(a[k], b[k])]
        allok &= not bad
        print(f"{name:24s} tensors {len(a):3d}  differing: {bad if bad else 'none'}", flush=True)
    print({"bit_identical": allok})


if __name__ == "__main__":
    main()
