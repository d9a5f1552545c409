"""A/B of the expert-FFN GEMM launches at the bench shape (N=1 layout): the forward pair and the
backward four as one multi-problem launch (parm_gemm_multi) vs one launch per GEMM, for each
library build given (tools/probes/build_variant.sh).  CUDA-graph replays, median of reps.

    python tools/probes/ffn_ab.py [lib.so ...]   ("" = the in-tree build; repeat to interleave)
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools" / "probes"))
import bench  # noqa: E402
from kbench import timeit  # noqa: E402
from paper_2407_00599_b200 import _lib  # noqa: E402
from paper_2407_00599_b200.config import MoEConfig  # noqa: E402
from paper_2407_00599_b200.runtime import MoELayer  # noqa: E402
from paper_2407_00599_b200.world import LocalWorld  # noqa: E402


def main():
    libs = sys.argv[1:] or [None]
    dev = torch.device("cuda", 0)
    cfg = MoEConfig(**bench.C2)
    layout = bench.layout_for(1)
    base = _lib.load()
    for path in libs:
        _lib._lib = _lib.load(path) if path else base   # "" = the in-tree build
        for fused in (True, False):
            layer = MoELayer(cfg, layout, LocalWorld(layout, dev), fused_ffn=fused)
            layer.init_random(0)
            x = torch.randn(cfg.tokens_per_rank, cfg.embed_dim, device=dev).to(torch.bfloat16)
            layer.forward("s1", {0: x})
            layer.backward({0: x})
            s = layer.st[0]
            b = s.bufs["_local"]
            rows = int(b["fill_in"].sum())
            fl = 2 * rows * layer.d.Mp * layer.d.Hsp
            tf = timeit(lambda: layer._ffn_fwd(s, b), inner=10)
            tb = timeit(lambda: layer._ffn_bwd(s, b), inner=10)
            print(f"{Path(path).name if path else 'in-tree':>16s} fused={fused!s:5s}  fwd {tf:7.1f} us "
                  f"({2 * fl / tf / 1e6:6.0f} TF/s)  bwd {tb:7.1f} us ({4 * fl / tb / 1e6:6.0f} TF/s)", flush=True)


if __name__ == "__main__":
    main()
