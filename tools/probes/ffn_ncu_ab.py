"""Expert-FFN multi-GEMM launches of several library builds, for an ncu A/B at locked clocks
(every launch in a fixed order: per build, `reps` forward launches then `reps` backward launches):

    ncu --metrics gpu__time_duration.sum -k regex:moe_gemm --csv --log-file out.csv \\
        python tools/probes/ffn_ncu_ab.py reps "" variant.so "" variant.so
    python tools/probes/ffn_ncu_ab.py --parse out.csv reps "" variant.so ...
"""
import csv
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))


def run(reps, libs):
    import torch
    import bench
    from paper_2407_00599_b200 import _lib
    from paper_2407_00599_b200.config import MoEConfig
    from paper_2407_00599_b200.runtime import MoELayer
    from paper_2407_00599_b200.world import LocalWorld
    dev = torch.device("cuda", 0)
    cfg = MoEConfig(**bench.C2)
    layout = bench.layout_for(1)
    base = _lib.load()
    for path in libs:
        _lib._lib = _lib.load(path) if path else base
        layer = MoELayer(cfg, layout, LocalWorld(layout, dev), fused_ffn=True)
        layer.init_random(0)
        x = torch.randn(cfg.tokens_per_rank, cfg.embed_dim, device=dev).to(torch.bfloat16)
        layer.forward("s1", {0: x})
        layer.backward({0: x})
        torch.cuda.synchronize()
        s = layer.st[0]
        b = s.bufs["_local"]
        for _ in range(reps):
            layer._ffn_fwd(s, b)
        for _ in range(reps):
            layer._ffn_bwd(s, b)
        torch.cuda.synchronize()


def parse(path, reps, libs):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    t = [float(r[vi].replace(",", "")) / 1e3 for r in rows[1:] if "moe_gemm" in r[ki]]
    per = 2 + 2 * reps   # warm-up forward + backward, then reps of each
    res = {}
    for i, lib in enumerate(libs):
        seg = t[i * per:(i + 1) * per][2:]
        name = Path(lib).stem if lib else "in-tree"
        res.setdefault(name, {"fwd": [], "bwd": []})
        res[name]["fwd"] += seg[:reps]
        res[name]["bwd"] += seg[reps:]
    for name, d in res.items():
        print(f"{name:>10s}  fwd median {statistics.median(d['fwd']):7.1f} us (n={len(d['fwd'])})  "
              f"bwd median {statistics.median(d['bwd']):7.1f} us (n={len(d['bwd'])})")


if __name__ == "__main__":
    if sys.argv[1] == "--parse":
        parse(sys.argv[2], int(sys.argv[3]), sys.argv[4:])
    else:
        run(int(sys.argv[1]), sys.argv[2:])
