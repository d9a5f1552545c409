"""Per-kernel CUDA time of one MoE-layer fwd+bwd step (torch.profiler / CUPTI), rank 0 printed.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/profile_step.py \
        --gpus N [--schedule s1] [--steps 5]
Works for N=1 without torchrun.  Eager launches (graph replays hide kernel names).
"""

from __future__ import annotations

import argparse
import os
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2407_00599_b200.config import MoEConfig  # noqa: E402
from paper_2407_00599_b200.runtime import MoELayer  # noqa: E402
from paper_2407_00599_b200.world import LocalWorld, NcclWorld, PeerWorld  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--schedule", default="s1")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--cfg", default=None, help="B,L,M,H,E,k,f (default: bench C2)")
    ap.add_argument("--layout", default=None, help="MP,EP,ESP (default: bench layout)")
    ap.add_argument("--transport", choices=("peer", "nccl"), default="peer")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    if args.cfg:
        b, l, m, h, e, k, f = args.cfg.split(",")
        cfg = MoEConfig(int(b), int(l), int(m), int(h), int(e), int(k), float(f))
    else:
        cfg = MoEConfig(**bench.C2)
    if args.layout:
        from paper_2407_00599_b200.config import ParallelLayout

        mp, ep, esp = (int(v) for v in args.layout.split(","))
        layout = ParallelLayout(mp, ep, esp, args.gpus)
    else:
        layout = bench.layout_for(args.gpus)
    peer = args.transport == "peer"
    w = ((PeerWorld if peer else NcclWorld)(layout, dev)) if world > 1 else LocalWorld(layout, dev)
    layer = MoELayer(cfg, layout, w)
    layer.init_random(0)
    x = torch.randn(cfg.tokens_per_rank, cfg.embed_dim, device=dev).to(torch.bfloat16)
    d = torch.randn(cfg.tokens_per_rank, cfg.embed_dim, device=dev).to(torch.bfloat16)
    for _ in range(3):
        layer.forward(args.schedule, {rank: x})
        layer.backward({rank: d})
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(args.steps):
            layer.forward(args.schedule, {rank: x})
            layer.backward({rank: d})
        torch.cuda.synchronize()
    if rank == 0:
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30, max_name_column_width=70))
        # GPU busy vs wall span
        evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
        if evs:
            t0 = min(e.time_range.start for e in evs)
            t1 = max(e.time_range.end for e in evs)
            busy = sum(e.time_range.end - e.time_range.start for e in evs)
            print(f"GPU span {(t1 - t0) / args.steps:.1f} us/step, summed kernel time {busy / args.steps:.1f} us/step")
    if world > 1:
        torch.distributed.barrier()
        torch.cuda.synchronize()
        sys.stdout.flush()
        os._exit(0)        # symmetric-memory mappings can stall process-group teardown


if __name__ == "__main__":
    main()
