"""Per-kernel time of one rank's step under torchrun (CUPTI via torch.profiler, CUDA-graph
replays of the bench layer): where the step goes at N > 1, where ncu (one process) cannot look.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        tools/probes/step_profile.py N [schedule] [peer|peer-<s1_return>|nccl]
"""
import collections
import json
import os
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2407_00599_b200.config import MoEConfig  # noqa: E402
from paper_2407_00599_b200.runtime import MoELayer  # noqa: E402
from paper_2407_00599_b200.world import NcclWorld, PeerWorld  # noqa: E402


def main():
    n = int(sys.argv[1])
    schedule = sys.argv[2] if len(sys.argv) > 2 else "s1"
    transport = sys.argv[3] if len(sys.argv) > 3 else "peer"
    rank, lrank = int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(lrank)
    dev = torch.device("cuda", lrank)
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=dev)
    cfg = MoEConfig(**bench.C2)
    layout = bench.layout_for(n)
    peer = transport.startswith("peer")
    opts = {"s1_return": transport.split("-", 1)[1]} if "-" in transport else {}
    layer = MoELayer(cfg, layout, PeerWorld(layout, dev) if peer else NcclWorld(layout, dev), peer=peer, **opts)
    layer.init_random(0)
    g = torch.Generator(device=dev).manual_seed(1000 + rank // layout.mp_size)
    x = torch.randn(cfg.tokens_per_rank, cfg.embed_dim, generator=g, device=dev).to(torch.bfloat16)
    d = torch.randn(cfg.tokens_per_rank, cfg.embed_dim, generator=g, device=dev).to(torch.bfloat16)
    graph = layer.capture_step(schedule, {rank: x}, {rank: d})
    for _ in range(5):
        graph.replay()
    torch.cuda.synchronize()
    dist.barrier()
    steps = 10
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            graph.replay()
        torch.cuda.synchronize()
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    span = [None, None]
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        tot[e.name[:70]] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
        cnt[e.name[:70]] += 1
    rows = sorted(tot.items(), key=lambda kv: -kv[1])
    # every kernel of the last profiled step in launch order, with its duration (barriers by position)
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    per_step = len(evs) // steps
    seq = [(e.name[:40], round(e.time_range.end - e.time_range.start, 2)) for e in evs[-per_step:]]
    if rank == 0:
        out = {"n": n, "schedule": schedule, "transport": transport, "steps": steps,
               "kernels_us_per_step": {k: round(v / steps, 2) for k, v in rows},
               "launches_per_step": {k: cnt[k] / steps for k, _ in rows},
               "sum_us_per_step": round(sum(tot.values()) / steps, 1),
               "last_step_sequence_us": seq}
        print(json.dumps(out, indent=1))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
