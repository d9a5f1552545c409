"""Selector vs measured-best schedule over a sub-grid of the paper's MoE-layer grid.

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 tools/selector_sweep.py \
        --profile profiles/nvlink_profile_p4.csv --out profiles/selector_sweep_p4.csv

Grid (Table 3 / moesched cli.SweepGrid:56-111, restricted to P GPUs of one box):
N_MP in {2, 4} (N_MP = 1 makes S1 == S2), N_ESP in {1, 2, 4}, N_EP = P / N_ESP,
(B, L) in {(2, 512), (2, 2048), (8, 2048)}, M/N_ESP and H/N_ESP in {1024, 4096}, f in {1.2, 2.4}, E = max(2, N_EP), k = 2.
Each point: baseline, S1, S2 forward+backward timed as CUDA-graph replays (max over ranks).
"""

from __future__ import annotations

import argparse
import itertools
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2407_00599_b200.config import MoEConfig, ParallelLayout, check_compatible  # noqa: E402
from paper_2407_00599_b200.runtime import MoELayer  # noqa: E402
from paper_2407_00599_b200.selector import load_profile, select_schedule  # noqa: E402
from paper_2407_00599_b200.world import NcclWorld, PeerWorld  # noqa: E402


def time_schedule(layer, schedule, x, d, dev, steps=5):
    r = layer.ranks[0]
    g = layer.capture_step(schedule, {r: x}, {r: d}, warmup=1)
    g.replay()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / steps], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    del g
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--profile", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--limit", type=int, default=0)
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    P, rank = dist.get_world_size(), dist.get_rank()
    prof = load_profile(args.profile)
    rows = []
    pts = []
    for mp, esp, (b, seq), m_sh, h_sh, f in itertools.product((2, 4), (1, 2, 4), ((2, 512), (2, 2048), (8, 2048)),
                                                              (1024, 4096), (1024, 4096), (1.2, 2.4)):
        if P % esp or P % mp:
            continue
        ep = P // esp
        try:
            cfg = MoEConfig(b, seq, m_sh * esp, h_sh * esp, max(2, ep), 2, f)
            lay = ParallelLayout(mp, ep, esp, P)
            check_compatible(cfg, lay)
        except ValueError:
            continue
        pts.append((cfg, lay))
    if args.limit:
        pts = pts[:args.limit]
    worlds = {}
    for i, (cfg, lay) in enumerate(pts):
        key = (lay.mp_size, lay.ep_size, lay.esp_size)
        if key not in worlds:                       # one set of communicators per layout
            peer = os.environ.get("PARM_PEER", "0") == "1"
            worlds[key] = (PeerWorld if peer else NcclWorld)(lay, dev)
        layer = MoELayer(cfg, lay, worlds[key])
        layer.init_random(i)
        gen = torch.Generator(device=dev).manual_seed(100 + rank // lay.mp_size)
        x = torch.randn(cfg.tokens_per_rank, cfg.embed_dim, generator=gen, device=dev).to(torch.bfloat16)
        dd = torch.randn(cfg.tokens_per_rank, cfg.embed_dim, generator=gen, device=dev).to(torch.bfloat16)
        t = {s: time_schedule(layer, s, x, dd, dev) for s in ("baseline", "s1", "s2")}
        rep = select_schedule(cfg, lay, prof)
        best = "s1" if t["s1"] <= t["s2"] else "s2"
        rows.append({"P": P, "MP": lay.mp_size, "EP": lay.ep_size, "ESP": lay.esp_size, "B": cfg.samples_per_rank,
                     "L": cfg.seq_len, "M": cfg.embed_dim, "H": cfg.hidden_dim, "E": cfg.num_experts,
                     "f": cfg.capacity_factor, "t_baseline_ms": t["baseline"], "t_s1_ms": t["s1"], "t_s2_ms": t["s2"],
                     "pred_s1_ms": rep.t_s1 * 1e3, "pred_s2_ms": rep.t_s2 * 1e3, "chosen": rep.chosen,
                     "measured_best": best, "speedup_chosen": t["baseline"] / t[rep.chosen],
                     "speedup_best": t["baseline"] / t[best]})
        del layer
        if isinstance(worlds[key], PeerWorld):
            worlds[key].release()
        torch.cuda.empty_cache()
        if rank == 0:
            print(json.dumps(rows[-1]), flush=True)
    if rank == 0:
        import csv

        with open(args.out, "w", newline="") as fh:
            w = csv.DictWriter(fh, fieldnames=list(rows[0]))
            w.writeheader()
            w.writerows(rows)
        n = len(rows)
        agree = sum(r["chosen"] == r["measured_best"] for r in rows)
        close = sum(r["chosen"] != r["measured_best"] and
                    abs(r["t_s1_ms"] - r["t_s2_ms"]) <= 0.03 * max(r["t_s1_ms"], r["t_s2_ms"]) for r in rows)
        worse = sorted((r["speedup_chosen"] for r in rows))
        summary = {"points": n, "agree": agree, "agree_frac": agree / n, "disagree_within_3pct": close,
                   "min_speedup_vs_baseline": worse[0], "mean_speedup_vs_baseline": sum(worse) / n,
                   "s1_best": sum(r["measured_best"] == "s1" for r in rows)}
        print("SUMMARY " + json.dumps(summary), flush=True)
        with open(args.out.replace(".csv", "_summary.json"), "w") as fh:
            json.dump(summary, fh, indent=1)
    dist.barrier()
    torch.cuda.synchronize()
    sys.stdout.flush()
    os._exit(0)        # symmetric-memory mappings can stall process-group teardown


if __name__ == "__main__":
    main()
