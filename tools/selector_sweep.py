"""Schedule selection on measured B200 steps: Algorithm 1 vs the B200 step model vs "always S1".

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 tools/selector_sweep.py \
        --profile profiles/nvlink_profile_p4.csv --peer-profile profiles/peer_profile_p4.json \
        --grid extended --transport both --out profiles/r2_selector_p4.csv
    python tools/selector_sweep.py --analyze profiles/r2_selector_p4.csv      # summary (no GPU)

Grid (Table 3 / moesched cli.SweepGrid:56-111, restricted to the P GPUs of one box):
  paper     N_MP in {2, 4} (N_MP = 1 makes S1 == S2), N_ESP in {1, 2, 4}, N_EP = P / N_ESP,
            (B, L) in {(2, 512), (2, 2048), (8, 2048)}, M/N_ESP and H/N_ESP in {1024, 4096},
            f in {1.2, 2.4}, E = max(2, N_EP), k = 2;
  extended  the paper grid plus k = 1 with f in {0.5, 1.0} (expert-slot volume E*T below the token
            volume B*L, the regime where S2's AllGather of slots is cheaper than S1's AllGather of
            tokens: paper §IV-D), (B, L) in {(2, 2048), (8, 2048)}, M/N_ESP = 1024.
Each point: baseline, S1 and S2 forward+backward as CUDA-graph replays (max over ranks), on the
NVLink peer transport and/or on NCCL collectives (the baseline always on NCCL).  The CSV keeps the
per-schedule features of selector.step_features so --analyze can fit and cross-validate the step
model offline.
"""

from __future__ import annotations

import argparse
import csv
import itertools
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2407_00599_b200 import selector as S  # noqa: E402
from paper_2407_00599_b200.config import MoEConfig, ParallelLayout, check_compatible  # noqa: E402


def grid(P: int, which: str):
    pts = []
    for mp, esp, (b, seq), m_sh, h_sh, f in itertools.product((2, 4), (1, 2, 4), ((2, 512), (2, 2048), (8, 2048)),
                                                              (1024, 4096), (1024, 4096), (1.2, 2.4)):
        pts.append((mp, esp, b, seq, m_sh, h_sh, 2, f))
    if which == "extended":
        for mp, esp, (b, seq), h_sh, f in itertools.product((2, 4), (1, 2, 4), ((2, 2048), (8, 2048)), (1024, 4096),
                                                            (0.5, 1.0)):
            pts.append((mp, esp, b, seq, 1024, h_sh, 1, f))
    out = []
    for mp, esp, b, seq, m_sh, h_sh, k, f in pts:
        if P % esp or P % mp:
            continue
        ep = P // esp
        try:
            cfg = MoEConfig(b, seq, m_sh * esp, h_sh * esp, max(2, ep), k, f)
            lay = ParallelLayout(mp, ep, esp, P)
            check_compatible(cfg, lay)
        except ValueError:
            continue
        out.append((cfg, lay))
    return out


def time_schedule(layer, schedule, x, d, dev, dist, steps=5):
    import torch

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


def measure(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2407_00599_b200.runtime import MoELayer
    from paper_2407_00599_b200.world import PeerWorld

    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    P, rank = dist.get_world_size(), dist.get_rank()
    prof = S.load_profile(args.profile)
    peer = json.loads(Path(args.peer_profile).read_text())
    pts = grid(P, args.grid)
    if args.limit:
        pts = pts[:args.limit]
    transports = ("peer", "nccl") if args.transport == "both" else (args.transport,)
    worlds = {}
    rows = []
    for i, (cfg, lay) in enumerate(pts):
        key = (lay.mp_size, lay.ep_size, lay.esp_size)
        if key not in worlds:                   # one set of communicators + symmetric buffers per layout
            worlds[key] = PeerWorld(lay, dev)
        gen = torch.Generator(device=dev).manual_seed(100 + rank // lay.mp_size)
        x = torch.randn(cfg.tokens_per_rank, cfg.embed_dim, generator=gen, device=dev).to(torch.bfloat16)
        dd = torch.randn(cfg.tokens_per_rank, cfg.embed_dim, generator=gen, device=dev).to(torch.bfloat16)
        t_base = None
        for tr in transports:
            layer = MoELayer(cfg, lay, worlds[key], peer=(tr == "peer"))
            layer.init_random(i)
            if t_base is None:
                t_base = time_schedule(layer, "baseline", x, dd, dev, dist)
            t = {"baseline": t_base, "s1": time_schedule(layer, "s1", x, dd, dev, dist),
                 "s2": time_schedule(layer, "s2", x, dd, dev, dist)}
            alg1 = S.select_schedule(cfg, lay, prof)
            row = {"transport": tr, "P": P, "MP": lay.mp_size, "EP": lay.ep_size, "ESP": lay.esp_size,
                   "B": cfg.samples_per_rank, "L": cfg.seq_len, "M": cfg.embed_dim, "H": cfg.hidden_dim,
                   "E": cfg.num_experts, "k": cfg.top_k, "f": cfg.capacity_factor,
                   "t_baseline_ms": t["baseline"], "t_s1_ms": t["s1"], "t_s2_ms": t["s2"],
                   "alg1_t_s1_ms": alg1.t_s1 * 1e3, "alg1_t_s2_ms": alg1.t_s2 * 1e3, "alg1_chosen": alg1.chosen,
                   "measured_best": "s1" if t["s1"] <= t["s2"] else "s2"}
            for s in ("baseline", "s1", "s2"):
                comm = (S._comm_nccl(cfg, lay, s, prof) if (s == "baseline" or tr == "nccl")
                        else S._comm_peer(cfg, lay, s, peer))
                for fk, fv in S.step_features(cfg, lay, s, comm).items():
                    row[f"{s}.{fk}"] = fv
            rows.append(row)
            if rank == 0:   # incremental: a failing point later in the grid keeps the rows measured so far
                new = not Path(args.out).exists() or len(rows) == 1
                with open(args.out, "w" if len(rows) == 1 else "a", newline="") as fh:
                    w = csv.DictWriter(fh, fieldnames=list(rows[0]))
                    if new:
                        w.writeheader()
                    w.writerow(row)
            del layer
            if tr == "peer":
                worlds[key].release()          # drop this layer's symmetric buffers (keeps the barrier's)
            torch.cuda.empty_cache()
            if rank == 0:
                print(json.dumps(row), flush=True)
    if rank == 0:
        for tr in transports:
            summ = analyze([r for r in rows if r["transport"] == tr])
            print("SUMMARY " + tr + " " + json.dumps(summ), flush=True)
    dist.barrier()
    torch.cuda.synchronize()
    sys.stdout.flush()
    os._exit(0)        # symmetric-memory mappings can stall process-group teardown


# ---------------------------------------------------------------- analysis (no GPU)
_PROFILES: dict = {}


def _feats(r: dict, s: str) -> dict:
    """Step-model features of schedule s at sweep row r: from the CSV when it carries the current
    feature set, else recomputed from the row's configuration and the calibrated profiles (so older
    sweeps can be re-analysed with a newer model)."""
    if all(f"{s}.{f}" in r for f in S.STEP_FEATURES):
        return {f: float(r[f"{s}.{f}"]) for f in S.STEP_FEATURES}
    if not _PROFILES:
        _PROFILES["nccl"] = S.load_profile(ROOT / "profiles" / "nvlink_profile_p4.csv")
        _PROFILES["peer"] = json.loads((ROOT / "profiles" / "peer_profile_p4.json").read_text())
    cfg = MoEConfig(int(r["B"]), int(r["L"]), int(r["M"]), int(r["H"]), int(r["E"]), int(r["k"]), float(r["f"]))
    lay = ParallelLayout(int(r["MP"]), int(r["EP"]), int(r["ESP"]), int(r["P"]))
    comm = (S._comm_nccl(cfg, lay, s, _PROFILES["nccl"]) if (s == "baseline" or r["transport"] == "nccl")
            else S._comm_peer(cfg, lay, s, _PROFILES["peer"]))
    return S.step_features(cfg, lay, s, comm)


def analyze(rows: list[dict], folds: int = 2) -> dict:
    """Agreement of each selector with the measured-faster of S1/S2, and the step model's
    accuracy.  The step model is fitted on (folds - 1) / folds of the points and evaluated on
    the held-out rest (k-fold by point index), so its agreement and error are out-of-sample."""
    n = len(rows)
    best = [r["measured_best"] for r in rows]
    pred_choice = [None] * n
    errs = []
    for fold in range(folds):
        train = [r for i, r in enumerate(rows) if i % folds != fold]
        samples = [(_feats(r, s), float(r[f"t_{s}_ms"]) / 1e3) for r in train for s in ("baseline", "s1", "s2")]
        model = S.fit_step_model(samples)
        for i, r in enumerate(rows):
            if i % folds != fold:
                continue
            p = {s: model.predict(_feats(r, s)) for s in ("baseline", "s1", "s2")}
            pred_choice[i] = "s1" if p["s1"] <= p["s2"] else "s2"
            for s in ("baseline", "s1", "s2"):
                m = float(r[f"t_{s}_ms"]) / 1e3
                errs.append(abs(p[s] - m) / m)
    full = S.fit_step_model([(_feats(r, s), float(r[f"t_{s}_ms"]) / 1e3) for r in rows
                             for s in ("baseline", "s1", "s2")])
    alg1_err = [abs(float(r[f"alg1_t_{s}_ms"]) - float(r[f"t_{s}_ms"])) / float(r[f"t_{s}_ms"])
                for r in rows for s in ("s1", "s2")]
    wins = {"s1": best.count("s1"), "s2": best.count("s2")}
    close = sum(abs(float(r["t_s1_ms"]) - float(r["t_s2_ms"])) <= 0.03 * max(float(r["t_s1_ms"]), float(r["t_s2_ms"]))
                for r in rows)
    chosen = lambda c, r: float(r[f"t_{c}_ms"])  # noqa: E731
    spd = [float(r["t_baseline_ms"]) / chosen(c, r) for c, r in zip(pred_choice, rows)]
    return {
        "points": n,
        "wins": wins,
        "c6_guard_each_wins_over_10pct": min(wins.values()) > 0.10 * n,
        "ties_within_3pct": close,
        "trivial_agree": wins["s1"] / n,                     # always choosing S1
        "alg1_agree": sum(r["alg1_chosen"] == b for r, b in zip(rows, best)) / n,
        "model_agree": sum(c == b for c, b in zip(pred_choice, best)) / n,
        "pred_vs_measured_err": {"model_mean": sum(errs) / len(errs), "model_max": max(errs),
                                 "alg1_comm_only_mean": sum(alg1_err) / len(alg1_err)},
        "model_coef_full_fit": dict(zip(S.STEP_FEATURES, full.coef)),
        "speedup_vs_baseline_model_choice": {"mean": sum(spd) / n, "min": min(spd)},
        "note": "model agreement and error are out-of-sample (2-fold by point index)",
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--profile", default="profiles/nvlink_profile_p4.csv")
    ap.add_argument("--peer-profile", default="profiles/peer_profile_p4.json")
    ap.add_argument("--grid", choices=("paper", "extended"), default="extended")
    ap.add_argument("--transport", choices=("peer", "nccl", "both"), default="both")
    ap.add_argument("--out", default="profiles/r2_selector_p4.csv")
    ap.add_argument("--limit", type=int, default=0)
    ap.add_argument("--analyze", default=None, help="summarise an existing sweep CSV (no GPU)")
    args = ap.parse_args()
    if args.analyze:
        rows = list(csv.DictReader(open(args.analyze)))
        summ = {tr: analyze([r for r in rows if r["transport"] == tr]) for tr in sorted({r["transport"] for r in rows})}
        print(json.dumps(summ, indent=1))
        Path(args.analyze.replace(".csv", "_summary.json")).write_text(json.dumps(summ, indent=1))
        return
    measure(args)


if __name__ == "__main__":
    main()
