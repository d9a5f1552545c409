"""Rank program for tests/test_world_gloo.py (torchrun, gloo backend, CPU tensors).

Exercises the NcclWorld plumbing (same class as on the GPUs, gloo instead of
NCCL) and the MoELayer message plans of every schedule against the oracle's
restated collectives (collectives.py semantics).  Exit code 0 = all checks
passed on every rank.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import moe_oracle as O  # noqa: E402
from paper_2407_00599_b200.config import MoEConfig, ParallelLayout, group_members  # noqa: E402
from paper_2407_00599_b200.runtime import MoELayer  # noqa: E402
from paper_2407_00599_b200.world import NcclWorld  # noqa: E402


def pattern(rank: int, shape, salt: int) -> torch.Tensor:
    n = int(np.prod(shape))
    return (torch.arange(n, dtype=torch.float32) * 0.001 + rank * 1000 + salt * 10).reshape(shape)


def gather_all(t: torch.Tensor) -> list[np.ndarray]:
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t.contiguous())
    return [o.numpy() for o in out]


def check_collectives(layout: ParallelLayout, fails: list) -> None:
    r = dist.get_rank()
    P = layout.world_size
    w = NcclWorld(layout, "cpu")
    ol = O.Layout(layout.mp_size, layout.ep_size, layout.esp_size, P, layout.esp_contiguous)
    for kind in ("mp", "esp", "ep"):
        g = len(group_members(layout, kind, r))
        x = pattern(r, (g * 3,), 1)
        allx = gather_all(x)
        out = torch.empty(g * g * 3)
        w.allgather(kind, {r: x}, {r: out})
        if not np.array_equal(out.numpy(), O.allgather(allx, ol, kind)[r]):
            fails.append(f"allgather {kind}")
        y = x.clone()
        w.allreduce(kind, {r: y})
        if not np.allclose(y.numpy(), O.allreduce(allx, ol, kind)[r]):
            fails.append(f"allreduce {kind}")
        rs = torch.empty(3)
        w.reduce_scatter(kind, {r: x}, {r: rs})
        if not np.allclose(rs.numpy(), O.reduce_scatter(allx, ol, kind)[r]):
            fails.append(f"reduce_scatter {kind}")


def check_plans(cfg: MoEConfig, layout: ParallelLayout, fails: list) -> None:
    """The runtime's message plans move exactly what the reference's fused collectives move."""
    r = dist.get_rank()
    P = layout.world_size
    ol = O.Layout(layout.mp_size, layout.ep_size, layout.esp_size, P, layout.esp_contiguous)
    layer = MoELayer(cfg, layout, NcclWorld(layout, "cpu"))
    d = layer.d
    for sched in ("s1", "s2"):
        b = layer._plan(sched, r)
        b["send"] = pattern(r, tuple(b["send"].shape), 2)
        b["route"].fill.copy_(torch.arange(d.E, dtype=torch.int32) + 10 * r)
        b["recv"] = torch.zeros_like(b["recv"], dtype=torch.float32)
        b["fill_in"].zero_()
        if sched == "s2":
            b["shard_fill"] = b["route"].fill.clone()
        layer.world.exchange(layer._fused_msgs(sched, "send", "recv", with_fill=True,
                                               fill_key="fill" if sched == "s1" else "shard_fill"))
        want = O.fused_dispatch(gather_all(b["send"].reshape(-1)), ol)[r]
        if not np.array_equal(b["recv"].reshape(-1).numpy(), want):
            fails.append(f"{sched} fused dispatch data")
        fills = gather_all(b["route"].fill.to(torch.float32))
        for s in range(P):
            j = layout.ep_pos(r)
            exp = fills[s][j * d.e_local:(j + 1) * d.e_local]
            if not np.array_equal(b["fill_in"][s, 0].numpy().astype(np.float32), exp):
                fails.append(f"{sched} fill counts from {s}")
        # return exchange == the A2A half of fused_combine; + the ESP sum == fused_combine
        b["y"] = pattern(r, tuple(b["y"].shape), 3)
        b["ret"] = torch.zeros_like(b["ret"], dtype=torch.float32)
        layer.world.exchange(layer._return_msgs(sched, "y", "ret"))
        ally = gather_all(b["y"].reshape(-1))
        if not np.array_equal(b["ret"].reshape(-1).numpy(), O.alltoall(ally, ol, "ep_esp")[r]):
            fails.append(f"{sched} return alltoall")
        ret = b["ret"].numpy()               # (P, e_local, q, M): ESP sum over sources of each EP block
        summed = []
        for j in range(layout.ep_size):
            srcs = [s for s in range(P) if layout.ep_pos(s) == j]
            acc = ret[srcs[0]].copy()
            for s in srcs[1:]:
                acc = acc + ret[s]
            summed.append(acc.reshape(-1))
        if not np.allclose(np.concatenate(summed), O.fused_combine(ally, ol)[r]):
            fails.append(f"{sched} fused combine")
    # baseline: EP AlltoAll of expert blocks per gathered block, and the whole-block return
    b = layer._plan("baseline", r)
    b["disp"] = pattern(r, tuple(b["disp"].shape), 4)
    b["recv"] = torch.zeros_like(b["recv"], dtype=torch.float32)
    b["blk_fill"].copy_(torch.arange(d.ESP * d.E, dtype=torch.int32).reshape(d.ESP, d.E) + 100 * r)
    layer.world.exchange(layer._ep_dispatch_msgs("disp", "recv", with_fill=True))
    alld = gather_all(b["disp"])
    allf = gather_all(b["blk_fill"])
    el = d.e_local
    for o in group_members(layout, "ep", r):
        j = group_members(layout, "ep", o).index(r)
        pos = layout.ep_pos(o)
        for q in range(d.ESP):
            if not np.array_equal(b["recv"][pos, q].numpy(), alld[o][q, j * el:(j + 1) * el]):
                fails.append(f"baseline dispatch from {o} block {q}")
            if not np.array_equal(b["fill_in"][pos, q].numpy(), allf[o][q, j * el:(j + 1) * el]):
                fails.append(f"baseline fills from {o} block {q}")
    b["y"] = pattern(r, tuple(b["y"].shape), 5)
    b["ret"] = torch.zeros_like(b["ret"], dtype=torch.float32)
    layer.world.exchange(layer._ep_return_msgs("y", "ret"))
    ally = gather_all(b["y"])
    for h in group_members(layout, "ep", r):
        if not np.array_equal(b["ret"][layout.ep_pos(h)].numpy(), ally[h][layout.ep_pos(r)]):
            fails.append(f"baseline return from {h}")


def main() -> int:
    dist.init_process_group("gloo")
    P = dist.get_world_size()
    fails: list[str] = []
    layouts = {2: [(2, 1, 2, True), (1, 2, 1, True), (2, 2, 1, True)],
               4: [(2, 2, 2, True), (2, 2, 2, False), (4, 4, 1, True), (1, 1, 4, True), (2, 4, 1, False)]}[P]
    for mp, ep, esp, contig in layouts:
        layout = ParallelLayout(mp, ep, esp, P, esp_contiguous=contig)
        check_collectives(layout, fails)
        E = max(2, ep) * 2
        check_plans(MoEConfig(2, 8, 16, 16 * esp, E, 2, 1.5), layout, fails)
    allf = [None] * P
    dist.all_gather_object(allf, fails)
    bad = sorted({x for fs in allf for x in fs})
    if dist.get_rank() == 0:
        print("\n".join(bad) if bad else f"GLOO OK P={P}")
    dist.barrier()
    dist.destroy_process_group()
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
