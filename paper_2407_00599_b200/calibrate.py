"""Measure the collectives' alpha/beta on the B200 box and fit the selector's profile.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        -m paper_2407_00599_b200.calibrate --layout 2,2,2 --out profiles/nvlink_profile.csv

Each (collective, group) key of the reference's cost model (costs.py:23-32) is
timed through the SAME NcclWorld primitives the schedule executors use (one
P2P message per peer for the AlltoAlls), over element counts 2^14..2^24
(bf16), CUDA-event timed, max over ranks, median of repeats.  Output: the
reference's fit-sample CSV (``collective,group,elements,seconds``, readable by
``moesched fit``) and the fitted profile CSV.  ``elements`` follows the
reference convention: gathered length for allgather, per-rank buffer length
otherwise.  The overlap key is fitted like the reference's acceptance suite
(test_acceptance.py:285-294): t(A2A(ep&esp, x) with AG(mp, x*MP/ESP)) - t(AG(mp, x*MP/ESP)),
the pair executed exactly as S2's return runs it (MoELayer._saa: sequential unless
the layer runs with saa="phased"; --saa here), so the selector prices the overlap this hardware actually delivers.
"""

from __future__ import annotations

import argparse
import os
import statistics
import sys

import torch
import torch.distributed as dist

from .config import ParallelLayout, group_members
from .selector import FIT_HEADER, fit_profile, write_profile_csv
from .world import Msg, NcclWorld

SIZES = [2 ** k for k in range(14, 25, 2)]


def _time(fn, dev, reps=5, inner=4, warm=2) -> float:
    """Device time of one `fn`, measured the way the schedules run: `inner`
    back-to-back calls captured in a CUDA graph (no host launch gaps), replayed
    `reps` times; max over ranks, median over replays."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(inner):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    samples = []
    for _ in range(reps):
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 1e3 / inner], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        samples.append(float(t.item()))
    return statistics.median(samples)


def _a2a_msgs(world: NcclWorld, kind: str, send: torch.Tensor, recv: torch.Tensor) -> list[Msg]:
    grp = group_members(world.layout, kind, world.rank)
    g = len(grp)
    cs, cr = send.view(g, -1), recv.view(g, -1)
    msgs = []
    me = grp.index(world.rank)
    for i, peer in enumerate(grp):
        if peer == world.rank:
            msgs.append(Msg(peer, peer, cs[me], cr[me]))
            continue
        msgs.append(Msg(world.rank, peer, cs[i], None))
        msgs.append(Msg(peer, world.rank, None, cr[i]))
    # every rank enumerates the pairs in the same global order
    msgs.sort(key=lambda m: (m.src, m.dst))
    return msgs


def measure(layout: ParallelLayout, dev, saa: str = "seq") -> list[tuple[str, str, float, float]]:
    world = NcclWorld(layout, dev)
    rows = []
    bf = dict(dtype=torch.bfloat16, device=dev)
    for x in SIZES:
        for kind in ("mp", "esp"):
            g = len(group_members(layout, kind, world.rank))
            if g == 1:
                continue
            n = max(g, x // g)
            src = torch.randn(n, **bf)
            out = torch.empty(n * g, **bf)
            rows.append(("allgather", kind, n * g, _time(lambda: world.allgather(kind, {world.rank: src},
                                                                                {world.rank: out}), dev)))
        g = len(group_members(layout, "esp", world.rank))
        if g > 1:
            buf = torch.randn(x - x % g, **bf)
            rs = torch.empty(buf.numel() // g, **bf)
            rows.append(("reducescatter", "esp", buf.numel(),
                         _time(lambda: world.reduce_scatter("esp", {world.rank: buf}, {world.rank: rs}), dev)))
            rows.append(("allreduce", "esp", buf.numel(), _time(lambda: world.allreduce("esp", {world.rank: buf}), dev)))
        for kind in ("ep", "ep_esp"):
            g = len(group_members(layout, kind, world.rank))
            if g == 1:
                continue
            n = x - x % g
            send, recv = torch.randn(n, **bf), torch.empty(n, **bf)
            msgs = _a2a_msgs(world, kind, send, recv)
            rows.append(("alltoall", kind, n, _time(lambda: world.exchange(msgs), dev)))
        # overlap: the S2 return as the runtime executes it (MoELayer._saa) -- A2A(ep&esp, x)
        # together with AG(mp, x*MP/ESP) -- minus the AG alone, as the reference's acceptance
        # suite defines the key (test_acceptance.py:285-294).  Sequential SAA (the default on
        # NVSwitch, where phasing measured slower) makes this the plain A2A cost.
        P = layout.world_size
        mp_g = len(group_members(layout, "mp", world.rank))
        if P > 1 and mp_g > 1:
            n = x - x % (P * layout.ep_size)
            send, recv = torch.randn(n, **bf), torch.empty(n, **bf)
            msgs = _a2a_msgs(world, "ep_esp", send, recv)
            ag_n = max(mp_g * layout.ep_size, int(n * layout.mp_size / layout.esp_size) // mp_g)
            ag_n -= ag_n % layout.ep_size
            ag_src, ag_out = torch.randn(ag_n, **bf), torch.empty(layout.ep_size, mp_g, ag_n // layout.ep_size, **bf)
            ag = lambda: world.allgather("mp", {world.rank: ag_src}, {world.rank: ag_out})  # noqa: E731
            if saa == "phased" and layout.ep_size > 1:
                src_blocks = ag_src.view(layout.ep_size, -1)

                def saa():
                    hs = []
                    for j in range(layout.ep_size):
                        world.exchange([m for m in msgs
                                        if layout.ep_pos(m.src) == (m.dst // layout.mp_size + j) % layout.ep_size])
                        bj = (world.rank // layout.mp_size + j) % layout.ep_size
                        hs.append(world.allgather_async("mp", {world.rank: src_blocks[bj]},
                                                        {world.rank: ag_out[bj]}))
                    for h in hs:
                        world.wait(h)
            else:
                def saa():
                    world.exchange(msgs)
                    ag()

            t_both = _time(saa, dev)
            t_ag = _time(ag, dev)
            rows.append(("overlap", "ep_esp", n, max(t_both - t_ag, 1e-7)))
    return rows


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--layout", default=None, help="MP,EP,ESP (default: bench layout for the world size)")
    ap.add_argument("--out", default="profiles/nvlink_profile.csv")
    ap.add_argument("--samples-out", default=None)
    ap.add_argument("--saa", choices=("seq", "phased"), default="seq", help="S2 return execution to price (overlap key)")
    args = ap.parse_args(argv)
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    P = dist.get_world_size()
    if args.layout:
        mp, ep, esp = (int(v) for v in args.layout.split(","))
    else:
        mp, ep, esp = {2: (2, 1, 2), 4: (2, 2, 2), 8: (2, 4, 2)}[P]
    layout = ParallelLayout(mp, ep, esp, P)
    rows = measure(layout, dev, args.saa)
    if dist.get_rank() == 0:
        lines = [",".join(FIT_HEADER)] + [f"{c},{g},{x},{t:.9g}" for c, g, x, t in rows]
        samples_path = args.samples_out or args.out.replace(".csv", "_samples.csv")
        with open(samples_path, "w") as f:
            f.write("\n".join(lines) + "\n")
        samples: dict = {}
        for c, g, x, t in rows:
            samples.setdefault((c, g), []).append((float(x), t))
        prof = fit_profile(samples)
        # keys a layout cannot exercise (group of one) inherit a neighbour's fit so the
        # profile stays complete for select_schedule (documented in the CSV header row order)
        from .selector import ALL_KEYS, AlphaBeta

        fallback = prof.entries.get(("alltoall", "ep_esp")) or next(iter(prof.entries.values()))
        for key in ALL_KEYS:
            if key not in prof.entries:
                prof.add(AlphaBeta(fallback.alpha, fallback.beta, key[0], key[1], fallback.r_squared))
        with open(args.out, "w") as f:
            f.write(write_profile_csv(prof))
        print(f"calibrated P={P} layout mp{mp}-ep{ep}-esp{esp}: {len(rows)} samples -> {args.out}")
        for key, ab in sorted(prof.entries.items()):
            print(f"  {key[0]:14s} {key[1]:7s} alpha={ab.alpha * 1e6:8.2f} us  beta={ab.beta * 1e12:8.3f} ps/elem "
                  f"({2 / ab.beta / 1e9:7.1f} GB/s)  r2={ab.r_squared:.4f}")
    dist.barrier()
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
