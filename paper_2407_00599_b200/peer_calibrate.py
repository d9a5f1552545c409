"""Calibrate the cost terms of the fused NVLink peer transport on the box.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        -m paper_2407_00599_b200.peer_calibrate --out profiles/peer_profile_p4.json

On the peer transport (world.PeerWorld) the schedules' collectives are loads and
stores inside the permute kernels.  This measures that transport's constants (the
evidence behind DESIGN.md §(e)), each CUDA-graph timed (max over ranks, median of
repeats):

  barrier   alpha of one parm_peer_barrier
  push      alpha/beta of posted NVLink stores (parm_push_rows of x bf16 elements
            spread over every peer, + barrier)
  pull      beta of gathering rows from peers through a peer slot view instead of
            locally (combine_fwd over the same picks, remote minus local)
  allreduce alpha of the MP all-reduce of the gate gradient (NCCL, 32 KB)
  token     per-token cost of the token-side kernels (gate, combine, combine
            backward, dispatch backward, gate weight gradient) per embed column,
            the work S2 duplicates over the MP group (from the N=1 profile)
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch
import torch.distributed as dist

from . import kernels as K
from .config import ParallelLayout
from .world import PeerWorld


def _time(fn, dev, reps=7, inner=8) -> float:
    for _ in range(2):
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
    out = []
    for _ in range(reps):
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 1e3 / inner], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out.append(float(t.item()))
    return statistics.median(out)


def _fit(xs, ts):
    A = np.vstack([np.ones(len(xs)), np.asarray(xs, dtype=np.float64)]).T
    (a, b), *_ = np.linalg.lstsq(A, np.asarray(ts), rcond=None)
    return float(max(a, 0.0)), float(max(b, 0.0))


def measure(world: PeerWorld, dev) -> dict:
    P, rank = world.layout.world_size, world.rank
    res = {"P": P}
    res["barrier_alpha"] = _time(world.peer_barrier, dev)
    # push: every rank stores rows of M=1024 into every peer's buffer (segment per destination)
    M, el = 1024, 1
    xs, ts = [], []
    for rows in (64, 256, 1024, 4096):
        src = torch.randn(P, 1, el, rows, M, device=dev).to(torch.bfloat16)
        fill = torch.full((P, 1, el), rows, dtype=torch.int32, device=dev)
        dst, peers = world.sym((P, el, rows, M))
        fan = [a + 2 * rank * el * rows * M for a in peers]

        def push():
            K.push_rows(src, fill, fan)
            world.peer_barrier()
        t = _time(push, dev) - res["barrier_alpha"]
        xs.append(P * rows * M * (P - 1) / P)          # remote elements stored per rank
        ts.append(t)
    res["push_alpha"], res["push_beta"] = _fit(xs, ts)
    # pull: combine over picks whose rows live on peers vs the same picks locally
    n, k, E, q = 8192, 2, 8, 2458
    y, peers = world.sym((P, 1, E, q, M))
    ei = torch.randint(0, E, (n, k), dtype=torch.int32, device=dev)
    si = torch.randint(0, q, (n, k), dtype=torch.int32, device=dev)
    cw = torch.rand(n, k, device=dev)
    out = torch.empty(n, M, dtype=torch.bfloat16, device=dev)
    local = K.SlotView(y, e_local=E, n_p=1, stride_i=q * M, stride_slo=M)
    other = (rank + 1) % P
    remote = K.SlotView(None, e_local=E, n_p=1, stride_i=q * M, stride_slo=M,
                        peers=(peers[other] + 2 * rank * E * q * M,), peer_ep=0, peer_p=0)
    t_loc = _time(lambda: K.combine_fwd(local, ei, si, cw, out), dev)
    t_rem = _time(lambda: K.combine_fwd(remote, ei, si, cw, out), dev)
    res["pull_beta"] = max(t_rem - t_loc, 0.0) / (n * k * M)
    # NCCL all-reduce of the gate gradient (E x M f32) over the MP group (here: the world)
    g = torch.zeros(E, M, device=dev)
    res["allreduce_alpha"] = _time(lambda: dist.all_reduce(g), dev)
    return res


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/peer_profile.json")
    ap.add_argument("--token-cost", type=float, default=None,
                    help="per-token per-embed-column seconds of the token-side kernels (default: measured at N=1 "
                         "from profiles/r1_launches_n1.csv numbers, 9.4e-12)")
    args = ap.parse_args(argv)
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    P = dist.get_world_size()
    world = PeerWorld(ParallelLayout(1, P, 1, P), dev)
    res = measure(world, dev)
    res["token_beta"] = args.token_cost if args.token_cost is not None else 9.4e-12
    if dist.get_rank() == 0:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)
        print(json.dumps(res))
    dist.barrier()
    torch.cuda.synchronize()
    sys.stdout.flush()
    os._exit(0)


if __name__ == "__main__":
    sys.exit(main())
