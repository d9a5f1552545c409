"""NCCL point-to-point strategies over NVLink (2+ ranks): GB/s per rank for one exchange.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/p2p_bench.py
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / reps], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    r, P = dist.get_rank(), dist.get_world_size()
    MB = 20
    n = MB * 1024 * 1024 // 2
    send = torch.randn(n, device="cuda").to(torch.bfloat16)
    recv = torch.empty(P * n, device="cuda", dtype=torch.bfloat16)
    res = {}
    for pieces in (1, 2, 8, 32):
        m = n // pieces

        def ex():
            ops = []
            for d in range(P):
                if d == r:
                    continue
                for i in range(pieces):
                    ops.append(dist.P2POp(dist.isend, send[i * m:(i + 1) * m], d))
                    ops.append(dist.P2POp(dist.irecv, recv[d * n + i * m:d * n + (i + 1) * m], d))
            for q in dist.batch_isend_irecv(ops):
                q.wait()

        ms = timeit(ex)
        res[f"p2p {pieces} msgs/peer"] = (P - 1) * n * 2 / (ms / 1e3) / 1e9
    a2a_in = torch.randn(P * n, device="cuda").to(torch.bfloat16)
    a2a_out = torch.empty_like(a2a_in)
    ms = timeit(lambda: dist.all_to_all_single(a2a_out, a2a_in))
    res["all_to_all_single"] = (P - 1) * n * 2 / (ms / 1e3) / 1e9
    ag_out = torch.empty(P * n, device="cuda", dtype=torch.bfloat16)
    ms = timeit(lambda: dist.all_gather_into_tensor(ag_out, send))
    res["all_gather (busbw)"] = (P - 1) * n * 2 / (ms / 1e3) / 1e9
    if r == 0:
        print(f"P={P} {MB} MB per peer, NCCL env: " + " ".join(f"{k}={v}" for k, v in os.environ.items()
                                                              if k.startswith("NCCL_")))
        for k, v in res.items():
            print(f"  {k:28s} {v:8.1f} GB/s per rank")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
