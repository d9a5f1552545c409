"""NCCL collective bus bandwidth on the box (nccl-tests conventions), CUDA-graph timed, max over ranks.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/nccl_busbw.py

all_gather / reduce_scatter: busbw = algbw * (n-1)/n; all_reduce: algbw * 2(n-1)/n;
all_to_all: algbw * (n-1)/n; algbw = bytes per rank / time.  bf16, 1 MiB .. 512 MiB per rank.
Printed as JSON lines (rank 0), for comparison with the fused peer kernels' NVLink GB/s
(tools/probes/nvlink_probe.py) and the 770 GB/s measured peer-copy reference.
"""

from __future__ import annotations

import json
import os
import statistics
import sys

import torch
import torch.distributed as dist


def timed(fn, dev, reps=5, inner=5):
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


def main() -> int:
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    n, rank = dist.get_world_size(), dist.get_rank()
    for mib in (1, 8, 64, 256, 512):
        elems = mib * 1024 * 1024 // 2
        elems -= elems % n
        x = torch.randn(elems, device=dev).to(torch.bfloat16)
        big = torch.empty(elems * n, device=dev, dtype=torch.bfloat16)
        small = torch.empty(elems // n, device=dev, dtype=torch.bfloat16)
        y = torch.empty_like(x)
        byt = elems * 2
        cases = {
            "all_gather": (lambda: dist.all_gather_into_tensor(big, x), byt, (n - 1) / n * n),
            "reduce_scatter": (lambda: dist.reduce_scatter_tensor(small, x), byt, (n - 1) / n),
            "all_reduce": (lambda: dist.all_reduce(y), byt, 2 * (n - 1) / n),
            "all_to_all": (lambda: dist.all_to_all_single(y, x), byt, (n - 1) / n),
        }
        for name, (fn, b, factor) in cases.items():
            t = timed(fn, dev)
            # all_gather moves the gathered size; nccl-tests' algbw uses the output bytes for it
            algbw = (b * n if name == "all_gather" else b) / t / 1e9
            bus = algbw * (factor / n if name == "all_gather" else factor)
            if rank == 0:
                print(json.dumps({"collective": name, "ranks": n, "bytes_per_rank": b, "us": t * 1e6,
                                  "algbw_gbs": algbw, "busbw_gbs": bus}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
