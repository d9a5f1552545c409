"""NVLink store throughput of the peer push vs the number of issuing CTAs (torchrun, PeerWorld).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/probes/push_sms.py

Every rank stores `rows` rows of M=1024 bf16 into each peer's buffer (and its own); the
question for overlapping the dispatch with the GEMM is how few SMs saturate NVLink.
"""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2407_00599_b200 import kernels as K  # noqa: E402
from paper_2407_00599_b200.config import ParallelLayout  # noqa: E402
from paper_2407_00599_b200.world import PeerWorld  # noqa: E402


def main():
    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    world = PeerWorld(ParallelLayout(1, P, 1, P), dev)
    M, el, rows = 1024, 1, 8192
    src = torch.randn(P, 1, el, rows, M, device=dev).to(torch.bfloat16)
    fill = torch.full((P, 1, el), rows, dtype=torch.int32, device=dev)
    dst, peers = world.sym((P, el, rows, M))
    fan = [a + 2 * rank * el * rows * M for a in peers]
    for cap in (8, 16, 24, 32, 48, 74, 148, 296, 0):
        os.environ["PARM_PUSH_MAX_CTAS"] = str(cap)
        for _ in range(3):
            K.push_rows(src, fill, fan)
        world.peer_barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            K.push_rows(src, fill, fan)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 10], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        remote = (P - 1) * rows * M * 2
        if rank == 0:
            print(f"ctas {cap or 'all'}: {t.item() * 1e3:.1f} us per push, remote {remote / 1e6:.1f} MB, "
                  f"{remote / (t.item() * 1e-3) / 1e9:.0f} GB/s out per rank", flush=True)
        world.peer_barrier()
    torch.cuda.synchronize()
    dist.barrier()
    os._exit(0)


if __name__ == "__main__":
    main()
