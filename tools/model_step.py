"""MoE transformer training steps around the hot path (BASELINE configs 4-5).

    python tools/model_step.py [--model bert|gpt2] [--moe parm|torch] [--steps 10]
    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/model_step.py \
        --model gpt2 --gpus 4          # E=16, MP=2 ESP=2 (EP=2), NVLink peer transport

24 pre-LN transformer blocks, hidden 1024, 16 heads, FFN 4096; every other FFN is an MoE
layer, top-2, f=1.2 (the paper's model-level setting): bert = bidirectional
attention, E=8; gpt2 = causal attention, E=16.  Multi-GPU (torchrun): the MoE layers run the
Parm schedule over the (MP, EP, ESP) layout; the dense blocks are replicated inside an MP group
(the paper's replicated-MP convention) and data-parallel across groups (gradient all-reduce).
Synthetic token embeddings (B=16, L=512 -> 8192 tokens), MSE loss, AdamW, bf16 autocast for the
dense parts.  ``--moe parm`` uses ParmMoE (the sm_100a hot path); ``--moe torch`` an eager
PyTorch MoE with the same routing rule (softmax top-2, capacity drop, scatter/gather + bmm
experts) as the comparison point.  Prints one JSON line with the step time.
"""

from __future__ import annotations

import argparse
import json
import math
import sys
import time
from pathlib import Path

import torch
import torch.nn.functional as F
from torch import nn

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2407_00599_b200.config import MoEConfig, ParallelLayout  # noqa: E402
from paper_2407_00599_b200.module import ParmMoE  # noqa: E402
from paper_2407_00599_b200.world import LocalWorld  # noqa: E402


class TorchMoE(nn.Module):
    """Eager reference MoE (same math: raw softmax top-k weights, token-major capacity drop)."""

    def __init__(self, M, H, E, k, f, n):
        super().__init__()
        self.E, self.k = E, k
        self.cap = max(1, math.ceil(f * k * n / E))
        self.gate = nn.Parameter(torch.randn(M, E) * 1.0)
        self.w1 = nn.Parameter(torch.randn(E, M, H) / math.sqrt(M))
        self.w2 = nn.Parameter(torch.randn(E, H, M) / math.sqrt(H))

    def forward(self, x):
        n, M = x.shape
        probs = torch.softmax(x.float() @ self.gate, dim=-1)
        w, idx = probs.topk(self.k, dim=-1)
        onehot = F.one_hot(idx.reshape(-1), self.E)                          # (n*k, E) token-major
        pos = (onehot.cumsum(0) - 1).gather(1, idx.reshape(-1, 1)).squeeze(1)
        keep = pos < self.cap
        slot = idx.reshape(-1) * self.cap + pos.clamp(max=self.cap - 1)
        disp = torch.zeros(self.E * self.cap, M, device=x.device, dtype=x.dtype)
        src = x.repeat_interleave(self.k, 0)
        disp.index_copy_(0, slot[keep], src[keep])
        h = torch.relu(torch.bmm(disp.view(self.E, self.cap, M), self.w1.to(x.dtype)))
        y = torch.bmm(h, self.w2.to(x.dtype)).view(self.E * self.cap, M)
        out = (y[slot] * (w.reshape(-1, 1) * keep.unsqueeze(1)).to(y.dtype)).view(n, self.k, M).sum(1)
        return out


class Block(nn.Module):
    def __init__(self, M, heads, H, moe: nn.Module | None, causal: bool = False):
        super().__init__()
        self.causal = causal
        self.ln1, self.ln2 = nn.LayerNorm(M), nn.LayerNorm(M)
        self.qkv, self.proj = nn.Linear(M, 3 * M), nn.Linear(M, M)
        self.heads = heads
        self.moe = moe
        if moe is None:
            self.fc1, self.fc2 = nn.Linear(M, H), nn.Linear(H, M)

    def forward(self, x, B, L):
        M = x.shape[-1]
        q, k, v = self.qkv(self.ln1(x)).view(B, L, 3, self.heads, M // self.heads).permute(2, 0, 3, 1, 4)
        a = F.scaled_dot_product_attention(q, k, v, is_causal=self.causal).transpose(1, 2).reshape(B * L, M)
        x = x + self.proj(a)
        h = self.ln2(x)
        if self.moe is None:
            return x + self.fc2(F.gelu(self.fc1(h)))
        return x + self.moe(h).to(x.dtype)


def main() -> int:
    import os

    ap = argparse.ArgumentParser()
    ap.add_argument("--model", choices=("bert", "gpt2"), default="bert")
    ap.add_argument("--layers", type=int, default=24)
    ap.add_argument("--moe", choices=("parm", "torch"), default="parm")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--schedule", choices=("s1", "s2", "baseline"), default="s1",
                    help="MoE-layer schedule (baseline = the DeepSpeed-MoE ordering on NCCL collectives)")
    ap.add_argument("--transport", choices=("peer", "nccl"), default="peer",
                    help="multi-GPU S1/S2 exchanges: NVLink peer memory or NCCL collectives")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    E = 8 if args.model == "bert" else 16
    B, L = (16, 512) if args.model == "bert" else (8, 1024)
    M, heads, H, k, f = 1024, 16, 4096, 2, 1.2
    n = B * L
    cfg = MoEConfig(B, L, M, H, E, k, f)
    layout = {1: ParallelLayout(1, 1, 1, 1), 2: ParallelLayout(2, 1, 2, 2), 4: ParallelLayout(2, 2, 2, 4),
              8: ParallelLayout(2, 4, 2, 8)}[world]
    if world > 1 and args.moe != "parm":
        raise SystemExit("the eager comparison MoE is single-GPU")
    torch.manual_seed(1234 + rank // layout.mp_size)    # MP ranks hold identical dense replicas and tokens
    mk_world = None
    if world > 1:
        from paper_2407_00599_b200.world import NcclWorld, PeerWorld

        mk_world = PeerWorld(layout, dev) if args.transport == "peer" else NcclWorld(layout, dev)
    blocks = []
    for i in range(args.layers):
        moe = None
        if i % 2 == 1:
            if args.moe == "parm":
                moe = ParmMoE(cfg, layout, mk_world if world > 1 else LocalWorld(layout, dev), schedule=args.schedule,
                              seed=i)
            else:
                moe = TorchMoE(M, H, E, k, f, n).to(dev)
        blocks.append(Block(M, heads, H, moe, causal=args.model == "gpt2").to(dev))
    model = nn.ModuleList(blocks)
    if world > 1:   # identical dense init on every rank
        for p_ in model.parameters():
            if not any(p_ is q_ for blk in blocks if blk.moe is not None for q_ in (blk.moe.w1, blk.moe.w2)):
                dist.broadcast(p_.data, 0)
    dense = [p_ for p_ in model.parameters()
             if not any(p_ is q_ for blk in blocks if blk.moe is not None for q_ in (blk.moe.w1, blk.moe.w2))]
    opt = torch.optim.AdamW(model.parameters(), lr=1e-4, fused=True)
    x0 = torch.randn(n, M, device=dev)
    target = torch.randn(n, M, device=dev)

    def step():
        opt.zero_grad(set_to_none=True)
        with torch.autocast("cuda", dtype=torch.bfloat16):
            x = x0
            for blk in model:
                x = blk(x, B, L)
            loss = F.mse_loss(x.float(), target)
        loss.backward()
        if world > 1:       # data-parallel dense (and gate) gradients; expert shards are unique per rank
            for p_ in dense:
                if p_.grad is not None:
                    dist.all_reduce(p_.grad, op=dist.ReduceOp.AVG)
        opt.step()
        return loss

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(args.steps):
        loss = step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if dist is not None:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    toks = (world // layout.mp_size) * n
    if rank == 0:
        name = {"bert": "BERT-large-MoE", "gpt2": "GPT-2-MoE"}[args.model]
        print(json.dumps({"model": f"{name} ({args.layers} blocks, MoE every other FFN, E={E} top-2 f=1.2)",
                          "moe_impl": args.moe, "schedule": args.schedule if args.moe == "parm" else None,
                          "transport": args.transport if world > 1 else "local", "n_gpus": world,
                          "layout": f"MP={layout.mp_size} EP={layout.ep_size} ESP={layout.esp_size}",
                          "tokens_per_step": toks, "ms_per_step": ms, "tokens_per_s": toks / ms * 1e3,
                          "wall_ms_per_step": (time.perf_counter() - t0) / args.steps * 1e3, "loss": float(loss),
                          "data": "synthetic embeddings, MSE loss, AdamW, bf16 autocast (dense), fp32 masters"}),
              flush=True)
    if dist is not None:
        dist.barrier()
        sys.stdout.flush()
        os._exit(0)
    return 0


if __name__ == "__main__":
    sys.exit(main())
