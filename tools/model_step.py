"""BERT-large-shaped MoE model training step on one B200 (BASELINE config 4).

    python tools/model_step.py [--layers 24] [--moe parm|torch] [--steps 10]

24 pre-LN transformer blocks, hidden 1024, 16 heads, FFN 4096; every other FFN is an MoE
layer with E=8 experts, top-2, f=1.2 (the paper's model-level setting).
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
    def __init__(self, M, heads, H, moe: nn.Module | None):
        super().__init__()
        self.ln1, self.ln2 = nn.LayerNorm(M), nn.LayerNorm(M)
        self.qkv, self.proj = nn.Linear(M, 3 * M), nn.Linear(M, M)
        self.heads = heads
        self.moe = moe
        if moe is None:
            self.fc1, self.fc2 = nn.Linear(M, H), nn.Linear(H, M)

    def forward(self, x, B, L):
        M = x.shape[-1]
        q, k, v = self.qkv(self.ln1(x)).view(B, L, 3, self.heads, M // self.heads).permute(2, 0, 3, 1, 4)
        a = F.scaled_dot_product_attention(q, k, v).transpose(1, 2).reshape(B * L, M)
        x = x + self.proj(a)
        h = self.ln2(x)
        if self.moe is None:
            return x + self.fc2(F.gelu(self.fc1(h)))
        return x + self.moe(h).to(x.dtype)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=24)
    ap.add_argument("--moe", choices=("parm", "torch"), default="parm")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.manual_seed(0)
    B, L, M, heads, H, E, k, f = 16, 512, 1024, 16, 4096, 8, 2, 1.2
    n = B * L
    cfg = MoEConfig(B, L, M, H, E, k, f)
    layout = ParallelLayout(1, 1, 1, 1)
    blocks = []
    for i in range(args.layers):
        moe = None
        if i % 2 == 1:
            moe = (ParmMoE(cfg, layout, LocalWorld(layout, dev), schedule="s1", seed=i) if args.moe == "parm"
                   else TorchMoE(M, H, E, k, f, n).to(dev))
        blocks.append(Block(M, heads, H, moe).to(dev))
    model = nn.ModuleList(blocks)
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
        opt.step()
        return loss

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(args.steps):
        loss = step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    print(json.dumps({"model": f"BERT-large-MoE ({args.layers} blocks, MoE every other FFN, E=8 top-2 f=1.2)",
                      "moe_impl": args.moe, "tokens_per_step": n, "ms_per_step": ms, "tokens_per_s": n / ms * 1e3,
                      "wall_ms_per_step": (time.perf_counter() - t0) / args.steps * 1e3, "loss": float(loss),
                      "data": "synthetic embeddings, MSE loss, AdamW, bf16 autocast (dense), fp32 masters"}))
    return 0


if __name__ == "__main__":
    sys.exit(main())
