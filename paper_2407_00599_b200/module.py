"""``ParmMoE``: the hot path as a ``torch.nn.Module`` for training loops.

One process per GPU.  The module owns this rank's shards as fp32 master parameters
(gate (E, M), w1 (e_local, M, H/N_ESP), w2 (e_local, H/N_ESP, M), the reference layout of
``ExpertWeights.w1_shard`` / ``w2_shard``) and runs the layer through ``runtime.MoELayer``:
the forward and backward are the sm_100a kernels and the schedule's exchanges, wrapped in
one ``torch.autograd.Function`` so any surrounding model (attention, dense FFNs, losses)
back-propagates through it.  Before each forward the bf16 compute copies are refreshed
from the masters; the weight gradients arrive in fp32 straight from the wgrad GEMMs.

The schedule is chosen once by Algorithm 1 (``selector.select_schedule``) with a measured
profile, or fixed by the caller.  With N_MP > 1 every MP rank passes the same tokens
(the replicated-MP convention of the paper) and gets the full output back.
"""

from __future__ import annotations

import math

import torch
from torch import nn

from .config import MoEConfig, ParallelLayout
from .runtime import MoELayer
from .world import World, make_world


class _MoEFunction(torch.autograd.Function):
    """The layer keeps ONE set of activation buffers (routing, received rows, H and its ReLU
    mask) per schedule, so a backward is only valid for the most recent forward.  Each forward
    stamps a generation number into ctx; a backward whose forward has since been overwritten
    (microbatch loops running all forwards first, an eval forward in between) raises instead
    of silently returning the gradients of another batch.  x is saved through
    save_for_backward so autograd's version counter catches in-place edits of the input (the
    gate weight gradient reads it)."""

    @staticmethod
    def forward(ctx, x, gate, w1, w2, mod):          # noqa: D401 - autograd signature
        mod._sync_compute_weights()
        r = mod.rank
        out = mod.layer.forward(mod.schedule, {r: x})[r]
        mod._generation += 1
        ctx.mod = mod
        ctx.generation = mod._generation
        ctx.save_for_backward(x)
        return out.clone()                           # the layer reuses its output buffer next call

    @staticmethod
    def backward(ctx, dout):
        mod = ctx.mod
        if ctx.generation != mod._generation:
            raise RuntimeError("ParmMoE: backward of a forward whose activations were overwritten by a later "
                               "forward (one outstanding forward per module; run backward before the next "
                               "forward, or use one ParmMoE per microbatch in flight)")
        ctx.saved_tensors                            # autograd's in-place check of x
        r = mod.rank
        dx = mod.layer.backward({r: dout.contiguous().to(torch.bfloat16)})[r].clone()
        d, s = mod.layer.d, mod.layer.st[r]
        dgate = s.dgate[:, :d.M].clone()                                   # (E, M)
        dw1 = s.dw1t[:, :d.Hs, :d.M].transpose(1, 2).contiguous()         # (e_local, M, Hs)
        dw2 = s.dw2t[:, :d.M, :d.Hs].transpose(1, 2).contiguous()         # (e_local, Hs, M)
        return dx, dgate, dw1, dw2, None


class ParmMoE(nn.Module):
    """Parm MoE layer (gate + E ReLU experts, top-k, capacity f) on this rank's GPU."""

    def __init__(self, cfg: MoEConfig, layout: ParallelLayout, world: World | None = None, device=None,
                 schedule: str = "s1", seed: int = 0):
        super().__init__()
        self.layer = MoELayer(cfg, layout, world if world is not None else make_world(layout, device))
        if len(self.layer.ranks) != 1:
            raise ValueError("ParmMoE runs one rank per process (torchrun); use MoELayer to emulate a layout")
        self.rank = self.layer.ranks[0]
        self.schedule = schedule
        d, dev = self.layer.d, self.layer.dev
        gen = torch.Generator(device=dev).manual_seed(seed * 7919 + self.rank)
        g0 = torch.Generator(device=dev).manual_seed(seed)
        self.gate = nn.Parameter(torch.randn(d.E, d.M, generator=g0, device=dev))
        self.w1 = nn.Parameter(torch.randn(d.e_local, d.M, d.Hs, generator=gen, device=dev) / math.sqrt(d.M))
        self.w2 = nn.Parameter(torch.randn(d.e_local, d.Hs, d.M, generator=gen, device=dev) / math.sqrt(d.H))
        self._synced = None
        self._generation = 0

    def _sync_compute_weights(self) -> None:
        """bf16 compute copies (transposed, padded layouts of MoELayer) from the fp32 masters."""
        key = (self.gate._version, self.w1._version, self.w2._version)
        if key == self._synced:
            return
        d, s = self.layer.d, self.layer.st[self.rank]
        with torch.no_grad():
            s.gate[:, :d.M].copy_(self.gate)
            s.w1t[:, :d.Hs, :d.M].copy_(self.w1.transpose(1, 2))
            s.w2t[:, :d.M, :d.Hs].copy_(self.w2.transpose(1, 2))
        self._synced = key

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        """x: (B*L, M) tokens of this rank's MP group, bf16 or fp32; returns (B*L, M) bf16."""
        return _MoEFunction.apply(x.to(torch.bfloat16).contiguous(), self.gate, self.w1, self.w2, self)


__all__ = ["ParmMoE"]
