"""ParmMoE (torch.nn.Module + autograd.Function around the hot path) on one GPU."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import moe_oracle as O

pytestmark = pytest.mark.gpu


def _module(cfg_t=(2, 64, 128, 256, 4, 2, 1.2)):
    from paper_2407_00599_b200.config import MoEConfig, ParallelLayout
    from paper_2407_00599_b200.module import ParmMoE
    from paper_2407_00599_b200.world import LocalWorld

    cfg = MoEConfig(*cfg_t)
    layout = ParallelLayout(1, 1, 1, 1)
    return ParmMoE(cfg, layout, LocalWorld(layout), schedule="s1", seed=3), cfg


def test_module_matches_oracle_and_autograd_grads(cuda_lib):
    mod, cfg = _module()
    n, M = cfg.tokens_per_rank, cfg.embed_dim
    rng = np.random.default_rng(0)
    x = torch.from_numpy(O.round_bf16(rng.normal(size=(n, M)))).float().cuda().requires_grad_(True)
    dout = torch.from_numpy(O.round_bf16(rng.normal(size=(n, M)))).float().cuda()
    out = mod(x)
    (out.float() * dout).sum().backward()
    # oracle on the same bf16-rounded master weights
    g = O.round_bf16(mod.gate.detach().cpu().double().numpy().T)                 # (M, E)
    w1 = O.round_bf16(mod.w1.detach().cpu().double().numpy())                    # (E, M, H)
    w2 = O.round_bf16(mod.w2.detach().cpu().double().numpy())                    # (E, H, M)
    w = O.Weights(g, w1, w2)
    lay = O.Layout(1, 1, 1, 1)
    ref, caches, _ = O.schedule_forward("s1", n, w, cfg.top_k, cfg.capacity_factor, lay,
                                        x.detach().cpu().double().numpy()[None])
    rg = O.schedule_backward("s1", caches, w, lay, dout.cpu().double().numpy()[None])[0]
    assert O.max_rel_error(out.detach().float().cpu().numpy(), ref[0]) <= 1e-2

    def nerr(a, b):
        b = np.asarray(b, dtype=np.float64)
        return np.linalg.norm(np.asarray(a, dtype=np.float64) - b) / max(np.linalg.norm(b), 1e-30)

    assert nerr(x.grad.cpu().numpy(), rg["dx"]) <= 2e-2
    assert nerr(mod.w1.grad.cpu().numpy(), rg["dw1"]) <= 2e-2
    assert nerr(mod.w2.grad.cpu().numpy(), rg["dw2"]) <= 2e-2
    assert nerr(mod.gate.grad.cpu().numpy().T, rg["dgate"]) <= 2e-2


def test_module_trains(cuda_lib):
    """A few SGD steps on a regression target lower the loss (weights re-synced every step)."""
    mod, cfg = _module()
    n, M = cfg.tokens_per_rank, cfg.embed_dim
    gen = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(n, M, generator=gen, device="cuda")
    target = torch.randn(n, M, generator=gen, device="cuda") * 0.1
    opt = torch.optim.SGD(mod.parameters(), lr=0.05)
    losses = []
    for _ in range(6):
        opt.zero_grad()
        loss = ((mod(x).float() - target) ** 2).mean()
        loss.backward()
        opt.step()
        losses.append(float(loss))
    assert losses[-1] < losses[0]


def test_module_rejects_backward_of_an_overwritten_forward(cuda_lib):
    """One activation set per module: a second forward before the first backward must not
    silently produce gradients of the second batch."""
    mod, cfg = _module()
    n, M = cfg.tokens_per_rank, cfg.embed_dim
    x1 = torch.randn(n, M, device="cuda", requires_grad=True)
    x2 = torch.randn(n, M, device="cuda", requires_grad=True)
    out1 = mod(x1)
    out2 = mod(x2)
    with pytest.raises(RuntimeError, match="overwritten by a later forward"):
        out1.float().sum().backward()
    out2.float().sum().backward()          # the latest forward is still valid
    assert x2.grad is not None and torch.isfinite(x2.grad).all()


def test_captured_step_sees_gate_weight_updates(cuda_lib):
    """refresh_gate() updates the f64 gate copy in place, so a captured step routes with the new
    weights (the graph's gate node keeps reading the same buffer)."""
    from paper_2407_00599_b200.config import MoEConfig, ParallelLayout
    from paper_2407_00599_b200.runtime import MoELayer
    from paper_2407_00599_b200.world import LocalWorld

    cfg = MoEConfig(2, 64, 128, 256, 4, 2, 1.2)
    layout = ParallelLayout(1, 1, 1, 1)
    layer = MoELayer(cfg, layout, LocalWorld(layout))
    layer.init_random(0)
    x = torch.randn(128, 128, device="cuda").to(torch.bfloat16)
    d = torch.randn(128, 128, device="cuda").to(torch.bfloat16)
    g = layer.capture_step("s1", {0: x}, {0: d}, warmup=1)
    g.replay()
    before = layer.routing(0).expert_idx.clone()
    layer.init_random(7)                    # new gate weights, refreshed in place
    g.replay()
    torch.cuda.synchronize()
    replayed = layer.routing(0).expert_idx.clone()
    layer.forward("s1", {0: x})
    eager = layer.routing(0).expert_idx.clone()
    assert torch.equal(replayed, eager)
    assert not torch.equal(before, eager)
