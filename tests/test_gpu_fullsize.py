"""Parity at the benchmark's full size (BASELINE config 2 per-rank shape, N=1, S1).

The oracle's whole-layer restatement at B*L = 8192, M = 1024, H = 4096 is minutes of f64
NumPy, so this checks what is size-independent: the routing of all 8192 tokens bit for bit
against the oracle gate, and then -- given that routing -- per-token forward outputs and
input gradients on a token sample, and the full weight gradients of two experts (every row
routed to them), all against f64 restatements of dataplane.py's formulas (`_combine`,
`expert_shard_forward`) and their adjoints.  Tolerances as in test_gpu_parity.py.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import moe_oracle as O

pytestmark = pytest.mark.gpu

B, L, M, H, E, K, F = 8, 1024, 1024, 4096, 8, 2, 1.2


def _rel(a, b):
    b = np.asarray(b, dtype=np.float64)
    return np.linalg.norm(np.asarray(a, dtype=np.float64) - b) / max(np.linalg.norm(b), 1e-30)


def test_bench_size_layer_matches_oracle(cuda_lib):
    from paper_2407_00599_b200.config import MoEConfig, ParallelLayout, derive_capacity
    from paper_2407_00599_b200.runtime import MoELayer
    from paper_2407_00599_b200.world import LocalWorld

    cfg = MoEConfig(B, L, M, H, E, K, F)
    layout = ParallelLayout(1, 1, 1, 1)
    n = B * L
    w = O.Weights.generate(M, H, E, seed=11)
    w = O.Weights(O.round_bf16(w.gate), O.round_bf16(w.w1), O.round_bf16(w.w2))
    rng = np.random.default_rng(12)
    x = O.round_bf16(rng.normal(size=(n, M)))
    dout = O.round_bf16(rng.normal(size=(n, M)))
    layer = MoELayer(cfg, layout, LocalWorld(layout))
    layer.load_weights(w)
    dev = layer.dev
    out = layer.forward("s1", {0: torch.from_numpy(x).to(dev).to(torch.bfloat16)})[0].float().cpu().numpy()
    rt = layer.routing(0)
    ei, si = rt.expert_idx.cpu().numpy(), rt.slot_idx.cpu().numpy()
    cw = rt.combine_w.cpu().numpy().astype(np.float64)
    dx = layer.backward({0: torch.from_numpy(dout).to(dev).to(torch.bfloat16)})[0].float().cpu().numpy()
    grads = {k: v.float().cpu().numpy() for k, v in layer.shard_grads(0).items()}

    # routing of every token, bit-exact (dataplane.py:86-119)
    ref = O.gate(x, w.gate, K, derive_capacity(cfg))
    np.testing.assert_array_equal(ei, ref.expert_index)
    np.testing.assert_array_equal(si, ref.slot_index)

    # per-token forward and input gradient on a sample, given that routing
    logits = x @ w.gate
    probs = np.exp(logits - logits.max(1, keepdims=True))
    probs /= probs.sum(1, keepdims=True)
    sample = np.random.default_rng(13).choice(n, 96, replace=False)
    out_ref, dx_ref = np.zeros((96, M)), np.zeros((96, M))
    for i, t in enumerate(sample):
        dS = np.zeros(E)
        for j in range(K):
            if si[t, j] < 0:
                continue
            e = ei[t, j]
            pre = x[t] @ w.w1[e]
            h = np.maximum(pre, 0.0)
            y = h @ w.w2[e]
            out_ref[i] += cw[t, j] * y
            dS[e] = dout[t] @ O.round_bf16(y)            # the GPU keeps expert outputs in bf16
            dh = (cw[t, j] * dout[t]) @ w.w2[e].T * (pre > 0)
            dx_ref[i] += dh @ w.w1[e].T
        dlog = probs[t] * (dS - probs[t] @ dS)          # softmax adjoint; dS is zero off the kept picks
        dx_ref[i] += w.gate @ dlog
    assert O.max_rel_error(out[sample], out_ref) <= 1e-2
    assert _rel(dx[sample], dx_ref) <= 2e-2

    # full weight gradients of two experts: every row routed to them
    for e in (0, E - 1):
        t_idx, j_idx = np.nonzero((ei == e) & (si >= 0))
        xe = x[t_idx]
        dye = cw[t_idx, j_idx][:, None] * dout[t_idx]
        pre = xe @ w.w1[e]
        he = np.maximum(pre, 0.0)
        dw2 = O.round_bf16(he).T @ O.round_bf16(dye)       # GEMM operands are bf16 on the GPU
        dh = (O.round_bf16(dye) @ w.w2[e].T) * (pre > 0)
        dw1 = xe.T @ O.round_bf16(dh)
        assert _rel(grads["dw2"][e], dw2) <= 2e-2
        assert _rel(grads["dw1"][e], dw1) <= 2e-2


@pytest.mark.parametrize("P,lay", [(2, (2, 1, 2)), (4, (2, 2, 2))])
def test_bench_size_peer_transport_emulated(cuda_lib, P, lay):
    """The bench's multi-GPU layouts at full size on one GPU: S1 over PeerLocalWorld (the NVLink
    transport's fused kernels, peer tables and GEMM-epilogue return, every rank's buffers on this
    device) -- each rank's slice routing bit-exact against the oracle gate with the S1 quota, and
    outputs, dx and expert weight gradients bit-identical to the copy-collective transport."""
    from paper_2407_00599_b200.config import MoEConfig, ParallelLayout, derive_capacity
    from paper_2407_00599_b200.runtime import MoELayer
    from paper_2407_00599_b200.world import LocalWorld, PeerLocalWorld

    cfg = MoEConfig(B, L, M, H, E, K, F)
    mp = lay[0]
    layout = ParallelLayout(*lay, P)
    n = B * L
    w = O.Weights.generate(M, H, E, seed=21)
    w = O.Weights(O.round_bf16(w.gate), O.round_bf16(w.w1), O.round_bf16(w.w2))
    G = P // mp
    rng = np.random.default_rng(22)
    xs = [O.round_bf16(rng.normal(size=(n, M))) for _ in range(G)]
    ds = [O.round_bf16(rng.normal(size=(n, M))) for _ in range(G)]
    res = {}
    for wk in ("local", "peer"):
        W = PeerLocalWorld(layout) if wk == "peer" else LocalWorld(layout)
        layer = MoELayer(cfg, layout, W)
        assert layer.peer == (wk == "peer")
        layer.load_weights(w)
        dev = layer.dev
        outs = layer.forward("s1", {r: torch.from_numpy(xs[r // mp]).to(dev).to(torch.bfloat16) for r in range(P)})
        outs = {r: v.clone() for r, v in outs.items()}
        routes = {r: (layer.routing(r).expert_idx.clone(), layer.routing(r).slot_idx.clone()) for r in range(P)}
        dxs = layer.backward({r: torch.from_numpy(ds[r // mp]).to(dev).to(torch.bfloat16) for r in range(P)})
        dxs = {r: v.clone() for r, v in dxs.items()}
        grads = {r: {k: v.clone() for k, v in layer.shard_grads(r).items()} for r in range(P)}
        res[wk] = (outs, routes, dxs, grads)
        del layer, W
        torch.cuda.empty_cache()
    q = -(-derive_capacity(cfg) // mp)
    sl = n // mp
    for r in range(P):
        m = layout.mp_pos(r)
        ref = O.gate(xs[r // mp][m * sl:(m + 1) * sl], w.gate, K, q, token_offset=m * sl)
        for wk in ("local", "peer"):
            ei, si = (v.cpu().numpy() for v in res[wk][1][r])
            np.testing.assert_array_equal(ei, ref.expert_index, err_msg=f"{wk} rank {r}")
            np.testing.assert_array_equal(si, ref.slot_index, err_msg=f"{wk} rank {r}")
        a, b = res["local"], res["peer"]
        assert torch.equal(a[0][r], b[0][r]), f"rank {r} outputs differ"
        assert torch.equal(a[2][r], b[2][r]), f"rank {r} dx differs"
        for key in ("dw1", "dw2"):
            assert torch.equal(a[3][r][key], b[3][r][key]), f"rank {r} {key} differs"
        torch.testing.assert_close(a[3][r]["dgate"], b[3][r]["dgate"], rtol=1e-5, atol=1e-6)
