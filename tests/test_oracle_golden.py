"""Pin the CPU oracle to the real reference (golden fixtures from tests/golden/make_golden.py)
and check its hand-derived backward against torch float64 autograd."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import moe_oracle as O

# The reference's own golden vector, test_dataplane.py:113-130 (cfg B=1 L=8 M=4 H=4 E=2 k=1 f=2,
# weight seed 2024, input seed 99), checked at the reference's rtol 1e-14.
GOLDEN_OUTPUT = np.array([
    [-0.05979384657637676, 0.15185705966043322, -0.10612337709716334, 0.11755696695576796],
    [-0.6429848273406604, 1.4031655429257417, 1.9546437606040847, 0.4486660339080583],
    [0.004660389732578047, 0.35631625640939363, 0.3376851614954176, 0.18945729801611136],
    [-0.01799903093222844, 0.12084517347324827, -0.1301303355427365, 0.05819028538223777],
    [-0.20225905409404188, -0.14007058509538675, -0.07143392262900716, -0.16565717872448996],
    [-0.012042422705751267, -0.09206698740876898, -0.26487397765697857, -0.1968289809241353],
    [-0.19378972066014516, 0.49216330537083797, -0.3439420739875189, 0.3809979302621517],
    [-0.04739256754969226, -0.048607725630537335, -0.2840253184788717, -0.14907690979535176],
])


def test_reference_golden_vector():
    w = O.Weights.generate(4, 4, 2, seed=2024)
    tokens = np.random.default_rng(99).normal(size=(8, 4))
    out, _ = O.block_forward(tokens, w, 1, O.derive_capacity(8, 2, 1, 2.0))
    np.testing.assert_allclose(out, GOLDEN_OUTPUT, rtol=1e-14, atol=1e-16)


def test_capacity_known_answers(golden):
    meta, _ = golden
    kat = meta["costs"]["capacity_kat"]
    assert kat == [308, 2458, 615, 4916]
    assert O.derive_capacity(512, 4, 2, 1.2) == 308
    assert O.derive_capacity(8192, 8, 2, 1.2) == 2458
    assert O.derive_capacity(512, 4, 2, 2.4) == 615
    assert O.derive_capacity(8192, 8, 2, 2.4) == 4916


def test_gate_matches_reference(golden):
    meta, arr = golden
    assert len(meta["gate"]) >= 8
    for case in meta["gate"]:
        r = O.gate(arr[case["tokens"]], arr[case["weights"]], case["k"], case["cap"], case["offset"])
        np.testing.assert_array_equal(r.expert_index, arr[case["expert_index"]], err_msg=case["name"])
        np.testing.assert_array_equal(r.slot_index, arr[case["slot_index"]], err_msg=case["name"])
        np.testing.assert_array_equal(r.combine_weights, arr[case["combine_weights"]], err_msg=case["name"])
        assert sorted(map(list, r.dropped)) == case["dropped"], case["name"]
        d = O.dispatch_tensor(arr[case["tokens"]], r, arr[case["weights"]].shape[1])
        assert d.sum() == pytest.approx(case["dispatch_sum"], rel=1e-12, abs=1e-12)


@pytest.mark.parametrize("seed", range(6))
def test_vectorised_slots_equal_reference_loop(seed):
    rng = np.random.default_rng(seed)
    n, M, E = int(rng.integers(1, 200)), 16, int(rng.integers(2, 9))
    k = int(rng.integers(1, E + 1))
    cap = int(rng.integers(1, 60))
    x, w = rng.normal(size=(n, M)), rng.normal(size=(M, E))
    a, b = O.gate(x, w, k, cap, 5), O.gate_loop(x, w, k, cap, 5)
    np.testing.assert_array_equal(a.expert_index, b.expert_index)
    np.testing.assert_array_equal(a.slot_index, b.slot_index)
    assert a.dropped == b.dropped


def test_forward_matches_reference(golden):
    meta, arr = golden
    case = meta["forward"][1]
    B, L, M, H, E, k, f = case["cfg"]
    w = O.Weights(arr[case["gate"]], arr[case["w1"]], arr[case["w2"]])
    out, _ = O.block_forward(arr[case["tokens"]], w, k, O.derive_capacity(B * L, E, k, f))
    np.testing.assert_allclose(out, arr[case["out"]], rtol=1e-12, atol=1e-14)


def test_schedule_outputs_and_drops_match_reference(golden):
    meta, arr = golden
    assert len(meta["schedules"]) >= 8
    for case in meta["schedules"]:
        B, L, M, H, E, k, f = case["cfg"]
        lay = O.Layout(*case["layout"], esp_contiguous=case["esp_contiguous"])
        w = O.Weights.generate(M, H, E, seed=case["seed"])
        inputs = np.random.default_rng(case["seed"] + 1).normal(size=(lay.world // lay.mp, B * L, M))
        if case["bf16"]:
            w = O.Weights(O.round_bf16(w.gate), O.round_bf16(w.w1), O.round_bf16(w.w2))
            inputs = O.round_bf16(inputs)
        assert case["capacity"] == O.derive_capacity(B * L, E, k, f)
        for s, rec in case["results"].items():
            outs, _, drops = O.schedule_forward(s, B * L, w, k, f, lay, inputs)
            assert sorted(map(list, drops)) == rec["dropped"], (case["name"], s)
            if "outputs" in rec:
                np.testing.assert_allclose(outs, arr[rec["outputs"]], rtol=1e-9, atol=1e-12,
                                           err_msg=f"{case['name']}/{s}")
            np.testing.assert_allclose(outs.sum(axis=2), arr[rec["row_sums"]], rtol=1e-9, atol=1e-9)
            assert rec["oracle_error"] < 1e-9 or s == "s1"


def test_collectives_match_reference(golden):
    meta, arr = golden
    for case in meta["collectives"]:
        lay = O.Layout(*case["layout"], esp_contiguous=case["esp_contiguous"])
        bufs = list(arr[case["inputs"]])
        checks = {
            "fused_dispatch": O.fused_dispatch(bufs, lay),
            "fused_combine": O.fused_combine(bufs, lay),
            "saa": O.saa(bufs, lay),
            "alltoall_ep": O.alltoall(bufs, lay, "ep"),
            "allgather_esp": O.allgather(bufs, lay, "esp"),
            "reduce_scatter_esp": O.reduce_scatter(bufs, lay, "esp"),
            "allreduce_mp": O.allreduce(bufs, lay, "mp"),
        }
        for key, got in checks.items():
            np.testing.assert_array_equal(np.stack(got), arr[case[key]], err_msg=f"{case['name']}/{key}")


def test_backward_matches_torch_autograd():
    """The hand-derived adjoint equals float64 autograd through the same fixed routing."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    n, M, H, E, k = 40, 12, 20, 4, 2
    w = O.Weights.generate(M, H, E, seed=1)
    x = rng.normal(size=(n, M))
    dout = rng.normal(size=(n, M))
    cap = 14  # forces some drops
    out, cache = O.block_forward(x, w, k, cap)
    g = O.block_backward(cache, w, dout)
    r = cache.routing
    assert r.dropped
    X = torch.tensor(x, requires_grad=True)
    G = torch.tensor(w.gate, requires_grad=True)
    W1 = torch.tensor(w.w1, requires_grad=True)
    W2 = torch.tensor(w.w2, requires_grad=True)
    p = torch.softmax(X @ G, dim=1)
    y = torch.zeros(n, M, dtype=torch.float64)
    for j in range(k):
        for t in range(n):
            s = int(r.slot_index[t, j])
            if s < 0:
                continue
            e = int(r.expert_index[t, j])
            h = torch.relu(X[t] @ W1[e])
            y[t] = y[t] + p[t, e] * (h @ W2[e])
    np.testing.assert_allclose(y.detach().numpy(), out, rtol=1e-12, atol=1e-12)
    (y * torch.tensor(dout)).sum().backward()
    np.testing.assert_allclose(g.dx, X.grad.numpy(), rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(g.dgate, G.grad.numpy(), rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(g.dw1, W1.grad.numpy(), rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(g.dw2, W2.grad.numpy(), rtol=1e-10, atol=1e-12)


def test_schedule_backward_consistent_across_schedules():
    """Without slice overflow all schedules compute one function, so their gradients agree."""
    M, H, E, k, f = 8, 16, 4, 2, 2.4
    lay = O.Layout(2, 2, 2, 4)
    w = O.Weights.generate(M, H, E, seed=3)
    rng = np.random.default_rng(4)
    inputs = rng.normal(size=(2, 32, M))
    douts = rng.normal(size=(2, 32, M))
    res = {}
    for s in ("baseline", "s1", "s2"):
        _, caches, drops = O.schedule_forward(s, 32, w, k, f, lay, inputs)
        assert not drops
        res[s] = O.schedule_backward(s, caches, w, lay, douts)
    for r in range(4):
        for key in ("dx", "dw1", "dw2", "dgate"):
            np.testing.assert_allclose(res["s1"][r][key], res["baseline"][r][key], rtol=1e-10, atol=1e-12)
            np.testing.assert_allclose(res["s2"][r][key], res["baseline"][r][key], rtol=1e-10, atol=1e-12)


def test_round_bf16_matches_torch():
    torch = pytest.importorskip("torch")
    a = np.random.default_rng(9).normal(size=1000) * 10
    ours = O.round_bf16(a)
    ref = torch.tensor(a, dtype=torch.float32).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(ours, ref)
