"""Drop-in data-plane API: the reference's ``moesched.dataplane`` surface on B200.

Same names, signatures, argument meaning and ValueError texts as
/root/reference/pkg/src/moesched/dataplane.py, with the work done by the
sm_100a kernels.  NumPy arrays in, NumPy float64 arrays out (the reference's
types); device tensors are accepted too.  Arithmetic is bf16 with f32/f64
accumulation: routing is bit-exact to the reference on
bf16-representable inputs, activations agree within the stated tolerance.

``run_schedule`` executes every rank: under torchrun with a world of exactly
``layout.world_size`` processes it drives this process's rank over NCCL and
gathers all ranks' outputs; otherwise it emulates all ranks on the current
GPU (``LocalWorld``), like the reference simulates them in one process.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import kernels as K
from .config import ClusterSpec, MoEConfig, ParallelLayout, check_compatible, derive_capacity
from .runtime import SCHEDULES, MoELayer
from .trace import CommTrace, schedule_ffn_rows
from .world import LocalWorld, make_world


# ---------------------------------------------------------------- weights
@dataclass(frozen=True)
class ExpertWeights:
    """Replicated gate weights plus per-expert two-layer FFN weights (dataplane.py:50-77)."""

    gate: np.ndarray  # (embed, num_experts)
    w1: np.ndarray    # (num_experts, embed, hidden)
    w2: np.ndarray    # (num_experts, hidden, embed)

    @classmethod
    def generate(cls, cfg: MoEConfig, seed: int = 0) -> "ExpertWeights":
        rng = np.random.default_rng(seed)
        g = rng.normal(size=(cfg.embed_dim, cfg.num_experts))
        w1 = rng.normal(scale=1.0 / math.sqrt(cfg.embed_dim),
                        size=(cfg.num_experts, cfg.embed_dim, cfg.hidden_dim))
        w2 = rng.normal(scale=1.0 / math.sqrt(cfg.hidden_dim),
                        size=(cfg.num_experts, cfg.hidden_dim, cfg.embed_dim))
        return cls(gate=g, w1=w1, w2=w2)

    def w1_shard(self, expert: int, shard: int, esp_size: int) -> np.ndarray:
        w = self.w1.shape[2] // esp_size
        return self.w1[expert][:, shard * w:(shard + 1) * w]

    def w2_shard(self, expert: int, shard: int, esp_size: int) -> np.ndarray:
        w = self.w2.shape[1] // esp_size
        return self.w2[expert][shard * w:(shard + 1) * w, :]


@dataclass
class GateOutput:
    """Routing decision for one token block (dataplane.py:38-47)."""

    dispatch: np.ndarray
    expert_index: np.ndarray
    combine_weights: np.ndarray
    slot_index: np.ndarray
    dropped: set
    token_offset: int = 0


@dataclass
class ScheduleResult:
    outputs: np.ndarray          # (world_size, tokens_per_rank, embed)
    trace: CommTrace
    dropped: set                 # (mp-group id, global token, expert)
    ffn_rows: int


def _dev() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2407_00599_b200 runs on a B200 GPU; no CUDA device is visible "
                           "(there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _bf16_dev(a, shape_cols_pad: int | None = None) -> torch.Tensor:
    """Host (NumPy / torch) or device array -> contiguous bf16 on the GPU; the dtype
    conversion runs on the device after one H2D of the caller's bytes."""
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
    t = t.to(device=_dev()).to(torch.bfloat16)
    if shape_cols_pad is not None and t.shape[-1] != shape_cols_pad:
        pad = torch.zeros(*t.shape[:-1], shape_cols_pad, dtype=torch.bfloat16, device=t.device)
        pad[..., :t.shape[-1]] = t
        t = pad
    return t.contiguous()


def _ceil(x: int, m: int) -> int:
    return (x + m - 1) // m * m


# ---------------------------------------------------------------- gate / expert shard
def gate(tokens, gate_weights, k: int, capacity: int, token_offset: int = 0) -> GateOutput:
    """Softmax routing with stable top-k and token-major per-expert slot quota (dataplane.py:86-119)."""
    n, embed = tuple(tokens.shape)
    n_experts = gate_weights.shape[1]
    if k > n_experts:
        raise ValueError(f"top_k ({k}) exceeds number of experts ({n_experts})")
    Mp = _ceil(embed, 8)
    x = _bf16_dev(tokens, Mp)
    wg = torch.zeros(n_experts, Mp, dtype=torch.bfloat16, device=x.device)   # transposed (E, M)
    wg[:, :embed] = _bf16_dev(np.ascontiguousarray(np.asarray(gate_weights).T))
    dev = x.device
    ei = torch.empty(n, k, dtype=torch.int32, device=dev)
    cw = torch.empty(n, k, dtype=torch.float32, device=dev)
    pr = torch.empty(n, n_experts, dtype=torch.float32, device=dev)
    si = torch.empty(n, k, dtype=torch.int32, device=dev)
    ss = torch.empty(n_experts, capacity, dtype=torch.int32, device=dev)
    fill = torch.empty(n_experts, dtype=torch.int32, device=dev)
    counts = torch.empty(max(1, (n + 7) // 8 * n_experts), dtype=torch.int32, device=dev)
    disp = torch.zeros(n_experts, capacity, Mp, dtype=torch.bfloat16, device=dev)
    if n:
        K.gate_fwd(x, wg, k, ei, cw, pr, counts)
        K.route_dispatch(x, ei, counts, capacity, si, ss, fill, 0, out=disp)
    else:
        ss.fill_(-1)
        fill.zero_()
    ei_h = ei.cpu().numpy().astype(np.int64)
    si_h = si.cpu().numpy().astype(np.int64)
    dropped = {(token_offset + int(t), int(ei_h[t, j])) for t, j in zip(*np.nonzero(si_h < 0))}
    return GateOutput(dispatch=disp[:, :, :embed].float().cpu().numpy().astype(np.float64),
                      expert_index=ei_h, combine_weights=cw.cpu().numpy().astype(np.float64),
                      slot_index=si_h, dropped=dropped, token_offset=token_offset)


def expert_shard_forward(rows, w1_shard, w2_shard) -> np.ndarray:
    """relu(rows @ w1_shard) @ w2_shard on the tcgen05 grouped GEMM (dataplane.py:122-128)."""
    if rows.shape[1] != w1_shard.shape[0]:
        raise ValueError(f"row width {rows.shape[1]} does not match weight rows {w1_shard.shape[0]}")
    n, M = rows.shape
    Hs = w1_shard.shape[1]
    Mp, Hp, Rp = _ceil(M, 128), _ceil(Hs, 128), _ceil(max(n, 1), 128)
    dev = _dev()
    x = torch.zeros(1, Rp, Mp, dtype=torch.bfloat16, device=dev)
    x[0, :n, :M] = _bf16_dev(rows)
    w1t = torch.zeros(1, Hp, Mp, dtype=torch.bfloat16, device=dev)
    w1t[0, :Hs, :M] = _bf16_dev(np.ascontiguousarray(np.asarray(w1_shard).T))
    w2t = torch.zeros(1, Mp, Hp, dtype=torch.bfloat16, device=dev)
    w2t[0, :M, :Hs] = _bf16_dev(np.ascontiguousarray(np.asarray(w2_shard).T))
    h = torch.empty(1, Rp, Hp, dtype=torch.bfloat16, device=dev)
    y = torch.empty(1, Rp, Mp, dtype=torch.bfloat16, device=dev)
    K.grouped_gemm(x, K.KMAJOR, w1t, K.KMAJOR, h, K.EPI_RELU)
    K.grouped_gemm(h, K.KMAJOR, w2t, K.KMAJOR, y, K.EPI_BF16)
    return y[0, :n, :M].float().cpu().numpy().astype(np.float64)


# ---------------------------------------------------------------- layers
_LAYER_CACHE: dict = {}


def _dist_key() -> tuple:
    """Which world make_world would build right now (process group size and rank, or local)."""
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            return ("dist", dist.get_world_size(), dist.get_rank())
    except ImportError:  # pragma: no cover
        pass
    return ("local",)


def _layer(cfg: MoEConfig, layout: ParallelLayout, weights) -> MoELayer:
    # The world (and, under torchrun, its NCCL sub-communicators) is built only on a cache miss
    # and lives with the cached layer: a hit creates no process groups.
    key = (cfg, layout, _dist_key())
    lay = _LAYER_CACHE.get(key)
    if lay is None:
        if len(_LAYER_CACHE) > 8:
            _LAYER_CACHE.clear()
        lay = MoELayer(cfg, layout, make_world(layout))
        _LAYER_CACHE[key] = lay
    if getattr(lay, "_weights_id", None) is not weights:
        lay.load_weights(weights)
        lay._weights_id = weights
    return lay


def reference_forward(cfg: MoEConfig, weights, tokens) -> np.ndarray:
    """Single-device forward: gate, unsharded expert FFNs, weighted combine (dataplane.py:146-159)."""
    if tuple(tokens.shape) != (cfg.tokens_per_rank, cfg.embed_dim):
        raise ValueError(f"expected input of shape {(cfg.tokens_per_rank, cfg.embed_dim)}, "
                         f"got {tuple(tokens.shape)}")
    lay = _layer(cfg, ParallelLayout(1, 1, 1, 1), weights)
    out = lay.forward("s1", {0: _bf16_dev(tokens)})
    return out[0].float().cpu().numpy().astype(np.float64)


def run_schedule(schedule: str, cfg: MoEConfig, layout: ParallelLayout, cluster: ClusterSpec, weights,
                 inputs) -> ScheduleResult:
    """Execute one schedule over all ranks (dataplane.py:183-207)."""
    if schedule not in SCHEDULES:
        raise ValueError(f"unknown schedule {schedule!r}")
    if cluster.world_size != layout.world_size:
        raise ValueError("cluster/layout world size mismatch")
    check_compatible(cfg, layout)
    expected = (layout.world_size // layout.mp_size, cfg.tokens_per_rank, cfg.embed_dim)
    if tuple(inputs.shape) != expected:
        raise ValueError(f"expected inputs of shape {expected}, got {tuple(inputs.shape)}")
    lay = _layer(cfg, layout, weights)
    xs = {r: _bf16_dev(inputs[r // layout.mp_size]) for r in lay.ranks}
    outs = lay.forward(schedule, xs)
    dropped = set()
    per_rank = {}
    for r in lay.ranks:
        per_rank[r] = outs[r].contiguous()      # bf16: gathered as is, widened exactly on the way out
        rt = lay.routing(r)
        si = rt.slot_idx.cpu().numpy()
        ei = rt.expert_idx.cpu().numpy()
        g = r // layout.mp_size
        dropped.update((g, rt.token_offset + int(t), int(ei[t, j])) for t, j in zip(*np.nonzero(si < 0)))
    outputs = np.empty((layout.world_size, cfg.tokens_per_rank, cfg.embed_dim))
    if isinstance(lay.world, LocalWorld):
        for r, o in per_rank.items():
            torch.from_numpy(outputs[r]).copy_(o.double())
    else:
        import torch.distributed as dist

        mine = per_rank[lay.ranks[0]].contiguous()
        gathered = [torch.empty_like(mine) for _ in range(layout.world_size)]
        dist.all_gather(gathered, mine)
        for r, o in enumerate(gathered):
            torch.from_numpy(outputs[r]).copy_(o.double())
        allsets = [None] * layout.world_size
        dist.all_gather_object(allsets, sorted(dropped))
        dropped = {tuple(x) for s in allsets for x in s}
    # S1 keeps one (slice-local) drop set per MP rank; all ranks of a group agree
    # on baseline/s2, so the union equals the reference's per-group record.
    # the trace is the one the executed exchanges emitted (MoELayer.last_trace)
    return ScheduleResult(outputs, lay.last_trace, dropped, schedule_ffn_rows(schedule, cfg, layout))


def max_rel_error(outputs, reference) -> float:
    """max |out - ref| scaled by the reference magnitude (floor 1) (dataplane.py:416-419)."""
    scale = max(1.0, float(np.abs(reference).max()))
    return float(np.abs(np.asarray(outputs) - np.asarray(reference)).max()) / scale


def oracle_errors(cfg: MoEConfig, layout: ParallelLayout, weights, inputs, result: ScheduleResult) -> float:
    """Worst max_rel_error of any rank vs reference_forward of its block (dataplane.py:422-431)."""
    refs = [reference_forward(cfg, weights, inputs[g]) for g in range(inputs.shape[0])]
    return max(max_rel_error(result.outputs[r], refs[r // layout.mp_size]) for r in range(layout.world_size))


__all__ = ["ExpertWeights", "GateOutput", "ScheduleResult", "SCHEDULES", "gate", "expert_shard_forward",
           "reference_forward", "run_schedule", "max_rel_error", "oracle_errors", "derive_capacity"]
