"""CPU oracle for the Parm MoE-layer hot path — TEST INFRASTRUCTURE ONLY.

A NumPy (float64) restatement of the reference simulator ``moesched``
(/root/reference/pkg/src/moesched) used as the checker for the B200 kernels.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import it; the product path never does.

Pinning: ``tests/golden/make_golden.py`` imports the real reference in the
build container and records its outputs (gate routing, reference_forward,
run_schedule outputs + traces + drops, fused collectives, selector reports)
into ``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this module
against every one of them plus the reference's own GOLDEN_OUTPUT vector
(test_dataplane.py:113-154).

The backward half (``block_backward``) has no reference: the reference is
forward-only.  It is the adjoint of ``block_forward`` derived by
hand and cross-checked against torch float64 autograd in
``tests/test_oracle_golden.py`` — gradient parity is "restated, unpinned by
the reference".
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np


# ---------------------------------------------------------------- config
def derive_capacity(tokens: int, num_experts: int, top_k: int, capacity_factor: float) -> int:
    """T = max(1, ceil(Fraction(str(f)) * k * tokens / E)) — config.py:54-63."""
    exact = Fraction(str(capacity_factor)) * top_k * tokens / num_experts
    return max(1, math.ceil(exact))


@dataclass(frozen=True)
class Layout:
    """Rank overlay of config.py:100-184 (ESP contiguous by default)."""

    mp: int
    ep: int
    esp: int
    world: int
    esp_contiguous: bool = True

    def ep_pos(self, r: int) -> int:
        return r // self.esp if self.esp_contiguous else r % self.ep

    def esp_pos(self, r: int) -> int:
        return r % self.esp if self.esp_contiguous else r // self.ep

    def mp_pos(self, r: int) -> int:
        return r % self.mp

    def rank_of(self, ep_pos: int, esp_pos: int) -> int:
        return ep_pos * self.esp + esp_pos if self.esp_contiguous else esp_pos * self.ep + ep_pos

    def group(self, kind: str, r: int) -> list[int]:
        if kind == "mp":
            b = (r // self.mp) * self.mp
            return list(range(b, b + self.mp))
        if kind == "ep_esp":
            return list(range(self.world))
        if kind == "esp":
            return sorted(self.rank_of(self.ep_pos(r), p) for p in range(self.esp))
        if kind == "ep":
            return sorted(self.rank_of(j, self.esp_pos(r)) for j in range(self.ep))
        raise ValueError(kind)

    def groups(self, kind: str) -> list[list[int]]:
        seen, out = set(), []
        for r in range(self.world):
            if r not in seen:
                g = self.group(kind, r)
                out.append(g)
                seen.update(g)
        return out


# ---------------------------------------------------------------- gate
def softmax(logits: np.ndarray) -> np.ndarray:
    """dataplane.py:80-83."""
    z = logits - logits.max(axis=-1, keepdims=True)
    ez = np.exp(z)
    return ez / ez.sum(axis=-1, keepdims=True)


@dataclass
class Routing:
    expert_index: np.ndarray      # (n, k) int64, selection order
    combine_weights: np.ndarray   # (n, k) f64 softmax score of each pick
    slot_index: np.ndarray        # (n, k) int64, -1 = dropped
    scores: np.ndarray            # (n, E) f64 full softmax
    dropped: set = field(default_factory=set)
    capacity: int = 0
    token_offset: int = 0


def gate(tokens: np.ndarray, gate_w: np.ndarray, k: int, capacity: int, token_offset: int = 0) -> Routing:
    """dataplane.py:86-119, vectorised.

    The reference walks (t asc, j asc) and gives each pick slot fill[e]++ while
    fill[e] < capacity.  Picks of one token hit distinct experts, so the slot of
    (t, e) equals the number of earlier tokens that picked e — an exclusive
    prefix count — and the pick is dropped iff that count >= capacity.
    ``gate_loop`` is the literal loop; tests assert both agree.
    """
    n, _ = tokens.shape
    E = gate_w.shape[1]
    if k > E:
        raise ValueError(f"top_k ({k}) exceeds number of experts ({E})")
    scores = softmax(tokens @ gate_w)
    ranked = np.argsort(-scores, axis=1, kind="stable")[:, :k]
    weights = np.take_along_axis(scores, ranked, axis=1)
    onehot = np.zeros((n, E), dtype=np.int64)
    np.put_along_axis(onehot, ranked, 1, axis=1)
    before = np.cumsum(onehot, axis=0) - onehot          # picks of e by earlier tokens
    slot = np.take_along_axis(before, ranked, axis=1)
    slot = np.where(slot < capacity, slot, -1).astype(np.int64)
    dropped = {(token_offset + int(t), int(ranked[t, j])) for t, j in zip(*np.nonzero(slot < 0))}
    return Routing(ranked.astype(np.int64), weights, slot, scores, dropped, capacity, token_offset)


def gate_loop(tokens: np.ndarray, gate_w: np.ndarray, k: int, capacity: int, token_offset: int = 0) -> Routing:
    """Literal per-pick loop of dataplane.py:104-116 (small inputs only)."""
    scores = softmax(tokens @ gate_w)
    ranked = np.argsort(-scores, axis=1, kind="stable")[:, :k]
    n, E = scores.shape
    slot = np.full((n, k), -1, dtype=np.int64)
    fill = [0] * E
    dropped = set()
    for t in range(n):
        for j in range(k):
            e = int(ranked[t, j])
            if fill[e] < capacity:
                slot[t, j] = fill[e]
                fill[e] += 1
            else:
                dropped.add((token_offset + t, e))
    return Routing(ranked.astype(np.int64), np.take_along_axis(scores, ranked, axis=1), slot, scores, dropped,
                   capacity, token_offset)


def dispatch_tensor(tokens: np.ndarray, r: Routing, E: int) -> np.ndarray:
    """(E, capacity, M) zero-padded slot tensor (dataplane.py:101,112)."""
    out = np.zeros((E, r.capacity, tokens.shape[1]))
    keep = r.slot_index >= 0
    t_idx, j_idx = np.nonzero(keep)
    out[r.expert_index[t_idx, j_idx], r.slot_index[t_idx, j_idx]] = tokens[t_idx]
    return out


# ---------------------------------------------------------------- weights
@dataclass
class Weights:
    gate: np.ndarray   # (M, E)
    w1: np.ndarray     # (E, M, H)
    w2: np.ndarray     # (E, H, M)

    @classmethod
    def generate(cls, M: int, H: int, E: int, seed: int = 0) -> "Weights":
        """ExpertWeights.generate (dataplane.py:58-69): one default_rng(seed),
        gate N(0,1), then w1 N(0, 1/sqrt(M)), then w2 N(0, 1/sqrt(H))."""
        rng = np.random.default_rng(seed)
        g = rng.normal(size=(M, E))
        w1 = rng.normal(scale=1.0 / math.sqrt(M), size=(E, M, H))
        w2 = rng.normal(scale=1.0 / math.sqrt(H), size=(E, H, M))
        return cls(g, w1, w2)

    def shard(self, e: int, p: int, esp: int) -> tuple[np.ndarray, np.ndarray]:
        """w1_shard / w2_shard (dataplane.py:71-77)."""
        h = self.w1.shape[2] // esp
        return self.w1[e][:, p * h:(p + 1) * h], self.w2[e][p * h:(p + 1) * h, :]


def round_bf16(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float64 (the GPU's inputs)."""
    f = np.asarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


# ---------------------------------------------------------------- forward / backward of one token block
@dataclass
class BlockCache:
    tokens: np.ndarray
    routing: Routing
    dispatch: np.ndarray     # (E, cap, M)
    hidden: np.ndarray       # (E, cap, H) post-ReLU
    expert_out: np.ndarray   # (E, cap, M)


def block_forward(tokens: np.ndarray, w: Weights, k: int, capacity: int, token_offset: int = 0):
    """gate -> unsharded expert FFNs -> weighted combine (dataplane.py:146-159)."""
    E = w.gate.shape[1]
    r = gate(tokens, w.gate, k, capacity, token_offset)
    d = dispatch_tensor(tokens, r, E)
    h = np.maximum(np.matmul(d, w.w1), 0.0)          # batched BLAS per expert
    y = np.matmul(h, w.w2)
    out = combine(r, y, tokens.shape[1])
    return out, BlockCache(tokens, r, d, h, y)


def combine(r: Routing, expert_out: np.ndarray, M: int) -> np.ndarray:
    """out[t] = sum_j w[t,j] * Y[e_j, s_j], j ascending, dropped -> 0 (dataplane.py:131-143)."""
    n, k = r.slot_index.shape
    out = np.zeros((n, M))
    for j in range(k):
        keep = r.slot_index[:, j] >= 0
        t = np.nonzero(keep)[0]
        out[t] += r.combine_weights[t, j, None] * expert_out[r.expert_index[t, j], r.slot_index[t, j]]
    return out


@dataclass
class BlockGrads:
    dx: np.ndarray     # (n, M)
    dw1: np.ndarray    # (E, M, H)
    dw2: np.ndarray    # (E, H, M)
    dgate: np.ndarray  # (M, E)


def block_backward(c: BlockCache, w: Weights, dout: np.ndarray) -> BlockGrads:
    """Adjoint of block_forward for a fixed (discrete) routing.

    dY[e,s] = w[t,j] dout[t];  dw[t,j] = <dout[t], Y[e_j,s_j]>
    dH = (dY W2^T) * [H > 0];  dW2 = H^T dY;  dW1 = R^T dH;  dR = dH W1^T
    dx[t] = sum_j dR[e_j, s_j] + (s * (dS - <s, dS>)) Wg^T;  dWg = x^T dlogits
    Gradients flow only through the kept picks' softmax scores (no aux loss,
    SPEC.md:322); routing decisions are piecewise constant.
    """
    r = c.routing
    n, k = r.slot_index.shape
    E, cap, M = c.dispatch.shape
    dY = np.zeros_like(c.expert_out)
    dS = np.zeros_like(r.scores)
    for j in range(k):
        t = np.nonzero(r.slot_index[:, j] >= 0)[0]
        e, s = r.expert_index[t, j], r.slot_index[t, j]
        dY[e, s] += r.combine_weights[t, j, None] * dout[t]
        dS[t, e] += np.einsum("tm,tm->t", dout[t], c.expert_out[e, s])
    dH = np.matmul(dY, w.w2.transpose(0, 2, 1)) * (c.hidden > 0)
    dw2 = np.matmul(c.hidden.transpose(0, 2, 1), dY)
    dw1 = np.matmul(c.dispatch.transpose(0, 2, 1), dH)
    dR = np.matmul(dH, w.w1.transpose(0, 2, 1))
    dx = np.zeros((n, M))
    for j in range(k):
        t = np.nonzero(r.slot_index[:, j] >= 0)[0]
        dx[t] += dR[r.expert_index[t, j], r.slot_index[t, j]]
    p = r.scores
    dlogits = p * (dS - (p * dS).sum(axis=1, keepdims=True))
    dx += dlogits @ w.gate.T
    dgate = c.tokens.T @ dlogits
    return BlockGrads(dx, dw1, dw2, dgate)


# ---------------------------------------------------------------- per-schedule semantics
def schedule_forward(schedule: str, tokens_per_rank: int, w: Weights, k: int, capacity_factor: float,
                     layout: Layout, inputs: np.ndarray):
    """Per-rank outputs of run_schedule (dataplane.py:183-413), computed directly.

    baseline / s2: every rank gates its full block with capacity T, so rank r's
    output is reference_forward(inputs[r // MP]) (baseline keeps its own slot
    range of identically-routed copies, dataplane.py:286-290; s2 pads and
    splits slots, dataplane.py:361-410).  s1: MP rank m gates token slice m
    with quota ceil(T / MP) and token_offset m * n / MP (dataplane.py:305-320);
    the MP AllGather concatenates the slices.
    Returns (outputs (P, n, M), per-rank list of (cache, offset) blocks, drops).
    """
    E = w.gate.shape[1]
    n = tokens_per_rank
    T = derive_capacity(n, E, k, capacity_factor)
    P = layout.world
    outs = np.zeros((P, n, w.gate.shape[0]))
    caches: list[list[tuple[BlockCache, int]]] = []
    drops = set()
    for rank in range(P):
        g = rank // layout.mp
        block = inputs[g]
        if schedule in ("baseline", "s2"):
            o, cch = block_forward(block, w, k, T)
            outs[rank] = o
            caches.append([(cch, 0)])
            drops.update((g, t, e) for t, e in cch.routing.dropped)
        elif schedule == "s1":
            quota = math.ceil(T / layout.mp)
            sl = n // layout.mp
            parts = []
            for m in range(layout.mp):
                o, cch = block_forward(block[m * sl:(m + 1) * sl], w, k, quota, token_offset=m * sl)
                outs[rank, m * sl:(m + 1) * sl] = o
                parts.append((cch, m * sl))
                drops.update((g, t, e) for t, e in cch.routing.dropped)
            caches.append(parts)
        else:
            raise ValueError(f"unknown schedule {schedule!r}")
    return outs, caches, drops


def schedule_backward(schedule: str, caches, w: Weights, layout: Layout, douts: np.ndarray):
    """Per-rank gradients under the replicated-MP convention.

    douts (P/MP, n, M): one upstream gradient per MP group, replicated on its ranks.
    Loss L = sum_g <out_g, dout_g> counts each group's output once.
      dx[r]     = dL/dX_g                   (g = r // MP, full block, every MP rank)
      dw1/dw2[r]= dL/d(rank r's expert shard), summed over all groups
      dgate[r]  = dL_g/dWg                  (own group; DP reduction excluded)
    """
    P = layout.world
    E = w.gate.shape[1]
    n_groups = P // layout.mp
    per_group = []
    for g in range(n_groups):
        parts = caches[g * layout.mp]
        dx = np.zeros_like(douts[g])
        acc = None
        for cch, off in parts:
            m = cch.tokens.shape[0]
            gr = block_backward(cch, w, douts[g][off:off + m])
            dx[off:off + m] = gr.dx
            if acc is None:
                acc = BlockGrads(None, gr.dw1, gr.dw2, gr.dgate)
            else:
                acc = BlockGrads(None, acc.dw1 + gr.dw1, acc.dw2 + gr.dw2, acc.dgate + gr.dgate)
        per_group.append((dx, acc))
    dw1_tot = sum(pg[1].dw1 for pg in per_group)
    dw2_tot = sum(pg[1].dw2 for pg in per_group)
    e_local = E // layout.ep
    H = w.w1.shape[2]
    hs = H // layout.esp
    res = []
    for rank in range(P):
        g = rank // layout.mp
        ep, p = layout.ep_pos(rank), layout.esp_pos(rank)
        experts = range(ep * e_local, (ep + 1) * e_local)
        dw1 = np.stack([dw1_tot[e][:, p * hs:(p + 1) * hs] for e in experts])
        dw2 = np.stack([dw2_tot[e][p * hs:(p + 1) * hs, :] for e in experts])
        res.append({"dx": per_group[g][0], "dw1": dw1, "dw2": dw2, "dgate": per_group[g][1].dgate})
    return res


def max_rel_error(out: np.ndarray, ref: np.ndarray) -> float:
    """dataplane.py:416-419: max|out-ref| / max(1, max|ref|)."""
    return float(np.abs(out - ref).max()) / max(1.0, float(np.abs(ref).max()))


# ---------------------------------------------------------------- collectives (checkers for the comm layer)
def allgather(bufs: list[np.ndarray], layout: Layout, kind: str) -> list[np.ndarray]:
    """collectives.py:142-157: concatenate in group rank order."""
    out = [None] * layout.world
    for grp in layout.groups(kind):
        cat = np.concatenate([bufs[r] for r in grp])
        for r in grp:
            out[r] = cat.copy()
    return out


def reduce_scatter(bufs, layout: Layout, kind: str):
    """collectives.py:160-183: member i keeps the sequential sum of chunk i."""
    out = [None] * layout.world
    for grp in layout.groups(kind):
        c = bufs[grp[0]].size // len(grp)
        for i, r in enumerate(grp):
            acc = bufs[grp[0]][i * c:(i + 1) * c].copy()
            for o in grp[1:]:
                acc = acc + bufs[o][i * c:(i + 1) * c]
            out[r] = acc
    return out


def allreduce(bufs, layout: Layout, kind: str):
    """collectives.py:186-199 (RS then AG)."""
    return allgather(reduce_scatter(bufs, layout, kind), layout, kind)


def alltoall(bufs, layout: Layout, kind: str):
    """collectives.py:202-219: chunk j of member i -> slot i of member j."""
    out = [None] * layout.world
    for grp in layout.groups(kind):
        c = bufs[grp[0]].size // len(grp)
        for i, r in enumerate(grp):
            out[r] = np.concatenate([bufs[s][i * c:(i + 1) * c] for s in grp])
    return out


def fused_dispatch(bufs, layout: Layout):
    """collectives.py:256-283: dump x N_ESP, arrange by (esp_pos(d), ep_pos(d)), A2A over the world."""
    n = bufs[0].size
    sub = n // layout.ep
    arranged = []
    for b in bufs:
        parts = b.reshape(layout.ep, sub)
        arranged.append(np.concatenate([parts[layout.ep_pos(d)] for d in range(layout.world)]))
    return alltoall(arranged, layout, "ep_esp")


def fused_combine(bufs, layout: Layout):
    """collectives.py:286-312: A2A over the world, then per EP position the
    sequential sum of the pieces from sources with that ep_pos (rank order)."""
    ret = alltoall(bufs, layout, "ep_esp")
    sub = ret[0].size // layout.world
    out = []
    for b in ret:
        pieces = b.reshape(layout.world, sub)
        blocks = []
        for j in range(layout.ep):
            srcs = [s for s in range(layout.world) if layout.ep_pos(s) == j]
            acc = pieces[srcs[0]].copy()
            for s in srcs[1:]:
                acc = acc + pieces[s]
            blocks.append(acc)
        out.append(np.concatenate(blocks))
    return out


def saa(bufs, layout: Layout):
    """collectives.py:315-353: data equals allgather(mp) of alltoall(ep_esp)."""
    return allgather(alltoall(bufs, layout, "ep_esp"), layout, "mp")
