"""The MoE layer on B200: per-rank device state and the three schedule executors.

``MoELayer`` owns, for every rank this process executes, the bf16 expert
shards (W1/W2 stored transposed so every forward GEMM operand is K-major),
the gate weights (stored transposed, (E, M)), f32 gradient buffers and one
preallocated buffer set per schedule.  ``forward(schedule, xs)`` /
``backward(douts)`` run the reference's schedules (moesched
dataplane.py:220-413) as sm_100a kernels (libparm_b200.so) plus collectives
from ``world.py``:

  baseline  gate | AG_esp(x) -> N_ESP gates -> dispatch -> A2A_ep -> FFN ->
            AR_esp -> A2A_ep -> own slot range -> combine           (DeepSpeed-MoE order)
  s1        MP split -> gate(slice, quota ceil(T/MP)) -> dispatch -> fused
            A2A(ep&esp) -> FFN -> A2A(ep&esp) + ESP sum fused into combine -> AG_mp
  s2        gate(block) -> dispatch of own slot shard (pad to ceil(T/MP)*MP) ->
            fused A2A -> FFN -> A2A -> ESP sum -> AG_mp(slots) -> combine

Data layout.  Every expert-row tensor (received tokens,
hidden, outputs and their gradients) is the AlltoAll receive layout
``[src_hi][src_lo][expert][row][col]`` — s1/s2: (P, 1, e_local, q, C) with
src = the token owner; baseline: (N_EP, N_ESP, e_local, T, C) with (owner,
gathered block) — so every exchange is ONE message per peer (NCCL P2P
throughput collapses with message count) and the grouped GEMM reads/writes
it directly through 5-D TMA maps.  Each source also ships its per-expert fill
counts, so the GEMM skips tiles of unfilled capacity slots.

Backward (no reference) is the adjoint of each sequence
under the replicated-MP convention the paper uses (split <-> AllGather,
AllReduce <-> identity, A2A <-> A2A, dump <-> local sum): every schedule
returns the gradient of L = sum_g <out_g, dout_g> with each MP group's output
counted once.  The baseline processes each token N_MP times (its duplicated
computation), so its expert weight gradients are scaled by 1/N_MP in the
wgrad GEMM epilogue to report the same quantity.

Padding: embed M and shard width H/ESP are padded to multiples of 128 with
zeros, so every shape meets the GEMM contract without changing results.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import kernels as K
from .config import MoEConfig, ParallelLayout, check_compatible, derive_capacity, group_members
from .trace import CommTrace, rec_allgather, rec_allreduce, rec_alltoall, rec_dump, rec_split
from .world import Msg, World, make_world

SCHEDULES = ("baseline", "s1", "s2")


def _ceil_to(x: int, m: int) -> int:
    return ((x + m - 1) // m) * m


@dataclass(frozen=True)
class Dims:
    n: int          # tokens per rank (B*L)
    M: int
    Mp: int         # padded embed
    H: int
    Hs: int         # shard width H / N_ESP
    Hsp: int        # padded shard width
    E: int
    k: int
    T: int          # capacity
    e_local: int
    P: int
    MP: int
    EP: int
    ESP: int

    @classmethod
    def of(cls, cfg: MoEConfig, layout: ParallelLayout) -> "Dims":
        Hs = cfg.hidden_dim // layout.esp_size
        return cls(cfg.tokens_per_rank, cfg.embed_dim, _ceil_to(cfg.embed_dim, 128), cfg.hidden_dim, Hs,
                   _ceil_to(Hs, 128), cfg.num_experts, cfg.top_k, derive_capacity(cfg),
                   cfg.num_experts // layout.ep_size, layout.world_size, layout.mp_size, layout.ep_size,
                   layout.esp_size)


@dataclass
class Routing:
    """Device-resident gate outputs of one token block."""

    expert_idx: torch.Tensor   # (n, k) int32
    combine_w: torch.Tensor    # (n, k) f32
    probs: torch.Tensor        # (n, E) f32
    slot_idx: torch.Tensor     # (n, k) int32, -1 dropped
    slot_src: torch.Tensor     # (E, cap) int32
    fill: torch.Tensor         # (E,) int32
    cap: int
    token_offset: int = 0
    counts: torch.Tensor | None = None   # per-8-token-tile pick counts (gate -> slot pass)

    @classmethod
    def alloc(cls, n: int, k: int, E: int, cap: int, dev, token_offset: int = 0,
              fill: torch.Tensor | None = None) -> "Routing":
        i32 = dict(dtype=torch.int32, device=dev)
        f32 = dict(dtype=torch.float32, device=dev)
        return cls(torch.empty(n, k, **i32), torch.empty(n, k, **f32), torch.empty(n, E, **f32),
                   torch.empty(n, k, **i32), torch.empty(E, max(cap, 1), **i32),
                   fill if fill is not None else torch.zeros(E, **i32), cap, token_offset,
                   torch.empty(max(1, (n + 7) // 8 * E), **i32))

    def run(self, x: torch.Tensor, wg_t: torch.Tensor, k: int, out: torch.Tensor | None = None, slot_lo: int = 0,
            dst: K.SlotView | None = None, slots_out: int | None = None, fill_fan: list | None = None) -> None:
        """Gate (f64 tensor-core logits, softmax, stable top-k, tile counts), then the slot pass
        fused with the dispatch of the token rows into ``out`` / the holders (``dst``), or the
        slot pass alone when neither is given."""
        K.gate_fwd(x, wg_t, k, self.expert_idx, self.combine_w, self.probs, self.counts)
        K.route_dispatch(x, self.expert_idx, self.counts, self.cap, self.slot_idx, self.slot_src, self.fill, slot_lo,
                         out=out, dst=dst, slots_out=slots_out, fill_fan=fill_fan)


@dataclass
class RankState:
    rank: int
    gate: torch.Tensor            # (E, Mp) bf16, transposed (one 16-B load per lane per expert)
    w1t: torch.Tensor             # (e_local, Hsp, Mp) bf16
    w2t: torch.Tensor             # (e_local, Mp, Hsp) bf16
    dgate: torch.Tensor           # (E, Mp) f32
    dw1t: torch.Tensor            # (e_local, Hsp, Mp) f32
    dw2t: torch.Tensor            # (e_local, Mp, Hsp) f32
    bufs: dict = field(default_factory=dict)


@dataclass
class StepGraph:
    """A captured forward+backward step; ``outs``/``dxs`` alias the layer's buffers."""

    graph: torch.cuda.CUDAGraph
    outs: dict
    dxs: dict
    schedule: str

    def replay(self) -> None:
        self.graph.replay()


S1_RETURNS = ("epilogue", "push", "pull")
S2_RETURNS = ("pull", "push")
SAA_MODES = ("seq", "phased")


class MoELayer:
    """One MoE layer under MP+EP+ESP on the ranks this process owns.

    Execution options (all paths are parity-tested against the oracle; the defaults are
    the measured-fastest on B200, DESIGN.md §(e)):

    ``s1_return``  peer-memory S1 only: how expert outputs (and dR) go back to the owners.
                   ``epilogue`` -- the second GEMM's TMA epilogue stores each tile straight
                   into the owner's receive block over NVLink (default); ``push`` -- a copy
                   kernel pushes the filled rows after the GEMM; ``pull`` -- the owners'
                   combine gathers from the holders through a peer slot view.
    ``s2_return``  peer-memory S2: ``pull`` (owners gather through the slot-shard view,
                   default; measured 0.84 vs 0.85 ms for ``push`` at N=4) or ``push``
                   (holders store MP copies of every row: the AllGather as pushes).
    ``saa``        NCCL/local S2 return: ``seq`` (A2A then AllGather, default; the phased
                   overlap measured 8% slower on NVSwitch, which shares the ports) or
                   ``phased`` (the paper's SAA, per-expert-block rotation).
    ``peer``       None (default): S1/S2 use the fused peer-memory path whenever the world
                   maps peers (PeerWorld / PeerLocalWorld); False: the separate collectives
                   even there (like-for-like schedule comparisons on one transport).  The
                   baseline (DeepSpeed-MoE ordering) always runs on the collectives."""

    def __init__(self, cfg: MoEConfig, layout: ParallelLayout, world: World | None = None, device=None, *,
                 s1_return: str = "epilogue", s2_return: str = "pull", saa: str = "seq", peer: bool | None = None,
                 fused_ffn: bool = True):
        check_compatible(cfg, layout)
        if cfg.top_k > 8 or cfg.num_experts > 32:
            raise ValueError("B200 kernels support top_k <= 8 and num_experts <= 32")
        for name, v, ok in (("s1_return", s1_return, S1_RETURNS), ("s2_return", s2_return, S2_RETURNS),
                            ("saa", saa, SAA_MODES)):
            if v not in ok:
                raise ValueError(f"{name} must be one of {ok}, got {v!r}")
        self.cfg = cfg
        self.layout = layout
        self.world = world if world is not None else make_world(layout, device)
        self.dev = self.world.device
        self.d = Dims.of(cfg, layout)
        d = self.d
        self.saa_phased = saa == "phased" and layout.mp_size > 1 and layout.ep_size > 1
        # S1/S2 over (NVLink) peer memory: dispatch/return/AllGather fused into the kernels
        if peer and not self.world.maps_peers:
            raise ValueError(f"peer=True needs a world that maps peer memory, got {type(self.world).__name__}")
        self.peer = self.world.maps_peers and d.P > 1 and peer is not False
        self.peer_push = s1_return in ("epilogue", "push")
        self.peer_epilogue = s1_return == "epilogue"
        self.peer_push_s2 = s2_return == "push"
        # expert FFN GEMMs as one persistent launch per pass (forward 2, backward 4; parm_gemm_multi)
        self.fused_ffn = fused_ffn and d.Mp % 256 == 0 and d.Hsp % 256 == 0
        self.options = {"s1_return": s1_return, "s2_return": s2_return, "saa": saa, "peer": self.peer,
                        "fused_ffn": self.fused_ffn}
        bf, f32 = dict(dtype=torch.bfloat16, device=self.dev), dict(dtype=torch.float32, device=self.dev)
        self.ranks = list(self.world.ranks)
        self.st: dict[int, RankState] = {}
        for r in self.ranks:
            self.st[r] = RankState(r, torch.zeros(d.E, d.Mp, **bf), torch.zeros(d.e_local, d.Hsp, d.Mp, **bf),
                                   torch.zeros(d.e_local, d.Mp, d.Hsp, **bf), torch.zeros(d.E, d.Mp, **f32),
                                   torch.zeros(d.e_local, d.Hsp, d.Mp, **f32),
                                   torch.zeros(d.e_local, d.Mp, d.Hsp, **f32))
        self._last: str | None = None
        self._ws_gate = None
        self._ws_gemm: dict[int, torch.Tensor] = {}   # per rank: tile queue + completion counters (kept zeroed)
        self._trace: CommTrace | None = None
        self.last_trace: CommTrace | None = None      # records of the last forward's exchanges

    # ------------------------------------------------------------ weights
    def local_experts(self, rank: int) -> range:
        j = self.layout.ep_pos(rank)
        return range(j * self.d.e_local, (j + 1) * self.d.e_local)

    def load_weights(self, weights) -> None:
        """Upload full f64 weights (gate (M,E), w1 (E,M,H), w2 (E,H,M)) as this rank's bf16 shards."""
        d = self.d
        for r, s in self.st.items():
            p = self.layout.esp_pos(r)
            g = torch.from_numpy(np.ascontiguousarray(weights.gate)).to(torch.float32)
            s.gate.zero_()
            s.gate[:, :d.M].copy_(g.t().to(self.dev).to(torch.bfloat16))
            s.w1t.zero_()
            s.w2t.zero_()
            for i, e in enumerate(self.local_experts(r)):
                w1 = np.ascontiguousarray(weights.w1[e][:, p * d.Hs:(p + 1) * d.Hs].T)   # (Hs, M)
                w2 = np.ascontiguousarray(weights.w2[e][p * d.Hs:(p + 1) * d.Hs, :].T)   # (M, Hs)
                s.w1t[i, :d.Hs, :d.M].copy_(torch.from_numpy(w1).to(torch.float32).to(self.dev).to(torch.bfloat16))
                s.w2t[i, :d.M, :d.Hs].copy_(torch.from_numpy(w2).to(torch.float32).to(self.dev).to(torch.bfloat16))

    def init_random(self, seed: int = 0) -> None:
        """Synthetic weights drawn directly on the device with the reference's
        scales (gate N(0,1), w1 N(0,1/sqrt(M)), w2 N(0,1/sqrt(H)), dataplane.py:58-69)."""
        d = self.d
        for r, s in self.st.items():
            gen = torch.Generator(device=self.dev).manual_seed(seed * 7919 + r)
            s.gate.zero_()
            s.gate[:, :d.M].copy_(torch.randn(d.M, d.E, generator=torch.Generator(device=self.dev).manual_seed(seed),
                                              device=self.dev).t())
            s.w1t.zero_()
            s.w2t.zero_()
            s.w1t[:, :d.Hs, :d.M].copy_(torch.randn(d.e_local, d.Hs, d.M, generator=gen, device=self.dev)
                                        / math.sqrt(d.M))
            s.w2t[:, :d.M, :d.Hs].copy_(torch.randn(d.e_local, d.M, d.Hs, generator=gen, device=self.dev)
                                        / math.sqrt(d.H))

    def shard_grads(self, rank: int) -> dict:
        """Gradients in the reference layout: dw1 (e_local, M, Hs), dw2 (e_local, Hs, M), dgate (M, E)."""
        d, s = self.d, self.st[rank]
        return {"dw1": s.dw1t[:, :d.Hs, :d.M].transpose(1, 2), "dw2": s.dw2t[:, :d.M, :d.Hs].transpose(1, 2),
                "dgate": s.dgate[:, :d.M].t()}

    # ------------------------------------------------------------ buffers
    def _plan(self, schedule: str, r: int) -> dict:
        s = self.st[r]
        if schedule in s.bufs:
            return s.bufs[schedule]
        d, dev = self.d, self.dev
        bf = dict(dtype=torch.bfloat16, device=dev)
        i32 = dict(dtype=torch.int32, device=dev)
        el = d.e_local
        peer = self.peer and schedule in ("s1", "s2")
        W = self.world
        b: dict = {}
        if peer and schedule == "s1":   # symmetric: every MP peer writes its slice rows into them (fused AllGather)
            b["out"], b["out_peers"] = W.sym((d.n, d.Mp), rank=r)
            b["dx"], b["dx_peers"] = W.sym((d.n, d.Mp), rank=r)
        else:
            b["out"], b["dx"] = torch.zeros(d.n, d.Mp, **bf), torch.zeros(d.n, d.Mp, **bf)
        if d.M != d.Mp:
            b["x"] = torch.zeros(d.n, d.Mp, **bf)
            b["dout"] = torch.zeros(d.n, d.Mp, **bf)
        if schedule == "_local" or schedule in ("s1", "s2"):
            q = math.ceil(d.T / d.MP)
            if schedule == "s2":
                b["route"] = Routing.alloc(d.n, d.k, d.E, d.T, dev)
            else:   # s1 (and P == 1): this MP rank's token slice, slot quota ceil(T / MP)
                sl = d.n // d.MP
                b["route"] = Routing.alloc(sl, d.k, d.E, q, dev, token_offset=self.layout.mp_pos(r) * sl)
            b["q"] = q
            if not peer:
                b["send"] = torch.zeros(d.E, q, d.Mp, **bf)
                b["dsend"] = torch.zeros(d.E, q, d.Mp, **bf)
            if peer:         # holders' receive buffers, written by the sources' dispatch kernels
                b["recv"], b["recv_peers"] = W.sym((d.P, 1, el, q, d.Mp), rank=r)
                b["dyrecv"], b["dyrecv_peers"] = W.sym((d.P, 1, el, q, d.Mp), rank=r)
                b["fill_in"], b["fill_in_peers"] = W.sym((d.P, 1, el), torch.int32, rank=r)
            elif d.P == 1:   # no exchange: the slot tensors ARE the GEMM operands
                b["recv"] = b["send"].view(1, 1, d.E, q, d.Mp)
                b["dyrecv"] = b["dsend"].view(1, 1, d.E, q, d.Mp)
                b["fill_in"] = b["route"].fill.view(1, 1, d.E)
            else:
                b["recv"] = torch.zeros(d.P, 1, el, q, d.Mp, **bf)
                b["dyrecv"] = torch.zeros(d.P, 1, el, q, d.Mp, **bf)
                b["fill_in"] = torch.zeros(d.P, 1, el, **i32)
            shape = (d.P, 1, el, q)
        else:  # baseline, P > 1
            b["q"] = d.T
            b["route"] = Routing.alloc(d.n, d.k, d.E, d.T, dev)
            b["blk_fill"] = torch.zeros(d.ESP, d.E, **i32)
            b["route_blk"] = [Routing.alloc(d.n, d.k, d.E, d.T, dev, fill=b["blk_fill"][q]) for q in range(d.ESP)]
            b["xg"] = torch.zeros(d.ESP, d.n, d.Mp, **bf)
            b["disp"] = torch.zeros(d.ESP, d.E, d.T, d.Mp, **bf)             # [block q][e][slot]
            b["recv"] = torch.zeros(d.EP, d.ESP, el, d.T, d.Mp, **bf)        # [owner][block][i][slot]
            b["dyrecv"] = torch.zeros(d.EP, d.ESP, el, d.T, d.Mp, **bf)
            b["fill_in"] = torch.zeros(d.EP, d.ESP, el, **i32)
            b["dyown"] = torch.zeros(d.E, d.T, d.Mp, **bf)
            b["dyg"] = torch.zeros(d.ESP, d.E, d.T, d.Mp, **bf)
            b["dg"] = torch.zeros(d.ESP, d.n, d.Mp, **bf)
            shape = (d.EP, d.ESP, el, d.T)
        b["h"] = torch.zeros(*shape, d.Hsp, **bf)
        b["hmask"] = torch.zeros(*shape, d.Hsp // 32, dtype=torch.int32, device=dev)   # H > 0, one bit each
        b["dh"] = torch.zeros(*shape, d.Hsp, **bf)
        if peer:             # expert outputs, gathered by the owners' combine / dispatch-backward kernels
            b["y"], b["y_peers"] = W.sym((*shape, d.Mp), rank=r)
            b["dr"], b["dr_peers"] = W.sym((*shape, d.Mp), rank=r)
        else:
            b["y"] = torch.zeros(*shape, d.Mp, **bf)
            b["dr"] = torch.zeros(*shape, d.Mp, **bf)
        if peer:
            if schedule == "s1" and d.MP > 1:           # MP members' gate-gradient partials [mp_pos][E][M]
                b["gsum"], b["gsum_peers"] = W.sym((d.MP, d.E, d.Mp), torch.float32, rank=r)
            if schedule == "s1" and self.peer_push:     # owners' receive blocks [holder][i][slot]
                b["ret"], b["ret_peers"] = W.sym((d.P, el, b["q"], d.Mp), rank=r)
                b["dret"], b["dret_peers"] = W.sym((d.P, el, b["q"], d.Mp), rank=r)
            if schedule == "s2" and self.peer_push_s2:  # owners' gathered slots [holder][MP shard][i][slot]
                b["gath"], b["gath_peers"] = W.sym((d.P, d.MP, el, b["q"], d.Mp), rank=r)
                b["dgath"], b["dgath_peers"] = W.sym((d.P, d.MP, el, b["q"], d.Mp), rank=r)
        elif schedule == "baseline":
            b["ret"] = torch.zeros(d.EP, d.ESP, el, d.T, d.Mp, **bf)        # owner side [holder j][block][i][slot]
            b["dd"] = torch.zeros(d.EP, d.ESP, el, d.T, d.Mp, **bf)
        elif d.P == 1:
            b["ret"] = b["y"].view(1, d.E, b["q"], d.Mp)
            b["dret"] = b["dr"].view(1, d.E, b["q"], d.Mp)
        else:
            b["ret"] = torch.zeros(d.P, el, b["q"], d.Mp, **bf)
            b["dret"] = torch.zeros(d.P, el, b["q"], d.Mp, **bf)
            if schedule == "s2":
                b["comb"] = torch.zeros(d.E, b["q"], d.Mp, **bf)
                # phased SAA gathers per expert block: (EP, MP, e_local, q, M); else (MP, E, q, M)
                gshape = (d.EP, d.MP, el, b["q"], d.Mp) if self.saa_phased else (d.MP, d.E, b["q"], d.Mp)
                b["gath"] = torch.zeros(gshape, **bf)
                b["dcomb"] = torch.zeros(d.E, b["q"], d.Mp, **bf)
                b["dgath"] = torch.zeros(gshape, **bf)
        nr = b["route"].expert_idx.shape[0]
        b["dlogits"] = torch.zeros(nr, d.E, dtype=torch.float32, device=dev)
        need = K.gate_wgrad_workspace(d.n, d.Mp, d.E)
        if self._ws_gate is None or self._ws_gate.numel() * 4 < need:
            self._ws_gate = torch.zeros(max(1, need // 4), dtype=torch.float32, device=dev)   # counters start at zero
        s.bufs[schedule] = b
        return b

    def _input(self, b: dict, x: torch.Tensor, key: str) -> torch.Tensor:
        d = self.d
        if x.dtype != torch.bfloat16 or x.device != self.dev:
            x = x.to(device=self.dev, dtype=torch.bfloat16)
        if tuple(x.shape) != (d.n, d.M):
            raise ValueError(f"expected input of shape {(d.n, d.M)}, got {tuple(x.shape)}")
        if d.Mp == d.M and x.is_contiguous():
            return x
        b[key][:, :d.M].copy_(x)
        return b[key]

    # ------------------------------------------------------------ FFN
    def _combine_bwd_dy(self, dout, yv, rt, dlogits, slot_lo: int, cap: int, out=None, dst=None,
                        slots_out=None) -> None:
        """Combine backward (dlogits) and the dispatch of combine_w * dOut into the slot rows the
        dH GEMM reads (``out``, or the holders' buffers through the peer view ``dst``) -- one
        fused pass over dOut."""
        K.combine_bwd_dispatch(dout, yv, rt.expert_idx, rt.slot_idx, rt.probs, rt.combine_w, dlogits, slot_lo,
                               rt.fill, out=out, dst=dst, slots_out=slots_out)

    def _gemm_ws(self, rank: int, gemms: list) -> torch.Tensor:
        need = K.gemm_multi_workspace(gemms)
        ws = self._ws_gemm.get(rank)
        if ws is None or ws.numel() * 4 < need:
            ws = self._ws_gemm[rank] = torch.zeros(max(need // 4, 64), dtype=torch.int32, device=self.dev)
        return ws

    def _ffn_fwd(self, s: RankState, b: dict, y_peer: tuple | None = None) -> None:
        """H = relu(R W1) (+ the H > 0 bit mask), Y = H W2 (dataplane.py:122-128): one persistent
        launch, each Y row-pair tile starting once its H row pair is stored."""
        f = b["fill_in"]
        if self.fused_ffn:
            gs = [K.Gemm.row(b["recv"], s.w1t, K.KMAJOR, b["h"], K.EPI_RELU_MASK, aux=b["hmask"], fill=f),
                  K.Gemm.row(b["h"], s.w2t, K.KMAJOR, b["y"], K.EPI_BF16, fill=f)]
            K.gemm_multi(gs, [None, (K.DEP_ROW_PAIR, 0)], self._gemm_ws(s.rank, gs), peer=y_peer, seg_prob=1)
            return
        K.gemm_rows(b["recv"], s.w1t, K.KMAJOR, b["h"], K.EPI_RELU_MASK, aux=b["hmask"], fill=f)
        K.gemm_rows(b["h"], s.w2t, K.KMAJOR, b["y"], K.EPI_BF16, fill=f, peer=y_peer)

    def _ffn_bwd(self, s: RankState, b: dict, wscale: float = 1.0, dr_peer: tuple | None = None) -> None:
        """dH = (dY W2^T) . [H > 0], dW2^T = dY^T H, dR = dH W1^T, dW1^T = dH^T R: one persistent
        launch in that queue order (dW2 has no dependency and fills in while dH rows complete)."""
        f = b["fill_in"]
        # ReLU' from the bit mask the forward GEMM wrote (1/16 of re-reading H)
        if self.fused_ffn:
            gs = [K.Gemm.row(b["dyrecv"], s.w2t, K.MNMAJOR, b["dh"], K.EPI_DMASK, aux=b["hmask"], fill=f),
                  K.Gemm.wgrad(b["dyrecv"], b["h"], s.dw2t, K.EPI_F32, fill=f, alpha=wscale),
                  K.Gemm.row(b["dh"], s.w1t, K.MNMAJOR, b["dr"], K.EPI_BF16, fill=f),
                  K.Gemm.wgrad(b["dh"], b["recv"], s.dw1t, K.EPI_F32, fill=f, alpha=wscale)]
            K.gemm_multi(gs, [None, None, (K.DEP_ROW_PAIR, 0), (K.DEP_COL_BLOCK, 0)], self._gemm_ws(s.rank, gs),
                         peer=dr_peer, seg_prob=2)
            return
        K.gemm_rows(b["dyrecv"], s.w2t, K.MNMAJOR, b["dh"], K.EPI_DMASK, aux=b["hmask"], fill=f)
        K.gemm_wgrad(b["dyrecv"], b["h"], s.dw2t, K.EPI_F32, fill=f, alpha=wscale)
        K.gemm_wgrad(b["dh"], b["recv"], s.dw1t, K.EPI_F32, fill=f, alpha=wscale)
        K.gemm_rows(b["dh"], s.w1t, K.MNMAJOR, b["dr"], K.EPI_BF16, fill=f, peer=dr_peer)

    # ------------------------------------------------------------ message plans
    def _owned(self, *ranks) -> bool:
        return any(self.world.owns(r) for r in ranks)

    def _buf(self, rank: int, schedule: str, key: str):
        return self.st[rank].bufs[schedule][key] if self.world.owns(rank) else None

    def _fused_msgs(self, schedule: str, send_key: str, recv_key: str, with_fill: bool,
                    fill_key: str = "fill") -> list[Msg]:
        """EP&ESP AlltoAll of the dumped dispatch (collectives.py:256-283): every
        destination d receives from every source s the expert block ep_pos(d) —
        one contiguous (e_local, q, M) message per pair — plus, forward, the
        source's fill counts of those experts."""
        L, d = self.layout, self.d
        el = d.e_local
        msgs = []
        for s in range(d.P):
            for dst in range(d.P):
                if not self._owned(s, dst):
                    continue
                j = L.ep_pos(dst)
                sv = self._buf(s, schedule, send_key)
                rv = self._buf(dst, schedule, recv_key)
                msgs.append(Msg(s, dst, None if sv is None else sv[j * el:(j + 1) * el],
                                None if rv is None else rv[s, 0]))
                if with_fill:
                    fs = None
                    if self.world.owns(s):
                        bs = self.st[s].bufs[schedule]
                        fs = bs["route"].fill if fill_key == "fill" else bs[fill_key]
                    fr = self._buf(dst, schedule, "fill_in")
                    msgs.append(Msg(s, dst, None if fs is None else fs[j * el:(j + 1) * el],
                                    None if fr is None else fr[s, 0]))
        return msgs

    def _return_msgs(self, schedule: str, src_key: str, dst_key: str) -> list[Msg]:
        """Return AlltoAll (fused_combine's exchange): holder h sends owner o's rows back."""
        d = self.d
        msgs = []
        for h in range(d.P):
            for o in range(d.P):
                if not self._owned(h, o):
                    continue
                sv = self._buf(h, schedule, src_key)
                rv = self._buf(o, schedule, dst_key)
                msgs.append(Msg(h, o, None if sv is None else sv[o, 0], None if rv is None else rv[h]))
        return msgs

    def _ret_view(self, b: dict, key: str) -> K.SlotView:
        """ESP partials of owner-side returned slots: row (e, s, p) = ret[rank_of(ep_e, p)][i_e][s]."""
        d, L = self.d, self.layout
        blk = d.e_local * b["q"] * d.Mp
        a, c = (d.ESP, 1) if L.esp_contiguous else (1, d.EP)
        return K.SlotView(b[key], e_local=d.e_local, n_p=d.ESP, stride_ep=a * blk, stride_i=b["q"] * d.Mp,
                          stride_p=c * blk, stride_slo=d.Mp)

    # ------------------------------------------------------------ public API
    # ------------------------------------------------------------ communication trace
    # Each exchange the executors run appends the reference's record for it (collectives.py
    # :131-139 semantics: elements = gathered length for allgather, per-rank buffer otherwise,
    # unpadded embed), its sizes taken from the buffers / message plan actually used -- so a
    # change of the message plan shows up in ``last_trace``.  NVTX ranges name every step.
    def _unpad(self, elems: int) -> int:
        return elems * self.d.M // self.d.Mp

    def _emit(self, rec) -> None:
        if self._trace is not None:
            self._trace.add(rec)

    def _sent(self, msgs: list[Msg]) -> int:
        """bf16 elements the first hosted rank sends in a message plan (unpadded embed)."""
        r0 = self.ranks[0]
        return self._unpad(sum(m.send.numel() for m in msgs
                               if m.src == r0 and m.send is not None and m.send.dtype == torch.bfloat16))

    @staticmethod
    def _nvtx(name: str):
        return torch.cuda.nvtx.range(f"parm.{name}")

    def forward(self, schedule: str, xs: dict) -> dict:
        if schedule not in SCHEDULES:
            raise ValueError(f"unknown schedule {schedule!r}")
        self._trace = CommTrace()
        with self._nvtx(f"{schedule}.fwd"):
            if self.d.P == 1:
                out = self._fwd_local(schedule, xs)
            else:
                out = {"baseline": self._fwd_baseline, "s1": self._fwd_s1, "s2": self._fwd_s2}[schedule](xs)
        self.last_trace, self._trace = self._trace, None
        return out

    def backward(self, douts: dict) -> dict:
        if self._last is None:
            raise RuntimeError("backward() needs a preceding forward()")
        if self.d.P == 1:
            return self._bwd_local(douts)
        fn = {"baseline": self._bwd_baseline, "s1": self._bwd_s1, "s2": self._bwd_s2}[self._last]
        with self._nvtx(f"{self._last}.bwd"):
            return fn(douts)

    def capture_step(self, schedule: str, xs: dict, douts: dict, warmup: int = 2) -> StepGraph:
        """Record one forward+backward of ``schedule`` (every kernel and every
        NCCL call) into a CUDA graph over the layer's static buffers; replaying
        it costs one host launch per step instead of ~30 kernel + comm launches.
        ``xs``/``douts`` are the device tensors the graph reads (refill them
        in place between replays)."""
        for _ in range(warmup):            # allocate plans and settle NCCL state outside capture
            self.forward(schedule, xs)
            self.backward(douts)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                outs = self.forward(schedule, xs)
                dxs = self.backward(douts)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        return StepGraph(g, outs, dxs, schedule)

    def routing(self, rank: int) -> Routing:
        """Routing of the last forward on ``rank``: its own block (baseline, s2)
        or its MP token slice (s1; ``token_offset`` locates the slice)."""
        b = self.st[rank].bufs[self._last if self.d.P > 1 else "_local"]
        return b["route"]

    # ------------------------------------------------------------ P == 1
    def _fwd_local(self, schedule: str, xs: dict) -> dict:
        d = self.d
        outs = {}
        for r in self.ranks:
            s = self.st[r]
            b = self._plan("_local", r)
            x = self._input(b, xs[r], "x")
            b["xin"] = x
            rt = b["route"]
            rt.run(x, s.gate, d.k, out=b["send"])
            self._ffn_fwd(s, b)
            K.combine_fwd(self._ret_view(b, "ret"), rt.expert_idx, rt.slot_idx, rt.combine_w, b["out"])
            outs[r] = b["out"][:, :d.M]
        self._emit_local(schedule, self.st[self.ranks[0]].bufs["_local"])
        self._last = schedule
        return outs

    def _emit_local(self, schedule: str, b: dict) -> None:
        """P = 1: every exchange is the identity; the records (zero wire) keep the schedule's shape."""
        x, send = self._unpad(b["xin"].numel()), self._unpad(b["send"].numel())
        if schedule == "baseline":
            self._emit(rec_allgather("esp", 1, x))
            self._emit(rec_alltoall("ep", 1, send))
            self._emit(rec_allreduce("esp", 1, send))
            self._emit(rec_alltoall("ep", 1, send))
            self._emit(rec_split("esp", 1, send))
            return
        self._emit(rec_split("mp", 1, x if schedule == "s1" else send))
        self._emit(rec_dump(1, send))
        self._emit(rec_alltoall("ep_esp", 1, send))
        self._emit(rec_alltoall("ep_esp", 1, send))
        if schedule == "s2":
            self._trace.retag_overlapped(1, 1)
            self._emit(rec_allgather("mp", 1, send))
            self._trace.retag_overlapped(1, 1)
        else:
            self._emit(rec_allgather("mp", 1, x))

    def _bwd_local(self, douts: dict) -> dict:
        d = self.d
        res = {}
        for r in self.ranks:
            s = self.st[r]
            b = s.bufs["_local"]
            dout = self._input(b, douts[r], "dout")
            rt = b["route"]
            self._combine_bwd_dy(dout, self._ret_view(b, "ret"), rt, b["dlogits"], 0, rt.cap, out=b["dsend"])
            self._ffn_bwd(s, b)
            K.dispatch_bwd(self._ret_view(b, "dret"), rt.expert_idx, rt.slot_idx, b["dlogits"], s.gate, d.E,
                           b["dx"])
            K.gate_wgrad(b["xin"], b["dlogits"], s.dgate, self._ws_gate)
            res[r] = b["dx"][:, :d.M]
        return res

    # ------------------------------------------------------------ S1 over peer memory
    def _peer_view(self, b: dict, key: str, r: int) -> K.SlotView:
        """Rows (e, s, p) of source r in the holders' (P, 1, e_local, q, M) buffers `key`:
        partial p of expert e lives on rank_of(ep_e, p), at that rank's segment [r]."""
        d, L = self.d, self.layout
        q, el = b["q"], d.e_local
        off = 2 * r * el * q * d.Mp
        pe, pp = (d.ESP, 1) if L.esp_contiguous else (1, d.EP)
        return K.SlotView(None, e_local=el, n_p=d.ESP, stride_i=q * d.Mp, stride_slo=d.Mp,
                          peers=tuple(a + off for a in b[key + "_peers"]), peer_ep=pe, peer_p=pp)

    def _epi_peer(self, b: dict, key: str, h: int) -> tuple:
        """GEMM-epilogue destinations: segment src of holder h's output -> owner src's block [h]."""
        d = self.d
        return (self._push_fan(b, key, h), b["q"] * d.Mp, d.Mp)

    def _push_fan(self, b: dict, key: str, h: int) -> list[int]:
        """Holder h's block in every owner's (P, e_local, q, M) receive buffer `key` (segment = owner)."""
        d = self.d
        off = 2 * h * d.e_local * b["q"] * d.Mp
        return [a + off for a in b[key + "_peers"]]

    def _mp_fan(self, b: dict, key: str, r: int) -> list[int]:
        """Row r-slice of every MP peer's (n, M) buffer `key` (the fused MP AllGather)."""
        d, L = self.d, self.layout
        off = 2 * L.mp_pos(r) * (d.n // d.MP) * d.Mp
        return [b[key + "_peers"][m] + off for m in group_members(L, "mp", r)]

    def _fwd_s1_peer(self, xs: dict) -> dict:
        d, L = self.d, self.layout
        sl, el = d.n // d.MP, d.e_local
        b0 = self._plan("s1", self.ranks[0])
        self._emit(rec_split("mp", d.MP, d.n * d.M))
        buf = d.E * b0["q"] * d.M                      # the dump-source slot tensor each rank dispatches
        self._emit(rec_dump(d.ESP, buf))
        self._emit(rec_alltoall("ep_esp", d.P, buf * d.ESP))   # rows stored into the N_ESP holders
        self._emit(rec_alltoall("ep_esp", d.P, self._unpad(b0["y"].numel())))   # epilogue / push return
        self._emit(rec_allgather("mp", d.MP, sl * d.M))         # combine's fan-out to the MP peers
        for r in self.ranks:
            s, b = self.st[r], self._plan("s1", r)
            x = self._input(b, xs[r], "x")
            m = L.mp_pos(r)
            xs_ = x[m * sl:(m + 1) * sl]
            b["xslice"] = xs_
            rt = b["route"]
            rt.run(xs_, s.gate, d.k, dst=self._peer_view(b, "recv", r), slots_out=b["q"],
                   fill_fan=[a + 4 * r * el for a in b["fill_in_peers"]])
        self.world.peer_barrier()                                     # receive buffers complete
        for r in self.ranks:
            b = self.st[r].bufs["s1"]
            if self.peer_push and self.peer_epilogue:      # the second GEMM stores into the owners directly
                self._ffn_fwd(self.st[r], b, y_peer=self._epi_peer(b, "ret", r))
            else:
                self._ffn_fwd(self.st[r], b)
                if self.peer_push:
                    K.push_rows(b["y"], b["fill_in"], self._push_fan(b, "ret", r))
        self.world.peer_barrier()                                     # expert outputs complete / delivered
        for r in self.ranks:
            b = self.st[r].bufs["s1"]
            rt = b["route"]
            yv = self._ret_view(b, "ret") if self.peer_push else self._peer_view(b, "y", r)
            K.combine_fwd_fan(yv, rt.expert_idx, rt.slot_idx, rt.combine_w, self._mp_fan(b, "out", r), sl, d.Mp, d.Mp)
        self.world.peer_barrier()                                     # every MP slice gathered
        self._last = "s1"
        return {r: self.st[r].bufs["s1"]["out"][:, :d.M] for r in self.ranks}

    def _bwd_s1_peer(self, douts: dict) -> dict:
        d, L = self.d, self.layout
        sl = d.n // d.MP
        for r in self.ranks:
            s, b = self.st[r], self.st[r].bufs["s1"]
            dout = self._input(b, douts[r], "dout")
            m = L.mp_pos(r)
            ds = dout[m * sl:(m + 1) * sl]
            rt = b["route"]
            yv = self._ret_view(b, "ret") if self.peer_push else self._peer_view(b, "y", r)
            self._combine_bwd_dy(ds, yv, rt, b["dlogits"], 0, rt.cap, dst=self._peer_view(b, "dyrecv", r),
                                 slots_out=b["q"])
        self.world.peer_barrier()
        for r in self.ranks:
            b = self.st[r].bufs["s1"]
            if self.peer_push and self.peer_epilogue:
                self._ffn_bwd(self.st[r], b, dr_peer=self._epi_peer(b, "dret", r))
            else:
                self._ffn_bwd(self.st[r], b)
                if self.peer_push:
                    K.push_rows(b["dr"], b["fill_in"], self._push_fan(b, "dret", r))
        self.world.peer_barrier()
        for r in self.ranks:
            s, b = self.st[r], self.st[r].bufs["s1"]
            rt = b["route"]
            dv = self._ret_view(b, "dret") if self.peer_push else self._peer_view(b, "dr", r)
            K.dispatch_bwd_fan(dv, rt.expert_idx, rt.slot_idx, b["dlogits"], s.gate, d.E,
                               self._mp_fan(b, "dx", r), sl, d.Mp, d.Mp)
            K.gate_wgrad(b["xslice"], b["dlogits"], s.dgate, self._ws_gate)
            if d.MP > 1:      # slices gate different tokens: replicate the partial to every MP peer
                off = 4 * L.mp_pos(r) * d.E * d.Mp
                K.fan_copy(s.dgate, [b["gsum_peers"][m] + off for m in group_members(L, "mp", r)])
        self.world.peer_barrier()                                        # dx slices and dWg partials landed
        if d.MP > 1:
            for r in self.ranks:                                         # fixed-order sum: identical on the group
                s, b = self.st[r], self.st[r].bufs["s1"]
                K.sum_chunks(b["gsum"], s.dgate)
        return {r: self.st[r].bufs["s1"]["dx"][:, :d.M] for r in self.ranks}

    # ------------------------------------------------------------ S1
    def _fwd_s1(self, xs: dict) -> dict:
        if self.peer:
            return self._fwd_s1_peer(xs)
        d, L = self.d, self.layout
        sl = d.n // d.MP
        for r in self.ranks:
            s, b = self.st[r], self._plan("s1", r)
            x = self._input(b, xs[r], "x")
            m = L.mp_pos(r)
            xs_ = x[m * sl:(m + 1) * sl]                # MP split: this rank's token slice
            b["xslice"] = xs_
            rt = b["route"]
            rt.run(xs_, s.gate, d.k, out=b["send"])
        self._emit(rec_split("mp", d.MP, xs[self.ranks[0]].numel()))
        msgs = self._fused_msgs("s1", "send", "recv", with_fill=True)
        sent = self._sent(msgs)                         # the dumped buffer posted to every destination
        self._emit(rec_dump(d.ESP, sent // d.ESP))
        self._emit(rec_alltoall("ep_esp", d.P, sent))
        self.world.exchange(msgs)
        for r in self.ranks:
            self._ffn_fwd(self.st[r], self.st[r].bufs["s1"])
        msgs = self._return_msgs("s1", "y", "ret")
        self._emit(rec_alltoall("ep_esp", d.P, self._sent(msgs)))
        self.world.exchange(msgs)
        ins, outs = {}, {}
        for r in self.ranks:
            b = self.st[r].bufs["s1"]
            m = L.mp_pos(r)
            rt = b["route"]
            K.combine_fwd(self._ret_view(b, "ret"), rt.expert_idx, rt.slot_idx, rt.combine_w,
                          b["out"][m * sl:(m + 1) * sl])
            ins[r], outs[r] = b["out"][m * sl:(m + 1) * sl], b["out"]
        self._emit(rec_allgather("mp", d.MP, self._unpad(ins[self.ranks[0]].numel())))
        self.world.allgather("mp", ins, outs)
        self._last = "s1"
        return {r: self.st[r].bufs["s1"]["out"][:, :d.M] for r in self.ranks}

    def _bwd_s1(self, douts: dict) -> dict:
        if self.peer:
            return self._bwd_s1_peer(douts)
        d, L = self.d, self.layout
        sl = d.n // d.MP
        for r in self.ranks:
            s, b = self.st[r], self.st[r].bufs["s1"]
            dout = self._input(b, douts[r], "dout")
            m = L.mp_pos(r)
            ds = dout[m * sl:(m + 1) * sl]          # adjoint of AG_mp: own slice
            rt = b["route"]
            self._combine_bwd_dy(ds, self._ret_view(b, "ret"), rt, b["dlogits"], 0, rt.cap, out=b["dsend"])
        self.world.exchange(self._fused_msgs("s1", "dsend", "dyrecv", with_fill=False))  # adjoint of ESP sum + A2A
        for r in self.ranks:
            self._ffn_bwd(self.st[r], self.st[r].bufs["s1"])
        self.world.exchange(self._return_msgs("s1", "dr", "dret"))                  # adjoint of dump + A2A
        ins, outs, gins = {}, {}, {}
        for r in self.ranks:
            s, b = self.st[r], self.st[r].bufs["s1"]
            m = L.mp_pos(r)
            rt = b["route"]
            K.dispatch_bwd(self._ret_view(b, "dret"), rt.expert_idx, rt.slot_idx, b["dlogits"], s.gate, d.E,
                           b["dx"][m * sl:(m + 1) * sl])
            K.gate_wgrad(b["xslice"], b["dlogits"], s.dgate, self._ws_gate)
            ins[r], outs[r] = b["dx"][m * sl:(m + 1) * sl], b["dx"]
            gins[r] = s.dgate
        self.world.allgather("mp", ins, outs)                            # adjoint of the MP split
        self.world.allreduce("mp", gins)                                 # slices gate different tokens
        return {r: self.st[r].bufs["s1"]["dx"][:, :d.M] for r in self.ranks}

    # ------------------------------------------------------------ S2
    def _gath_view(self, b: dict, key: str) -> K.SlotView:
        """MP-gathered slots: row (e, s) = g[ep_e][s // q][i_e][s % q] (phased SAA, per-block
        gathers) or g[s // q][e][s % q] (one gather)."""
        d = self.d
        q, el = b["q"], d.e_local
        if self.saa_phased:
            return K.SlotView(b[key], e_local=el, slot_div=q, stride_ep=d.MP * el * q * d.Mp, stride_i=q * d.Mp,
                              stride_shi=el * q * d.Mp, stride_slo=d.Mp)
        return K.SlotView(b[key], e_local=d.E, slot_div=q, stride_i=q * d.Mp, stride_shi=d.E * q * d.Mp,
                          stride_slo=d.Mp)

    def _saa(self, src_key: str, ret_key: str, comb_key: str, gath_key: str) -> None:
        """S2's return AlltoAll + MP AllGather (SAA, collectives.py:315-353, paper §IV-D).

        Phased: the return is cut into N_EP phases.  In phase j, MP group g (ranks
        g*N_MP ...) receives expert block (g + j) mod N_EP from its N_ESP holders, ESP-sums
        it and starts that block's MP AllGather on the MP communicator while phase j+1
        is on the wire.  The reference phases by source rank (every rank receives from
        rank p in phase p), which on a switch leaves all but one sender idle per phase;
        the per-group rotation keeps every holder sending in every phase (exactly
        balanced when N_EP divides the number of MP groups).  Sequential (default, see
        _saa_phased): the A2A, one ESP sum, one AllGather.  Either way the data is
        identical to AllGather(ESP-sum(AlltoAll)), as the reference's is."""
        d, L = self.d, self.layout
        el = d.e_local
        msgs = self._return_msgs("s2", src_key, ret_key)
        if self._trace is not None:       # forward: the SAA pair, both overlapped over P phases
            self._emit(rec_alltoall("ep_esp", d.P, self._sent(msgs)))
            self._trace.retag_overlapped(1, d.P)
            self._emit(rec_allgather("mp", d.MP, self._unpad(self.st[self.ranks[0]].bufs["s2"][comb_key].numel())))
            self._trace.retag_overlapped(1, d.P)
        if not self.saa_phased:
            self.world.exchange(msgs)
            ins, outs = {}, {}
            for r in self.ranks:
                b = self.st[r].bufs["s2"]
                K.esp_sum(self._ret_view(b, ret_key), b[comb_key])
                ins[r], outs[r] = b[comb_key], b[gath_key]
            self.world.allgather("mp", ins, outs)
            return
        a, c = (d.ESP, 1) if L.esp_contiguous else (1, d.EP)
        handles = []
        for j in range(d.EP):
            self.world.exchange([m for m in msgs if L.ep_pos(m.src) == (m.dst // d.MP + j) % d.EP])
            ins, outs = {}, {}
            for r in self.ranks:
                bj = (r // d.MP + j) % d.EP
                b = self.st[r].bufs["s2"]
                blk = el * b["q"] * d.Mp
                view = K.SlotView(b[ret_key], e_local=el, n_p=d.ESP, stride_i=b["q"] * d.Mp, stride_p=c * blk,
                                  stride_slo=d.Mp, offset=bj * a * blk)
                K.esp_sum(view, b[comb_key][bj * el:(bj + 1) * el])
                ins[r], outs[r] = b[comb_key][bj * el:(bj + 1) * el], b[gath_key][bj]
            handles.append(self.world.allgather_async("mp", ins, outs))
        for h in handles:
            self.world.wait(h)

    def _shard_view(self, b: dict, key: str, r: int) -> K.SlotView:
        """S2 over peer memory: slot s of expert e (full-block capacity) was dispatched by MP
        member s // q of r's group, so its row lives on holder rank_of(ep_e, p) in that member's
        segment; the MP members are consecutive ranks, so the shard index is a plain stride."""
        d, L = self.d, self.layout
        q, el = b["q"], d.e_local
        seg = el * q * d.Mp
        r0 = group_members(L, "mp", r)[0]
        pe, pp = (d.ESP, 1) if L.esp_contiguous else (1, d.EP)
        return K.SlotView(None, e_local=el, n_p=d.ESP, slot_div=q, stride_i=q * d.Mp, stride_shi=seg,
                          stride_slo=d.Mp, peers=tuple(a + 2 * r0 * seg for a in b[key + "_peers"]),
                          peer_ep=pe, peer_p=pp)

    def _push_s2(self, b: dict, src_key: str, dst_key: str, h: int) -> None:
        """S2's return + MP AllGather as pushes: holder h stores segment src's rows into the
        [h][mp_pos(src)] block of every member of src's MP group (one launch per member index)."""
        d = self.d
        blk = d.e_local * b["q"] * d.Mp
        for j in range(d.MP):
            fan = [b[dst_key + "_peers"][(src // d.MP) * d.MP + j] + 2 * (h * d.MP + src % d.MP) * blk
                   for src in range(d.P)]
            K.push_rows(b[src_key], b["fill_in"], fan)

    def _gath_push_view(self, b: dict, key: str) -> K.SlotView:
        """Owner-side pushed slots: row (e, s, p) = buf[rank_of(ep_e, p)][s // q][i_e][s % q]."""
        d, L = self.d, self.layout
        q, el = b["q"], d.e_local
        blk = d.MP * el * q * d.Mp
        a, c = (d.ESP, 1) if L.esp_contiguous else (1, d.EP)
        return K.SlotView(b[key], e_local=el, n_p=d.ESP, slot_div=q, stride_ep=a * blk, stride_i=q * d.Mp,
                          stride_p=c * blk, stride_shi=el * q * d.Mp, stride_slo=d.Mp)

    def _fwd_s2_peer(self, xs: dict) -> dict:
        d, L = self.d, self.layout
        el = d.e_local
        b0 = self._plan("s2", self.ranks[0])
        buf = d.E * b0["q"] * d.M                      # this rank's slot shard [m q, (m + 1) q)
        self._emit(rec_split("mp", d.MP, buf * d.MP))
        self._emit(rec_dump(d.ESP, buf))
        self._emit(rec_alltoall("ep_esp", d.P, buf * d.ESP))
        self._emit(rec_alltoall("ep_esp", d.P, self._unpad(b0["y"].numel())))   # combine gathers from holders
        self._trace.retag_overlapped(1, d.P)
        self._emit(rec_allgather("mp", d.MP, buf))                              # ... of every MP shard
        self._trace.retag_overlapped(1, d.P)
        for r in self.ranks:
            s, b = self.st[r], self._plan("s2", r)
            x = self._input(b, xs[r], "x")
            b["xin"] = x
            rt = b["route"]
            # this MP rank's slot shard [m q, (m+1) q) straight into the holders (dispatch + A2A + dump)
            rt.run(x, s.gate, d.k, slot_lo=L.mp_pos(r) * b["q"], dst=self._peer_view(b, "recv", r), slots_out=b["q"],
                   fill_fan=[a + 4 * r * el for a in b["fill_in_peers"]])
        self.world.peer_barrier()
        for r in self.ranks:
            b = self.st[r].bufs["s2"]
            self._ffn_fwd(self.st[r], b)
            if self.peer_push_s2:
                self._push_s2(b, "y", "gath", r)
        self.world.peer_barrier()
        for r in self.ranks:      # return A2A + ESP sum + MP AllGather of the slots, fused into the combine
            b = self.st[r].bufs["s2"]
            rt = b["route"]
            yv = self._gath_push_view(b, "gath") if self.peer_push_s2 else self._shard_view(b, "y", r)
            K.combine_fwd(yv, rt.expert_idx, rt.slot_idx, rt.combine_w, b["out"])
        self._last = "s2"
        return {r: self.st[r].bufs["s2"]["out"][:, :d.M] for r in self.ranks}

    def _bwd_s2_peer(self, douts: dict) -> dict:
        d, L = self.d, self.layout
        for r in self.ranks:
            s, b = self.st[r], self.st[r].bufs["s2"]
            dout = self._input(b, douts[r], "dout")
            rt = b["route"]
            yv = self._gath_push_view(b, "gath") if self.peer_push_s2 else self._shard_view(b, "y", r)
            self._combine_bwd_dy(dout, yv, rt, b["dlogits"], L.mp_pos(r) * b["q"], rt.cap,
                                 dst=self._peer_view(b, "dyrecv", r), slots_out=b["q"])
        self.world.peer_barrier()
        for r in self.ranks:
            b = self.st[r].bufs["s2"]
            self._ffn_bwd(self.st[r], b)
            if self.peer_push_s2:
                self._push_s2(b, "dr", "dgath", r)
        self.world.peer_barrier()
        for r in self.ranks:
            s, b = self.st[r], self.st[r].bufs["s2"]
            rt = b["route"]
            dv = self._gath_push_view(b, "dgath") if self.peer_push_s2 else self._shard_view(b, "dr", r)
            K.dispatch_bwd(dv, rt.expert_idx, rt.slot_idx, b["dlogits"], s.gate, d.E, b["dx"])
            K.gate_wgrad(b["xin"], b["dlogits"], s.dgate, self._ws_gate)
        return {r: self.st[r].bufs["s2"]["dx"][:, :d.M] for r in self.ranks}

    def _fwd_s2(self, xs: dict) -> dict:
        if self.peer:
            return self._fwd_s2_peer(xs)
        d, L = self.d, self.layout
        for r in self.ranks:
            s, b = self.st[r], self._plan("s2", r)
            x = self._input(b, xs[r], "x")
            b["xin"] = x
            rt = b["route"]
            # this rank's slot shard [m*q, (m+1)*q), and its fill clamp(fill - m*q, 0, q) per expert
            if "shard_fill" not in b:
                b["shard_fill"] = torch.zeros(d.E, dtype=torch.int32, device=self.dev)
            rt.run(x, s.gate, d.k, out=b["send"], slot_lo=L.mp_pos(r) * b["q"], fill_fan=[b["shard_fill"].data_ptr()])
        b0 = self.st[self.ranks[0]].bufs["s2"]
        self._emit(rec_split("mp", d.MP, self._unpad(b0["send"].numel()) * d.MP))
        msgs = self._fused_msgs("s2", "send", "recv", with_fill=True, fill_key="shard_fill")
        sent = self._sent(msgs)
        self._emit(rec_dump(d.ESP, sent // d.ESP))
        self._emit(rec_alltoall("ep_esp", d.P, sent))
        self.world.exchange(msgs)
        for r in self.ranks:
            self._ffn_fwd(self.st[r], self.st[r].bufs["s2"])
        self._saa("y", "ret", "comb", "gath")
        for r in self.ranks:
            b = self.st[r].bufs["s2"]
            rt = b["route"]
            K.combine_fwd(self._gath_view(b, "gath"), rt.expert_idx, rt.slot_idx, rt.combine_w, b["out"])
        self._last = "s2"
        return {r: self.st[r].bufs["s2"]["out"][:, :d.M] for r in self.ranks}

    def _bwd_s2(self, douts: dict) -> dict:
        if self.peer:
            return self._bwd_s2_peer(douts)
        d, L = self.d, self.layout
        for r in self.ranks:
            s, b = self.st[r], self.st[r].bufs["s2"]
            dout = self._input(b, douts[r], "dout")
            rt = b["route"]
            # adjoint of AG_mp over slots: only this rank's slot shard
            self._combine_bwd_dy(dout, self._gath_view(b, "gath"), rt, b["dlogits"], L.mp_pos(r) * b["q"], rt.cap,
                                 out=b["dsend"])
        self.world.exchange(self._fused_msgs("s2", "dsend", "dyrecv", with_fill=False))
        for r in self.ranks:
            self._ffn_bwd(self.st[r], self.st[r].bufs["s2"])
        self._saa("dr", "dret", "dcomb", "dgath")                       # A2A + adjoint of the slot split
        for r in self.ranks:
            s, b = self.st[r], self.st[r].bufs["s2"]
            rt = b["route"]
            K.dispatch_bwd(self._gath_view(b, "dgath"), rt.expert_idx, rt.slot_idx, b["dlogits"], s.gate, d.E,
                           b["dx"])
            K.gate_wgrad(b["xin"], b["dlogits"], s.dgate, self._ws_gate)
        return {r: self.st[r].bufs["s2"]["dx"][:, :d.M] for r in self.ranks}

    # ------------------------------------------------------------ baseline
    def _ret_own_view(self, b: dict, key: str, q: int) -> K.SlotView:
        """Owner-side slots of gathered block q: row (e, s) = buf[ep_e][q][i_e][s]."""
        d = self.d
        el = d.e_local
        return K.SlotView(b[key], e_local=el, stride_ep=d.ESP * el * d.T * d.Mp, stride_i=d.T * d.Mp,
                          stride_slo=d.Mp, offset=q * el * d.T * d.Mp)

    def _fwd_baseline(self, xs: dict) -> dict:
        d, L = self.d, self.layout
        ins, outs = {}, {}
        for r in self.ranks:
            s, b = self.st[r], self._plan("baseline", r)
            x = self._input(b, xs[r], "x")
            b["xin"] = x
            b["route"].run(x, s.gate, d.k)                         # routing of the own block (slot pass only)
            ins[r], outs[r] = x, b["xg"]
        self._emit(rec_allgather("esp", d.ESP, self._unpad(ins[self.ranks[0]].numel())))
        self.world.allgather("esp", ins, outs)                   # ESP-AllGather of raw tokens
        for r in self.ranks:
            s, b = self.st[r], self.st[r].bufs["baseline"]
            for q in range(d.ESP):                               # re-gate every gathered block
                rt = b["route_blk"][q]
                rt.run(b["xg"][q], s.gate, d.k, out=b["disp"][q])
        msgs = self._ep_dispatch_msgs("disp", "recv", with_fill=True)
        self._emit(rec_alltoall("ep", d.EP, self._sent(msgs)))
        self.world.exchange(msgs)
        ys = {}
        for r in self.ranks:
            b = self.st[r].bufs["baseline"]
            self._ffn_fwd(self.st[r], b)
            ys[r] = b["y"]
        self._emit(rec_allreduce("esp", d.ESP, self._unpad(ys[self.ranks[0]].numel())))
        self.world.allreduce("esp", ys)                          # ESP-AllReduce of shard partials
        msgs = self._ep_return_msgs("y", "ret")
        self._emit(rec_alltoall("ep", d.EP, self._sent(msgs)))
        self.world.exchange(msgs)
        self._emit(rec_split("esp", d.ESP, self._unpad(ys[self.ranks[0]].numel())))   # own slot range kept
        for r in self.ranks:
            b = self.st[r].bufs["baseline"]
            rt = b["route"]
            K.combine_fwd(self._ret_own_view(b, "ret", L.esp_pos(r)), rt.expert_idx, rt.slot_idx, rt.combine_w,
                          b["out"])                              # own slot range (ESP split)
        self._last = "baseline"
        return {r: self.st[r].bufs["baseline"]["out"][:, :d.M] for r in self.ranks}

    def _ep_dispatch_msgs(self, src_key: str, dst_key: str, with_fill: bool) -> list[Msg]:
        """EP-AlltoAll of expert blocks: owner o -> holder h (EP member j), one
        message per gathered block q (src [q][j-block] is contiguous)."""
        d, L = self.d, self.layout
        el = d.e_local
        msgs = []
        for o in range(d.P):
            for j, h in enumerate(group_members(L, "ep", o)):
                if not self._owned(o, h):
                    continue
                pos = L.ep_pos(o)
                sv = self._buf(o, "baseline", src_key)
                rv = self._buf(h, "baseline", dst_key)
                bf = self._buf(o, "baseline", "blk_fill")
                rf = self._buf(h, "baseline", "fill_in")
                for q in range(d.ESP):
                    msgs.append(Msg(o, h, None if sv is None else sv[q, j * el:(j + 1) * el],
                                    None if rv is None else rv[pos, q]))
                    if with_fill:
                        msgs.append(Msg(o, h, None if bf is None else bf[q, j * el:(j + 1) * el],
                                        None if rf is None else rf[pos, q]))
        return msgs

    def _ep_return_msgs(self, src_key: str, dst_key: str) -> list[Msg]:
        """Return EP-AlltoAll: holder h sends owner o's (N_ESP, e_local, T) block in one message."""
        d, L = self.d, self.layout
        msgs = []
        for h in range(d.P):
            for o in group_members(L, "ep", h):
                if not self._owned(o, h):
                    continue
                sv = self._buf(h, "baseline", src_key)
                rv = self._buf(o, "baseline", dst_key)
                msgs.append(Msg(h, o, None if sv is None else sv[L.ep_pos(o)],
                                None if rv is None else rv[L.ep_pos(h)]))
        return msgs

    def _bwd_baseline(self, douts: dict) -> dict:
        d, L = self.d, self.layout
        ins, outs = {}, {}
        for r in self.ranks:
            s, b = self.st[r], self.st[r].bufs["baseline"]
            dout = self._input(b, douts[r], "dout")
            rt = b["route"]
            self._combine_bwd_dy(dout, self._ret_own_view(b, "ret", L.esp_pos(r)), rt, b["dlogits"], 0, d.T,
                                 out=b["dyown"])
            ins[r], outs[r] = b["dyown"], b["dyg"]
        self.world.allgather("esp", ins, outs)                   # adjoint of the ESP split
        self.world.exchange(self._ep_dispatch_msgs("dyg", "dyrecv", with_fill=False))  # adjoint of return A2A
        for r in self.ranks:                                     # AR adjoint = identity
            self._ffn_bwd(self.st[r], self.st[r].bufs["baseline"], wscale=1.0 / d.MP)
        self.world.exchange(self._ep_return_msgs("dr", "dd"))    # adjoint of the dispatch EP-A2A
        gins, gouts = {}, {}
        for r in self.ranks:
            s, b = self.st[r], self.st[r].bufs["baseline"]
            for q in range(d.ESP):
                rt = b["route_blk"][q]
                own = q == L.esp_pos(r)
                K.dispatch_bwd(self._ret_own_view(b, "dd", q), rt.expert_idx, rt.slot_idx,
                               b["dlogits"] if own else None, s.gate if own else None, d.E, b["dg"][q])
            K.gate_wgrad(b["xin"], b["dlogits"], s.dgate, self._ws_gate)
            gins[r], gouts[r] = b["dg"], b["dx"]
        self.world.reduce_scatter("esp", gins, gouts)            # adjoint of the ESP-AllGather
        return {r: self.st[r].bufs["baseline"]["dx"][:, :d.M] for r in self.ranks}
