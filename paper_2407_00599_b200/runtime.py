"""The MoE layer on B200: per-rank device state and the three schedule executors.

``MoELayer`` owns, for every rank this process executes, the bf16 expert
shards (W1/W2 stored transposed so every forward GEMM operand is K-major),
the gate weights, f32 gradient buffers and one preallocated buffer set per
schedule.  ``forward(schedule, xs)`` / ``backward(douts)`` run the
reference's schedules (moesched dataplane.py:220-413) as sm_100a kernels
(libparm_b200.so) plus collectives from ``world.py``:

  baseline  gate | AG_esp(x) -> N_ESP gates -> dispatch -> A2A_ep -> FFN ->
            AR_esp -> A2A_ep -> own slot range -> combine           (DeepSpeed-MoE order)
  s1        MP split -> gate(slice, quota ceil(T/MP)) -> dispatch -> fused
            A2A(ep&esp) -> FFN -> A2A(ep&esp) + ESP sum fused into combine -> AG_mp
  s2        gate(block) -> dispatch of own slot shard (pad to ceil(T/MP)*MP) ->
            fused A2A -> FFN -> A2A -> ESP sum -> AG_mp(slots) -> combine

Backward (no reference) is the adjoint of each sequence
under the replicated-MP convention the paper uses (split <-> AllGather,
AllReduce <-> identity, A2A <-> A2A, dump <-> local sum): every schedule
returns the gradient of L = sum_g <out_g, dout_g> with each MP group's output
counted once.  The baseline processes each token N_MP times (its duplicated
computation), so its expert weight gradients are scaled by 1/N_MP in the
wgrad GEMM epilogue to report the same quantity.

Padding: embed M and shard width H/ESP are padded to multiples of 128 and the
per-expert row count to a multiple of 128 with zeros, so every shape meets
the GEMM contract without changing results (zero rows/columns contribute 0).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import kernels as K
from .config import MoEConfig, ParallelLayout, check_compatible, derive_capacity, group_members
from .world import LocalWorld, Msg, World, make_world

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

    @classmethod
    def alloc(cls, n: int, k: int, E: int, cap: int, dev, token_offset: int = 0) -> "Routing":
        i32 = dict(dtype=torch.int32, device=dev)
        f32 = dict(dtype=torch.float32, device=dev)
        return cls(torch.empty(n, k, **i32), torch.empty(n, k, **f32), torch.empty(n, E, **f32),
                   torch.empty(n, k, **i32), torch.empty(E, max(cap, 1), **i32), torch.empty(E, **i32), cap,
                   token_offset)

    def run(self, x: torch.Tensor, wg: torch.Tensor, k: int) -> None:
        K.gate_fwd(x, wg, k, self.expert_idx, self.combine_w, self.probs)
        K.gate_slots(self.expert_idx, wg.shape[1], self.cap, self.slot_idx, self.slot_src, self.fill)


@dataclass
class RankState:
    rank: int
    gate: torch.Tensor            # (Mp, E) bf16
    w1t: torch.Tensor             # (e_local, Hsp, Mp) bf16
    w2t: torch.Tensor             # (e_local, Mp, Hsp) bf16
    dgate: torch.Tensor           # (Mp, E) f32
    dw1t: torch.Tensor            # (e_local, Hsp, Mp) f32
    dw2t: torch.Tensor            # (e_local, Mp, Hsp) f32
    bufs: dict = field(default_factory=dict)


class MoELayer:
    """One MoE layer under MP+EP+ESP on the ranks this process owns."""

    def __init__(self, cfg: MoEConfig, layout: ParallelLayout, world: World | None = None, device=None):
        check_compatible(cfg, layout)
        if cfg.top_k > 8 or cfg.num_experts > 32:
            raise ValueError("B200 kernels support top_k <= 8 and num_experts <= 32")
        self.cfg = cfg
        self.layout = layout
        self.world = world if world is not None else make_world(layout, device)
        self.dev = self.world.device
        self.d = Dims.of(cfg, layout)
        d = self.d
        bf, f32 = dict(dtype=torch.bfloat16, device=self.dev), dict(dtype=torch.float32, device=self.dev)
        self.ranks = list(self.world.ranks)
        self.st: dict[int, RankState] = {}
        for r in self.ranks:
            self.st[r] = RankState(r, torch.zeros(d.Mp, d.E, **bf), torch.zeros(d.e_local, d.Hsp, d.Mp, **bf),
                                   torch.zeros(d.e_local, d.Mp, d.Hsp, **bf), torch.zeros(d.Mp, d.E, **f32),
                                   torch.zeros(d.e_local, d.Hsp, d.Mp, **f32),
                                   torch.zeros(d.e_local, d.Mp, d.Hsp, **f32))
        self._last: str | None = None
        self._ws_gate = None

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
            s.gate[:d.M].copy_(g.to(self.dev).to(torch.bfloat16))
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
            s.gate[:d.M].copy_(torch.randn(d.M, d.E, generator=torch.Generator(device=self.dev).manual_seed(seed),
                                           device=self.dev))
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
                "dgate": s.dgate[:d.M]}

    # ------------------------------------------------------------ buffers
    def _plan(self, schedule: str, r: int) -> dict:
        s = self.st[r]
        if schedule in s.bufs:
            return s.bufs[schedule]
        d, dev = self.d, self.dev
        bf = dict(dtype=torch.bfloat16, device=dev)
        b: dict = {}
        b["x"] = torch.zeros(d.n, d.Mp, **bf)          # padded input (alias of caller's when M == Mp)
        b["out"] = torch.zeros(d.n, d.Mp, **bf)
        b["dout"] = torch.zeros(d.n, d.Mp, **bf)
        b["dx"] = torch.zeros(d.n, d.Mp, **bf)
        if schedule in ("s1", "s2") or d.P == 1:
            if schedule == "s1" or d.P == 1:
                q = math.ceil(d.T / d.MP)
                rows_tok = d.n // d.MP
                b["route"] = Routing.alloc(rows_tok, d.k, d.E, q, dev, token_offset=self.layout.mp_pos(r) * rows_tok)
            else:
                q = math.ceil(d.T / d.MP)
                b["route"] = Routing.alloc(d.n, d.k, d.E, d.T, dev)
            rows = d.P * q
            rows_pad = _ceil_to(rows, 128)
            b.update(q=q, rows=rows, rows_pad=rows_pad)
            b["send"] = torch.zeros(d.E, q, d.Mp, **bf)
            b["recv"] = torch.zeros(d.e_local, rows_pad, d.Mp, **bf)
            b["dyrecv"] = torch.zeros(d.e_local, rows_pad, d.Mp, **bf)
            b["ret"] = torch.zeros(d.P, d.e_local, q, d.Mp, **bf)
            b["dret"] = torch.zeros(d.P, d.e_local, q, d.Mp, **bf)
            if schedule == "s2" and d.P > 1:
                b["comb"] = torch.zeros(d.E, q, d.Mp, **bf)
                b["gath"] = torch.zeros(d.MP, d.E, q, d.Mp, **bf)
                b["dcomb"] = torch.zeros(d.E, q, d.Mp, **bf)
                b["dgath"] = torch.zeros(d.MP, d.E, q, d.Mp, **bf)
        else:  # baseline, P > 1
            gs = d.ESP * d.T
            rows = d.EP * gs
            rows_pad = _ceil_to(rows, 128)
            b.update(q=d.T, gs=gs, rows=rows, rows_pad=rows_pad)
            b["route"] = Routing.alloc(d.n, d.k, d.E, d.T, dev)
            b["route_blk"] = [Routing.alloc(d.n, d.k, d.E, d.T, dev) for _ in range(d.ESP)]
            b["xg"] = torch.zeros(d.ESP, d.n, d.Mp, **bf)
            b["disp"] = torch.zeros(d.E, gs, d.Mp, **bf)
            b["recv"] = torch.zeros(d.e_local, rows_pad, d.Mp, **bf)
            b["dyrecv"] = torch.zeros(d.e_local, rows_pad, d.Mp, **bf)
            b["ret"] = torch.zeros(d.E, gs, d.Mp, **bf)
            b["dyown"] = torch.zeros(d.E, d.T, d.Mp, **bf)
            b["dyg"] = torch.zeros(d.ESP, d.E, d.T, d.Mp, **bf)
            b["dd"] = torch.zeros(d.E, gs, d.Mp, **bf)
            b["dg"] = torch.zeros(d.ESP, d.n, d.Mp, **bf)
        rp = b["rows_pad"]
        b["h"] = torch.zeros(d.e_local, rp, d.Hsp, **bf)
        b["y"] = torch.zeros(d.e_local, rp, d.Mp, **bf)
        b["dh"] = torch.zeros(d.e_local, rp, d.Hsp, **bf)
        b["dr"] = torch.zeros(d.e_local, rp, d.Mp, **bf)
        nr = b["route"].expert_idx.shape[0]
        b["dlogits"] = torch.zeros(nr, d.E, dtype=torch.float32, device=dev)
        if self._ws_gate is None or self._ws_gate.numel() * 4 < K.gate_wgrad_workspace(d.n, d.Mp, d.E):
            self._ws_gate = torch.empty(max(1, K.gate_wgrad_workspace(d.n, d.Mp, d.E) // 4), dtype=torch.float32,
                                        device=dev)
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
    def _ffn_fwd(self, s: RankState, b: dict) -> None:
        K.grouped_gemm(b["recv"], K.KMAJOR, s.w1t, K.KMAJOR, b["h"], K.EPI_RELU)
        K.grouped_gemm(b["h"], K.KMAJOR, s.w2t, K.KMAJOR, b["y"], K.EPI_BF16)

    def _ffn_bwd(self, s: RankState, b: dict, wscale: float = 1.0) -> None:
        K.grouped_gemm(b["dyrecv"], K.KMAJOR, s.w2t, K.MNMAJOR, b["dh"], K.EPI_DRELU, aux=b["h"])
        K.grouped_gemm(b["dyrecv"], K.MNMAJOR, b["h"], K.MNMAJOR, s.dw2t, K.EPI_F32, alpha=wscale)
        K.grouped_gemm(b["dh"], K.MNMAJOR, b["recv"], K.MNMAJOR, s.dw1t, K.EPI_F32, alpha=wscale)
        K.grouped_gemm(b["dh"], K.KMAJOR, s.w1t, K.MNMAJOR, b["dr"], K.EPI_BF16)

    # ------------------------------------------------------------ message plans
    def _fused_msgs(self, src_key: str, dst_key: str, schedule: str) -> list[Msg]:
        """EP&ESP AlltoAll of the dumped dispatch (collectives.py:256-283):
        destination d gets source s's expert block ep_pos(d); expert-major receive."""
        L, d = self.layout, self.d
        msgs = []
        for s in range(d.P):
            for dst in range(d.P):
                if not (self.world.owns(s) or self.world.owns(dst)):
                    continue
                for i in range(d.e_local):
                    e = L.ep_pos(dst) * d.e_local + i
                    sv = self.st[s].bufs[schedule][src_key][e] if self.world.owns(s) else None
                    if self.world.owns(dst):
                        bq = self.st[dst].bufs[schedule]
                        rv = bq[dst_key][i, s * bq["q"]:(s + 1) * bq["q"]]
                    else:
                        rv = None
                    msgs.append(Msg(s, dst, sv, rv))
        return msgs

    def _return_msgs(self, src_key: str, dst_key: str, schedule: str) -> list[Msg]:
        """Return AlltoAll (fused_combine's exchange): holder h sends rows of
        owner o back to o, landing at ret[o][h][i]."""
        d = self.d
        msgs = []
        for h in range(d.P):
            for o in range(d.P):
                if not (self.world.owns(h) or self.world.owns(o)):
                    continue
                for i in range(d.e_local):
                    if self.world.owns(h):
                        bh = self.st[h].bufs[schedule]
                        sv = bh[src_key][i, o * bh["q"]:(o + 1) * bh["q"]]
                    else:
                        sv = None
                    rv = self.st[o].bufs[schedule][dst_key][h, i] if self.world.owns(o) else None
                    msgs.append(Msg(h, o, sv, rv))
        return msgs

    def _ret_view(self, b: dict, key: str) -> K.SlotView:
        """ESP partials of owner-side returned slots: row (e, s, p) = ret[rank_of(ep_e, p)][i_e][s]."""
        d, L = self.d, self.layout
        blk = d.e_local * b["q"] * d.Mp
        a, c = (d.ESP, 1) if L.esp_contiguous else (1, d.EP)
        return K.SlotView(b[key], e_local=d.e_local, n_p=d.ESP, stride_ep=a * blk, stride_i=b["q"] * d.Mp,
                          stride_p=c * blk, stride_slo=d.Mp)

    # ------------------------------------------------------------ public API
    def forward(self, schedule: str, xs: dict) -> dict:
        if schedule not in SCHEDULES:
            raise ValueError(f"unknown schedule {schedule!r}")
        if self.d.P == 1:
            return self._fwd_local(schedule, xs)
        fn = {"baseline": self._fwd_baseline, "s1": self._fwd_s1, "s2": self._fwd_s2}[schedule]
        return fn(xs)

    def backward(self, douts: dict) -> dict:
        if self._last is None:
            raise RuntimeError("backward() needs a preceding forward()")
        if self.d.P == 1:
            return self._bwd_local(douts)
        fn = {"baseline": self._bwd_baseline, "s1": self._bwd_s1, "s2": self._bwd_s2}[self._last]
        return fn(douts)

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
            rt.run(x, s.gate, d.k)
            # slots straight into the expert-major FFN input (no exchange at P = 1)
            K.dispatch_rows(x, rt.slot_src, d.k, rt.cap, 0, b["recv"][:, :b["q"]])
            self._ffn_fwd(s, b)
            view = K.SlotView(b["y"], e_local=d.E, stride_i=b["rows_pad"] * d.Mp, stride_slo=d.Mp)
            K.combine_fwd(view, rt.expert_idx, rt.slot_idx, rt.combine_w, b["out"])
            outs[r] = b["out"][:, :d.M]
        self._last = schedule
        return outs

    def _bwd_local(self, douts: dict) -> dict:
        d = self.d
        res = {}
        for r in self.ranks:
            s = self.st[r]
            b = s.bufs["_local"]
            dout = self._input(b, douts[r], "dout")
            rt = b["route"]
            view = K.SlotView(b["y"], e_local=d.E, stride_i=b["rows_pad"] * d.Mp, stride_slo=d.Mp)
            K.combine_bwd(dout, view, rt.expert_idx, rt.slot_idx, rt.probs, b["dlogits"])
            K.dispatch_rows(dout, rt.slot_src, d.k, rt.cap, 0, b["dyrecv"][:, :b["q"]], scale=rt.combine_w)
            self._ffn_bwd(s, b)
            dview = K.SlotView(b["dr"], e_local=d.E, stride_i=b["rows_pad"] * d.Mp, stride_slo=d.Mp)
            K.dispatch_bwd(dview, rt.expert_idx, rt.slot_idx, b["dlogits"], s.gate, d.E, b["dx"])
            K.gate_wgrad(b["xin"], b["dlogits"], s.dgate, self._ws_gate)
            res[r] = b["dx"][:, :d.M]
        return res

    # ------------------------------------------------------------ S1
    def _fwd_s1(self, xs: dict) -> dict:
        d, L = self.d, self.layout
        sl = d.n // d.MP
        for r in self.ranks:
            s, b = self.st[r], self._plan("s1", r)
            x = self._input(b, xs[r], "x")
            b["xin"] = x
            m = L.mp_pos(r)
            xs_ = x[m * sl:(m + 1) * sl]
            b["xslice"] = xs_
            rt = b["route"]
            rt.run(xs_, s.gate, d.k)
            K.dispatch_rows(xs_, rt.slot_src, d.k, rt.cap, 0, b["send"])
        self.world.exchange(self._fused_msgs("send", "recv", "s1"))
        for r in self.ranks:
            self._ffn_fwd(self.st[r], self.st[r].bufs["s1"])
        self.world.exchange(self._return_msgs("y", "ret", "s1"))
        ins, outs = {}, {}
        for r in self.ranks:
            b = self.st[r].bufs["s1"]
            m = L.mp_pos(r)
            rt = b["route"]
            K.combine_fwd(self._ret_view(b, "ret"), rt.expert_idx, rt.slot_idx, rt.combine_w,
                          b["out"][m * sl:(m + 1) * sl])
            ins[r], outs[r] = b["out"][m * sl:(m + 1) * sl], b["out"]
        self.world.allgather("mp", ins, outs)
        self._last = "s1"
        return {r: self.st[r].bufs["s1"]["out"][:, :d.M] for r in self.ranks}

    def _bwd_s1(self, douts: dict) -> dict:
        d, L = self.d, self.layout
        sl = d.n // d.MP
        for r in self.ranks:
            s, b = self.st[r], self.st[r].bufs["s1"]
            dout = self._input(b, douts[r], "dout")
            m = L.mp_pos(r)
            ds = dout[m * sl:(m + 1) * sl]          # adjoint of AG_mp: own slice
            rt = b["route"]
            K.combine_bwd(ds, self._ret_view(b, "ret"), rt.expert_idx, rt.slot_idx, rt.probs, b["dlogits"])
            K.dispatch_rows(ds, rt.slot_src, d.k, rt.cap, 0, b["send"], scale=rt.combine_w)
        self.world.exchange(self._fused_msgs("send", "dyrecv", "s1"))   # adjoint of ESP sum + A2A
        for r in self.ranks:
            self._ffn_bwd(self.st[r], self.st[r].bufs["s1"])
        self.world.exchange(self._return_msgs("dr", "dret", "s1"))      # adjoint of dump + A2A
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
        d = self.d
        q = b["q"]
        return K.SlotView(b[key], e_local=d.E, slot_div=q, stride_i=q * d.Mp, stride_shi=d.E * q * d.Mp,
                          stride_slo=d.Mp)

    def _fwd_s2(self, xs: dict) -> dict:
        d, L = self.d, self.layout
        for r in self.ranks:
            s, b = self.st[r], self._plan("s2", r)
            x = self._input(b, xs[r], "x")
            b["xin"] = x
            rt = b["route"]
            rt.run(x, s.gate, d.k)
            K.dispatch_rows(x, rt.slot_src, d.k, rt.cap, L.mp_pos(r) * b["q"], b["send"])
        self.world.exchange(self._fused_msgs("send", "recv", "s2"))
        for r in self.ranks:
            self._ffn_fwd(self.st[r], self.st[r].bufs["s2"])
        self.world.exchange(self._return_msgs("y", "ret", "s2"))
        ins, outs = {}, {}
        for r in self.ranks:
            b = self.st[r].bufs["s2"]
            K.esp_sum(self._ret_view(b, "ret"), b["comb"])
            ins[r], outs[r] = b["comb"], b["gath"]
        self.world.allgather("mp", ins, outs)
        for r in self.ranks:
            b = self.st[r].bufs["s2"]
            rt = b["route"]
            K.combine_fwd(self._gath_view(b, "gath"), rt.expert_idx, rt.slot_idx, rt.combine_w, b["out"])
        self._last = "s2"
        return {r: self.st[r].bufs["s2"]["out"][:, :d.M] for r in self.ranks}

    def _bwd_s2(self, douts: dict) -> dict:
        d, L = self.d, self.layout
        for r in self.ranks:
            s, b = self.st[r], self.st[r].bufs["s2"]
            dout = self._input(b, douts[r], "dout")
            rt = b["route"]
            K.combine_bwd(dout, self._gath_view(b, "gath"), rt.expert_idx, rt.slot_idx, rt.probs, b["dlogits"])
            # adjoint of AG_mp over slots: only this rank's slot shard
            K.dispatch_rows(dout, rt.slot_src, d.k, rt.cap, L.mp_pos(r) * b["q"], b["send"], scale=rt.combine_w)
        self.world.exchange(self._fused_msgs("send", "dyrecv", "s2"))
        for r in self.ranks:
            self._ffn_bwd(self.st[r], self.st[r].bufs["s2"])
        self.world.exchange(self._return_msgs("dr", "dret", "s2"))
        ins, outs = {}, {}
        for r in self.ranks:
            b = self.st[r].bufs["s2"]
            K.esp_sum(self._ret_view(b, "dret"), b["dcomb"])
            ins[r], outs[r] = b["dcomb"], b["dgath"]
        self.world.allgather("mp", ins, outs)                            # adjoint of the slot split
        for r in self.ranks:
            s, b = self.st[r], self.st[r].bufs["s2"]
            rt = b["route"]
            K.dispatch_bwd(self._gath_view(b, "dgath"), rt.expert_idx, rt.slot_idx, b["dlogits"], s.gate, d.E,
                           b["dx"])
            K.gate_wgrad(b["xin"], b["dlogits"], s.dgate, self._ws_gate)
        return {r: self.st[r].bufs["s2"]["dx"][:, :d.M] for r in self.ranks}

    # ------------------------------------------------------------ baseline
    def _fwd_baseline(self, xs: dict) -> dict:
        d, L = self.d, self.layout
        ins, outs = {}, {}
        for r in self.ranks:
            s, b = self.st[r], self._plan("baseline", r)
            x = self._input(b, xs[r], "x")
            b["xin"] = x
            b["route"].run(x, s.gate, d.k)                       # combine weights of the own block
            ins[r], outs[r] = x, b["xg"]
        self.world.allgather("esp", ins, outs)                   # ESP-AllGather of raw tokens
        for r in self.ranks:
            s, b = self.st[r], self.st[r].bufs["baseline"]
            for q in range(d.ESP):                               # re-gate every gathered block
                rt = b["route_blk"][q]
                rt.run(b["xg"][q], s.gate, d.k)
                K.dispatch_rows(b["xg"][q], rt.slot_src, d.k, d.T, 0, b["disp"][:, q * d.T:(q + 1) * d.T])
        self.world.exchange(self._ep_msgs_fwd())
        ys = {}
        for r in self.ranks:
            b = self.st[r].bufs["baseline"]
            self._ffn_fwd(self.st[r], b)
            ys[r] = b["y"]
        self.world.allreduce("esp", ys)                          # ESP-AllReduce of shard partials
        self.world.exchange(self._ep_msgs_ret())
        for r in self.ranks:
            b = self.st[r].bufs["baseline"]
            rt = b["route"]
            view = K.SlotView(b["ret"], e_local=d.E, stride_i=b["gs"] * d.Mp, stride_slo=d.Mp,
                              offset=L.esp_pos(r) * d.T * d.Mp)  # own slot range (ESP split)
            K.combine_fwd(view, rt.expert_idx, rt.slot_idx, rt.combine_w, b["out"])
        self._last = "baseline"
        return {r: self.st[r].bufs["baseline"]["out"][:, :d.M] for r in self.ranks}

    def _ep_msgs_fwd(self) -> list[Msg]:
        """EP-AlltoAll of whole expert blocks: owner o -> holder h = EP member j."""
        d, L = self.d, self.layout
        msgs = []
        for o in range(d.P):
            grp = group_members(L, "ep", o)
            for j, h in enumerate(grp):
                if not (self.world.owns(o) or self.world.owns(h)):
                    continue
                for i in range(d.e_local):
                    sv = self.st[o].bufs["baseline"]["disp"][j * d.e_local + i] if self.world.owns(o) else None
                    if self.world.owns(h):
                        bh = self.st[h].bufs["baseline"]
                        pos = L.ep_pos(o)
                        rv = bh["recv"][i, pos * bh["gs"]:(pos + 1) * bh["gs"]]
                    else:
                        rv = None
                    msgs.append(Msg(o, h, sv, rv))
        return msgs

    def _ep_msgs_ret(self, src_key: str = "y", dst_key: str = "ret") -> list[Msg]:
        d, L = self.d, self.layout
        msgs = []
        for h in range(d.P):
            grp = group_members(L, "ep", h)
            for j, o in enumerate(grp):
                if not (self.world.owns(o) or self.world.owns(h)):
                    continue
                for i in range(d.e_local):
                    if self.world.owns(h):
                        bh = self.st[h].bufs["baseline"]
                        sv = bh[src_key][i, j * bh["gs"]:(j + 1) * bh["gs"]]
                    else:
                        sv = None
                    rv = self.st[o].bufs["baseline"][dst_key][L.ep_pos(h) * d.e_local + i] \
                        if self.world.owns(o) else None
                    msgs.append(Msg(h, o, sv, rv))
        return msgs

    def _bwd_baseline(self, douts: dict) -> dict:
        d, L = self.d, self.layout
        ins, outs = {}, {}
        for r in self.ranks:
            s, b = self.st[r], self.st[r].bufs["baseline"]
            dout = self._input(b, douts[r], "dout")
            rt = b["route"]
            view = K.SlotView(b["ret"], e_local=d.E, stride_i=b["gs"] * d.Mp, stride_slo=d.Mp,
                              offset=L.esp_pos(r) * d.T * d.Mp)
            K.combine_bwd(dout, view, rt.expert_idx, rt.slot_idx, rt.probs, b["dlogits"])
            K.dispatch_rows(dout, rt.slot_src, d.k, d.T, 0, b["dyown"], scale=rt.combine_w)
            ins[r], outs[r] = b["dyown"], b["dyg"]
        self.world.allgather("esp", ins, outs)                   # adjoint of the ESP split
        # adjoint of the return EP-A2A: owner o sends range q of holder-h experts
        msgs = []
        for o in range(d.P):
            grp = group_members(L, "ep", o)
            for j, h in enumerate(grp):
                if not (self.world.owns(o) or self.world.owns(h)):
                    continue
                for i in range(d.e_local):
                    for q in range(d.ESP):
                        sv = self.st[o].bufs["baseline"]["dyg"][q, j * d.e_local + i] if self.world.owns(o) else None
                        if self.world.owns(h):
                            bh = self.st[h].bufs["baseline"]
                            lo = L.ep_pos(o) * bh["gs"] + q * d.T
                            rv = bh["dyrecv"][i, lo:lo + d.T]
                        else:
                            rv = None
                        msgs.append(Msg(o, h, sv, rv))
        self.world.exchange(msgs)
        for r in self.ranks:                                     # AR adjoint = identity
            self._ffn_bwd(self.st[r], self.st[r].bufs["baseline"], wscale=1.0 / d.MP)
        self.world.exchange(self._ep_msgs_ret("dr", "dd"))       # adjoint of the dispatch EP-A2A
        gins, gouts = {}, {}
        for r in self.ranks:
            s, b = self.st[r], self.st[r].bufs["baseline"]
            for q in range(d.ESP):
                rt = b["route_blk"][q]
                view = K.SlotView(b["dd"], e_local=d.E, stride_i=b["gs"] * d.Mp, stride_slo=d.Mp,
                                  offset=q * d.T * d.Mp)
                own = q == L.esp_pos(r)
                K.dispatch_bwd(view, rt.expert_idx, rt.slot_idx, b["dlogits"] if own else None,
                               s.gate if own else None, d.E, b["dg"][q])
            K.gate_wgrad(b["xin"], b["dlogits"], s.dgate, self._ws_gate)
            gins[r], gouts[r] = b["dg"], b["dx"]
        self.world.reduce_scatter("esp", gins, gouts)            # adjoint of the ESP-AllGather
        return {r: self.st[r].bufs["baseline"]["dx"][:, :d.M] for r in self.ranks}
