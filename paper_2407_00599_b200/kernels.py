"""Thin typed wrappers: torch device tensors -> C-ABI calls on the current stream.

Each wrapper validates dtypes/devices/contiguity on the host (cheap) and hands
raw pointers to ``libparm_b200.so``.  Nothing here computes on the CPU.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib

KMAJOR, MNMAJOR = 0, 1
EPI_BF16, EPI_RELU, EPI_DRELU, EPI_F32, EPI_F32_ACC, EPI_RELU_MASK, EPI_DMASK = 0, 1, 2, 3, 4, 5, 6


def _stream(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _need(t: torch.Tensor, dtype: torch.dtype, name: str) -> None:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path exists)")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")


@dataclass
class SlotView:
    """Python side of ``parm_slot_view`` (see include/parm_b200.h)."""

    base: torch.Tensor           # bf16 storage the strides index into
    e_local: int
    n_p: int = 1
    slot_div: int = 1 << 30
    stride_ep: int = 0
    stride_i: int = 0
    stride_p: int = 0
    stride_shi: int = 0
    stride_slo: int = 0
    offset: int = 0              # element offset added to base
    peers: tuple | None = None   # peer view: per-rank buffer addresses (already offset), indexed ep*peer_ep + p*peer_p
    peer_ep: int = 0
    peer_p: int = 0

    def c(self) -> _lib.SlotViewC:
        v = _lib.SlotViewC()
        if self.peers is None:
            _need(self.base, torch.bfloat16, "slot view base")
            v.ptr = self.base.data_ptr() + 2 * self.offset
        else:
            if not 1 <= len(self.peers) <= _lib.MAX_PEERS:
                raise ValueError(f"peer view over {len(self.peers)} ranks (max {_lib.MAX_PEERS})")
            v.n_peer = len(self.peers)
            for i, a in enumerate(self.peers):
                v.peer[i] = a
            v.peer_ep, v.peer_p = self.peer_ep, self.peer_p
        v.e_local, v.n_p, v.slot_div = self.e_local, self.n_p, self.slot_div
        v.stride_ep, v.stride_i, v.stride_p = self.stride_ep, self.stride_i, self.stride_p
        v.stride_shi, v.stride_slo = self.stride_shi, self.stride_slo
        return v


def _fan(ptrs, cls=None):
    f = (cls or _lib.RowFanC)()
    if not 1 <= len(ptrs) <= _lib.MAX_PEERS:
        raise ValueError(f"fan over {len(ptrs)} buffers (max {_lib.MAX_PEERS})")
    for i, a in enumerate(ptrs):
        f.ptr[i] = a
    if hasattr(f, "n"):
        f.n = len(ptrs)
    return f


def plain_view(t: torch.Tensor, e_local: int | None = None) -> SlotView:
    """(E, S, M) contiguous slot tensor, one partial."""
    E, S, M = t.shape
    el = E if e_local is None else e_local
    return SlotView(t, e_local=el, stride_ep=el * S * M, stride_i=S * M, stride_slo=M)


def gate_fwd(x: torch.Tensor, wg: torch.Tensor, k: int, expert_idx: torch.Tensor, combine_w: torch.Tensor,
             probs: torch.Tensor | None, counts: torch.Tensor | None = None) -> None:
    """wg: gate weights transposed, (E, M) bf16.  counts: int32 (ceil(n/8), E) per-tile pick counts."""
    _need(x, torch.bfloat16, "tokens")
    _need(wg, torch.bfloat16, "gate weights (bf16, transposed (E, M))")
    n, M = x.shape
    E = wg.shape[0]          # gate weights are stored transposed: (E, M)
    if x.stride(1) != 1 or not wg.is_contiguous() or wg.shape[1] != M:
        raise ValueError("tokens rows and (E, M) gate weights must be contiguous")
    if counts is not None and (counts.dtype != torch.int32 or counts.numel() < (n + 7) // 8 * E):
        raise ValueError("counts must be int32 with ceil(n/8) * E entries")
    _lib.call("parm_gate_fwd", x.data_ptr(), x.stride(0), wg.data_ptr(), n, M, E, k, expert_idx.data_ptr(),
              combine_w.data_ptr(), _ptr(probs), _ptr(counts), _stream())


def route_dispatch(x: torch.Tensor, expert_idx: torch.Tensor, counts: torch.Tensor, cap: int, slot_idx: torch.Tensor,
                   slot_src: torch.Tensor, fill: torch.Tensor, slot_lo: int = 0, out: torch.Tensor | None = None,
                   dst: SlotView | None = None, slots_out: int | None = None, fill_fan: list | None = None) -> None:
    """Slot pass + dispatch (one kernel): slots from the gate's tile counts, and every kept pick's
    token row into ``out`` (E, S_out, M) rows [slot_lo, slot_lo + S_out) -- or, with ``dst``, into
    the holders' receive buffers (peer view; per-segment fill counts to ``fill_fan``)."""
    _need(x, torch.bfloat16, "tokens")
    n, k = expert_idx.shape
    E = slot_src.shape[0]
    if x.shape[0] != n or x.stride(1) != 1:
        raise ValueError("route_dispatch: x must be (n, M) with unit inner stride")
    if dst is not None:
        if slots_out is None:
            raise ValueError("route_dispatch: slots_out required with a peer destination")
        dv = dst.c()
        ff = _fan(fill_fan, _lib.IntFanC) if fill_fan is not None else None
        _lib.call("parm_route_dispatch", x.data_ptr(), x.stride(0), expert_idx.data_ptr(), counts.data_ptr(), n, k, E,
                  cap, x.shape[1], slot_idx.data_ptr(), slot_src.data_ptr(), fill.data_ptr(), slot_lo, slots_out, None,
                  0, 0, ctypes.byref(dv), None if ff is None else ctypes.byref(ff), _stream())
        return
    ff = _fan(fill_fan, _lib.IntFanC) if fill_fan is not None else None
    if out is None:                      # slot pass only
        _lib.call("parm_route_dispatch", x.data_ptr(), x.stride(0), expert_idx.data_ptr(), counts.data_ptr(), n, k, E,
                  cap, x.shape[1], slot_idx.data_ptr(), slot_src.data_ptr(), fill.data_ptr(), slot_lo, 0, None, 0, 0,
                  None, None if ff is None else ctypes.byref(ff), _stream())
        return
    _need(out, torch.bfloat16, "dispatch out")
    if out.stride(2) != 1 or out.shape[0] != E:
        raise ValueError("route_dispatch: out must be (E, S_out, M) with unit inner stride")
    _lib.call("parm_route_dispatch", x.data_ptr(), x.stride(0), expert_idx.data_ptr(), counts.data_ptr(), n, k, E,
              cap, x.shape[1], slot_idx.data_ptr(), slot_src.data_ptr(), fill.data_ptr(), slot_lo, out.shape[1],
              out.data_ptr(), out.stride(0), out.stride(1), None, None if ff is None else ctypes.byref(ff), _stream())


def combine_fwd(view: SlotView, expert_idx: torch.Tensor, slot_idx: torch.Tensor, combine_w: torch.Tensor,
                out: torch.Tensor) -> None:
    n, M = out.shape
    k = expert_idx.shape[1]
    v = view.c()
    _lib.call("parm_combine_fwd", ctypes.byref(v), expert_idx.data_ptr(), slot_idx.data_ptr(),
              combine_w.data_ptr(), n, k, M, out.data_ptr(), out.stride(0), _stream())


def combine_bwd_dispatch(dout: torch.Tensor, view: SlotView, expert_idx: torch.Tensor, slot_idx: torch.Tensor,
                         probs: torch.Tensor, combine_w: torch.Tensor, dlogits: torch.Tensor, slot_lo: int,
                         fill: torch.Tensor, out: torch.Tensor | None = None, dst: SlotView | None = None,
                         slots_out: int | None = None) -> None:
    """Combine backward (dlogits) and the dispatch of combine_w * dOut into slot rows in one pass
    over dOut: the rows go to ``out`` (E, S_out, M) or, with ``dst``, to the holders (peer view)."""
    _need(dout, torch.bfloat16, "dOut")
    n, M = dout.shape
    k = expert_idx.shape[1]
    E = probs.shape[1]
    v = view.c()
    if dst is not None:
        if slots_out is None:
            raise ValueError("combine_bwd_dispatch: slots_out required with a peer destination")
        dv = dst.c()
        _lib.call("parm_combine_bwd_dispatch", dout.data_ptr(), dout.stride(0), ctypes.byref(v),
                  expert_idx.data_ptr(), slot_idx.data_ptr(), probs.data_ptr(), combine_w.data_ptr(), n, k, E, M,
                  dlogits.data_ptr(), slot_lo, slots_out, fill.data_ptr(), None, 0, 0, ctypes.byref(dv), _stream())
    else:
        _need(out, torch.bfloat16, "dispatch out")
        if out.stride(2) != 1:
            raise ValueError("dispatch rows need unit inner stride")
        _lib.call("parm_combine_bwd_dispatch", dout.data_ptr(), dout.stride(0), ctypes.byref(v),
                  expert_idx.data_ptr(), slot_idx.data_ptr(), probs.data_ptr(), combine_w.data_ptr(), n, k, E, M,
                  dlogits.data_ptr(), slot_lo, out.shape[1], fill.data_ptr(), out.data_ptr(), out.stride(0),
                  out.stride(1), None, _stream())


def dispatch_bwd(view: SlotView, expert_idx: torch.Tensor, slot_idx: torch.Tensor, dlogits: torch.Tensor | None,
                 wg: torch.Tensor | None, E: int, dx: torch.Tensor) -> None:
    """wg: the transposed (E, M) bf16 gate weights (or None with dlogits None)."""
    if wg is not None:
        _need(wg, torch.bfloat16, "gate weights (bf16, transposed (E, M))")
    n, M = dx.shape
    k = expert_idx.shape[1]
    v = view.c()
    _lib.call("parm_dispatch_bwd", ctypes.byref(v), expert_idx.data_ptr(), slot_idx.data_ptr(), _ptr(dlogits),
              _ptr(wg), n, k, E, M, dx.data_ptr(), dx.stride(0), _stream())


def combine_fwd_fan(view: SlotView, expert_idx: torch.Tensor, slot_idx: torch.Tensor, combine_w: torch.Tensor,
                    out_ptrs: list, n: int, M: int, ldo: int) -> None:
    """combine_fwd writing every output row to each address in ``out_ptrs`` (fused AllGather)."""
    k = expert_idx.shape[1]
    v = view.c()
    f = _fan(out_ptrs)
    _lib.call("parm_combine_fwd_fan", ctypes.byref(v), expert_idx.data_ptr(), slot_idx.data_ptr(),
              combine_w.data_ptr(), n, k, M, ctypes.byref(f), ldo, _stream())


def dispatch_bwd_fan(view: SlotView, expert_idx: torch.Tensor, slot_idx: torch.Tensor, dlogits: torch.Tensor | None,
                     wg: torch.Tensor | None, E: int, dx_ptrs: list, n: int, M: int, ldx: int) -> None:
    if wg is not None:
        _need(wg, torch.bfloat16, "gate weights (bf16, transposed (E, M))")
    k = expert_idx.shape[1]
    v = view.c()
    f = _fan(dx_ptrs)
    _lib.call("parm_dispatch_bwd_fan", ctypes.byref(v), expert_idx.data_ptr(), slot_idx.data_ptr(), _ptr(dlogits),
              _ptr(wg), n, k, E, M, ctypes.byref(f), ldx, _stream())


def push_rows(src: torch.Tensor, fill: torch.Tensor, dst_ptrs: list) -> None:
    """src (nseg, 1, e_local, rows, M) holder rows; rows s < fill[seg, i] go to dst_ptrs[seg] + (i*rows+s)*M."""
    _need(src, torch.bfloat16, "push source")
    nseg, _, el, rows, M = src.shape
    f = _fan(dst_ptrs)
    _lib.call("parm_push_rows", src.data_ptr(), nseg, el, rows, M, fill.data_ptr(), ctypes.byref(f), _stream())


def fan_copy(src: torch.Tensor, dst_ptrs: list) -> None:
    """Replicate the bytes of contiguous ``src`` into every address of ``dst_ptrs``."""
    if not src.is_contiguous():
        raise ValueError("fan_copy needs a contiguous source")
    f = _fan(dst_ptrs)
    _lib.call("parm_fan_copy", src.data_ptr(), src.numel() * src.element_size(), ctypes.byref(f), _stream())


def peer_barrier(pads: list, counters: list, ranks: list, timeout_s: float = 300.0) -> None:
    """Device-side barrier of len(pads) ranks (signal-pad addresses of every rank) for the ranks
    this process hosts (``ranks``, each with its epoch counter tensor in ``counters``): one launch,
    cooperative when it hosts several; a rank still waiting after ``timeout_s`` traps rather than
    hanging the GPU."""
    sigs = (_lib.PeerSignalC * len(ranks))()
    for s, c, r in zip(sigs, counters, ranks):
        for i, a in enumerate(pads):
            s.pad[i] = a
        s.counter = c.data_ptr()
        s.rank, s.n = r, len(pads)
        s.timeout_ns = int(timeout_s * 1e9)
    _lib.call("parm_peer_barrier", sigs, len(ranks), _stream())


def esp_sum(view: SlotView, out: torch.Tensor) -> None:
    E, S, M = out.shape
    v = view.c()
    _lib.call("parm_esp_sum", ctypes.byref(v), E, S, M, out.data_ptr(), _stream())


def sum_chunks(src: torch.Tensor, out: torch.Tensor, accumulate: bool = False) -> None:
    """out (+)= src.sum(0) for a contiguous f32 (chunks, ...) tensor, in a fixed chunk order."""
    _need(src, torch.float32, "chunks")
    _need(out, torch.float32, "out")
    if not (src.is_contiguous() and out.is_contiguous()) or src[0].numel() != out.numel():
        raise ValueError("sum_chunks: contiguous (chunks, ...) source and an output of one chunk's size")
    _lib.call("parm_sum_chunks", src.data_ptr(), src.shape[0], out.numel(), out.data_ptr(), int(accumulate),
              _stream())


def gate_wgrad_workspace(n: int, M: int, E: int) -> int:
    return int(_lib.load().parm_gate_wgrad_workspace(n, M, E))


def gate_wgrad(x: torch.Tensor, dlogits: torch.Tensor, dwg: torch.Tensor, workspace: torch.Tensor,
               accumulate: bool = False) -> None:
    n, M = x.shape
    E = dlogits.shape[1]
    _lib.call("parm_gate_wgrad", x.data_ptr(), x.stride(0), dlogits.data_ptr(), n, M, E, workspace.data_ptr(),
              workspace.numel() * workspace.element_size(), dwg.data_ptr(), int(accumulate), _stream())


class GemmTimer:
    """Optional CUDA-event bracketing of every GEMM launch (bench.py roofline).

    Events are recorded on the launching (current) stream, so the measured
    interval is the kernel's own duration in stream order.
    """

    def __init__(self) -> None:
        self.pairs: list[tuple[torch.cuda.Event, torch.cuda.Event, int]] = []

    def total_ms(self) -> tuple[float, int, int]:
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b, _ in self.pairs)
        flops = sum(f for _, _, f in self.pairs)
        return ms, len(self.pairs), flops


gemm_timer: GemmTimer | None = None

ROW, WGT = 0, 1


def _rows(t: torch.Tensor | None) -> _lib.RowsC:
    """parm_rows for a 5-D [hi][lo][g][r][c] view or a 3-D [g][r][c] tensor (unit inner stride)."""
    if t is None:
        return _lib.RowsC(None, 0, 0, 0, 0)
    if t.stride(-1) != 1:
        raise ValueError("GEMM operands need a unit inner stride")
    if t.dim() == 5:
        return _lib.RowsC(t.data_ptr(), t.stride(3), t.stride(2), t.stride(1), t.stride(0))
    if t.dim() == 3:
        return _lib.RowsC(t.data_ptr(), t.stride(1), t.stride(0), 0, 0)
    raise ValueError(f"GEMM operand must be 3-D or 5-D, got {t.dim()}-D")


def _desc(kind, epi, b_major, G, nhi, nlo, L, M, N, Kd, alpha, a, b, d, aux, fill):
    return _lib.GemmDescC(kind, epi, b_major, G, nhi, nlo, L, M, N, Kd, float(alpha), 0, _rows(a), _rows(b),
                          _rows(d), _rows(aux), _ptr(fill))


def _timed(launch, flops) -> None:
    if gemm_timer is not None:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        launch()
        e1.record()
        gemm_timer.pairs.append((e0, e1, flops))
        return
    launch()


def _gemm(kind, epi, b_major, G, nhi, nlo, L, M, N, Kd, alpha, a, b, d, aux, fill, flops, peer=None) -> None:
    desc = _desc(kind, epi, b_major, G, nhi, nlo, L, M, N, Kd, alpha, a, b, d, aux, fill)

    def launch():
        if peer is None:
            _lib.call("parm_gemm", ctypes.byref(desc), _stream())
        else:
            ptrs, g_stride, ld = peer
            f = _fan(ptrs)
            _lib.call("parm_gemm_peer", ctypes.byref(desc), ctypes.byref(f), g_stride, ld, _stream())

    _timed(launch, flops)


class Gemm:
    """One GEMM of a multi-problem launch (``row`` / ``wgrad`` build it with the checks of
    gemm_rows / gemm_wgrad; ``flops`` counts every row of the row space)."""

    def __init__(self, desc, flops: int, tensors: tuple):
        self.desc, self.flops, self._keep = desc, flops, tensors

    @staticmethod
    def row(a, b, b_major, d, epi, aux=None, fill=None, alpha=1.0) -> "Gemm":
        nhi, nlo, G, L, Kd, N = _check_rows(a, b, b_major, d, epi, aux)
        return Gemm(_desc(ROW, epi, b_major, G, nhi, nlo, L, 0, N, Kd, alpha, a, b, d, aux, fill),
                    2 * nhi * nlo * G * L * N * Kd, (a, b, d, aux, fill))

    @staticmethod
    def wgrad(a, b, d, epi=None, fill=None, alpha=1.0) -> "Gemm":
        epi = EPI_F32 if epi is None else epi
        nhi, nlo, G, L, M, N = _check_wgrad(a, b, d)
        return Gemm(_desc(WGT, epi, MNMAJOR, G, nhi, nlo, L, M, N, 0, alpha, a, b, d, None, fill),
                    2 * nhi * nlo * G * L * M * N, (a, b, d, fill))


DEP_NONE, DEP_ROW_PAIR, DEP_COL_BLOCK = 0, 1, 2


def gemm_multi_workspace(gemms: list) -> int:
    arr = (_lib.GemmDescC * len(gemms))(*[g.desc for g in gemms])
    return int(_lib.load().parm_gemm_multi_workspace(arr, len(gemms)))


def gemm_multi(gemms: list, deps: list | None, ws: torch.Tensor, peer: tuple | None = None,
               seg_prob: int = -1) -> None:
    """``gemms`` as one persistent launch over one tile queue (parm_gemm_multi).  ``deps``: per
    problem None or (DEP_ROW_PAIR | DEP_COL_BLOCK, index of an earlier problem); with dependencies
    the launch is cooperative.  ``ws``: a zeroed workspace of >= gemm_multi_workspace bytes that
    stays zeroed between launches (the dependency counters).  ``peer``
    (addresses, g_stride, ld): problem ``seg_prob``'s outputs go to the owners' receive blocks."""
    n = len(gemms)
    arr = (_lib.GemmDescC * n)(*[g.desc for g in gemms])
    dep = (_lib._c_int * (2 * n))()
    for i, dd in enumerate(deps or [None] * n):
        if dd is not None:
            dep[2 * i], dep[2 * i + 1] = dd
    need = gemm_multi_workspace(gemms)
    if ws.numel() * ws.element_size() < need:
        raise ValueError(f"gemm_multi: workspace of {ws.numel() * ws.element_size()} bytes < {need}")

    def launch():
        if peer is None:
            _lib.call("parm_gemm_multi", arr, n, dep, ws.data_ptr(), need, -1, None, 0, 0, _stream())
        else:
            ptrs, g_stride, ld = peer
            f = _fan(ptrs)
            _lib.call("parm_gemm_multi", arr, n, dep, ws.data_ptr(), need, seg_prob, ctypes.byref(f), g_stride, ld,
                      _stream())

    _timed(launch, sum(g.flops for g in gemms))


def _check_rows(a, b, b_major, d, epi, aux):
    _need(a, torch.bfloat16, "A")
    _need(b, torch.bfloat16, "B")
    _need(d, torch.bfloat16, "D")
    nhi, nlo, G, L, Kd = a.shape
    N = b.shape[1] if b_major == KMAJOR else b.shape[2]
    if tuple(d.shape) != (nhi, nlo, G, L, N) or b.shape[0] != G:
        raise ValueError(f"gemm_rows shape mismatch: A{tuple(a.shape)} B{tuple(b.shape)} D{tuple(d.shape)}")
    if epi in (EPI_RELU_MASK, EPI_DMASK):
        if aux is None or aux.dtype != torch.int32 or tuple(aux.shape) != (nhi, nlo, G, L, N // 32):
            raise ValueError("bit-mask epilogues need an int32 aux of shape D[..., N/32]")
    elif aux is not None and tuple(aux.shape) != tuple(d.shape):
        raise ValueError("aux must be shaped like D")
    return nhi, nlo, G, L, Kd, N


def _check_wgrad(a, b, d):
    _need(a, torch.bfloat16, "A")
    _need(b, torch.bfloat16, "B")
    _need(d, torch.float32, "D")
    nhi, nlo, G, L, M = a.shape
    N = b.shape[4]
    if tuple(b.shape[:4]) != (nhi, nlo, G, L) or tuple(d.shape) != (G, M, N):
        raise ValueError(f"gemm_wgrad shape mismatch: A{tuple(a.shape)} B{tuple(b.shape)} D{tuple(d.shape)}")
    return nhi, nlo, G, L, M, N


def gemm_rows(a: torch.Tensor, b: torch.Tensor, b_major: int, d: torch.Tensor, epi: int,
              aux: torch.Tensor | None = None, fill: torch.Tensor | None = None, alpha: float = 1.0,
              peer: tuple | None = None) -> None:
    """ROW GEMM: D[hi][lo][g][r][n] = alpha * A[hi][lo][g][r][:] . B[g][n][:] (5-D A/D, 3-D weights B).
    ``peer=(addresses, g_stride, ld)``: rows of segment hi*nlo+lo go to addresses[seg] + g*g_stride + r*ld
    instead of D (the epilogue stores into the owners' receive blocks over NVLink)."""
    nhi, nlo, G, L, Kd, N = _check_rows(a, b, b_major, d, epi, aux)
    _gemm(ROW, epi, b_major, G, nhi, nlo, L, 0, N, Kd, alpha, a, b, d, aux, fill,
          2 * nhi * nlo * G * L * N * Kd, peer)


def gemm_wgrad(a: torch.Tensor, b: torch.Tensor, d: torch.Tensor, epi: int = EPI_F32,
               fill: torch.Tensor | None = None, alpha: float = 1.0) -> None:
    """WGT GEMM: D[g][m][n] = alpha * sum_{hi,lo,r} A[hi][lo][g][r][m] * B[hi][lo][g][r][n] (f32 D)."""
    nhi, nlo, G, L, M, N = _check_wgrad(a, b, d)
    _gemm(WGT, epi, MNMAJOR, G, nhi, nlo, L, M, N, 0, alpha, a, b, d, None, fill, 2 * nhi * nlo * G * L * M * N)


def grouped_gemm(a: torch.Tensor, major_a: int, b: torch.Tensor, major_b: int, d: torch.Tensor, epi: int,
                 aux: torch.Tensor | None = None, alpha: float = 1.0) -> None:
    """Plain 3-D grouped GEMM D_g = A_g B_g^T (K-major A: (G, M, K); MN-major A: (G, K, M); same for B)."""
    if major_a == KMAJOR:
        u = lambda t: t.unsqueeze(0).unsqueeze(0)  # noqa: E731  (G, R, C) -> (1, 1, G, R, C)
        gemm_rows(u(a), b, major_b, u(d), epi, aux=u(aux) if aux is not None else None, alpha=alpha)
    else:
        if major_b != MNMAJOR:
            raise ValueError("MN-major A needs MN-major B")
        u = lambda t: t.unsqueeze(0).unsqueeze(0)  # noqa: E731
        gemm_wgrad(u(a), u(b), d, epi, alpha=alpha)
