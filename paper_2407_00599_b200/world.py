"""Communication backends for the schedule executors.

Executors are written once, per rank, against four primitives:

* ``exchange(msgs)``  point-to-point messages (every AlltoAll, including the
  fused EP&ESP dispatch/combine whose "dump" is just the same send buffer
  posted to N_ESP peers — collectives.py:256-312 without materialising copies);
* ``allgather(kind, ins, outs)``, ``allreduce(kind, bufs)``,
  ``reduce_scatter(kind, ins, outs)`` over the MP / EP / ESP groups.

Implementations:

``NcclWorld``   one process per GPU (torchrun), torch.distributed over NCCL on
                NVLink/NVSwitch; one sub-communicator per MP/EP/ESP group.
``PeerWorld``   NcclWorld plus NVLink peer memory (torch symmetric memory):
                S1/S2's exchanges become loads/stores inside the kernels.
``LocalWorld``  every rank of a layout emulated on ONE device with
                device-to-device copies in place of the wire — the same
                kernels and buffers per rank, used for single-GPU parity runs
                over layouts the box cannot host (P up to 16), exactly as the
                reference simulates all ranks in one process.
``PeerLocalWorld``  LocalWorld whose ranks' "symmetric" buffers are mapped to each
                other on the one device: the PeerWorld data path (peer-pointer
                tables, fused kernels, device barrier) on a single GPU.
A ``GlooWorld`` variant of NcclWorld (CPU tensors) exercises the multi-process
message plumbing in the CPU test suite.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .config import ParallelLayout, group_members, groups_of


@dataclass
class Msg:
    src: int              # sending rank
    dst: int              # receiving rank
    send: torch.Tensor    # contiguous view on the sender
    recv: torch.Tensor    # contiguous view on the receiver


class World:
    layout: ParallelLayout
    ranks: list[int]
    device: torch.device
    maps_peers = False   # True: ``sym``/``peer_barrier`` exist and S1/S2 run the fused peer-memory path

    @property
    def world_size(self) -> int:
        return self.layout.world_size

    def owns(self, rank: int) -> bool:
        return rank in self._owned

    def exchange(self, msgs: list[Msg]) -> None:
        raise NotImplementedError

    def allgather(self, kind: str, ins: dict, outs: dict) -> None:
        raise NotImplementedError

    def allreduce(self, kind: str, bufs: dict) -> None:
        raise NotImplementedError

    def reduce_scatter(self, kind: str, ins: dict, outs: dict) -> None:
        raise NotImplementedError

    def allgather_async(self, kind: str, ins: dict, outs: dict):
        """Start an allgather that may overlap later exchanges; finish with wait()."""
        self.allgather(kind, ins, outs)
        return None

    def wait(self, handle) -> None:
        pass

    def barrier(self) -> None:
        pass


class LocalWorld(World):
    """All P ranks in this process on one device; the wire is a D2D copy."""

    def __init__(self, layout: ParallelLayout, device: torch.device | str | None = None):
        self.layout = layout
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.ranks = list(range(layout.world_size))
        self._owned = set(self.ranks)

    def exchange(self, msgs: list[Msg]) -> None:
        for m in msgs:
            m.recv.copy_(m.send)

    def allgather(self, kind: str, ins: dict, outs: dict) -> None:
        for grp in groups_of(self.layout, kind):
            for r in grp:
                chunks = outs[r].view(len(grp), -1)
                for i, s in enumerate(grp):
                    src = ins[s].reshape(-1)
                    if chunks[i].data_ptr() != src.data_ptr():
                        chunks[i].copy_(src)

    # Reductions round to the buffer dtype after every addition, as NCCL's ring does for
    # bf16 (each hop adds in f32 and stores bf16): the emulated ranks see the numerics the
    # NCCL transport ships (for a 2-member group, bit for bit: round(a + b)).
    @staticmethod
    def _sum(parts: list) -> torch.Tensor:
        acc = parts[0]
        for p in parts[1:]:
            acc = (acc.float() + p.float()).to(p.dtype)
        return acc

    def allreduce(self, kind: str, bufs: dict) -> None:
        for grp in groups_of(self.layout, kind):
            if len(grp) == 1:
                continue
            acc = self._sum([bufs[s] for s in grp])
            for r in grp:
                bufs[r].copy_(acc)

    def reduce_scatter(self, kind: str, ins: dict, outs: dict) -> None:
        for grp in groups_of(self.layout, kind):
            for i, r in enumerate(grp):
                acc = self._sum([ins[s].reshape(len(grp), -1)[i] for s in grp])
                outs[r].reshape(-1).copy_(acc)


class PeerLocalWorld(LocalWorld):
    """Every rank of a layout on ONE device, running the NVLink peer-memory data path.

    ``sym`` hands each emulated rank its own zeroed copy of a "symmetric" buffer plus
    the addresses of every rank's copy -- exactly what ``PeerWorld`` gets from torch
    symmetric memory, except that the peers' copies live on the same GPU.  So the
    fused kernels (``route_dispatch`` into the holders, the GEMM's peer-epilogue stores,
    ``combine_fwd_fan``, ``combine_bwd_dispatch`` into the holders, ``dispatch_bwd_fan``,
    ``fan_copy``, ``push_rows``) run with the same peer-pointer tables, segment
    offsets and layouts as on a multi-GPU box and can be checked against the oracle on
    a single GPU.  ``peer_barrier`` runs the real device barrier for all emulated
    ranks as ONE cooperative launch (a CTA per rank, co-resident by construction), so
    the epoch/signal-pad protocol runs too (graph-capturable)."""

    maps_peers = True

    def __init__(self, layout: ParallelLayout, device: torch.device | str | None = None,
                 barrier_timeout_s: float = 300.0):
        super().__init__(layout, device)
        if layout.world_size > 8:
            raise ValueError("peer memory is supported within one 8-GPU box")
        P = layout.world_size
        self._groups: list[list[torch.Tensor]] = []        # allocation index -> every rank's copy
        self._next = {r: 0 for r in self.ranks}
        self._pads = torch.zeros(P, 64, dtype=torch.int32, device=self.device)   # pad[r][j]: epoch of j seen by r
        self.pads = [self._pads[r].data_ptr() for r in range(P)]
        self.counters = torch.zeros(P, 16, dtype=torch.int32, device=self.device)
        self.timeout_s = barrier_timeout_s

    def sym(self, shape, dtype=torch.bfloat16, rank: int = 0) -> tuple[torch.Tensor, list[int]]:
        """Rank ``rank``'s copy of the next symmetric buffer and every rank's address.
        Like PeerWorld.sym this is 'collective': the i-th call of each rank names the
        same buffer, so every rank must request the same buffers in the same order."""
        i = self._next[rank]
        self._next[rank] = i + 1
        if i == len(self._groups):
            self._groups.append([torch.zeros(tuple(shape), dtype=dtype, device=self.device) for _ in self.ranks])
        grp = self._groups[i]
        if tuple(grp[rank].shape) != tuple(shape) or grp[rank].dtype != dtype:
            raise RuntimeError(f"symmetric allocation {i}: rank {rank} asked for {tuple(shape)} {dtype}, "
                               f"the group holds {tuple(grp[rank].shape)} {grp[rank].dtype}")
        return grp[rank], [t.data_ptr() for t in grp]

    def peer_barrier(self) -> None:
        from . import kernels as K

        K.peer_barrier(self.pads, [self.counters[r] for r in self.ranks], self.ranks, self.timeout_s)


class NcclWorld(World):
    """One rank per process over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, layout: ParallelLayout, device: torch.device | str | None = None):
        import torch.distributed as dist

        if not dist.is_initialized():
            raise RuntimeError("NcclWorld needs torch.distributed initialised (torchrun)")
        if dist.get_world_size() != layout.world_size:
            raise ValueError(f"process group has {dist.get_world_size()} ranks, layout expects "
                             f"{layout.world_size}")
        self.dist = dist
        self.layout = layout
        self.rank = dist.get_rank()
        self.ranks = [self.rank]
        self._owned = {self.rank}
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl"
            else torch.device("cpu"))
        # Every process must create every group, in the same order.
        self.groups = {}
        for kind in ("mp", "ep", "esp"):
            for grp in groups_of(layout, kind):
                pg = dist.new_group(grp) if len(grp) > 1 else None
                if self.rank in grp:
                    self.groups[kind] = (grp, pg)
        self.groups["ep_esp"] = (list(range(layout.world_size)), dist.group.WORLD)

    def exchange(self, msgs: list[Msg]) -> None:
        ops = []
        for m in msgs:
            if m.src == self.rank and m.dst == self.rank:
                m.recv.copy_(m.send)
            elif m.src == self.rank:
                ops.append(self.dist.P2POp(self.dist.isend, m.send, m.dst))
            elif m.dst == self.rank:
                ops.append(self.dist.P2POp(self.dist.irecv, m.recv, m.src))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()

    def allgather(self, kind: str, ins: dict, outs: dict) -> None:
        grp, pg = self.groups[kind]
        src, dst = ins[self.rank], outs[self.rank]
        if len(grp) == 1:
            if dst.data_ptr() != src.data_ptr():
                dst.reshape(-1).copy_(src.reshape(-1))
            return
        self.dist.all_gather_into_tensor(dst.reshape(-1), src.reshape(-1), group=pg)

    def allgather_async(self, kind: str, ins: dict, outs: dict):
        # Runs on the group's own NCCL stream: it overlaps P2P exchanges issued
        # after it on the world communicator until wait() joins it back.
        grp, pg = self.groups[kind]
        src, dst = ins[self.rank], outs[self.rank]
        if len(grp) == 1:
            if dst.data_ptr() != src.data_ptr():
                dst.reshape(-1).copy_(src.reshape(-1))
            return None
        return self.dist.all_gather_into_tensor(dst.reshape(-1), src.reshape(-1), group=pg, async_op=True)

    def wait(self, handle) -> None:
        if handle is not None:
            handle.wait()

    def allreduce(self, kind: str, bufs: dict) -> None:
        grp, pg = self.groups[kind]
        if len(grp) > 1:
            self.dist.all_reduce(bufs[self.rank], group=pg)

    def reduce_scatter(self, kind: str, ins: dict, outs: dict) -> None:
        grp, pg = self.groups[kind]
        src, dst = ins[self.rank], outs[self.rank]
        if len(grp) == 1:
            dst.reshape(-1).copy_(src.reshape(-1))
            return
        self.dist.reduce_scatter_tensor(dst.reshape(-1), src.reshape(-1), group=pg)

    def barrier(self) -> None:
        self.dist.barrier()


class PeerWorld(NcclWorld):
    """NcclWorld plus NVLink peer memory: buffers allocated as torch symmetric
    memory are mapped into every rank of the box, so the permute kernels store
    dispatch rows straight into the holders' receive buffers and gather expert
    outputs straight from them (the schedules' AlltoAlls and MP AllGathers fused
    into the kernels, DESIGN.md §(e)).  Ordering is a device-side barrier over
    the symmetric signal pads (``parm_peer_barrier``, one tiny kernel, graph-
    capturable).  NCCL stays for the small gate-gradient AllReduce and for the
    baseline schedule (the DeepSpeed-ordered reference stays on NCCL)."""

    PAD_SLOT = 2048          # u32 index of this runtime's barrier slots inside each signal pad
    maps_peers = True

    def __init__(self, layout: ParallelLayout, device: torch.device | str | None = None,
                 barrier_timeout_s: float = 300.0):
        """``barrier_timeout_s``: how long a device barrier waits for a peer before it traps
        (a dead peer must not hang the GPU forever; host-side skew between ranks -- a
        checkpoint save, an eval pass -- must stay well inside it)."""
        super().__init__(layout, device)
        self.timeout_s = barrier_timeout_s
        import torch.distributed._symmetric_memory as symm_mem

        if layout.world_size > 8:
            raise ValueError("peer memory is supported within one 8-GPU box")
        self.symm = symm_mem
        self.group_name = self.dist.group.WORLD.group_name
        self._handles = []
        sync, hs = self._alloc((64,), torch.int32)
        self._sync = sync
        pad = hs.get_signal_pad(self.rank, (layout.world_size,), torch.int32, self.PAD_SLOT)
        pad.zero_()
        self.pads = [a + 4 * self.PAD_SLOT for a in hs.signal_pad_ptrs]
        self.counter = torch.zeros(1, dtype=torch.int32, device=self.device)
        torch.cuda.synchronize(self.device)
        self.dist.barrier()

    def _alloc(self, shape, dtype):
        t = self.symm.empty(*shape, dtype=dtype, device=self.device)
        t.zero_()
        torch.cuda.synchronize(self.device)      # zeroed before any peer can see (and write) it
        h = self.symm.rendezvous(t, self.group_name)
        self._handles.append(h)
        return t, h

    def sym(self, shape, dtype=torch.bfloat16, rank: int | None = None) -> tuple[torch.Tensor, list[int]]:
        """A zeroed symmetric buffer and the address of every rank's copy (rank order).
        Collective: every rank allocates the same buffers in the same order."""
        t, h = self._alloc(tuple(shape), dtype)
        return t, [int(a) for a in h.buffer_ptrs]

    def peer_barrier(self) -> None:
        from . import kernels as K

        K.peer_barrier(self.pads, [self.counter], [self.rank], self.timeout_s)

    def release(self) -> None:
        """Drop every symmetric buffer but the barrier's (after the layers using them are gone)."""
        torch.cuda.synchronize(self.device)
        self.dist.barrier()
        del self._handles[1:]


def make_world(layout: ParallelLayout, device=None) -> World:
    """NCCL world when torch.distributed spans exactly the layout, else emulate locally."""
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized() and dist.get_world_size() == layout.world_size \
                and layout.world_size > 1:
            return NcclWorld(layout, device)
    except ImportError:  # pragma: no cover
        pass
    return LocalWorld(layout, device)


__all__ = ["Msg", "World", "LocalWorld", "PeerLocalWorld", "NcclWorld", "PeerWorld", "make_world", "group_members"]
