"""Communication backends for the schedule executors.

Executors are written once, per rank, against four primitives:

* ``exchange(msgs)``  point-to-point messages (every AlltoAll, including the
  fused EP&ESP dispatch/combine whose "dump" is just the same send buffer
  posted to N_ESP peers — collectives.py:256-312 without materialising copies);
* ``allgather(kind, ins, outs)``, ``allreduce(kind, bufs)``,
  ``reduce_scatter(kind, ins, outs)`` over the MP / EP / ESP groups.

Two implementations:

``NcclWorld``   one process per GPU (torchrun), torch.distributed over NCCL on
                NVLink/NVSwitch; one sub-communicator per MP/EP/ESP group.
``LocalWorld``  every rank of a layout emulated on ONE device with
                device-to-device copies in place of the wire — the same
                kernels and buffers per rank, used for single-GPU parity runs
                over layouts the box cannot host (P up to 16), exactly as the
                reference simulates all ranks in one process.
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

    def allreduce(self, kind: str, bufs: dict) -> None:
        for grp in groups_of(self.layout, kind):
            if len(grp) == 1:
                continue
            acc = bufs[grp[0]].float()
            for s in grp[1:]:
                acc += bufs[s].float()
            for r in grp:
                bufs[r].copy_(acc)

    def reduce_scatter(self, kind: str, ins: dict, outs: dict) -> None:
        for grp in groups_of(self.layout, kind):
            for i, r in enumerate(grp):
                acc = ins[grp[0]].reshape(len(grp), -1)[i].float()
                for s in grp[1:]:
                    acc = acc + ins[s].reshape(len(grp), -1)[i].float()
                outs[r].reshape(-1).copy_(acc)


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

    def __init__(self, layout: ParallelLayout, device: torch.device | str | None = None):
        super().__init__(layout, device)
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

    def sym(self, shape, dtype=torch.bfloat16) -> tuple[torch.Tensor, list[int]]:
        """A zeroed symmetric buffer and the address of every rank's copy (rank order).
        Collective: every rank allocates the same buffers in the same order."""
        t, h = self._alloc(tuple(shape), dtype)
        return t, [int(a) for a in h.buffer_ptrs]

    def peer_barrier(self) -> None:
        from . import kernels as K

        K.peer_barrier(self.pads, self.counter, self.rank)

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


__all__ = ["Msg", "World", "LocalWorld", "NcclWorld", "PeerWorld", "make_world", "group_members"]
