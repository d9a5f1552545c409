"""Communication trace records (reference collectives.py:60-107 semantics).

``elements`` is the cost-model argument: the gathered length for allgather,
the per-rank buffer length otherwise.  ``wire_per_rank`` counts elements that
actually cross links per rank: AG n(G-1), A2A/RS n(G-1)/G, AR 2n(G-1)/G,
split/dump 0.  The B200 executors (runtime.MoELayer) append these records as
they run each exchange, sized from the message plans and buffers actually used
(``MoELayer.last_trace``, returned by ``api.run_schedule``); ``schedule_trace``
is the analytic expectation of the same sequence, so trace-structure tests
written against ``moesched`` apply to both.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .config import MoEConfig, ParallelLayout, derive_capacity


@dataclass(frozen=True)
class TraceRecord:
    collective: str
    group: str
    group_size: int
    elements: int
    wire_per_rank: float
    phases: int = 1
    overlapped: bool = False

    def __post_init__(self) -> None:
        if self.elements < 0 or self.wire_per_rank < 0:
            raise ValueError("element counts must be non-negative")


class CommTrace:
    """Append-only list of the collectives one schedule issued."""

    def __init__(self) -> None:
        self.records: list[TraceRecord] = []

    def add(self, record: TraceRecord) -> None:
        self.records.append(record)

    def comm_records(self) -> list[TraceRecord]:
        return [r for r in self.records if r.wire_per_rank > 0]

    def retag_overlapped(self, count: int, phases: int) -> None:
        if count > len(self.records):
            raise ValueError("fewer records than requested")
        tail = self.records[len(self.records) - count:]
        self.records[len(self.records) - count:] = [
            TraceRecord(r.collective, r.group, r.group_size, r.elements, r.wire_per_rank, phases, True)
            for r in tail]

    def count(self, collective: str, group: str | None = None) -> int:
        return sum(r.collective == collective and (group is None or r.group == group) for r in self.records)

    def total_wire(self) -> float:
        return sum(r.wire_per_rank for r in self.records)

    def __iter__(self):
        return iter(self.records)

    def __len__(self) -> int:
        return len(self.records)


# ---- record constructors (one per collective kind)
def rec_allgather(kind: str, size: int, n: int) -> TraceRecord:
    return TraceRecord("allgather", kind, size, n * size, n * (size - 1))


def rec_alltoall(kind: str, size: int, n: int) -> TraceRecord:
    return TraceRecord("alltoall", kind, size, n, n * (size - 1) / size)


def rec_reducescatter(kind: str, size: int, n: int) -> TraceRecord:
    return TraceRecord("reducescatter", kind, size, n, n * (size - 1) / size)


def rec_allreduce(kind: str, size: int, n: int) -> TraceRecord:
    return TraceRecord("allreduce", kind, size, n, 2 * n * (size - 1) / size, phases=2)


def rec_split(kind: str, size: int, n: int) -> TraceRecord:
    return TraceRecord("split", kind, size, n, 0.0)


def rec_dump(replication: int, n: int) -> TraceRecord:
    return TraceRecord("dump", "local", replication, n * replication, 0.0)


def schedule_trace(schedule: str, cfg: MoEConfig, layout: ParallelLayout) -> CommTrace:
    """The forward trace of one schedule, exactly as the reference records it
    (dataplane.py:220-413 with collectives.py accounting)."""
    P, MP, EP, ESP = layout.world_size, layout.mp_size, layout.ep_size, layout.esp_size
    E, M, n = cfg.num_experts, cfg.embed_dim, cfg.tokens_per_rank
    T = derive_capacity(cfg)
    tr = CommTrace()
    if schedule == "baseline":
        slots = ESP * T
        disp = E * slots * M
        tr.add(rec_allgather("esp", ESP, n * M))
        tr.add(rec_alltoall("ep", EP, disp))
        tr.add(rec_allreduce("esp", ESP, disp))
        tr.add(rec_alltoall("ep", EP, disp))
        tr.add(rec_split("esp", ESP, disp))
    elif schedule == "s1":
        q = math.ceil(T / MP)
        buf = E * q * M
        tr.add(rec_split("mp", MP, n * M))
        tr.add(rec_dump(ESP, buf))
        tr.add(rec_alltoall("ep_esp", P, buf * ESP))
        tr.add(rec_alltoall("ep_esp", P, buf * ESP))
        tr.add(rec_allgather("mp", MP, (n // MP) * M))
    elif schedule == "s2":
        ts = math.ceil(T / MP)
        buf = E * ts * M
        tr.add(rec_split("mp", MP, E * ts * MP * M))
        tr.add(rec_dump(ESP, buf))
        tr.add(rec_alltoall("ep_esp", P, buf * ESP))
        tr.add(rec_alltoall("ep_esp", P, buf * ESP))
        tr.retag_overlapped(1, P)
        tr.add(rec_allgather("mp", MP, buf))
        tr.retag_overlapped(1, P)
    else:
        raise ValueError(f"unknown schedule {schedule!r}")
    return tr


def schedule_ffn_rows(schedule: str, cfg: MoEConfig, layout: ParallelLayout) -> int:
    """Expert rows processed, summed over ranks (ScheduleResult.ffn_rows)."""
    P, MP, EP, ESP = layout.world_size, layout.mp_size, layout.ep_size, layout.esp_size
    T = derive_capacity(cfg)
    e_local = cfg.num_experts // EP
    if schedule == "baseline":
        per_rank = e_local * EP * ESP * T
    else:
        per_rank = e_local * P * math.ceil(T / MP)
    return P * per_rank
