"""The executors' communication trace and FFN row counts equal the reference's records
(golden run_schedule traces) — CPU only."""

from __future__ import annotations

import pytest

from paper_2407_00599_b200.config import MoEConfig, ParallelLayout
from paper_2407_00599_b200.trace import CommTrace, TraceRecord, schedule_ffn_rows, schedule_trace


def test_traces_match_reference(golden):
    meta, _ = golden
    n = 0
    for case in meta["schedules"]:
        cfg = MoEConfig(*case["cfg"])
        lay = ParallelLayout(*case["layout"], esp_contiguous=case["esp_contiguous"])
        for s, rec in case["results"].items():
            tr = schedule_trace(s, cfg, lay)
            got = [[r.collective, r.group, r.group_size, r.elements, r.wire_per_rank, r.phases, r.overlapped]
                   for r in tr]
            assert got == rec["trace"], (case["name"], s)
            assert schedule_ffn_rows(s, cfg, lay) == rec["ffn_rows"], (case["name"], s)
            n += 1
    assert n >= 27


def test_trace_structure_fig2():
    cfg = MoEConfig(1, 8, 4, 4, 2, 1, 2.0)
    lay = ParallelLayout(2, 2, 2, 4)
    base = [(r.collective, r.group) for r in schedule_trace("baseline", cfg, lay).comm_records()]
    assert base == [("allgather", "esp"), ("alltoall", "ep"), ("allreduce", "esp"), ("alltoall", "ep")]
    for s in ("s1", "s2"):
        tr = schedule_trace(s, cfg, lay)
        assert [(r.collective, r.group) for r in tr.comm_records()] == [
            ("alltoall", "ep_esp"), ("alltoall", "ep_esp"), ("allgather", "mp")]
        assert tr.count("dump") == 1 and tr.count("split", "mp") == 1
    ov = [r for r in schedule_trace("s2", cfg, lay) if r.overlapped]
    assert [(r.collective, r.group, r.phases) for r in ov] == [("alltoall", "ep_esp", 4), ("allgather", "mp", 4)]
    # S1 halves the AlltoAll volume and the FFN rows of the baseline (capacity divisible by MP)
    b_a2a = [r.elements for r in schedule_trace("baseline", cfg, lay) if r.collective == "alltoall"]
    s1_a2a = [r.elements for r in schedule_trace("s1", cfg, lay) if r.collective == "alltoall"]
    assert 2 * s1_a2a[0] == b_a2a[0]
    assert schedule_ffn_rows("baseline", cfg, lay) == 2 * schedule_ffn_rows("s1", cfg, lay)


def test_trace_record_validation_and_retag():
    with pytest.raises(ValueError):
        TraceRecord("alltoall", "ep", 2, -1, 0.0)
    tr = CommTrace()
    tr.add(TraceRecord("alltoall", "ep_esp", 4, 8, 6.0))
    tr.retag_overlapped(1, 4)
    assert tr.records[0].overlapped and tr.records[0].phases == 4 and tr.total_wire() == 6.0
    with pytest.raises(ValueError):
        tr.retag_overlapped(2, 4)
    with pytest.raises(ValueError, match="unknown schedule"):
        schedule_trace("s3", MoEConfig(1, 8, 4, 4, 2, 1, 2.0), ParallelLayout(1, 2, 2, 4))
