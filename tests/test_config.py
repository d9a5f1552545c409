"""Host-side configuration: capacity, rank overlay, groups, placement, compatibility and the
config-file parser behave like the reference's (moesched config.py) — CPU only."""

from __future__ import annotations

import itertools

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2407_00599_b200.config import (
    ClusterSpec,
    ConfigError,
    MoEConfig,
    ParallelLayout,
    PlacementCase,
    check_compatible,
    classify_placement,
    derive_capacity,
    group_members,
    groups_of,
    load_config,
    mp_groups_intra_node,
    parse_config_text,
)

from oracle import moe_oracle as O


def cfg(**kw):
    base = dict(samples_per_rank=4, seq_len=128, embed_dim=256, hidden_dim=512, num_experts=4, top_k=2,
                capacity_factor=1.2)
    base.update(kw)
    return MoEConfig(**base)


def test_capacity_known_answers(golden):
    meta, _ = golden
    kat = meta["costs"]["capacity_kat"]
    assert derive_capacity(cfg()) == kat[0] == 308
    assert derive_capacity(MoEConfig(8, 1024, 1024, 4096, 8, 2, 1.2)) == kat[1] == 2458
    assert derive_capacity(cfg(capacity_factor=2.4)) == kat[2]
    assert derive_capacity(MoEConfig(8, 1024, 1024, 4096, 8, 2, 2.4)) == kat[3]
    assert derive_capacity(cfg(capacity_factor=1e-6)) == 1                        # floor of one slot
    assert derive_capacity(cfg(top_k=1, capacity_factor=4.0, num_experts=4)) == 512   # exact rational, no float creep


@given(b=st.integers(1, 16), seq=st.integers(1, 512), e=st.integers(1, 16), k=st.integers(1, 4),
       f=st.sampled_from([0.5, 1.0, 1.2, 1.25, 2.4, 3.0]))
@settings(max_examples=200, deadline=None)
def test_capacity_matches_oracle_and_is_monotone(b, seq, e, k, f):
    if k > e:
        return
    c = MoEConfig(b, seq, 8, 8, e, k, f)
    assert derive_capacity(c) == O.derive_capacity(b * seq, e, k, f)
    assert derive_capacity(MoEConfig(b + 1, seq, 8, 8, e, k, f)) >= derive_capacity(c)


@pytest.mark.parametrize("bad", [dict(samples_per_rank=0), dict(top_k=5), dict(capacity_factor=0.0),
                                 dict(embed_dim=-1), dict(seq_len=1.5)])
def test_moe_config_validation(bad):
    with pytest.raises(ValueError):
        cfg(**bad)


LAYOUTS = [ParallelLayout(mp, ep, esp, ep * esp, esp_contiguous=c)
           for ep, esp in itertools.product((1, 2, 4, 8), (1, 2, 4)) for mp in (1, 2, 4)
           for c in (True, False) if (ep * esp) % mp == 0]


@pytest.mark.parametrize("lay", LAYOUTS, ids=lambda l: f"mp{l.mp_size}ep{l.ep_size}esp{l.esp_size}"
                                                        f"{'c' if l.esp_contiguous else 'f'}")
def test_overlay_matches_oracle_and_partitions(lay):
    o = O.Layout(lay.mp_size, lay.ep_size, lay.esp_size, lay.world_size, lay.esp_contiguous)
    seen_pairs = set()
    for r in range(lay.world_size):
        assert (lay.ep_pos(r), lay.esp_pos(r), lay.mp_pos(r)) == (o.ep_pos(r), o.esp_pos(r), o.mp_pos(r))
        assert lay.rank_of(lay.ep_pos(r), lay.esp_pos(r)) == r
        seen_pairs.add((lay.ep_pos(r), lay.esp_pos(r)))
        for kind in ("mp", "ep", "esp", "ep_esp"):
            assert group_members(lay, kind, r) == o.group(kind, r)
            assert r in group_members(lay, kind, r)
    assert len(seen_pairs) == lay.world_size
    for kind in ("mp", "ep", "esp", "ep_esp"):
        grps = groups_of(lay, kind)
        flat = sorted(x for g in grps for x in g)
        assert flat == list(range(lay.world_size))
        assert len({len(g) for g in grps}) == 1


def test_layout_validation_messages():
    with pytest.raises(ValueError, match="must equal"):
        ParallelLayout(1, 2, 2, 8)
    with pytest.raises(ValueError, match="must divide"):
        ParallelLayout(3, 2, 2, 4)
    with pytest.raises(ValueError, match="out of range"):
        ParallelLayout(1, 2, 2, 4).ep_pos(4)
    with pytest.raises(ValueError, match="unknown group kind"):
        group_members(ParallelLayout(1, 2, 2, 4), "dp", 0)


def test_check_compatible_messages():
    lay = ParallelLayout(2, 2, 2, 4)
    check_compatible(cfg(), lay)
    with pytest.raises(ValueError, match="num_experts .* divisible by ep_size"):
        check_compatible(cfg(num_experts=3, top_k=1), lay)
    with pytest.raises(ValueError, match="hidden_dim .* divisible by esp_size"):
        check_compatible(cfg(hidden_dim=511), lay)
    with pytest.raises(ValueError, match="tokens per rank .* divisible by mp_size"):
        check_compatible(cfg(samples_per_rank=1, seq_len=7), lay)


def test_cluster_and_placement():
    with pytest.raises(ValueError):
        ClusterSpec(1, 4, 4e-9, 4e-10)          # beta_intra must be < beta_inter
    one = ClusterSpec(1, 8, 4e-10, 4e-9)
    assert classify_placement(one, ParallelLayout(2, 4, 2, 8)) is PlacementCase.SINGLE_NODE
    two = ClusterSpec(2, 4, 4e-10, 4e-9)
    assert two.node_of(3) == 0 and two.node_of(4) == 1
    assert two.link_class(0, 3) == "intra" and two.link_class(3, 4) == "inter"
    assert classify_placement(two, ParallelLayout(2, 2, 4, 8)) is PlacementCase.ESP_INTRA_NODE
    assert classify_placement(two, ParallelLayout(2, 4, 2, 8, esp_contiguous=False)) is PlacementCase.EP_INTRA_NODE
    assert classify_placement(ClusterSpec(4, 2, 4e-10, 4e-9), ParallelLayout(1, 1, 8, 8)) is PlacementCase.OTHER
    assert mp_groups_intra_node(two, ParallelLayout(4, 4, 2, 8))
    with pytest.raises(ValueError):
        classify_placement(one, ParallelLayout(1, 2, 2, 4))


FIG2 = """# fig2
B = 1
L = 8
M = 4
H = 4
E = 2
k = 1
f = 2.0
N_MP = 2
N_EP = 2
N_ESP = 2
num_nodes = 2
devices_per_node = 2
beta_intra = 4e-10
beta_inter = 4e-9
alpha_link = 0.0
seed = 7
"""


def test_config_parser_roundtrip(tmp_path):
    p = tmp_path / "fig2.cfg"
    p.write_text(FIG2)
    exp = load_config(p)
    assert exp.moe == MoEConfig(1, 8, 4, 4, 2, 1, 2.0)
    assert exp.layout == ParallelLayout(2, 2, 2, 4)
    assert exp.cluster.world_size == 4 and exp.seed == 7
    flipped = parse_config_text(FIG2 + "overlay = ep_contiguous\n")
    assert not flipped.layout.esp_contiguous


@pytest.mark.parametrize("text,match", [
    (FIG2.replace("B = 1\n", ""), "missing keys"),
    (FIG2 + "Q = 3\n", "unknown key"),
    (FIG2.replace("L = 8", "L = eight"), "bad value"),
    (FIG2 + "B = 2\n", "duplicate"),
    (FIG2 + "just words\n", "expected 'key = value'"),
    (FIG2 + "overlay = diagonal\n", "overlay must be"),
    (FIG2.replace("N_EP = 2", "N_EP = 3"), "must equal"),
])
def test_config_parser_errors(text, match):
    with pytest.raises(ConfigError, match=match):
        parse_config_text(text)
