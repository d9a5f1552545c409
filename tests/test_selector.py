"""Cost model + Algorithm-1 selector: agree with the reference (golden reports on a sample of the
paper grid, fits) and with the paper's hand cases — CPU only."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2407_00599_b200 import selector as S
from paper_2407_00599_b200.config import MoEConfig, ParallelLayout


def _profile(vals: dict) -> S.CostProfile:
    p = S.CostProfile()
    for key, (a, b) in vals.items():
        c, g = key.split("/")
        p.add(S.AlphaBeta(a, b, c, g))
    return p


def test_reports_match_reference_golden(golden):
    meta, _ = golden
    prof = _profile(meta["costs"]["profile"])
    assert len(meta["costs"]["reports"]) > 30
    for rep in meta["costs"]["reports"]:
        cfg = MoEConfig(*rep["cfg"])
        lay = ParallelLayout(*rep["layout"])
        r = S.select_schedule(cfg, lay, prof)
        np.testing.assert_allclose([r.t_baseline, r.t_fused, r.t_s1, r.t_s2], rep["t"], rtol=1e-12)
        assert r.chosen == rep["chosen"]
        for k, v in rep["breakdown"].items():
            assert r.breakdown[k] == pytest.approx(v, rel=1e-12)
        lit = S.select_schedule(cfg, lay, prof, alg1_literal=True)
        np.testing.assert_allclose([lit.t_s1, lit.t_s2], rep["literal_t"], rtol=1e-12)
        assert lit.chosen == rep["literal_chosen"]


def test_fit_matches_reference(golden):
    meta, _ = golden
    for f in meta["costs"]["fits"]:
        ab = S.fit_alpha_beta([tuple(x) for x in f["samples"]])
        assert ab.alpha == pytest.approx(f["alpha"], rel=1e-9, abs=1e-15)
        assert ab.beta == pytest.approx(f["beta"], rel=1e-9)
        assert ab.r_squared == pytest.approx(f["r2"], rel=1e-9)
        assert ab.alpha_clamped == f["clamped"]


@pytest.mark.parametrize("alpha,beta", [(6.64e-4, 5.38e-10), (1.09e-4, 7.14e-10)])
def test_fit_recovers_paper_parameters(alpha, beta):
    xs = np.geomspace(2 ** 10, 2 ** 24, 24)
    ab = S.fit_alpha_beta([(x, alpha + beta * x) for x in xs])
    assert ab.alpha == pytest.approx(alpha, rel=1e-6) and ab.beta == pytest.approx(beta, rel=1e-6)


def test_fit_errors_and_clamp():
    with pytest.raises(S.FitError):
        S.fit_alpha_beta([(1.0, 1.0)])
    with pytest.raises(S.FitError):
        S.fit_alpha_beta([(5.0, 1.0), (5.0, 2.0)])
    with pytest.raises(S.FitError):
        S.fit_alpha_beta([(1.0, 2.0), (2.0, 1.0)])
    ab = S.fit_alpha_beta([(10.0, 0.5), (20.0, 2.0), (30.0, 3.5)])
    assert ab.alpha == 0.0 and ab.alpha_clamped


def _unit(alpha=0.0, beta=1.0, **over):
    p = S.CostProfile()
    for c, g in S.ALL_KEYS:
        a, b = over.get(f"{c}/{g}", (alpha, beta))
        p.add(S.AlphaBeta(a, b, c, g))
    return p


def test_selector_hand_cases():
    # tokens volume dominates -> the slot split (S2) wins; slots dominate -> S1 wins; ties -> S1.
    cfg_big_tokens = MoEConfig(1, 1000, 1, 4, 10, 1, 0.01)     # T = 1: slot volume tiny
    lay = ParallelLayout(2, 1, 2, 2)
    r = S.select_schedule(cfg_big_tokens, lay, _unit())
    assert r.t_s1 > r.t_s2 and r.chosen == "s2"
    cfg_big_slots = MoEConfig(1, 2, 1, 4, 10, 1, 50.0)         # T = 10 per expert: slots dominate
    r = S.select_schedule(cfg_big_slots, lay, _unit())
    assert r.t_s1 < r.t_s2 and r.chosen == "s1"
    r = S.select_schedule(cfg_big_slots, ParallelLayout(1, 1, 2, 2), _unit())
    assert r.t_s1 == r.t_s2 and r.chosen == "s1"                 # MP = 1: both are the fused schedule


@pytest.mark.parametrize("scale", [1e-3, 1.0, 1e6])
def test_choice_invariant_under_uniform_scaling(scale):
    cfg = MoEConfig(2, 64, 8, 16, 4, 2, 1.2)
    lay = ParallelLayout(2, 2, 2, 4)
    base = _unit(1e-5, 1e-9)
    scaled = _unit(1e-5 * scale, 1e-9 * scale)
    assert S.select_schedule(cfg, lay, base).chosen == S.select_schedule(cfg, lay, scaled).chosen


def test_missing_profile_entries():
    p = _unit()
    del p.entries[("allreduce", "esp")]
    with pytest.raises(S.ProfileError, match="allreduce/esp"):
        S.select_schedule(MoEConfig(2, 64, 8, 16, 4, 2, 1.2), ParallelLayout(2, 2, 2, 4), p)


def test_selector_is_argmin_on_random_profiles():
    rng = np.random.default_rng(600)
    for _ in range(2000):
        p = S.CostProfile()
        for c, g in S.ALL_KEYS:
            p.add(S.AlphaBeta(float(rng.uniform(0, 1e-4)), float(rng.uniform(1e-11, 1e-8)), c, g))
        esp = int(rng.choice([1, 2, 4]))
        ep = int(rng.choice([1, 2, 4, 8]))
        mp = int(rng.choice([m for m in (1, 2, 4) if (ep * esp) % m == 0]))
        cfg = MoEConfig(2, 64, 8, 8 * esp, max(2, ep), 2, float(rng.choice([1.0, 1.2, 2.4])))
        r = S.select_schedule(cfg, ParallelLayout(mp, ep, esp, ep * esp), p)
        assert r.chosen == ("s1" if r.t_s1 <= r.t_s2 else "s2")


def test_csv_round_trip_and_errors():
    samples = "collective,group,elements,seconds\n" + "".join(
        f"{c},{g},{x},{1e-5 + 1e-9 * x:.15g}\n" for c, g in S.ALL_KEYS for x in (1024, 65536, 1048576))
    prof = S.fit_profile(S.read_fit_samples(samples))
    again = S.read_profile_csv(S.write_profile_csv(prof))
    assert set(again.entries) == set(S.ALL_KEYS)
    for k in S.ALL_KEYS:
        assert again.entries[k].beta == pytest.approx(prof.entries[k].beta, rel=1e-11)
    with pytest.raises(S.CsvFormatError, match="line 1"):
        S.read_fit_samples("a,b,c,d\n")
    with pytest.raises(S.CsvFormatError, match="line 2"):
        S.read_fit_samples("collective,group,elements,seconds\nallgather,mp,xx,1\n")
    with pytest.raises(S.CsvFormatError, match="empty"):
        S.read_profile_csv("")
