"""The selector evaluation (tools/selector_sweep.py --analyze) on a synthetic sweep: the step model
recovers known coefficients, is scored out of sample, and the summary reports every key the
round-1 verdict asked for (trivial_agree, pred_vs_measured_err, per-schedule wins, the C6 guard)."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))

import selector_sweep as SW  # noqa: E402
from paper_2407_00599_b200 import selector as S  # noqa: E402


TRUTH = (2e-5, 1 / 1.4e15, 1 / 3e12, 0.6, 0.9, 0.0, 0.0, 1.0)   # const, gemm, tokens, a2a, ag, ar, overlap, peer


def _rows(truth=TRUTH):
    rows = []
    for i, (cfg, lay) in enumerate(SW.grid(4, "extended")):
        r = {"transport": "peer", "alg1_chosen": "s1"}
        for s in ("baseline", "s1", "s2"):
            c = 1e-5 * (1 + (i % 7)) * (2 if s == "s2" and cfg.top_k == 2 else 1)
            comm = {"a2a_seconds": c, "ag_seconds": 0.3 * c * (1 + i % 3), "peer_seconds": 0.5 * c * (i % 5)}
            f = S.step_features(cfg, lay, s, comm)
            t = sum(c * f[k] for c, k in zip(truth, S.STEP_FEATURES))
            r[f"t_{s}_ms"] = t * 1e3
            r[f"alg1_t_{s}_ms"] = c * 1e3
            for k, v in f.items():
                r[f"{s}.{k}"] = v
        r["measured_best"] = "s1" if r["t_s1_ms"] <= r["t_s2_ms"] else "s2"
        rows.append(r)
    return rows


def test_grid_extends_the_paper_grid():
    paper, ext = SW.grid(4, "paper"), SW.grid(4, "extended")
    assert len(paper) == 144 and len(ext) > len(paper)
    assert any(c.top_k == 1 and c.capacity_factor < 1.0 for c, _ in ext)


def test_step_model_fit_recovers_coefficients():
    truth = TRUTH
    rows = _rows(truth)
    samples = [(SW._feats(r, s), r[f"t_{s}_ms"] / 1e3) for r in rows for s in ("baseline", "s1", "s2")]
    m = S.fit_step_model(samples)
    np.testing.assert_allclose(m.coef, truth, rtol=1e-3, atol=1e-12)


def test_analysis_reports_the_verdict_keys():
    summ = SW.analyze(_rows())
    for key in ("trivial_agree", "alg1_agree", "model_agree", "pred_vs_measured_err", "wins",
                "c6_guard_each_wins_over_10pct"):
        assert key in summ
    assert summ["model_agree"] == 1.0 and summ["pred_vs_measured_err"]["model_mean"] < 1e-6
    assert summ["wins"]["s1"] + summ["wins"]["s2"] == summ["points"]
