"""Drop-in surface: every name of the reference's hot-path API exists with the same call shape,
host-only modules import without a GPU, and the data plane refuses to run without CUDA (no CPU
fallback) — CPU only.  Also checks bench.py's CPU reference arm contract."""

from __future__ import annotations

import inspect
import json
import subprocess
import sys
from pathlib import Path

import pytest
import torch

import paper_2407_00599_b200 as P

ROOT = Path(__file__).resolve().parents[1]

REFERENCE_HOT_PATH_API = [
    # dataplane.py
    "ExpertWeights", "GateOutput", "ScheduleResult", "SCHEDULES", "gate", "expert_shard_forward",
    "reference_forward", "run_schedule", "oracle_errors", "max_rel_error",
    # config.py
    "MoEConfig", "ParallelLayout", "ClusterSpec", "PlacementCase", "ConfigError", "ExperimentConfig",
    "derive_capacity", "check_compatible", "classify_placement", "group_members", "groups_of", "load_config",
    # collectives.py trace types
    "CommTrace", "TraceRecord",
    # costs.py
    "AlphaBeta", "CostProfile", "CostReport", "ProfileError", "FitError", "CsvFormatError", "cost_baseline",
    "cost_fused", "cost_s1", "cost_s2", "fit_alpha_beta", "fit_profile", "load_profile", "predict_collective",
    "select_schedule",
]


@pytest.mark.parametrize("name", REFERENCE_HOT_PATH_API)
def test_name_exists(name):
    assert getattr(P, name) is not None


def test_signatures_match_reference_shape():
    def params(f):
        return list(inspect.signature(f).parameters)

    assert params(P.gate) == ["tokens", "gate_weights", "k", "capacity", "token_offset"]
    assert params(P.run_schedule) == ["schedule", "cfg", "layout", "cluster", "weights", "inputs"]
    assert params(P.reference_forward) == ["cfg", "weights", "tokens"]
    assert params(P.expert_shard_forward) == ["rows", "w1_shard", "w2_shard"]
    assert params(P.select_schedule) == ["cfg", "layout", "profile", "alg1_literal"]
    assert P.SCHEDULES == ("baseline", "s1", "s2")


def test_expert_weights_generation_matches_reference_rng(golden):
    from oracle import moe_oracle as O

    cfg = P.MoEConfig(1, 8, 4, 4, 2, 1, 2.0)
    w = P.ExpertWeights.generate(cfg, seed=2024)
    o = O.Weights.generate(4, 4, 2, seed=2024)
    assert (w.gate == o.gate).all() and (w.w1 == o.w1).all() and (w.w2 == o.w2).all()
    assert (w.w1_shard(1, 1, 2) == o.shard(1, 1, 2)[0]).all()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_data_plane_refuses_cpu():
    import numpy as np

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.gate(np.ones((4, 8)), np.ones((8, 2)), k=1, capacity=4)
    from paper_2407_00599_b200 import kernels as K

    with pytest.raises(ValueError, match="CUDA tensor"):
        K.gate_fwd(torch.ones(4, 8, dtype=torch.bfloat16), torch.ones(2, 8, dtype=torch.bfloat16), 1,
                   torch.empty(4, 1, dtype=torch.int32), torch.empty(4, 1), None)


def test_bench_reference_arm_contract():
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["unit"] == "tokens/s" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
    assert "workload" in line["config"]
