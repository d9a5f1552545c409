"""B200-native Parm MoE-layer hot path (arXiv 2407.00599).

Drop-in for the reference simulator ``moesched``'s hot path: one MoE layer
under MP+EP+ESP with the baseline / S1 / S2 schedules and the Algorithm-1
selector, executed by hand-written sm_100a kernels (``libparm_b200.so``,
C ABI in ``include/parm_b200.h``) and NCCL over NVLink.

Host-only modules (config, trace, selector) import without a GPU; the data
plane (``api``, ``runtime``, ``kernels``) needs the CUDA library and raises
when it is missing — there is no CPU fallback.
"""

from .config import (
    ClusterSpec,
    ConfigError,
    ExperimentConfig,
    MoEConfig,
    ParallelLayout,
    PlacementCase,
    check_compatible,
    classify_placement,
    derive_capacity,
    group_members,
    groups_of,
    load_config,
    parse_config_text,
)
from .selector import (
    ALL_KEYS,
    AlphaBeta,
    CostProfile,
    CostReport,
    CsvFormatError,
    FitError,
    ProfileError,
    cost_baseline,
    cost_fused,
    cost_s1,
    cost_s2,
    fit_alpha_beta,
    fit_profile,
    load_profile,
    predict_collective,
    read_fit_samples,
    read_profile_csv,
    select_schedule,
    write_profile_csv,
)
from .trace import CommTrace, TraceRecord, schedule_ffn_rows, schedule_trace

SCHEDULES = ("baseline", "s1", "s2")

_DATA_PLANE = {
    "ExpertWeights", "GateOutput", "ScheduleResult", "gate", "expert_shard_forward", "reference_forward",
    "run_schedule", "max_rel_error", "oracle_errors",
}


def __getattr__(name):
    # The data plane loads torch + the CUDA library lazily so that host-only
    # users (selector sweeps, config parsing) never need a GPU.
    if name in _DATA_PLANE:
        from . import api

        return getattr(api, name)
    if name in ("MoELayer",):
        from .runtime import MoELayer

        return MoELayer
    if name in ("ParmMoE",):
        from .module import ParmMoE

        return ParmMoE
    raise AttributeError(name)
