#!/usr/bin/env python
"""Benchmark: Parm MoE-layer forward+backward on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl parm|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

A step = forward + backward of ONE MoE layer (gate -> dispatch -> expert FFN
-> combine and its adjoint, weight gradients included) over one batch of
synthetic tokens of the BASELINE config-2 per-rank shape (B=8 L=1024 M=1024
H=4096 E=8 top-2 f=1.2), weak-scaled over the measurement plan's layouts
(BASELINE.md §3): N=1 (MP,EP,ESP)=(1,1,1), N=2 (2,1,2), N=4 (2,2,2),
N=8 (2,4,2).  The headline schedule is the one the Algorithm-1 selector picks
with the calibrated NVLink profile (profiles/nvlink_profile.csv, else a
nominal NVLink profile); baseline/S1/S2 are all timed and reported.

value = distinct tokens processed by the whole job per second
      = (P / N_MP) * B * L / t_step,  t_step = max over ranks (CUDA events).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MoE layer fwd+bwd ms & tokens/s at 1/2/4/8 B200; speedup vs baseline sched"
C2 = dict(samples_per_rank=8, seq_len=1024, embed_dim=1024, hidden_dim=4096, num_experts=8, top_k=2,
          capacity_factor=1.2)
LAYOUTS = {1: (1, 1, 1), 2: (2, 1, 2), 4: (2, 2, 2), 8: (2, 4, 2)}   # (MP, EP, ESP)
CPU_SAMPLE_TOKENS = 2048


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("parm", "reference"), default="parm")
    ap.add_argument("--schedule", default="auto", help="auto (selector) | baseline | s1 | s2")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-compare", action="store_true", help="time only the headline schedule")
    ap.add_argument("--eager", action="store_true", help="launch kernels eagerly instead of replaying a CUDA graph")
    ap.add_argument("--transport", choices=("peer", "nccl"), default="peer",
                    help="N>1: S1/S2 over NVLink peer memory (fused kernels; default) or NCCL collectives")
    ap.add_argument("--no-api-e2e", action="store_true", help="skip the api.run_schedule (NumPy) e2e leg")
    return ap.parse_args()


def layout_for(n: int):
    from paper_2407_00599_b200.config import ParallelLayout

    if n not in LAYOUTS:
        raise SystemExit(f"--gpus must be one of {sorted(LAYOUTS)}")
    mp, ep, esp = LAYOUTS[n]
    return ParallelLayout(mp, ep, esp, n)


def tokens_per_step(cfg, layout) -> int:
    return layout.world_size // layout.mp_size * cfg.tokens_per_rank


# ---------------------------------------------------------------- reference (CPU) arm
def oracle_step_rate(cfg, layout, sample_tokens: int, reps: int, warmup: int = 0):
    """The reference algorithm (oracle port of moesched's data plane + restated
    backward) on the host cores: fwd+bwd of (P/MP) blocks of ``sample_tokens``
    tokens with the full M/H/E.  Returns (tokens/s, seconds per step, cores)."""
    import numpy as np

    from oracle import moe_oracle as O

    try:
        from threadpoolctl import threadpool_info

        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:  # pragma: no cover
        cores = os.cpu_count() or 1
    M, H, E, k, f = cfg.embed_dim, cfg.hidden_dim, cfg.num_experts, cfg.top_k, cfg.capacity_factor
    w = O.Weights.generate(M, H, E, seed=0)
    blocks = layout.world_size // layout.mp_size
    rng = np.random.default_rng(0)
    xs = [rng.normal(size=(sample_tokens, M)) for _ in range(blocks)]
    ds = [rng.normal(size=(sample_tokens, M)) for _ in range(blocks)]
    cap = O.derive_capacity(sample_tokens, E, k, f)

    def step():
        for x, d in zip(xs, ds):
            _, c = O.block_forward(x, w, k, cap)
            O.block_backward(c, w, d)

    for _ in range(warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(reps):
        step()
    dt = (time.perf_counter() - t0) / reps
    return blocks * sample_tokens / dt, dt, cores


def run_reference_arm(args, rank: int, world: int) -> None:
    from paper_2407_00599_b200.config import MoEConfig

    if rank != 0:
        return
    cfg = MoEConfig(**C2)
    layout = layout_for(args.gpus)
    rate, dt, cores = oracle_step_rate(cfg, layout, CPU_SAMPLE_TOKENS, max(1, args.steps), warmup=min(args.warmup, 1))
    sample = (f"{layout.world_size // layout.mp_size} block(s) x {CPU_SAMPLE_TOKENS} tokens (of "
              f"{cfg.tokens_per_rank}) per step, full M/H/E, f64 NumPy oracle fwd+bwd")
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(cfg, layout, "oracle"),
        "cpu_baseline": {"value": rate, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": sample,
                         "reference_anchor": reference_anchor()},
        "e2e": {"value": rate, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


def reference_anchor() -> dict | None:
    """profiles/cpu_anchor.json (tools/cpu_anchor.py, build container): the oracle port's forward
    timed beside the real reference's reference_forward on the same inputs and host."""
    try:
        a = json.loads((ROOT / "profiles" / "cpu_anchor.json").read_text())
    except (OSError, ValueError):
        return None
    return {"port_speed_over_reference": {str(r["tokens"]): round(r["port_over_reference_speed"], 3)
                                          for r in a["rows"]},
            "outputs_identical": all(r["max_rel_error_port_vs_reference"] == 0.0 for r in a["rows"]),
            "source": "profiles/cpu_anchor.json (moesched.reference_forward vs the port, same host, forward)"}


def config_block(cfg, layout, schedule) -> dict:
    return {
        "workload": "BASELINE config 2 per-rank shape: one MoE layer B=8 L=1024 M=1024 H=4096 E=8 top-2 f=1.2",
        "layout": f"MP={layout.mp_size} EP={layout.ep_size} ESP={layout.esp_size} P={layout.world_size}",
        "schedule": schedule,
        "global_batch_tokens": tokens_per_step(cfg, layout),
        "seq_len": cfg.seq_len,
        "parallelism": f"mp{layout.mp_size}-ep{layout.ep_size}-esp{layout.esp_size}",
        "l2": "per-step working set (weights + activations ~0.5 GB/rank) >> 126 MB L2; no explicit flush",
    }


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.samples: list[list[str]] = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for s in self.samples:
            try:
                sm.append(float(s[0]))
                mx.append(float(s[1]))
            except ValueError:
                continue
            for nm, v in zip(names, s[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [v for v in sm if v > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- GPU arm
def pick_schedule(cfg, layout, requested: str):
    from paper_2407_00599_b200 import selector

    if requested != "auto":
        return requested, None
    # the profile calibrated at this world size (paper_2407_00599_b200/calibrate.py), else the
    # another calibrated one (NVSwitch: per-pair bandwidth barely depends on P)
    cands = [ROOT / "profiles" / f"nvlink_profile_p{p}.csv" for p in (layout.world_size, 8, 4, 2)]
    cands = [c for c in cands if c.exists()]
    prof_path = cands[0] if cands else ROOT / "profiles" / "nvlink_profile.csv"
    if prof_path.exists():
        prof = selector.load_profile(prof_path)
        src = str(prof_path.relative_to(ROOT))
    else:
        prof = selector.CostProfile()
        beta = 2.0 / 700e9           # bf16 element over ~700 GB/s NVLink (nominal)
        for c, g in selector.ALL_KEYS:
            prof.add(selector.AlphaBeta(2e-5, beta, c, g))
        src = "nominal NVLink profile (alpha 20us, 700 GB/s)"
    rep = selector.select_schedule(cfg, layout, prof)
    return rep.chosen, {"profile": src, "t_s1_pred_ms": rep.t_s1 * 1e3, "t_s2_pred_ms": rep.t_s2 * 1e3,
                        "t_baseline_pred_ms": rep.t_baseline * 1e3}


def make_step(layer, schedule, xs, ds, use_graph: bool):
    """One fwd+bwd step: a replayed CUDA graph (default) or eager launches.
    Returns (step, outs, dxs): the layer's output / input-gradient buffers the step writes."""
    if use_graph:
        g = layer.capture_step(schedule, xs, ds)
        return g.replay, g.outs, g.dxs
    outs = layer.forward(schedule, xs)
    dxs = layer.backward(ds)
    return (lambda: (layer.forward(schedule, xs), layer.backward(ds))), outs, dxs


def time_steps(layer, schedule, xs, ds, steps, warmup, dist, dev, use_graph=True):
    import torch

    step = make_step(layer, schedule, xs, ds, use_graph)[0]
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ms = e0.elapsed_time(e1) / steps
    if dist is not None:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def bind_numa_local(dev) -> str | None:
    """Pin this process to the CPUs local to the GPU's PCIe root so pinned host
    buffers (allocated after this) sit on the GPU's NUMA node; returns the cpulist."""
    import torch

    p = torch.cuda.get_device_properties(dev)
    path = Path(f"/sys/bus/pci/devices/{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0/local_cpulist")
    try:
        spec = path.read_text().strip()
        cpus = set()
        for part in spec.split(","):
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
            return spec
    except (OSError, ValueError):
        pass
    return None


def h2d_bandwidth(host, dev) -> float:
    """GB/s of one pinned host -> device copy of `host` (CUDA events)."""
    import torch

    buf = torch.empty(host.shape, dtype=host.dtype, device=dev)
    buf.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        buf.copy_(host, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    return 5 * host.numel() * host.element_size() / (e0.elapsed_time(e1) / 1e3) / 1e9


def peaks_hbm() -> float:
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0                           # B200_PROFILING.md fallback


NVLINK_GBS = 770.0        # measured peer copy per direction per GPU (B200_PROFILING.md)


def layer_roofline(cfg, layout, schedule: str, ms: float, tc_peak: float, hbm_gbs: float) -> dict:
    """serialized-sum roofline of the whole layer step on one GPU,
    t_roof = FLOP_alg / tensor peak + wire bytes / NVLink + token-side HBM bytes / HBM,
    frac = t_roof / t_measured (Parm has no intra-layer pipelining)."""
    from paper_2407_00599_b200.trace import schedule_trace

    P, MP, ESP, k = layout.world_size, layout.mp_size, layout.esp_size, cfg.top_k
    n, M, H = cfg.tokens_per_rank, cfg.embed_dim, cfg.hidden_dim
    flops = (P // MP) * n * k * 12 * M * H / P                     # useful assignments, fwd 4MH + bwd 8MH
    wire = 0.0
    if P > 1:
        wire = 2 * 2 * sum(r.wire_per_rank for r in schedule_trace(schedule, cfg, layout).records)  # bf16, fwd+bwd
    ng = n // MP if schedule == "s1" else n                         # tokens this rank gates / combines
    row = M * 2
    hbm = ng * row * (1 + 2 * k + (k * ESP + 1) + (1 + k * ESP) + 2 * k + (k * ESP + 1) + 1)
    t_tc, t_nvl, t_hbm = flops / (tc_peak * 1e12), wire / (NVLINK_GBS * 1e9), hbm / (hbm_gbs * 1e9)
    t_roof = t_tc + t_nvl + t_hbm
    return {"t_roof_ms": t_roof * 1e3, "frac": t_roof * 1e3 / ms, "tensor_ms": t_tc * 1e3, "nvlink_ms": t_nvl * 1e3,
            "hbm_ms": t_hbm * 1e3, "flop_alg": flops, "wire_bytes": wire, "hbm_bytes": hbm,
            "peaks": {"tensor_tflops": tc_peak, "nvlink_gbs": NVLINK_GBS, "hbm_gbs": hbm_gbs},
            "note": "HBM bytes = token-side kernels (gate, dispatch x2, combine, combine-bwd, dispatch-bwd, gate wgrad)"}


def time_e2e(layer, schedule, host_x, host_d, steps, warmup, dist, dev, use_graph=True):
    """The step as a user runs it, a full round trip every step: the step's tokens and upstream
    gradient copied H2D from pinned host memory, forward + backward through the layer API,
    and the step's results -- the layer output and the input gradient -- copied back D2H into
    pinned host memory.  Copies are double-buffered on two copy streams (H2D of step i+1 and
    D2H of step i-1 overlap step i); each step's results are first snapshotted on the device
    (two D2D copies inside the timed region) so the next step may overwrite the layer's
    buffers.  S1 splits the MP group's tokens (paper §IV-C): a rank gates, dispatches and
    back-propagates only its slice, so only the slice's rows cross PCIe (the MP group as a
    whole moves every token once)."""
    import torch

    r = layer.ranks[0]
    lo, hi = 0, host_x.shape[0]
    if schedule == "s1" and layer.d.MP > 1:
        sl = layer.d.n // layer.d.MP
        lo = layer.layout.mp_pos(r) * sl
        hi = lo + sl
    M = host_x.shape[1]
    comp = torch.cuda.current_stream()
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    bx = [torch.empty(host_x.shape, dtype=torch.bfloat16, device=dev) for _ in range(2)]
    bd = [torch.empty(host_d.shape, dtype=torch.bfloat16, device=dev) for _ in range(2)]
    so = [torch.empty(hi - lo, M, dtype=torch.bfloat16, device=dev) for _ in range(2)]     # result snapshots
    sd = [torch.empty(hi - lo, M, dtype=torch.bfloat16, device=dev) for _ in range(2)]
    ho = [torch.empty(hi - lo, M, dtype=torch.bfloat16).pin_memory() for _ in range(2)]   # host results
    hdx = [torch.empty(hi - lo, M, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    back = [torch.cuda.Event() for _ in range(2)]
    for e in free + back:
        e.record(comp)
    fns = [make_step(layer, schedule, {r: bx[k]}, {r: bd[k]}, use_graph) for k in range(2)]
    copy_ev = []

    def prefetch(k):
        with torch.cuda.stream(h2d_s):
            h2d_s.wait_event(free[k])
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(h2d_s)
            bx[k][lo:hi].copy_(host_x[lo:hi], non_blocking=True)
            bd[k][lo:hi].copy_(host_d[lo:hi], non_blocking=True)
            c1.record(h2d_s)
            copy_ev.append((c0, c1))
            ready[k].record(h2d_s)

    def run(total):
        prefetch(0)
        for i in range(total):
            k = i % 2
            if i + 1 < total:
                prefetch((i + 1) % 2)
            comp.wait_event(ready[k])
            fn, outs, dxs = fns[k]
            fn()
            free[k].record(comp)
            comp.wait_event(back[k])                  # snapshot k's previous contents are on the host
            so[k].copy_(outs[r][lo:hi])
            sd[k].copy_(dxs[r][lo:hi])
            done[k].record(comp)
            with torch.cuda.stream(d2h_s):
                d2h_s.wait_event(done[k])
                ho[k].copy_(so[k], non_blocking=True)
                hdx[k].copy_(sd[k], non_blocking=True)
                back[k].record(d2h_s)
        comp.wait_stream(d2h_s)

    run(warmup)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    copy_ev.clear()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    h2d_s.wait_event(e0)
    run(steps)
    e1.record(comp)                                   # after the last step's results reached the host
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    time_e2e.h2d_ms = statistics.median(a.elapsed_time(b) for a, b in copy_ev)   # copy engine time per step
    time_e2e.result_check = (torch.equal(ho[(steps - 1) % 2], so[(steps - 1) % 2].cpu()) and
                             torch.equal(hdx[(steps - 1) % 2], sd[(steps - 1) % 2].cpu()))
    if dist is not None:
        dist.barrier()
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    h2d = 2 * (hi - lo) * M * 2
    d2h = 2 * (hi - lo) * M * 2
    return ms, h2d, d2h


def time_api_e2e(cfg, layout, rank, dist, calls: int = 3) -> dict:
    """The reference's own entry point: api.run_schedule (moesched dataplane.py:183), NumPy f64
    inputs (P/MP, B*L, M) in, NumPy f64 outputs (P, B*L, M) + trace + drop set out -- forward
    only, like the reference.  Wall clock per call (host API, synchronous), max over ranks."""
    import numpy as np
    import torch

    from paper_2407_00599_b200 import api
    from paper_2407_00599_b200.config import ClusterSpec

    w = api.ExpertWeights.generate(cfg, seed=0)
    inputs = np.random.default_rng(1).normal(size=(layout.world_size // layout.mp_size, cfg.tokens_per_rank,
                                                   cfg.embed_dim))
    cluster = ClusterSpec(1, layout.world_size, 4e-10, 4e-9)
    api.run_schedule("s1", cfg, layout, cluster, w, inputs)          # weights uploaded, buffers built
    samples = []
    for _ in range(calls):
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = api.run_schedule("s1", cfg, layout, cluster, w, inputs)
        samples.append(time.perf_counter() - t0)
    s = statistics.median(samples)
    if dist is not None:
        t = torch.tensor([s], device=torch.device("cuda", torch.cuda.current_device()), dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        s = float(t.item())
    tokens = layout.world_size // layout.mp_size * cfg.tokens_per_rank
    return {"value": tokens / s, "unit": "tokens/s (forward only)", "ms_per_call": s * 1e3,
            "h2d_bytes_per_call": int(inputs.nbytes), "d2h_bytes_per_call": int(res.outputs.nbytes),
            "api": "api.run_schedule('s1', ...) -- the reference's NumPy float64 boundary (dataplane.py:183), "
                   "forward only as in the reference; every rank returns all ranks' outputs"}


def gemm_roofline(layer, schedule, xs, ds, steps, dist, dev):
    """Average tcgen05 grouped-GEMM launch over `steps` steps, CUDA events on the launching stream."""
    import torch

    from paper_2407_00599_b200 import kernels as K

    K.gemm_timer = K.GemmTimer()
    try:
        # queue every launch behind a device-side sleep so the host is ahead of the GPU: the
        # per-GEMM event pairs then bracket back-to-back kernels, not host launch gaps
        torch.cuda.synchronize()
        torch.cuda._sleep(int(1.9e9 * 0.05))      # ~50 ms of spinning at 1.9 GHz
        for _ in range(steps):
            layer.forward(schedule, xs)
            layer.backward(ds)
        ms, launches, padded_flops = K.gemm_timer.total_ms()
    finally:
        K.gemm_timer = None
    d = layer.d
    r = layer.ranks[0]
    b = layer.st[r].bufs[schedule if d.P > 1 else "_local"]
    useful_rows = int((b["recv"].abs().amax(dim=-1) > 0).sum().item())   # real (kept) assignment rows
    alg_flops_step = 6 * 2 * useful_rows * d.M * d.Hs                   # 6 GEMMs per step (fwd 2, bwd 4)
    per_step = launches / steps                                         # 2 when fused (fwd pair, bwd four)
    per_launch_alg = alg_flops_step / per_step
    avg_ms = ms / launches
    return {"kernel": "moe_gemm_pair_kernel (tcgen05.mma.cta_group::2 kind::f16, TMA, TMEM; "
                      + ("forward pair and backward four as one persistent launch each)" if layer.fused_ffn
                         else "one launch per GEMM)"),
            "avg_launch_ms": avg_ms, "alg_flops_per_launch": per_launch_alg,
            "capacity_flops_per_launch": padded_flops / launches, "launches": launches,
            "launches_per_step": per_step, "useful_rows": useful_rows, "gemm_ms_per_step": ms / steps,
            "alg_flops_per_step": alg_flops_step}


def run_gpu_arm(args, rank: int, world: int, local_rank: int) -> None:
    import numpy as np
    import torch

    from paper_2407_00599_b200 import _lib
    from paper_2407_00599_b200.config import MoEConfig
    from paper_2407_00599_b200.runtime import MoELayer
    from paper_2407_00599_b200.world import LocalWorld, NcclWorld, PeerWorld

    dist = None
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        import torch.distributed as tdist

        tdist.init_process_group("nccl", device_id=dev)
        dist = tdist
    cfg = MoEConfig(**C2)
    layout = layout_for(args.gpus)
    if layout.world_size != world:
        raise SystemExit(f"--gpus {args.gpus} needs {args.gpus} ranks (got {world})")
    transport = "local"
    if world > 1:
        transport = "nccl"
        w = None
        if args.transport == "peer":
            try:
                w = PeerWorld(layout, dev)
                transport = "nvlink-peer (S1, S2) + nccl (baseline)"
            except Exception as exc:   # symmetric memory unavailable: NCCL for every exchange
                print(f"peer memory unavailable ({exc}); using NCCL", file=sys.stderr)
        if w is None:
            w = NcclWorld(layout, dev)
    else:
        w = LocalWorld(layout, dev)
    layer = MoELayer(cfg, layout, w)
    layer.init_random(seed=0)
    # like-for-like: the same schedules over NCCL collectives (same world, same communicators)
    layer_nccl = None
    if world > 1 and layer.peer and not args.no_compare:
        layer_nccl = MoELayer(cfg, layout, w, peer=False)
        layer_nccl.init_random(seed=0)
    g = torch.Generator(device=dev).manual_seed(1000 + rank // layout.mp_size)
    x = torch.randn(cfg.tokens_per_rank, cfg.embed_dim, generator=g, device=dev).to(torch.bfloat16)
    dout = torch.randn(cfg.tokens_per_rank, cfg.embed_dim, generator=g, device=dev).to(torch.bfloat16)
    xs, ds = {rank: x}, {rank: dout}

    schedule, sel = pick_schedule(cfg, layout, args.schedule)
    others = [] if args.no_compare or layout.world_size == 1 else [s for s in ("baseline", "s1", "s2")
                                                                     if s != schedule]
    sched_ms = {}
    clocks = ClockSampler(local_rank) if rank == 0 else None
    use_graph = not args.eager
    n0 = _lib.launch_count
    layer.forward(schedule, xs)
    layer.backward(ds)
    launches = (_lib.launch_count - n0) * args.steps          # our kernels per step x timed steps
    ms = time_steps(layer, schedule, xs, ds, args.steps, args.warmup, dist, dev, use_graph)
    sched_ms[schedule] = ms
    for s in others:
        sched_ms[s] = time_steps(layer, s, xs, ds, args.steps, args.warmup, dist, dev, use_graph)
    # the dominant kernel's roofline, inside the same clock record as the timed steps
    roof = gemm_roofline(layer, schedule, xs, ds, max(3, min(args.steps, 10)), dist, dev)
    clk = clocks.stop() if clocks else None
    sched_ms_nccl = {}
    if layer_nccl is not None:
        for s in ("baseline", "s1", "s2"):
            sched_ms_nccl[s] = time_steps(layer_nccl, s, xs, ds, args.steps, args.warmup, dist, dev, use_graph)
    api_e2e = None
    if not args.no_api_e2e:
        api_e2e = time_api_e2e(cfg, layout, rank, dist)
    e2e = None
    if not args.no_e2e:
        aff = os.sched_getaffinity(0)
        numa = bind_numa_local(dev)                 # host buffers on the GPU's NUMA node
        hx = x.cpu().pin_memory()
        hd = dout.cpu().pin_memory()
        os.sched_setaffinity(0, aff)
        h2d_gbs = h2d_bandwidth(hx, dev)
        # one untimed repetition first: the per-step H2D time falls over the first pass through the
        # pinned buffers (DMA address translation warm-up), 1.2 -> 0.8 ms on some boxes
        time_e2e(layer, schedule, hx, hd, args.steps, args.warmup, dist, dev, use_graph)
        reps = [time_e2e(layer, schedule, hx, hd, args.steps, args.warmup, dist, dev, use_graph) + (time_e2e.h2d_ms,)
                for _ in range(5)]
        e_ms, h2d, d2h, h2d_ms = sorted(reps)[2]                      # median of 5 repetitions
        tps = tokens_per_step(cfg, layout)
        e2e = {"value": tps / (e_ms / 1e3), "unit": "tokens/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
               "api": "MoELayer.forward/backward; every step: tokens + upstream gradient H2D from pinned host "
                      "memory, layer output + input gradient D2H into pinned host memory (double-buffered on "
                      "copy streams; S1: each rank moves its MP token slice)",
               "results_on_host_verified": bool(time_e2e.result_check),
               "h2d_gbs_measured": h2d_gbs, "host_numa_cpus": numa, "h2d_ms_per_step_in_loop": h2d_ms,
               "repetitions_ms": [r[0] for r in reps]}
        if api_e2e is not None:
            e2e["run_schedule"] = api_e2e
    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    burst = peaks.get("bf16_tflops")
    sustained = peaks.get("bf16_tflops_sustained")
    if burst is None or sustained is None:
        burst, sustained = 1590.0, 1590.0
        src = "fallback 1.59 PFLOP/s (B200_PROFILING.md)"
    # the burst figure applies when the clock record shows the SMs at (or within 3% of) max clock
    # during the timed steps and the GEMM timing; the sustained one when they ran clocked down
    at_max = bool(clk and clk.get("sm_mhz") and clk.get("sm_max_mhz") and clk["sm_mhz"] >= 0.97 * clk["sm_max_mhz"])
    if burst != sustained:
        peak = burst if at_max else sustained
        src = ("MEASURED_PEAKS.json bf16_tflops (burst): median SM clock at max during the measurement"
               if at_max else "MEASURED_PEAKS.json bf16_tflops_sustained: SM clock below max during the measurement")
    peak_src = src
    achieved = roof["alg_flops_per_launch"] / (roof["avg_launch_ms"] / 1e3) / 1e12
    traffic = None
    tfile = ROOT / "profiles" / "gemm_traffic.json"
    if tfile.exists():   # ncu dram bytes per launch of the same launch structure (fused or one per GEMM)
        tj = json.loads(tfile.read_text())
        traffic = tj.get("dram_bytes_per_launch_fused" if layer.fused_ffn else "dram_bytes_per_launch")
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "frac_burst": achieved / burst, "frac_sustained": achieved / sustained,
                "traffic": traffic, "peak_source": peak_src, "kernel": roof["kernel"],
                "avg_launch_ms": roof["avg_launch_ms"], "launches_sampled": roof["launches"],
                "alg_flops_per_launch": roof["alg_flops_per_launch"],
                "timing": "CUDA events around each GEMM launch on the launching stream, launches queued behind a "
                          "device sleep (no host gaps inside the intervals)",
                "gemm_share_of_step": roof["gemm_ms_per_step"] / ms,
                "launches_per_step": roof["launches_per_step"],
                "units": "alg FLOPs = 2 * kept assignment rows * M * (H/N_ESP) per GEMM; 6 GEMMs per step "
                         "in launches_per_step launches"}
    roofline["layer"] = layer_roofline(cfg, layout, schedule, ms, peak, peaks_hbm())
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        rate, dt, cores = oracle_step_rate(cfg, layout, CPU_SAMPLE_TOKENS, 3)
        cpu = {"value": rate, "unit": "tokens/s", "cores": cores, "kind": "port",
               "sample": f"{CPU_SAMPLE_TOKENS} of {cfg.tokens_per_rank} tokens, full M/H/E, f64 NumPy oracle "
                         f"fwd+bwd, 3 steps ({dt:.2f} s/step)", "reference_anchor": reference_anchor()}
    tps = tokens_per_step(cfg, layout)
    line = {
        "metric": METRIC, "value": tps / (ms / 1e3), "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (N(0,1) tokens, reference-scaled random weights)",
        "config": config_block(cfg, layout, schedule),
        "schedules_ms": sched_ms,
        "speedup_vs_baseline_schedule": (sched_ms["baseline"] / ms) if "baseline" in sched_ms and
                                        schedule != "baseline" else None,
        "schedules_ms_nccl": sched_ms_nccl or None,
        "speedup_vs_baseline_schedule_same_transport": (
            sched_ms_nccl["baseline"] / sched_ms_nccl[schedule]) if sched_ms_nccl and schedule != "baseline" else (
            sched_ms["baseline"] / ms if "baseline" in sched_ms and not layer.peer and schedule != "baseline"
            else None),
        "speedup_note": ("speedup_vs_baseline_schedule: the selected schedule on this run's transport vs the "
                         "baseline (DeepSpeed-MoE order, always on NCCL collectives); _same_transport: both on "
                         "NCCL collectives" if world > 1 else None),
        "selector": sel,
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
        "launch_mode": "eager" if args.eager else "cuda_graph (one replay per step; NCCL calls captured)",
        "transport": transport,
    }
    emit(line)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


_JSON_OUT = None


def emit(line: dict) -> None:
    """The one stdout line: the JSON result (written to the saved stdout; see main)."""
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    # stdout carries exactly one JSON line.  Everything else the process prints -- including
    # libraries writing straight to file descriptor 1, such as NCCL's "NCCL version ..." when
    # NCCL_DEBUG is set in the environment -- is sent to stderr: fd 1 is pointed at stderr for the
    # whole run and the result goes to a saved copy of the original stdout.
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    args = parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    run_gpu_arm(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
