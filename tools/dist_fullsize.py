"""Multi-GPU parity at the benchmark's full size (torchrun, P = 2 or 4, bench layouts).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/dist_fullsize.py

BASELINE config 2 per-rank shape (B*L = 8192, M = 1024, H = 4096, E = 8, top-2, f = 1.2) with the
bench layout, S1.  The whole-layer oracle is minutes of f64 NumPy at this size, so this checks:
each rank's slice routing bit-exact against the oracle gate with the S1 quota
(dataplane.py:305,319-320); and the NVLink peer transport (fused kernels) against the NCCL
transport (separate collectives) on the same inputs -- outputs, input gradients and expert weight
gradients bit for bit (same arithmetic, different data movement), the gate gradient (an MP
all-reduce in NCCL's order vs a fixed-order local sum) to 1e-5.  Rank 0 prints OK.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import moe_oracle as O  # noqa: E402
from paper_2407_00599_b200.config import MoEConfig, ParallelLayout, derive_capacity  # noqa: E402
from paper_2407_00599_b200.runtime import MoELayer  # noqa: E402
from paper_2407_00599_b200.world import NcclWorld, PeerWorld  # noqa: E402

LAYOUTS = {2: (2, 1, 2), 4: (2, 2, 2), 8: (2, 4, 2)}


def main() -> int:
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, P = dist.get_rank(), dist.get_world_size()
    mp, ep, esp = LAYOUTS[P]
    cfg = MoEConfig(8, 1024, 1024, 4096, 8, 2, 1.2)
    layout = ParallelLayout(mp, ep, esp, P)
    n, M = cfg.tokens_per_rank, cfg.embed_dim
    w = O.Weights.generate(M, cfg.hidden_dim, cfg.num_experts, seed=21)
    w = O.Weights(O.round_bf16(w.gate), O.round_bf16(w.w1), O.round_bf16(w.w2))
    rng = np.random.default_rng(22 + rank // mp)          # MP ranks share their group's tokens
    x = O.round_bf16(rng.normal(size=(n, M)))
    dout = O.round_bf16(rng.normal(size=(n, M)))
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev).to(torch.bfloat16)  # noqa
    res = {}
    failures = []
    for wk in ("nccl", "peer"):
        layer = MoELayer(cfg, layout, (PeerWorld if wk == "peer" else NcclWorld)(layout, dev))
        layer.load_weights(w)
        out = layer.forward("s1", {rank: t(x)})[rank].float().cpu().numpy()
        rt = layer.routing(rank)
        ei, si = rt.expert_idx.cpu().numpy(), rt.slot_idx.cpu().numpy()
        dx = layer.backward({rank: t(dout)})[rank].float().cpu().numpy()
        gr = {k: v.float().cpu().numpy() for k, v in layer.shard_grads(rank).items()}
        torch.cuda.synchronize()
        res[wk] = (out, ei, si, dx, gr)
    # S1 slice gate with quota ceil(T / N_MP), token offset of the MP position
    sl = n // mp
    m = layout.mp_pos(rank)
    quota = -(-derive_capacity(cfg) // mp)
    ref = O.gate(x[m * sl:(m + 1) * sl], w.gate, cfg.top_k, quota, token_offset=m * sl)
    for wk in ("nccl", "peer"):
        if not (np.array_equal(res[wk][1], ref.expert_index) and np.array_equal(res[wk][2], ref.slot_index)):
            failures.append(f"rank {rank} {wk}: slice routing differs from the oracle gate")
    a, b = res["nccl"], res["peer"]
    for name, i in (("out", 0), ("dx", 3)):
        if not np.array_equal(a[i], b[i]):
            failures.append(f"rank {rank}: {name} peer != nccl (max |diff| {np.abs(a[i] - b[i]).max():.3e})")
    for key in ("dw1", "dw2"):
        if not np.array_equal(a[4][key], b[4][key]):
            failures.append(f"rank {rank}: {key} peer != nccl (max |diff| {np.abs(a[4][key] - b[4][key]).max():.3e})")
    g_a, g_b = a[4]["dgate"], b[4]["dgate"]
    ge = np.linalg.norm(g_a - g_b) / max(np.linalg.norm(g_a), 1e-30)
    if ge > 1e-5:
        failures.append(f"rank {rank}: dgate peer vs nccl rel {ge:.3e}")
    if not np.isfinite(a[0]).all() or np.abs(a[0]).max() == 0:
        failures.append(f"rank {rank}: degenerate output")
    allf = [None] * P
    dist.all_gather_object(allf, failures)
    bad = [f for fs in allf for f in fs]
    if rank == 0:
        print("\n".join(bad) if bad else f"FULLSIZE OK (P={P}, layout MP={mp} EP={ep} ESP={esp}, S1, nccl == peer)")
    dist.barrier()
    torch.cuda.synchronize()
    sys.stdout.flush()
    os._exit(1 if bad else 0)


if __name__ == "__main__":
    sys.exit(main())
