"""Anchor the CPU arm (the oracle port, oracle/moe_oracle.py) to the real reference package.

    python tools/cpu_anchor.py        # build container only: imports moesched from /root/reference

bench.py's CPU legs time the NumPy oracle port, because /root/reference does not travel to the
GPU box.  This times the reference's own ``moesched.dataplane.reference_forward`` (the single-
device forward, dataplane.py:146-159) and the port's ``block_forward`` on the same inputs and
host, at the bench workload's per-rank shape (B*L = 8192, M = 1024, H = 4096, E = 8, top-2,
f = 1.2) and at the bench CPU sample (2048 tokens), and records the ratio in
profiles/cpu_anchor.json, which bench.py quotes next to its CPU numbers.
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

from moesched import config as CF  # noqa: E402
from moesched import dataplane as D  # noqa: E402

from oracle import moe_oracle as O  # noqa: E402


def best(fn, reps):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def main() -> None:
    try:
        from threadpoolctl import threadpool_info

        threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:  # pragma: no cover
        threads = os.cpu_count() or 1
    rows = []
    for n in (2048, 8192):
        cfg = CF.MoEConfig(n // 1024 if n >= 1024 else 1, 1024, 1024, 4096, 8, 2, 1.2)
        w = D.ExpertWeights.generate(cfg, seed=0)
        x = np.random.default_rng(1).normal(size=(cfg.tokens_per_rank, 1024))
        ow = O.Weights(w.gate, w.w1, w.w2)
        cap = CF.derive_capacity(cfg)
        t_ref = best(lambda: D.reference_forward(cfg, w, x), 2)
        t_port = best(lambda: O.block_forward(x, ow, 2, cap), 2)
        ref_out = D.reference_forward(cfg, w, x)
        port_out = O.block_forward(x, ow, 2, cap)[0]
        rows.append({"tokens": cfg.tokens_per_rank, "reference_forward_s": t_ref, "oracle_block_forward_s": t_port,
                     "port_over_reference_speed": t_ref / t_port,
                     "max_rel_error_port_vs_reference": float(np.abs(port_out - ref_out).max() /
                                                              max(1.0, np.abs(ref_out).max()))})
        print(json.dumps(rows[-1]), flush=True)
    out = {"host_threads": threads, "cpu_count": os.cpu_count(), "rows": rows,
           "what": "moesched.dataplane.reference_forward (the real reference, f64) vs oracle block_forward "
                   "(the port bench.py times) on the same inputs, forward only, best of 2, this build host"}
    (ROOT / "profiles" / "cpu_anchor.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
