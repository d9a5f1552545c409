"""Phase timeline of the tensor-core gate (variant build with -DPARM_GATE_TRACE): per CTA, the
%globaltimer at launch entry, after the Wg staging barrier, after the MMA loop, before and after
the ranking, and at the end of the tile (thread 0 only), relative to the earliest entry.

    bash tools/probes/build_variant.sh gtrace -DPARM_GATE_TRACE
    python tools/probes/gate_trace.py tools/probes/variants/gtrace.so
"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2407_00599_b200 import _lib  # noqa: E402
from paper_2407_00599_b200 import kernels as K  # noqa: E402


def main():
    lib = ctypes.CDLL(sys.argv[1])
    for name, (res, args) in _lib.SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is not None:
            fn.restype, fn.argtypes = res, args
    _lib._lib = lib
    dev = torch.device("cuda", 0)
    n, M, E, k = 8192, 1024, 8, 2
    x = torch.randn(n, M, device=dev).to(torch.bfloat16)
    wg = (torch.randn(E, M, device=dev) * 0.03).to(torch.bfloat16)
    ei = torch.empty(n, k, dtype=torch.int32, device=dev)
    cw = torch.empty(n, k, device=dev)
    pr = torch.empty(n, E, device=dev)
    counts = torch.empty((n + 7) // 8 * E, dtype=torch.int32, device=dev)
    for _ in range(5):   # (the trace's redo counters accumulate over these 5 + 1 launches)
        K.gate_fwd(x, wg, k, ei, cw, pr, counts)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    K.gate_fwd(x, wg, k, ei, cw, pr, counts)
    e1.record()
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (148 * 8))()
    assert lib.parm_debug_gate_trace(buf) == 0
    a = np.array(buf, dtype=np.float64).reshape(148, 8)
    t = a[:, :6]
    redo = a[t[:, 0] > 0, 6]
    redo_ns = a[t[:, 0] > 0, 7]
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    print(f"event time {e0.elapsed_time(e1) * 1e3:.1f} us, {len(t)} CTAs, {int(redo.sum() / 6)} tokens recomputed "
          f"exactly per launch (max {int(redo.max() / 6)} in one CTA); longest recompute+re-rank "
          f"{redo_ns.max() / 1e3:.2f} us")
    names = ["entry", "staged", "mma done", "partials summed", "ranked", "tile end"]
    for i, nm in enumerate(names):
        col = rel[:, i]
        print(f"{nm:16s} min {col.min():6.2f}  median {np.median(col):6.2f}  max {col.max():6.2f} us")


if __name__ == "__main__":
    main()
