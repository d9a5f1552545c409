"""Time the token-side kernels in isolation at the bench shape (CUDA events, warm and cold L2).

    python tools/probes/kbench.py [path/to/libparm_b200.so] [--n 8192 --M 1024 --E 8 --k 2]

Loads the given library build (default: the in-tree one) -- used to A/B kernel variants built
with different -D flags (tools/probes/build_variant.sh).
"""
import argparse
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2407_00599_b200 import _lib  # noqa: E402
from paper_2407_00599_b200 import kernels as K  # noqa: E402


def timeit(fn, reps=20, inner=20, flush=None):
    """Median over replays of a CUDA graph of `inner` back-to-back launches (no host gaps);
    with `flush`, an L2-sized memset precedes every launch and is timed separately and subtracted."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()

    def body():
        for _ in range(inner):
            if flush is not None:
                flush.zero_()
            fn()

    def graph_of(f):
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                f()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        return g

    def med(g):
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / inner)
        ts.sort()
        return ts[len(ts) // 2]

    t = med(graph_of(body))
    if flush is not None:
        t -= med(graph_of(lambda: [flush.zero_() for _ in range(inner)]))
    return t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("lib", nargs="?", default=None)
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--M", type=int, default=1024)
    ap.add_argument("--E", type=int, default=8)
    ap.add_argument("--k", type=int, default=2)
    ap.add_argument("--f", type=float, default=1.2)
    a = ap.parse_args()
    if a.lib:   # any build, also of another ABI version: type only the symbols it has
        import ctypes
        lib = ctypes.CDLL(a.lib)
        for name, (res, args) in _lib.SIGNATURES.items():
            fn = getattr(lib, name, None)
            if fn is not None:
                fn.restype, fn.argtypes = res, args
        _lib._lib = lib
    dev = torch.device("cuda", 0)
    n, M, E, k = a.n, a.M, a.E, a.k
    cap = -(-int(a.f * k * n) // E)
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(n, M, generator=g, device=dev).to(torch.bfloat16)
    wg = torch.randn(E, M, generator=g, device=dev).to(torch.bfloat16)
    ei = torch.empty(n, k, dtype=torch.int32, device=dev)
    cw = torch.empty(n, k, device=dev)
    pr = torch.empty(n, E, device=dev)
    si = torch.empty(n, k, dtype=torch.int32, device=dev)
    ss = torch.empty(E, cap, dtype=torch.int32, device=dev)
    fill = torch.empty(E, dtype=torch.int32, device=dev)
    counts = torch.empty((n + 7) // 8 * E, dtype=torch.int32, device=dev)
    out = torch.empty(E, cap, M, dtype=torch.bfloat16, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    gate = lambda: K.gate_fwd(x, wg, k, ei, cw, pr, counts)  # noqa: E731
    route = lambda: K.route_dispatch(x, ei, counts, cap, si, ss, fill, 0, out=out)  # noqa: E731
    gate()
    route()
    dl = torch.randn(n, E, generator=g, device=dev)
    dwg = torch.empty(E, M, device=dev)
    ws = torch.zeros(K.gate_wgrad_workspace(n, M, E) // 4, device=dev)
    wgrad = lambda: K.gate_wgrad(x, dl, dwg, ws)  # noqa: E731
    view = K.SlotView(out, e_local=E, stride_i=cap * M, stride_slo=M)
    y = torch.empty(n, M, dtype=torch.bfloat16, device=dev)
    comb = lambda: K.combine_fwd(view, ei, si, cw, y)  # noqa: E731
    dbwd = lambda: K.dispatch_bwd(view, ei, si, dl, wg, E, y)  # noqa: E731
    dy = torch.randn(n, M, generator=g, device=dev).to(torch.bfloat16)
    cbd = lambda: K.combine_bwd_dispatch(dy, view, ei, si, pr, cw, dl, 0, fill, out=out)  # noqa: E731
    for name, fn, alg in (("gate_fwd", gate, n * M * 2), ("route_dispatch", route, n * M * 2 * (1 + k)),
                          ("gate_wgrad", wgrad, n * M * 2), ("combine_fwd", comb, n * M * 2 * (1 + k)),
                          ("dispatch_bwd", dbwd, n * M * 2 * (1 + k)), ("combine_bwd_disp", cbd, n * M * 2 * (1 + 2 * k))):
        w = timeit(fn)
        c = timeit(fn, flush=flush)
        print(f"{name:16s} warm {w:7.2f} us  cold {c:7.2f} us   alg {alg / 1e6:6.1f} MB -> {alg / c / 1e3:7.1f} GB/s cold")


if __name__ == "__main__":
    main()
