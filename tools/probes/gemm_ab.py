"""Per-GEMM A/B of library builds at the bench shape (N=1 layout, E=8, 8192 tokens, top-2, f=1.2):
the six expert-FFN GEMMs each launched alone through parm_gemm (CUDA-graph replays, median), and
the fused multi-problem launches when the build has them.

    python tools/probes/gemm_ab.py lib_a.so [lib_b.so ...]     ("" = the in-tree build)
Older builds (other ABI versions) are loaded with only the symbols this probe needs.
"""
import ctypes
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools" / "probes"))
from kbench import timeit  # noqa: E402
from paper_2407_00599_b200 import _lib  # noqa: E402
from paper_2407_00599_b200 import kernels as K  # noqa: E402


def load_any(path):
    lib = ctypes.CDLL(path)
    for name, (res, args) in _lib.SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is not None:
            fn.restype, fn.argtypes = res, args
    return lib


def main():
    dev = torch.device("cuda", 0)
    E, q, M, H = 8, 2458, 1024, 4096
    bf = dict(dtype=torch.bfloat16, device=dev)
    g = torch.Generator(device=dev).manual_seed(0)
    fill = torch.full((1, 1, E), 2048, dtype=torch.int32, device=dev)
    R = (torch.randn(1, 1, E, q, M, generator=g, device=dev) * 0.5).to(torch.bfloat16)
    w1t = (torch.randn(E, H, M, generator=g, device=dev) * 0.03).to(torch.bfloat16)
    w2t = (torch.randn(E, M, H, generator=g, device=dev) * 0.03).to(torch.bfloat16)
    h = torch.empty(1, 1, E, q, H, **bf)
    mask = torch.zeros(1, 1, E, q, H // 32, dtype=torch.int32, device=dev)
    y = torch.empty(1, 1, E, q, M, **bf)
    dy = (torch.randn(1, 1, E, q, M, generator=g, device=dev) * 0.5).to(torch.bfloat16)
    dh = torch.empty(1, 1, E, q, H, **bf)
    dr = torch.empty(1, 1, E, q, M, **bf)
    dw1 = torch.empty(E, H, M, device=dev)
    dw2 = torch.empty(E, M, H, device=dev)
    fl = 2 * E * 2048 * M * H
    cases = [
        ("up   (ROW K=1024 relu-mask)", lambda: K.gemm_rows(R, w1t, K.KMAJOR, h, K.EPI_RELU_MASK, aux=mask, fill=fill)),
        ("down (ROW K=4096)", lambda: K.gemm_rows(h, w2t, K.KMAJOR, y, K.EPI_BF16, fill=fill)),
        ("dH   (ROW K=1024 MN-B mask)", lambda: K.gemm_rows(dy, w2t, K.MNMAJOR, dh, K.EPI_DMASK, aux=mask, fill=fill)),
        ("dW2  (WGT)", lambda: K.gemm_wgrad(dy, h, dw2, K.EPI_F32, fill=fill)),
        ("dR   (ROW K=4096 MN-B)", lambda: K.gemm_rows(dh, w1t, K.MNMAJOR, dr, K.EPI_BF16, fill=fill)),
        ("dW1  (WGT)", lambda: K.gemm_wgrad(dh, R, dw1, K.EPI_F32, fill=fill)),
    ]
    eager = "--eager" in sys.argv      # one eager launch each (for ncu --metrics gpu__time_duration at locked clocks)
    paths = [a for a in sys.argv[1:] if a != "--eager"] or [""]
    global timeit
    if eager:
        def timeit(fn, inner=1):   # noqa: F811
            fn()
            torch.cuda.synchronize()
            return 1.0
    for path in paths * (1 if eager else 2):   # interleaved twice (clocks drift under sustained GEMM load)
        _lib._lib = load_any(str(_lib.LIB_PATH) if not path else path)
        name = Path(path).name if path else "in-tree"
        tot = 0.0
        for label, fn in cases:
            t = timeit(fn, inner=10)
            tot += t
            print(f"{name:>14s} {label:30s} {t:7.1f} us  {fl / t / 1e6:6.0f} TF/s", flush=True)
        print(f"{name:>14s} {'sum of six':30s} {tot:7.1f} us  {6 * fl / tot / 1e6:6.0f} TF/s", flush=True)
        if hasattr(_lib._lib, "parm_gemm_multi"):
            ws = torch.zeros(4096, dtype=torch.int32, device=dev)
            fwd = [K.Gemm.row(R, w1t, K.KMAJOR, h, K.EPI_RELU_MASK, aux=mask, fill=fill),
                   K.Gemm.row(h, w2t, K.KMAJOR, y, K.EPI_BF16, fill=fill)]
            bwd = [K.Gemm.row(dy, w2t, K.MNMAJOR, dh, K.EPI_DMASK, aux=mask, fill=fill),
                   K.Gemm.wgrad(dy, h, dw2, K.EPI_F32, fill=fill),
                   K.Gemm.row(dh, w1t, K.MNMAJOR, dr, K.EPI_BF16, fill=fill),
                   K.Gemm.wgrad(dh, R, dw1, K.EPI_F32, fill=fill)]
            tf = timeit(lambda: K.gemm_multi(fwd, [None, (K.DEP_ROW_PAIR, 0)], ws), inner=10)
            tb = timeit(lambda: K.gemm_multi(bwd, [None, None, (K.DEP_ROW_PAIR, 0), (K.DEP_COL_BLOCK, 0)], ws),
                        inner=10)
            print(f"{name:>14s} {'fused fwd (up+down)':30s} {tf:7.1f} us  {2 * fl / tf / 1e6:6.0f} TF/s")
            print(f"{name:>14s} {'fused bwd (dH,dW2,dR,dW1)':30s} {tb:7.1f} us  {4 * fl / tb / 1e6:6.0f} TF/s")


if __name__ == "__main__":
    main()
