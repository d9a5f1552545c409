"""Why is the weight-gradient GEMM slower than the row GEMMs?  Same FLOPs, two operand layouts.

    PARM_GEMM_DEBUG=<bits> python tools/wgrad_probe.py     (bits: 1 = no epilogue stores, 2 = no TMA loads)

  wgt    dW1[g] (H x M) = sum_r dH[g][r][h] X[g][r][m]   both operands MN-major (the layer's wgrad)
  row    the same product from pre-transposed copies dH^T (H x R), X^T (M x R): both K-major
"""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2407_00599_b200 import kernels as K  # noqa: E402

dev = "cuda"
G, R, M, H = 8, 2048, 1024, 4096
u = lambda t: t.unsqueeze(0).unsqueeze(0)  # noqa: E731
dh = torch.randn(G, R, H, device=dev).bfloat16()
x = torch.randn(G, R, M, device=dev).bfloat16()
dht, xt = dh.transpose(1, 2).contiguous(), x.transpose(1, 2).contiguous()
dw = torch.empty(G, H, M, device=dev)
dwb = torch.empty(G, H, M, device=dev, dtype=torch.bfloat16)
fl = 2 * G * R * M * H
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def bench(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


dbg = os.environ.get("PARM_GEMM_DEBUG", "0")
for name, fn in (("wgt  MN-major f32", lambda: K.gemm_wgrad(u(dh), u(x), dw)),
                 ("row  K-major  bf16", lambda: K.gemm_rows(u(dht), xt, K.KMAJOR, u(dwb), K.EPI_BF16)),
                 ("row  A K-major, B MN-major", lambda: K.gemm_rows(u(dht), x, K.MNMAJOR, u(dwb), K.EPI_BF16))):
    ms = bench(fn)
    print(f"debug={dbg} {name:28s} {ms * 1e3:8.1f} us  {fl / ms / 1e9:8.1f} TFLOP/s", flush=True)
if dbg == "0":
    K.gemm_wgrad(u(dh), u(x), dw)
    ref = torch.bmm(dht.float(), x.float())
    print("wgt max rel err", ((dw - ref).abs().max() / ref.abs().max()).item())
