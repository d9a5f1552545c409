"""GPU smoke/accuracy/throughput check of the tcgen05 grouped GEMM (all variants)."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2407_00599_b200 import kernels as K

torch.manual_seed(0)
dev = "cuda"

def ref(a, ma, b, mb):
    A = a.float() if ma == K.KMAJOR else a.float().transpose(1, 2)
    B = b.float() if mb == K.KMAJOR else b.float().transpose(1, 2)
    return torch.bmm(A, B.transpose(1, 2))

def check(G, M, N, Kd, ma, mb, epi):
    a = torch.randn(G, M, Kd, device=dev).bfloat16() if ma == K.KMAJOR else torch.randn(G, Kd, M, device=dev).bfloat16()
    b = torch.randn(G, N, Kd, device=dev).bfloat16() if mb == K.KMAJOR else torch.randn(G, Kd, N, device=dev).bfloat16()
    r = ref(a, ma, b, mb)
    aux = None
    if epi == K.EPI_DRELU:
        aux = torch.randn(G, M, N, device=dev).bfloat16()
    dt = torch.float32 if epi in (K.EPI_F32, K.EPI_F32_ACC) else torch.bfloat16
    d = torch.zeros(G, M, N, device=dev, dtype=dt)
    if epi == K.EPI_F32_ACC:
        d.fill_(1.0); r = r + 1.0
    K.grouped_gemm(a, ma, b, mb, d, epi, aux)
    torch.cuda.synchronize()
    if epi == K.EPI_RELU: r = r.clamp_min(0)
    if epi == K.EPI_DRELU: r = torch.where(aux.float() > 0, r, torch.zeros_like(r))
    err = (d.float() - r).abs().max().item() / max(1.0, r.abs().max().item())
    ok = err < 1e-2
    print(f"G={G} M={M} N={N} K={Kd} ma={ma} mb={mb} epi={epi}: rel_err={err:.3e} {'OK' if ok else 'FAIL'}", flush=True)
    return ok

def check_mask(G, M, N, Kd):
    """ReLU bit-mask epilogues: fwd writes relu(x w) + bits, bwd keeps dy w^T where the bit is set."""
    u = lambda t: t.unsqueeze(0).unsqueeze(0)
    x = torch.randn(G, M, Kd, device=dev).bfloat16(); w = torch.randn(G, N, Kd, device=dev).bfloat16()
    h = torch.empty(G, M, N, device=dev, dtype=torch.bfloat16)
    mask = torch.zeros(G, M, N // 32, device=dev, dtype=torch.int32)
    K.gemm_rows(u(x), w, K.KMAJOR, u(h), K.EPI_RELU_MASK, aux=u(mask))
    wb = torch.randn(G, N, Kd, device=dev).bfloat16()          # MN-major B for the masked GEMM: (G, K=Kd?, N)
    dy = torch.randn(G, M, Kd, device=dev).bfloat16()
    bm = torch.randn(G, Kd, N, device=dev).bfloat16()
    dh = torch.empty(G, M, N, device=dev, dtype=torch.bfloat16)
    K.gemm_rows(u(dy), bm, K.MNMAJOR, u(dh), K.EPI_DMASK, aux=u(mask))
    torch.cuda.synchronize()
    ref_h = torch.bmm(x.float(), w.float().transpose(1, 2)).clamp_min(0)
    bits = ((mask.unsqueeze(-1) >> torch.arange(32, device=dev)) & 1).reshape(G, M, N).bool()
    ok1 = torch.equal(bits, h.float() > 0)
    ref_dh = torch.where(h.float() > 0, torch.bmm(dy.float(), bm.float()), torch.zeros_like(ref_h))
    e1 = (h.float() - ref_h).abs().max().item() / max(1.0, ref_h.abs().max().item())
    e2 = (dh.float() - ref_dh).abs().max().item() / max(1.0, ref_dh.abs().max().item())
    ok = ok1 and e1 < 1e-2 and e2 < 1e-2
    print(f"mask G={G} M={M} N={N} K={Kd}: bits_exact={ok1} fwd={e1:.3e} bwd={e2:.3e} {'OK' if ok else 'FAIL'}", flush=True)
    return ok

allok = True
for (G, M, N, Kd) in [(1,128,64,64),(2,256,128,128),(3,512,512,320)]:
    allok &= check_mask(G, M, N, Kd)
for (ma, mb, epi) in [(0,0,1),(0,0,0),(0,1,2),(0,1,0),(1,1,3),(1,1,4)]:
    for (G, M, N, Kd) in [(1,128,64,64),(2,256,128,128),(2,384,256,192),(3,512,512,320)]:
        allok &= check(G, M, N, Kd, ma, mb, epi)
print("ALL_OK" if allok else "SOME_FAIL", flush=True)

# throughput at the C2 per-rank expert FFN shape
G, R, Mm, Hs = 2, 9856, 1024, 2048
x = torch.randn(G, R, Mm, device=dev).bfloat16()
w1t = torch.randn(G, Hs, Mm, device=dev).bfloat16()
h = torch.empty(G, R, Hs, device=dev, dtype=torch.bfloat16)
for _ in range(3): K.grouped_gemm(x, 0, w1t, 0, h, K.EPI_RELU)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): K.grouped_gemm(x, 0, w1t, 0, h, K.EPI_RELU)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
fl = 2 * G * R * Mm * Hs
print(f"fwd1 GEMM {G}x{R}x{Hs}x{Mm}: {ms*1e3:.1f} us  {fl/ms/1e9:.1f} TFLOP/s", flush=True)
xs = x.float()
e0.record()
for _ in range(20): torch.bmm(x, w1t.transpose(1,2))
e1.record(); torch.cuda.synchronize()
ms2 = e0.elapsed_time(e1) / 20
print(f"torch.bmm same shape: {ms2*1e3:.1f} us  {fl/ms2/1e9:.1f} TFLOP/s", flush=True)

# all six FFN GEMM shapes of the C2 P=1 step (8 experts, 2458 rows (+OOB tail), M=1024, H=4096), no fill skip
E_, R_, M_, H_ = 8, 2458, 1024, 4096
u = lambda t: t.unsqueeze(0).unsqueeze(0)
xr = torch.randn(E_, R_, M_, device=dev).bfloat16(); w1 = torch.randn(E_, H_, M_, device=dev).bfloat16()
w2 = torch.randn(E_, M_, H_, device=dev).bfloat16(); hh = torch.empty(E_, R_, H_, device=dev).bfloat16()
yy = torch.empty(E_, R_, M_, device=dev).bfloat16(); dw1 = torch.empty(E_, H_, M_, device=dev)
dw2 = torch.empty(E_, M_, H_, device=dev)
cases = {
    "fwd1 relu(X W1)": lambda: K.gemm_rows(u(xr), w1, K.KMAJOR, u(hh), K.EPI_RELU),
    "fwd2 H W2":       lambda: K.gemm_rows(u(hh), w2, K.KMAJOR, u(yy), K.EPI_BF16),
    "bwd dH (drelu)":  lambda: K.gemm_rows(u(yy), w2, K.MNMAJOR, u(hh), K.EPI_DRELU, aux=u(hh)),
    "bwd dR":          lambda: K.gemm_rows(u(hh), w1, K.MNMAJOR, u(yy), K.EPI_BF16),
    "wgrad dW2":       lambda: K.gemm_wgrad(u(yy), u(hh), dw2),
    "wgrad dW1":       lambda: K.gemm_wgrad(u(hh), u(xr), dw1),
}
fl = 2 * E_ * R_ * M_ * H_
for name, fn in cases.items():
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name:18s} {ms*1e3:8.1f} us  {fl/ms/1e9:8.1f} TFLOP/s", flush=True)
