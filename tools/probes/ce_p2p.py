"""Copy-engine peer copies over NVLink (one process, 2+ GPUs): GB/s alone and under a GEMM."""
import torch

n = torch.cuda.device_count()
assert n >= 2
for a in range(n):
    for b in range(n):
        if a != b:
            assert torch.cuda.can_device_access_peer(a, b)
MB = 1 << 20
sizes = [4 * MB, 16 * MB, 64 * MB]
src = [torch.randn(64 * MB // 2, device=f"cuda:{i}", dtype=torch.bfloat16) for i in range(2)]
dst = [torch.empty(64 * MB // 2, device=f"cuda:{i}", dtype=torch.bfloat16) for i in range(2)]
streams = [torch.cuda.Stream(device=f"cuda:{i}") for i in range(2)]


def bidir(nbytes, reps=20):
    el = nbytes // 2
    ev = []
    for i in range(2):
        with torch.cuda.device(i):
            torch.cuda.synchronize()
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for i in range(2):
        with torch.cuda.device(i), torch.cuda.stream(streams[i]):
            e0[i].record()
            for _ in range(reps):
                dst[1 - i][:el].copy_(src[i][:el], non_blocking=True)   # push i -> 1-i
            e1[i].record()
    for i in range(2):
        with torch.cuda.device(i):
            torch.cuda.synchronize()
    return max(e0[i].elapsed_time(e1[i]) for i in range(2)) / reps


for s in sizes:
    t = bidir(s)
    print(f"CE push both directions {s // MB} MB: {t * 1e3:.1f} us, {s / t / 1e6:.0f} GB/s per direction", flush=True)

# under a concurrent GEMM on each GPU
A = [torch.randn(8192, 8192, device=f"cuda:{i}", dtype=torch.bfloat16) for i in range(2)]
gs = [torch.cuda.Stream(device=f"cuda:{i}") for i in range(2)]


def gemm_time(with_copy):
    for i in range(2):
        with torch.cuda.device(i):
            torch.cuda.synchronize()
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    c0 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    c1 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for i in range(2):
        with torch.cuda.device(i):
            with torch.cuda.stream(gs[i]):
                e0[i].record()
                for _ in range(5):
                    torch.mm(A[i], A[i])
                e1[i].record()
            if with_copy:
                with torch.cuda.stream(streams[i]):
                    c0[i].record()
                    for _ in range(20):
                        dst[1 - i][: 16 * MB // 2].copy_(src[i][: 16 * MB // 2], non_blocking=True)
                    c1[i].record()
    for i in range(2):
        with torch.cuda.device(i):
            torch.cuda.synchronize()
    g = max(e0[i].elapsed_time(e1[i]) for i in range(2)) / 5
    c = max(c0[i].elapsed_time(c1[i]) for i in range(2)) / 20 if with_copy else 0
    return g, c


gemm_time(False)
g0, _ = gemm_time(False)
g1, c = gemm_time(True)
print(f"GEMM 8192^3 alone {g0 * 1e3:.0f} us; with CE copies alongside {g1 * 1e3:.0f} us; "
      f"copy 16 MB under GEMM {c * 1e3:.1f} us ({16 * MB / c / 1e6:.0f} GB/s)", flush=True)
