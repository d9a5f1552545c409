"""NVLink evidence for the fused peer-memory kernels, from ONE process driving all GPUs.

    python tools/probes/nvlink_probe.py                 # CUDA-event timing, achieved NVLink GB/s
    ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum \
        -k regex:"route_dispatch|moe_gemm_pair|combine_fwd|dispatch_bwd" python tools/probes/nvlink_probe.py

Rank 0 of the bench layout at N = device_count (2: MP=2 EP=1 ESP=2; 4: MP=2 EP=2 ESP=2) runs its
S1 peer kernels at the bench shape (B*L = 8192, M = 1024, H = 4096, E = 8, top-2, f = 1.2) with
the other ranks' receive buffers on the other GPUs (peer access enabled, so the device pointers
are NVLink-mapped exactly as torch symmetric memory maps them under torchrun):
  route_dispatch   token rows into the N_ESP holders' receive buffers (EP&ESP dispatch + dump)
  gemm_peer        the second expert GEMM storing each output tile into its owner (return A2A)
  combine_fwd      combine gathering expert outputs from the holders (the pull return) + MP fan-out
  dispatch_bwd     dispatch backward gathering dR rows from the holders + MP fan-out of dx
One process and no cross-GPU waits inside any kernel, so ncu can replay each kernel safely.
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_2407_00599_b200 import kernels as K  # noqa: E402
from paper_2407_00599_b200.config import MoEConfig, ParallelLayout, derive_capacity, group_members  # noqa: E402

LAYOUTS = {2: (2, 1, 2), 4: (2, 2, 2), 8: (2, 4, 2)}


def enable_peer_access(G: int) -> None:
    from cuda.bindings import runtime as rt

    for i in range(G):
        rt.cudaSetDevice(i)
        for j in range(G):
            if i != j:
                err, = rt.cudaDeviceEnablePeerAccess(j, 0)
                if int(err) not in (0, 704):      # 704: already enabled
                    raise RuntimeError(f"cudaDeviceEnablePeerAccess({i}->{j}) failed: {err}")
    rt.cudaSetDevice(0)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3          # us


def main() -> None:
    G = torch.cuda.device_count()
    if G not in LAYOUTS:
        raise SystemExit(f"needs 2, 4 or 8 GPUs (have {G})")
    enable_peer_access(G)
    mp, ep, esp = LAYOUTS[G]
    L = ParallelLayout(mp, ep, esp, G)
    cfg = MoEConfig(8, 1024, 1024, 4096, 8, 2, 1.2)
    n, M, H, E, k = cfg.tokens_per_rank, cfg.embed_dim, cfg.hidden_dim, cfg.num_experts, cfg.top_k
    el, Hs = E // ep, H // esp
    T = derive_capacity(cfg)
    q = math.ceil(T / mp)
    sl = n // mp
    devs = [torch.device("cuda", d) for d in range(G)]
    bf = torch.bfloat16
    torch.cuda.set_device(0)
    d0 = devs[0]
    r = 0
    # every rank's receive / expert-output / return / output buffers on its own GPU
    recv = [torch.zeros(G, 1, el, q, M, dtype=bf, device=d) for d in devs]
    fill_in = [torch.zeros(G, 1, el, dtype=torch.int32, device=d) for d in devs]
    ret = [torch.zeros(G, el, q, M, dtype=bf, device=d) for d in devs]
    yb = [torch.randn(G, 1, el, q, M, device=d).to(bf) for d in devs]
    outb = [torch.zeros(n, M, dtype=bf, device=d) for d in devs]
    # rank 0's routing of its token slice
    x = torch.randn(n, M, device=d0).to(bf)[r * sl:(r + 1) * sl]
    wg = torch.randn(E, M, device=d0).to(bf)
    ei = torch.empty(sl, k, dtype=torch.int32, device=d0)
    cw = torch.empty(sl, k, device=d0)
    pr = torch.empty(sl, E, device=d0)
    si = torch.empty(sl, k, dtype=torch.int32, device=d0)
    ss = torch.empty(E, q, dtype=torch.int32, device=d0)
    fill = torch.empty(E, dtype=torch.int32, device=d0)
    counts = torch.empty((sl + 7) // 8 * E, dtype=torch.int32, device=d0)
    K.gate_fwd(x, wg, k, ei, cw, pr, counts)
    pe, pp = (esp, 1) if L.esp_contiguous else (1, ep)
    off = 2 * r * el * q * M
    view = K.SlotView(None, e_local=el, n_p=esp, stride_i=q * M, stride_slo=M,
                      peers=tuple(t.data_ptr() + off for t in recv), peer_ep=pe, peer_p=pp)
    fan = [t.data_ptr() + 4 * r * el for t in fill_in]

    def dispatch():
        K.route_dispatch(x, ei, counts, q, si, ss, fill, 0, dst=view, slots_out=q, fill_fan=fan)

    dispatch()
    torch.cuda.synchronize()
    kept = int((si >= 0).sum())
    results = {"G": G, "layout": f"MP={mp} EP={ep} ESP={esp}", "rank": r}
    # dispatch: each kept pick stored to N_ESP holders; the ones on other GPUs cross NVLink
    remote_frac = (G - 1) / G       # (expert block, partial) holders other than rank 0, uniform routing
    t = timed(dispatch)
    byt = kept * esp * M * 2 * remote_frac
    results["route_dispatch"] = {"us": t, "remote_bytes": byt, "nvlink_gbs": byt / t / 1e3}
    # second expert GEMM with the return AlltoAll in its epilogue: holder 0's output tiles -> owners
    h = torch.randn(G, 1, el, q, Hs, device=d0).to(bf)
    w2t = (torch.randn(el, M, Hs, device=d0) / math.sqrt(H)).to(bf)
    y = torch.empty(G, 1, el, q, M, dtype=bf, device=d0)
    f_in = torch.full((G, 1, el), q, dtype=torch.int32, device=d0)
    seg = [t.data_ptr() + 2 * r * el * q * M for t in ret]

    def gemm_peer():
        K.gemm_rows(h, w2t, K.KMAJOR, y, K.EPI_BF16, fill=f_in, peer=(seg, q * M, M))

    t = timed(gemm_peer)
    byt = G * el * q * M * 2 * (G - 1) / G
    results["gemm_peer"] = {"us": t, "remote_bytes": byt, "nvlink_gbs": byt / t / 1e3,
                            "tflops": 2 * G * el * q * M * Hs / t / 1e6}
    # combine pulling expert outputs from the holders + fan-out of the slice to the MP peers
    yview = K.SlotView(None, e_local=el, n_p=esp, stride_i=q * M, stride_slo=M,
                       peers=tuple(t_.data_ptr() + off for t_ in yb), peer_ep=pe, peer_p=pp)
    mp_fan = [outb[m].data_ptr() + 2 * L.mp_pos(r) * sl * M for m in group_members(L, "mp", r)]

    def combine():
        K.combine_fwd_fan(yview, ei, si, cw, mp_fan, sl, M, M)

    t = timed(combine)
    remote_rows = kept * esp * remote_frac
    byt = remote_rows * M * 2 + sl * M * 2 * (mp - 1)
    results["combine_fwd_pull_fan"] = {"us": t, "remote_bytes": byt, "nvlink_gbs": byt / t / 1e3}
    dl = torch.randn(sl, E, device=d0)

    def dbwd():
        K.dispatch_bwd_fan(yview, ei, si, dl, wg, E, mp_fan, sl, M, M)

    t = timed(dbwd)
    results["dispatch_bwd_pull_fan"] = {"us": t, "remote_bytes": byt, "nvlink_gbs": byt / t / 1e3}
    results["reference_peak"] = "770 GB/s measured peer copy per direction per GPU (B200_PROFILING.md), 900 nominal"
    print(json.dumps(results), flush=True)


if __name__ == "__main__":
    main()
