// Bulk-copy ring variants of the token-side gathers (included by permute.cu).
//
// The register gathers in permute.cu keep one token (or four slot rows) of
// loads in flight per warp, so every warp pays one HBM round trip per token
// and the short kernels ran at 1-3 TB/s.  (Measured in the N=1 step:
// dispatch_bwd 30.9 -> 26.3 us, combine_fwd 15.9 -> 14.3, dispatch 14.6 ->
// 13.9; combine_bwd, with a third row per stage and two CTAs per SM, was
// slower as a ring, 12.8 -> 14.9 us, and keeps the register kernel.  What is
// left is mostly launch ramp and tail: ncu shows the SMs active for ~60% of
// these 14-26 us kernels.)  Here each warp owns a ring of
// kStages shared-memory stages; lane 0 streams row chunks (512 columns =
// 1 KB) into them with cp.async.bulk (the TMA bulk engine, completion on a
// per-stage mbarrier) kStages-1 items ahead of the consumer, so a warp keeps
// several KB in flight without holding them in registers.  The routing of a
// warp's tokens is fetched once, one token per lane, and broadcast with
// shuffles.  Arithmetic, order of accumulation and outputs are those of the
// register kernels; every row must be 16-byte aligned (local or peer views) --
// otherwise the host launches the register kernels.
// (Measured against an 8-token-group variant that issued one bulk copy per
// (token, pick) lane: bulk-copy operands must be warp-uniform, so per-lane
// copies serialise in a waterfall loop -- 22 vs 14 us for combine_fwd.)
#pragma once

namespace ring {

constexpr int kCols = 512;                 // columns per row chunk (1 KB of bf16)
constexpr int kWarps = kRowThreads / 32;   // warps per CTA

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bar_init(uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void bar_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "RING_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra RING_WAIT;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

__device__ __forceinline__ void init_bars(uint32_t bar0, int stages, int lane) {
    if (lane == 0) {
        for (int s = 0; s < stages; ++s) bar_init(bar0 + 8 * s);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
}

// The stage about to be refilled was read through the generic proxy; order
// those reads before the bulk engine's writes.
__device__ __forceinline__ void proxy_fence() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ int4 lds16(const bf16* p) { return *reinterpret_cast<const int4*>(p); }

__device__ __forceinline__ long long shfl_ll(long long v, int src) {
    int lo = __shfl_sync(0xffffffffu, (int)(v & 0xffffffffll), src);
    int hi = __shfl_sync(0xffffffffu, (int)(v >> 32), src);
    return ((long long)hi << 32) | (unsigned int)lo;
}

template <int KT>
struct PickB {   // one token's picks, broadcast from the lane that fetched them
    int sl[KT];
    int ex[KT];
    int ep[KT];
    long long off[KT];
    float w[KT];
};

template <int KT>
__device__ __forceinline__ PickB<KT> bcast(const Picks<KT>& mine, int i) {
    PickB<KT> b;
#pragma unroll
    for (int j = 0; j < KT; ++j) {
        b.sl[j] = __shfl_sync(0xffffffffu, mine.sl[j], i);
        b.ex[j] = __shfl_sync(0xffffffffu, mine.ex[j], i);
        b.ep[j] = __shfl_sync(0xffffffffu, mine.ep[j], i);
        b.off[j] = shfl_ll(mine.off[j], i);
        b.w[j] = __shfl_sync(0xffffffffu, mine.w[j], i);
    }
    return b;
}

__device__ __forceinline__ void invalidate(Picks<2>& p) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        p.sl[j] = -1;
        p.ex[j] = 0;
        p.ep[j] = 0;
        p.off[j] = 0;
        p.w[j] = 0.0f;
    }
}

// Shared-memory footprint of a ring kernel: kWarps x stages x rows x kCols
// bf16, plus per-stage extra bytes, plus the barriers.
__host__ __device__ constexpr int ring_smem(int stages, int rows, int extra) {
    return kWarps * stages * (rows * kCols * 2 + extra) + kWarps * stages * 8;
}

// ---------------------------------------------------------------- combine forward
// out[t, c] = sum_p sum_j w_j Y_p[e_j, s_j, c]   (k <= 2; rows = 2 * NP)
template <int NP, int S>
__global__ void __launch_bounds__(kRowThreads, 3) combine_fwd_ring(const __grid_constant__ SlotView y,
                                                                const int* __restrict__ expert_idx,
                                                                const int* __restrict__ slot_idx,
                                                                const float* __restrict__ combine_w, int n, int k,
                                                                int M, const __grid_constant__ RowFan out,
                                                                long long ldo) {
        constexpr int KT = 2, R = KT * NP, STAGE = R * kCols;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    bf16* ring = reinterpret_cast<bf16*>(smem) + (size_t)warp * S * STAGE;
    const uint32_t bar0 = saddr(smem + (size_t)kWarps * S * STAGE * 2) + warp * S * 8;
    init_bars(bar0, S, lane);
    const long long wg = (long long)blockIdx.x * kWarps + warp, nw = (long long)gridDim.x * kWarps;
    const int nch = (M + kCols - 1) / kCols;
    uint32_t phase_base = 0;   // items completed so far on this warp's ring (parity bookkeeping)
    for (long long base = wg; base < n; base += 32 * nw) {
        const long long left = (n - 1 - base) / nw + 1;
        const int ntok = left < 32 ? (int)left : 32;
        Picks<KT> mine;
        if (lane < ntok)
            mine.load(base + lane * nw, k, slot_idx, expert_idx, combine_w, y);
        else
            invalidate(mine);
        const int items = ntok * nch;
        auto issue = [&](int q) {
            const int i = q / nch, c0 = (q - i * nch) * kCols;
            const int cols = min(kCols, M - c0);
            const uint32_t qs = phase_base + q, st = qs % S;
            const PickB<KT> b = bcast(mine, i);
            uint32_t bytes = 0;
#pragma unroll
            for (int j = 0; j < KT; ++j) bytes += b.sl[j] >= 0 ? NP * cols * 2 : 0;
            if (lane == 0) {
                proxy_fence();
                bar_expect(bar0 + 8 * st, bytes);
#pragma unroll
                for (int j = 0; j < KT; ++j)
                    if (b.sl[j] >= 0)
#pragma unroll
                        for (int p = 0; p < NP; ++p)
                            bulk_g2s(saddr(ring + st * STAGE + (j * NP + p) * kCols),
                                     slot_base(y, b.ep[j], p) + b.off[j] + c0, cols * 2, bar0 + 8 * st);
            }
        };
        const int pre = items < S - 1 ? items : S - 1;
        for (int q = 0; q < pre; ++q) issue(q);
        for (int q = 0; q < items; ++q) {
            if (q + S - 1 < items) issue(q + S - 1);
            const int i = q / nch, c0 = (q - i * nch) * kCols;
            const int cols = min(kCols, M - c0);
            const uint32_t qs = phase_base + q, st = qs % S;
            const PickB<KT> b = bcast(mine, i);
            bar_wait(bar0 + 8 * st, (qs / S) & 1);
            const bf16* sb = ring + st * STAGE;
            float acc[2][8];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int u = 0; u < 8; ++u) acc[h][u] = 0.0f;
#pragma unroll
            for (int p = 0; p < NP; ++p)
#pragma unroll
                for (int j = 0; j < KT; ++j) {   // j ascending, like the reference's _combine
                    if (b.sl[j] < 0) continue;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int c = lane * 8 + h * 256;
                        if (c < cols) fma2_bf16x8(acc[h], b.w[j], lds16(sb + (j * NP + p) * kCols + c));
                    }
                }
            const long long t = base + i * nw;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = lane * 8 + h * 256;
                if (c >= cols) continue;
                const Vec8 v8 = f32_to_vec8(acc[h]);
                for (int f = 0; f < out.n; ++f) st_vec8(out.ptr[f] + t * ldo + c0 + c, v8);
            }
            __syncwarp();
        }
        phase_base += items;
    }
}

// ---------------------------------------------------------------- dispatch backward
// dx[t] = sum_j sum_p dR_p[e_j, s_j] + dlogits[t] . Wg^T  (E <= 32, E % 4 == 0:
// the token's logit gradients ride in each stage as E floats).
template <int NP, int S>
__global__ void __launch_bounds__(kRowThreads, 3) dispatch_bwd_ring(const __grid_constant__ SlotView dr,
                                                                 const int* __restrict__ expert_idx,
                                                                 const int* __restrict__ slot_idx,
                                                                 const float* __restrict__ dlogits,
                                                                 const bf16* __restrict__ wgT, int n, int k, int E,
                                                                 int M, const __grid_constant__ RowFan dx,
                                                                 long long ldx) {
        constexpr int KT = 2, R = KT * NP, STAGE = R * kCols + 64;   // + 32 f32 of logit gradients (as bf16 units)
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    bf16* ring = reinterpret_cast<bf16*>(smem) + (size_t)warp * S * STAGE;
    const uint32_t bar0 = saddr(smem + (size_t)kWarps * S * STAGE * 2) + warp * S * 8;
    init_bars(bar0, S, lane);
    const long long wg = (long long)blockIdx.x * kWarps + warp, nw = (long long)gridDim.x * kWarps;
    const int nch = (M + kCols - 1) / kCols;
    const bool gate = dlogits != nullptr;
    uint32_t phase_base = 0;
    for (long long base = wg; base < n; base += 32 * nw) {
        const long long left = (n - 1 - base) / nw + 1;
        const int ntok = left < 32 ? (int)left : 32;
        Picks<KT> mine;
        if (lane < ntok)
            mine.load(base + lane * nw, k, slot_idx, expert_idx, nullptr, dr);
        else
            invalidate(mine);
        const int items = ntok * nch;
        auto issue = [&](int q) {
            const int i = q / nch, c0 = (q - i * nch) * kCols;
            const int cols = min(kCols, M - c0);
            const uint32_t qs = phase_base + q, st = qs % S;
            const PickB<KT> b = bcast(mine, i);
            uint32_t bytes = gate ? E * 4 : 0;
#pragma unroll
            for (int j = 0; j < KT; ++j) bytes += b.sl[j] >= 0 ? NP * cols * 2 : 0;
            if (lane == 0) {
                proxy_fence();
                bar_expect(bar0 + 8 * st, bytes);
                bf16* sb = ring + st * STAGE;
                if (gate) bulk_g2s(saddr(sb + R * kCols), dlogits + (base + i * nw) * E, E * 4, bar0 + 8 * st);
#pragma unroll
                for (int j = 0; j < KT; ++j)
                    if (b.sl[j] >= 0)
#pragma unroll
                        for (int p = 0; p < NP; ++p)
                            bulk_g2s(saddr(sb + (j * NP + p) * kCols), slot_base(dr, b.ep[j], p) + b.off[j] + c0,
                                     cols * 2, bar0 + 8 * st);
            }
        };
        const int pre = items < S - 1 ? items : S - 1;
        for (int q = 0; q < pre; ++q) issue(q);
        for (int q = 0; q < items; ++q) {
            if (q + S - 1 < items) issue(q + S - 1);
            const int i = q / nch, c0 = (q - i * nch) * kCols;
            const int cols = min(kCols, M - c0);
            const uint32_t qs = phase_base + q, st = qs % S;
            const PickB<KT> b = bcast(mine, i);
            bar_wait(bar0 + 8 * st, (qs / S) & 1);
            const bf16* sb = ring + st * STAGE;
            float acc[2][8];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int u = 0; u < 8; ++u) acc[h][u] = 0.0f;
#pragma unroll
            for (int p = 0; p < NP; ++p)
#pragma unroll
                for (int j = 0; j < KT; ++j) {
                    if (b.sl[j] < 0) continue;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int c = lane * 8 + h * 256;
                        if (c < cols) add_bf16x8(acc[h], lds16(sb + (j * NP + p) * kCols + c));
                    }
                }
            if (gate) {
                const float* dl = reinterpret_cast<const float*>(sb + R * kCols);
#pragma unroll 4
                for (int e = 0; e < E; ++e) {
                    const float d = dl[e];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int c = lane * 8 + h * 256;
                        if (c < cols) fma2_bf16x8(acc[h], d, ldg16(wgT + (long long)e * M + c0 + c));
                    }
                }
            }
            const long long t = base + i * nw;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = lane * 8 + h * 256;
                if (c >= cols) continue;
                const Vec8 v8 = f32_to_vec8(acc[h]);
                for (int f = 0; f < dx.n; ++f) st_vec8(dx.ptr[f] + t * ldx + c0 + c, v8);
            }
            __syncwarp();
        }
        phase_base += items;
    }
}

// ---------------------------------------------------------------- host side
// Every row 16-byte aligned.  Peer views qualify too: cp.async.bulk reads a peer GPU's
// NVLink-mapped memory like local HBM (tools/probes/peer_bulk_probe.cu: scattered 1 KB rows from
// the peer at 705 GB/s, byte-exact), so the pulls of the peer transport stream through the ring.
inline bool view_aligned(const SlotView& v) {
    if (v.stride_i % 8 != 0 || v.stride_shi % 8 != 0 || v.stride_slo % 8 != 0) return false;
    if (v.n_peer != 0) {
        for (int i = 0; i < v.n_peer; ++i)
            if (reinterpret_cast<uintptr_t>(v.peer[i]) & 15) return false;
        return true;
    }
    return v.stride_ep % 8 == 0 && v.stride_p % 8 == 0 && (reinterpret_cast<uintptr_t>(v.ptr) & 15) == 0;
}

// Grid of a ring kernel: as many CTAs as fit on the SMs (by shared memory),
// never more than one warp per unit.  per_sm caches the occupancy per kernel.
template <typename K>
inline int grid_for(K kernel, int smem, long long units, int& per_sm) {
    if (per_sm <= 0) {
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kRowThreads, smem);
        per_sm = b < 1 ? 1 : b;
    }
    long long g = (units + kWarps - 1) / kWarps;
    const long long cap = (long long)kNumSMs * per_sm;
    if (g > cap) g = cap;
    return (int)(g < 1 ? 1 : g);
}

inline bool fan_aligned(const RowFan& f, long long ld) {
    if (ld % 8 != 0) return false;
    for (int i = 0; i < f.n; ++i)
        if (reinterpret_cast<uintptr_t>(f.ptr[i]) & 15) return false;
    return true;
}

}  // namespace ring
