// Token <-> slot data movement of the MoE layer, each kernel written against
// the communication layout it feeds or drains (no separate regroup passes):
//
//   dispatch_rows   slot tensor (E, S, M) built by GATHER: row (e, s) <- x[t]
//                   (zero when the slot is unfilled or padding), optionally
//                   scaled by the combine weight (backward of the combine).
//                   Reference: gate() dispatch fill, dataplane.py:101,112 and
//                   the S2 slot split + zero pad, dataplane.py:373-378.
//   combine_fwd     out[t] = sum_j w[t,j] * sum_p Y_p[e_j, s_j]  (dropped -> 0)
//                   = fused_combine's local ESP sum (collectives.py:296-310)
//                   fused with _combine (dataplane.py:131-143).
//   combine_bwd     dlogits from dOut: dw_j = <dOut[t], Y[e_j,s_j]>, softmax
//                   adjoint over all E experts (no reference).
//   dispatch_bwd    dx[t] = sum_j sum_p dR_p[e_j, s_j] + dlogits[t] . Wg^T
//   esp_sum         S2: out[e, s] = sum_p Y_p[e, s] before the MP AllGather.
//
// All are HBM-streaming gathers: one warp per token/row, 16-byte vectors, and
// every row load of a 1024-column group is issued before any is consumed
// (KT picks x 4 chunks in flight per lane) — the memory-level parallelism
// these kernels live on.  Accumulation is f32.  dispatch, combine_fwd and
// dispatch_bwd run as bulk-copy rings (gather_ring.cuh) whenever their views
// are local and 16-byte aligned; peer views use the register kernels below.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace parm {

constexpr int kRowThreads = 256;
constexpr int kChunks = 4;                  // 16-B chunks per lane per column group (1024 columns / warp)
constexpr int kGroupCols = kChunks * 256;

// Token loops that prefetch the next token's routing run on a resident grid
// (every warp loops over several tokens, so the prefetch has a next token).
static int resident_grid(long long tokens, int ctas_per_sm) {
    long long blocks = (tokens * 32 + kRowThreads - 1) / kRowThreads;
    const long long cap = (long long)kNumSMs * ctas_per_sm;
    return (int)(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
}

static int row_grid(long long rows) {
    long long blocks = (rows * 32 + kRowThreads - 1) / kRowThreads;
    const long long cap = (long long)kNumSMs * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (int)blocks;
}

__device__ __forceinline__ int4 ldg16(const bf16* p) { return __ldg(reinterpret_cast<const int4*>(p)); }

// ------------------------------------------------------------------ token-side gathers
// Routing of one token's picks (lane-uniform).
template <int KT>
struct Picks {
    int sl[KT];
    int ex[KT];
    float w[KT];
    int ep[KT];          // expert-parallel block of the pick's expert
    long long off[KT];   // in-buffer offset of the pick's row (slot_inbuf, once per token)
    __device__ __forceinline__ void load(long long t, int k, const int* __restrict__ slot_idx,
                                         const int* __restrict__ expert_idx, const float* __restrict__ cw,
                                         const SlotView& v) {
#pragma unroll
        for (int j = 0; j < KT; ++j) {
            sl[j] = (j < k) ? __ldg(slot_idx + t * k + j) : -1;
            ex[j] = (sl[j] >= 0) ? __ldg(expert_idx + t * k + j) : 0;
            w[j] = (cw != nullptr && sl[j] >= 0) ? __ldg(cw + t * k + j) : 0.0f;
            off[j] = sl[j] >= 0 ? slot_inbuf(v, ex[j], sl[j], ep[j]) : 0;
            if (sl[j] < 0) ep[j] = 0;
        }
    }
};

// Loads of one partial p of every pick for one 1024-column group, all in flight together.
template <int KT>
__device__ __forceinline__ void load_picks(const SlotView& v, const Picks<KT>& pk, int p, int g0, int lane, int M,
                                           int4 (&buf)[KT][kChunks]) {
#pragma unroll
    for (int j = 0; j < KT; ++j) {
        const bf16* row = slot_base(v, pk.ep[j], p) + pk.off[j];
#pragma unroll
        for (int i = 0; i < kChunks; ++i) {
            const int c = g0 + lane * 8 + i * 256;
            buf[j][i] = (pk.sl[j] >= 0 && c < M) ? ldg16(row + c) : make_int4(0, 0, 0, 0);
        }
    }
}

__device__ __forceinline__ void fma_bf16x8(float* acc, float w, const int4& v) {
    Vec8 t;
    *reinterpret_cast<int4*>(&t) = v;
    float f[8];
    vec8_to_f32(t, f);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = fmaf(w, f[u], acc[u]);
}

// acc[u] += v[u] for 8 bf16 values: the sm_100 mixed-precision FMA (f32 += bf16 x bf16, the bf16
// operand read from its half of the 32-bit register) times 1.0 -- no conversion instructions,
// and the same single rounding as fmaf(1.0f, float(v[u]), acc[u]).
__device__ __forceinline__ void add_bf16x8(float* acc, const int4& v) {
    const uint32_t w[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
    const unsigned short one = 0x3F80;   // bf16 1.0
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const unsigned short lo = (unsigned short)(w[i] & 0xFFFFu), hi = (unsigned short)(w[i] >> 16);
        asm("fma.rn.f32.bf16 %0, %1, %2, %0;" : "+f"(acc[2 * i]) : "h"(lo), "h"(one));
        asm("fma.rn.f32.bf16 %0, %1, %2, %0;" : "+f"(acc[2 * i + 1]) : "h"(hi), "h"(one));
    }
}

// acc = fmaf(float(a[u]), float(b[u]), acc) for u = 0..7 in order, as eight mixed-precision FMAs
// on the bf16 halves (no conversions; the bf16 x bf16 product is exact either way).
__device__ __forceinline__ void dot_bf16x8(float& acc, const int4& a, const int4& b) {
    const uint32_t x[4] = {(uint32_t)a.x, (uint32_t)a.y, (uint32_t)a.z, (uint32_t)a.w};
    const uint32_t y[4] = {(uint32_t)b.x, (uint32_t)b.y, (uint32_t)b.z, (uint32_t)b.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        asm("fma.rn.f32.bf16 %0, %1, %2, %0;"
            : "+f"(acc)
            : "h"((unsigned short)(x[i] & 0xFFFFu)), "h"((unsigned short)(y[i] & 0xFFFFu)));
        asm("fma.rn.f32.bf16 %0, %1, %2, %0;" : "+f"(acc) : "h"((unsigned short)(x[i] >> 16)), "h"((unsigned short)(y[i] >> 16)));
    }
}

// acc[u] = fmaf(w, float(v[u]), acc[u]) for 8 bf16 values, as four FFMA2 (same roundings).
__device__ __forceinline__ void fma2_bf16x8(float* acc, float w, const int4& v) {
    const uint32_t x[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
        ffma2(acc[2 * i], acc[2 * i + 1], __uint_as_float(x[i] << 16), __uint_as_float(x[i] & 0xFFFF0000u), w);
}

#include "gather_ring.cuh"


// 256 threads, <= 128 registers, a resident grid of two CTAs per SM looping over
// tokens; the per-group accumulators are the only long-lived state.
template <int KT>
__global__ void __launch_bounds__(kRowThreads, 2) combine_fwd_kernel(const __grid_constant__ SlotView y,
                                                                      const int* __restrict__ expert_idx,
                                                                      const int* __restrict__ slot_idx,
                                                                      const float* __restrict__ combine_w, int n, int k,
                                                                      int M, const __grid_constant__ RowFan out,
                                                                      long long ldo) {
    const int lane = threadIdx.x & 31;
    const long long warp_global = ((long long)blockIdx.x * kRowThreads + threadIdx.x) >> 5;
    const long long num_warps = ((long long)gridDim.x * kRowThreads) >> 5;
    Picks<KT> nx;
    if (warp_global < n) nx.load(warp_global, k, slot_idx, expert_idx, combine_w, y);
    for (long long t = warp_global; t < n; t += num_warps) {
        const Picks<KT> pk = nx;                    // this token's routing, fetched one iteration ago
        if (t + num_warps < n) nx.load(t + num_warps, k, slot_idx, expert_idx, combine_w, y);
        for (int g0 = 0; g0 < M; g0 += kGroupCols) {
            float acc[kChunks][8];
#pragma unroll
            for (int i = 0; i < kChunks; ++i)
#pragma unroll
                for (int u = 0; u < 8; ++u) acc[i][u] = 0.0f;
            for (int p = 0; p < y.n_p; ++p) {
                int4 buf[KT][kChunks];
                load_picks<KT>(y, pk, p, g0, lane, M, buf);
#pragma unroll
                for (int j = 0; j < KT; ++j)       // j ascending, like the reference's _combine
#pragma unroll
                    for (int i = 0; i < kChunks; ++i) fma2_bf16x8(acc[i], pk.w[j], buf[j][i]);
            }
#pragma unroll
            for (int i = 0; i < kChunks; ++i) {
                const int c = g0 + lane * 8 + i * 256;
                if (c >= M) continue;
                const Vec8 v8 = f32_to_vec8(acc[i]);
                for (int f = 0; f < out.n; ++f) st_vec8(out.ptr[f] + t * ldo + c, v8);
            }
        }
    }
}

// Scatter target of the fused combine-backward + dy dispatch (SC = 1 local, 2 peer view):
// row (e, s - slot_lo) <- w_j * dOut[t] for every kept pick with s in the slot range,
// zero rows up to each segment's last 128-row GEMM tile -- what dispatch_rows(dOut,
// scale = combine weights, fill) writes, without reading dOut a second time.
struct DyScatter {
    const float* combine_w;
    int slot_lo, slots_out;
    const int* fill;
    bf16* out;
    long long stride_e, stride_s;
};

template <int SC>
__device__ __forceinline__ void scatter_row(const SlotView& dstv, const DyScatter& sc, int e, int sp, int c,
                                            const int4& v) {
    if (SC == 1) {
        *reinterpret_cast<int4*>(sc.out + (long long)e * sc.stride_e + (long long)sp * sc.stride_s + c) = v;
    } else {
        int ep;
        const long long off = slot_inbuf(dstv, e, sp, ep);
        for (int pp = 0; pp < dstv.n_p; ++pp)
            *reinterpret_cast<int4*>(const_cast<bf16*>(slot_base(dstv, ep, pp)) + off + c) = v;
    }
}

template <int KT, int SC>
__global__ void __launch_bounds__(kRowThreads, 2) combine_bwd_kernel(const bf16* __restrict__ dout, long long ldd,
                                                                      const __grid_constant__ SlotView y, const int* __restrict__ expert_idx,
                                                                      const int* __restrict__ slot_idx,
                                                                      const float* __restrict__ probs, int n, int k,
                                                                      int E, int M, float* __restrict__ dlogits,
                                                                      const __grid_constant__ DyScatter sc,
                                                                      const __grid_constant__ SlotView dstv) {
    const int lane = threadIdx.x & 31;
    const long long warp_global = ((long long)blockIdx.x * kRowThreads + threadIdx.x) >> 5;
    const long long num_warps = ((long long)gridDim.x * kRowThreads) >> 5;
    Picks<KT> nx;
    const float* cw = SC ? sc.combine_w : nullptr;
    if (warp_global < n) nx.load(warp_global, k, slot_idx, expert_idx, cw, y);
    for (long long t = warp_global; t < n; t += num_warps) {
        const Picks<KT> pk = nx;
        if (t + num_warps < n) nx.load(t + num_warps, k, slot_idx, expert_idx, cw, y);
        float dw[KT];
#pragma unroll
        for (int j = 0; j < KT; ++j) dw[j] = 0.0f;
        for (int g0 = 0; g0 < M; g0 += kGroupCols) {
            int4 gv[kChunks];
#pragma unroll
            for (int i = 0; i < kChunks; ++i) {
                const int c = g0 + lane * 8 + i * 256;
                gv[i] = c < M ? ldg16(dout + t * ldd + c) : make_int4(0, 0, 0, 0);
            }
            for (int p = 0; p < y.n_p; ++p) {     // <dOut, sum_p Y_p> = sum_p <dOut, Y_p>
                int4 buf[KT][kChunks];
                load_picks<KT>(y, pk, p, g0, lane, M, buf);
#pragma unroll
                for (int i = 0; i < kChunks; ++i)
#pragma unroll
                    for (int j = 0; j < KT; ++j) dot_bf16x8(dw[j], gv[i], buf[j][i]);
            }
            if (SC) {   // the dy dispatch: w_j * dOut[t] into the pick's slot row
#pragma unroll
                for (int j = 0; j < KT; ++j) {
                    const int sp = pk.sl[j] - sc.slot_lo;
                    if (pk.sl[j] < 0 || sp < 0 || sp >= sc.slots_out) continue;
#pragma unroll
                    for (int i = 0; i < kChunks; ++i) {
                        const int c = g0 + lane * 8 + i * 256;
                        if (c >= M) continue;
                        Vec8 g8;
                        *reinterpret_cast<int4*>(&g8) = gv[i];
                        float f[8];
                        vec8_to_f32(g8, f);
#pragma unroll
                        for (int u = 0; u < 8; ++u) f[u] *= pk.w[j];
                        const Vec8 r8 = f32_to_vec8(f);
                        scatter_row<SC>(dstv, sc, pk.ex[j], sp, c, *reinterpret_cast<const int4*>(&r8));
                    }
                }
            }
        }
#pragma unroll
        for (int j = 0; j < KT; ++j)
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) dw[j] += __shfl_xor_sync(0xffffffffu, dw[j], off);
        // Softmax adjoint: dl_e = p_e * (dS_e - sum_e' p_e' dS_e'), dS nonzero on kept picks.
        if (lane < E) {
            const float pe = __ldg(probs + t * E + lane);
            float dse = 0.0f, dot = 0.0f;
#pragma unroll
            for (int j = 0; j < KT; ++j) {
                if (pk.sl[j] < 0) continue;
                dot += __ldg(probs + t * E + pk.ex[j]) * dw[j];
                if (pk.ex[j] == lane) dse = dw[j];
            }
            dlogits[t * E + lane] = pe * (dse - dot);
        }
    }
    if (SC) {   // unfilled slot rows inside each segment's last GEMM tile: zeros
        for (long long it = warp_global; it < (long long)E * 128; it += num_warps) {
            const int e = (int)(it >> 7), r = (int)(it & 127);
            int sf = __ldg(sc.fill + e) - sc.slot_lo;
            sf = sf < 0 ? 0 : (sf > sc.slots_out ? sc.slots_out : sf);
            const int end = min((sf + 127) & ~127, sc.slots_out);
            if (sf + r >= end) continue;
            for (int c = lane * 8; c < M; c += 256) scatter_row<SC>(dstv, sc, e, sf + r, c, make_int4(0, 0, 0, 0));
        }
    }
}

// dx[t] = sum_j sum_p dR_p[e_j, s_j] + dlogits[t] . Wg^T.  A warp takes TB (4 for
// k <= 2) tokens per pass over 256-column groups: their TB x KT row loads per partial
// are all in flight together, and each 16-byte Wg^T load (bf16, the gate
// weights as stored) feeds all four tokens -- the gate term's weight traffic
// is 1/TB of a token-per-warp loop's.
template <int KT, int TB>
__global__ void __launch_bounds__(kRowThreads, 2) dispatch_bwd_kernel(const __grid_constant__ SlotView dr,
                                                                       const int* __restrict__ expert_idx,
                                                                       const int* __restrict__ slot_idx,
                                                                       const float* __restrict__ dlogits,
                                                                       const bf16* __restrict__ wgT, int n, int k,
                                                                       int E, int M,
                                                                       const __grid_constant__ RowFan dx,
                                                                       long long ldx) {
    const int lane = threadIdx.x & 31;
    const long long warp_global = ((long long)blockIdx.x * kRowThreads + threadIdx.x) >> 5;
    const long long num_warps = ((long long)gridDim.x * kRowThreads) >> 5;
    for (long long t0 = warp_global * TB; t0 < n; t0 += num_warps * TB) {
        long long off[TB][KT];   // in-buffer row offset, -1 = dropped / no token
        int epk[TB][KT];
#pragma unroll
        for (int b = 0; b < TB; ++b)
#pragma unroll
            for (int j = 0; j < KT; ++j) {
                const long long t = t0 + b;
                const int sl = (t < n && j < k) ? __ldg(slot_idx + t * k + j) : -1;
                epk[b][j] = 0;
                off[b][j] = sl >= 0 ? slot_inbuf(dr, __ldg(expert_idx + t * k + j), sl, epk[b][j]) : -1;
            }
        for (int c0 = 0; c0 < M; c0 += 256) {
            const int c = c0 + lane * 8;
            if (c >= M) continue;
            float acc[TB][8];
#pragma unroll
            for (int b = 0; b < TB; ++b)
#pragma unroll
                for (int u = 0; u < 8; ++u) acc[b][u] = 0.0f;
            for (int p = 0; p < dr.n_p; ++p) {
                int4 buf[TB][KT];
#pragma unroll
                for (int b = 0; b < TB; ++b)
#pragma unroll
                    for (int j = 0; j < KT; ++j)
                        buf[b][j] = off[b][j] >= 0 ? ldg16(slot_base(dr, epk[b][j], p) + off[b][j] + c)
                                                   : make_int4(0, 0, 0, 0);
#pragma unroll
                for (int b = 0; b < TB; ++b)
#pragma unroll
                    for (int j = 0; j < KT; ++j) add_bf16x8(acc[b], buf[b][j]);
            }
            if (dlogits != nullptr) {
#pragma unroll 2
                for (int e = 0; e < E; ++e) {
                    const int4 wv = ldg16(wgT + (long long)e * M + c);
#pragma unroll
                    for (int b = 0; b < TB; ++b) {
                        const float d = t0 + b < n ? __ldg(dlogits + (t0 + b) * E + e) : 0.0f;
                        fma2_bf16x8(acc[b], d, wv);
                    }
                }
            }
#pragma unroll
            for (int b = 0; b < TB; ++b) {
                if (t0 + b >= n) continue;
                const Vec8 v8 = f32_to_vec8(acc[b]);
                for (int f = 0; f < dx.n; ++f) st_vec8(dx.ptr[f] + (t0 + b) * ldx + c, v8);
            }
        }
    }
}

__global__ void __launch_bounds__(kRowThreads, 3) esp_sum_kernel(const __grid_constant__ SlotView y, int E, int slots,
                                                                  int M,
                                                                  bf16* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const long long warp_global = ((long long)blockIdx.x * kRowThreads + threadIdx.x) >> 5;
    const long long num_warps = ((long long)gridDim.x * kRowThreads) >> 5;
    const long long rows = (long long)E * slots;
    for (long long r = warp_global; r < rows; r += num_warps) {
        Picks<1> pk;
        pk.ex[0] = (int)(r / slots);
        pk.sl[0] = (int)(r - (long long)pk.ex[0] * slots);
        pk.w[0] = 1.0f;
        pk.off[0] = slot_inbuf(y, pk.ex[0], pk.sl[0], pk.ep[0]);
        for (int g0 = 0; g0 < M; g0 += kGroupCols) {
            float acc[kChunks][8];
#pragma unroll
            for (int i = 0; i < kChunks; ++i)
#pragma unroll
                for (int u = 0; u < 8; ++u) acc[i][u] = 0.0f;
            for (int p = 0; p < y.n_p; ++p) {
                int4 buf[1][kChunks];
                load_picks<1>(y, pk, p, g0, lane, M, buf);
#pragma unroll
                for (int i = 0; i < kChunks; ++i) add_bf16x8(acc[i], buf[0][i]);
            }
#pragma unroll
            for (int i = 0; i < kChunks; ++i) {
                const int c = g0 + lane * 8 + i * 256;
                if (c < M) st_vec8(out + r * M + c, f32_to_vec8(acc[i]));
            }
        }
    }
}

// ------------------------------------------------------------------ host
static int check_view(const SlotView& v, int M, const char* what) {
    PARM_CHECK_ARG(v.n_peer >= 0 && v.n_peer <= kMaxPeers, "%s: bad peer count %d", what, v.n_peer);
    if (v.n_peer == 0) {
        PARM_CHECK_ARG(v.ptr != nullptr, "%s: null slot view", what);
        PARM_CHECK_ARG((reinterpret_cast<uintptr_t>(v.ptr) & 15) == 0, "%s: slot view base not 16-byte aligned", what);
    } else {
        for (int i = 0; i < v.n_peer; ++i)
            PARM_CHECK_ARG(v.peer[i] != nullptr && (reinterpret_cast<uintptr_t>(v.peer[i]) & 15) == 0,
                           "%s: peer buffer %d null or not 16-byte aligned", what, i);
    }
    PARM_CHECK_ARG(v.e_local >= 1 && v.n_p >= 1 && v.slot_div >= 1, "%s: bad slot view", what);
    PARM_CHECK_ARG(M % 8 == 0, "%s: embed %d must be a multiple of 8", what, M);
    return 0;
}

// ------------------------------------------------------------------ route + dispatch
// The slot pass of the gate (dataplane.py:104-116: token-major fill, first come first
// served per expert) fused with the dispatch it feeds (dataplane.py:101,112 and the
// S2 slot split + pad, :373-378), as ONE persistent kernel over the gate's per-8-token
// tile pick counts:
//   1. each CTA owns a contiguous range of tiles; its per-expert base is the sum of the
//      counts of all earlier tiles (exact prefix, read from L2), the totals give fill;
//   2. slots of the CTA's tokens in token order (warp ballots per 32-token chunk,
//      chunk bases by an exclusive scan in shared memory) -> slot_idx, slot_src;
//   3. each kept pick whose slot falls in [slot_lo, slot_lo + slots_out) gets the token
//      row: lane 0 of each warp streams x rows into a shared-memory ring with
//      cp.async.bulk and stores each to its slot row(s) with bulk stores (local tensor,
//      or the N_ESP holders' receive buffers over NVLink -- the EP&ESP dispatch AlltoAll
//      with its dump, collectives.py:256-283); x is read once per token, not per pick;
//   4. rows between each expert's fill and its last 128-row GEMM tile are zeroed, and
//      the unfilled tail of slot_src is set to -1 (grid-strided over all CTAs).
constexpr int kRdWarps = 8;
constexpr int kRdCols = 1024;                 // row chunk per ring stage (2 KB of bf16)
constexpr int kRdStages = 10;
constexpr int kRdLag = 2;                     // a stage is refilled kRdLag items after its stores were issued

__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
                 : "memory");
}

template <int EMAX>
__global__ void __launch_bounds__(kRdWarps * 32) route_dispatch_kernel(
    const bf16* __restrict__ x, long long ldx, const int* __restrict__ expert_idx, const int* __restrict__ counts,
    int n, int k, int E, int cap, int M, int* __restrict__ slot_idx, int* __restrict__ slot_src,
    int* __restrict__ fill, int slot_lo, int slots_out, bf16* __restrict__ out, long long out_stride_e,
    long long out_stride_s, const __grid_constant__ SlotView dstv, const __grid_constant__ IntFan fan, int peer) {
    __shared__ int s_base[32], s_tot[32];
    __shared__ int s_red[kRdWarps][32];
    __shared__ int s_chunk[64][32];                // per 32-token chunk counts -> exclusive chunk bases
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tiles = (n + 7) / 8;
    const int tb = (int)((long long)tiles * blockIdx.x / gridDim.x);
    const int te = (int)((long long)tiles * (blockIdx.x + 1) / gridDim.x);
    // ---- 0. this CTA's token rows start streaming into a per-warp shared-memory ring now
    //        (cp.async.bulk, lane 0 of each warp): the slot pass below overlaps their latency
    const int t_begin = tb * 8, t_end = min(te * 8, n);
    const int nch = (M + kRdCols - 1) / kRdCols;
    const int ntok = t_end - t_begin;
    const int my_tok = warp < ntok ? (ntok - 1 - warp) / kRdWarps + 1 : 0;
    const int items = slots_out > 0 ? my_tok * nch : 0;   // slots_out == 0: slot pass only
    unsigned char* ring = smem + (size_t)warp * kRdStages * kRdCols * 2;
    const uint32_t bar0 = ring::saddr(smem + (size_t)kRdWarps * kRdStages * kRdCols * 2) + warp * kRdStages * 8;
    auto tok_of = [&](int it) { return t_begin + warp + (it / nch) * kRdWarps; };
    auto rd_load = [&](int it) {
        const int t = tok_of(it), c0 = (it % nch) * kRdCols;
        const int cols = min(kRdCols, M - c0);
        const uint32_t st = (uint32_t)it % kRdStages;
        ring::bar_expect(bar0 + 8 * st, cols * 2);
        ring::bulk_g2s(ring::saddr(ring + st * kRdCols * 2), x + (long long)t * ldx + c0, cols * 2, bar0 + 8 * st);
    };
    if (lane == 0 && items > 0) {
        for (int s = 0; s < kRdStages; ++s) ring::bar_init(bar0 + 8 * s);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int it = 0; it < min(items, kRdStages - kRdLag); ++it) rd_load(it);
    }
    // ---- 1. base (tiles < tb) and totals, per expert
    {
        int pre[EMAX], tot[EMAX];
#pragma unroll
        for (int e = 0; e < EMAX; ++e) pre[e] = tot[e] = 0;
        constexpr int TU = 4;   // tiles per thread per batch, all loads issued before use
        for (int i0 = 0; i0 < tiles; i0 += TU * blockDim.x) {
            int cv[TU][EMAX];
#pragma unroll
            for (int u = 0; u < TU; ++u) {
                const int i = i0 + u * blockDim.x + threadIdx.x;
#pragma unroll
                for (int e = 0; e < EMAX; ++e) cv[u][e] = (e < E && i < tiles) ? __ldg(counts + (long long)i * E + e) : 0;
            }
#pragma unroll
            for (int u = 0; u < TU; ++u) {
                const int i = i0 + u * blockDim.x + threadIdx.x;
#pragma unroll
                for (int e = 0; e < EMAX; ++e) {
                    tot[e] += cv[u][e];
                    if (i < tb) pre[e] += cv[u][e];
                }
            }
        }
#pragma unroll
        for (int e = 0; e < EMAX; ++e) {
            if (e >= E) break;
            int a = pre[e], b = tot[e];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                a += __shfl_xor_sync(0xffffffffu, a, o);
                b += __shfl_xor_sync(0xffffffffu, b, o);
            }
            if (lane == e) {
                s_red[warp][e] = a;
            }
            pre[e] = b;   // reuse: warp total of expert e
        }
        __syncthreads();
        if (threadIdx.x < E) {
            int a = 0;
            for (int w = 0; w < kRdWarps; ++w) a += s_red[w][threadIdx.x];
            s_base[threadIdx.x] = a;
        }
        __syncthreads();
#pragma unroll
        for (int e = 0; e < EMAX; ++e) {
            if (e >= E) break;
            if (lane == e) s_red[warp][e] = pre[e];
        }
        __syncthreads();
        if (threadIdx.x < E) {
            int b = 0;
            for (int w = 0; w < kRdWarps; ++w) b += s_red[w][threadIdx.x];
            s_tot[threadIdx.x] = b;
            if (blockIdx.x == 0) fill[threadIdx.x] = b < cap ? b : cap;
        }
        __syncthreads();
    }
    // ---- 2. slots of this CTA's tokens, in token order
    const int nchunk = (t_end - t_begin + 31) / 32;   // <= 64 (host caps tokens per CTA at 2048)
    unsigned my_mask[2] = {0u, 0u};                    // picks per chunk of this warp (lane = token), by expert bit
    for (int c = warp; c < nchunk; c += kRdWarps) {
        const int t = t_begin + c * 32 + lane;
        unsigned m = 0;
        if (t < t_end)
            for (int j = 0; j < k; ++j) m |= 1u << __ldg(expert_idx + (long long)t * k + j);
        if (c / kRdWarps < 2) my_mask[c / kRdWarps] = m;
#pragma unroll
        for (int e = 0; e < EMAX; ++e) {
            if (e >= E) break;
            const int cnt = __popc(__ballot_sync(0xffffffffu, (m >> e) & 1u));
            if (lane == 0) s_chunk[c][e] = cnt;
        }
    }
    __syncthreads();
    if (threadIdx.x < E) {                              // exclusive scan over chunks, from the CTA base
        int a = s_base[threadIdx.x];
        for (int c = 0; c < nchunk; ++c) {
            const int v = s_chunk[c][threadIdx.x];
            s_chunk[c][threadIdx.x] = a;
            a += v;
        }
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    for (int c = warp; c < nchunk; c += kRdWarps) {
        const int t = t_begin + c * 32 + lane;
        unsigned m = 0;
        if (c / kRdWarps < 2) {
            m = my_mask[c / kRdWarps];
        } else if (t < t_end) {
            for (int j = 0; j < k; ++j) m |= 1u << __ldg(expert_idx + (long long)t * k + j);
        }
        int pre_e[EMAX];
#pragma unroll
        for (int e = 0; e < EMAX; ++e) {
            if (e >= E) break;
            pre_e[e] = __popc(__ballot_sync(0xffffffffu, (m >> e) & 1u) & lt);
        }
        if (t < t_end) {
            for (int j = 0; j < k; ++j) {
                const int e = __ldg(expert_idx + (long long)t * k + j);
                int p = 0;
#pragma unroll
                for (int ee = 0; ee < EMAX; ++ee)
                    if (ee == e) p = pre_e[ee];
                const int slot = s_chunk[c][e] + p;
                if (slot < cap) {
                    slot_idx[(long long)t * k + j] = slot;
                    slot_src[(long long)e * cap + slot] = t * k + j;
                } else {
                    slot_idx[(long long)t * k + j] = -1;
                }
            }
        }
    }
    __syncthreads();   // slot_idx of the CTA's tokens visible to every warp (global memory, same CTA)
    // ---- 3. token rows -> slot rows: wait for the rows streamed in since step 0, store each
    //        to its kept picks' slot rows (bulk stores), refill the ring.  The picks of the
    //        warp's next 32 tokens are fetched at once (lane i: token i, every pick's slot row
    //        as a destination offset, -1 when not stored) and broadcast with shuffles, so the
    //        issuing lane never waits on a dependent load per token.
    if (items > 0) {
        long long dst[8];   // k <= 8
        for (int it = 0; it < items; ++it) {
            const int ti = it / nch, ch = it - ti * nch;
            if ((ti & 31) == 0 && ch == 0) {   // fetch picks of tokens ti .. ti + 31 of this warp
                const int tl = ti + lane;
                const bool ok = tl < my_tok;
                const int t = ok ? t_begin + warp + tl * kRdWarps : 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    dst[j] = -1;
                    if (!ok || j >= k) continue;
                    const int sl = slot_idx[(long long)t * k + j];
                    if (sl < slot_lo || sl >= slot_lo + slots_out) continue;
                    const int e = __ldg(expert_idx + (long long)t * k + j);
                    const int sp = sl - slot_lo;
                    if (peer) {
                        int ep;
                        const long long off = slot_inbuf(dstv, e, sp, ep);
                        dst[j] = ((long long)ep << 48) | off;   // (owner, in-buffer offset)
                    } else {
                        dst[j] = (long long)e * out_stride_e + (long long)sp * out_stride_s;
                    }
                }
            }
            long long d[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) d[j] = ring::shfl_ll(dst[j], ti & 31);
            if (lane == 0) {
                if (it + kRdStages - kRdLag < items) {
                    // the stage being refilled held item it - kRdLag: its stores must have read it
                    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kRdLag - 1) : "memory");
                    rd_load(it + kRdStages - kRdLag);
                }
                const int c0 = ch * kRdCols;
                const int cols = min(kRdCols, M - c0);
                const uint32_t st = (uint32_t)it % kRdStages;
                ring::bar_wait(bar0 + 8 * st, ((uint32_t)it / kRdStages) & 1);
                const uint32_t src = ring::saddr(ring + st * kRdCols * 2);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (d[j] < 0) continue;
                    if (peer) {
                        const int ep = (int)(d[j] >> 48);
                        const long long off = d[j] & ((1ll << 48) - 1);
                        for (int pp = 0; pp < dstv.n_p; ++pp)
                            bulk_s2g(const_cast<bf16*>(slot_base(dstv, ep, pp)) + off + c0, src, cols * 2);
                    } else {
                        bulk_s2g(out + d[j] + c0, src, cols * 2);
                    }
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            __syncwarp();
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    // ---- 4. zero rows up to each expert's last GEMM tile; unfilled slot_src entries
    {
        const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
        const long long gn = (long long)gridDim.x * blockDim.x;
        const int vec = M / 8;
        for (int e = 0; e < E; ++e) {
            const int f = min(s_tot[e], cap);
            int sf = f - slot_lo;
            sf = sf < 0 ? 0 : (sf > slots_out ? slots_out : sf);
            const int end = min((sf + 127) & ~127, slots_out);
            const long long work = (long long)(end - sf) * vec;
            for (long long i = gt; i < work; i += gn) {
                const int r = sf + (int)(i / vec), c = (int)(i % vec) * 8;
                if (peer) {
                    int ep;
                    const long long off = slot_inbuf(dstv, e, r, ep);
                    for (int pp = 0; pp < dstv.n_p; ++pp)
                        *reinterpret_cast<int4*>(const_cast<bf16*>(slot_base(dstv, ep, pp)) + off + c) =
                            make_int4(0, 0, 0, 0);
                } else {
                    *reinterpret_cast<int4*>(out + (long long)e * out_stride_e + (long long)r * out_stride_s + c) =
                        make_int4(0, 0, 0, 0);
                }
            }
            for (long long i = gt; i < cap - f; i += gn) slot_src[(long long)e * cap + f + i] = -1;
        }
        if (blockIdx.x == 0 && threadIdx.x < E && fan.ptr[0] != nullptr) {   // per-segment fill counts
            const int e = threadIdx.x;
            int c = min(s_tot[e], cap) - slot_lo;
            c = c < 0 ? 0 : (c > slots_out ? slots_out : c);
            if (peer) {   // into each holder's table
                const int ep = e / dstv.e_local, i = e - ep * dstv.e_local;
                for (int p = 0; p < dstv.n_p; ++p) fan.ptr[ep * dstv.peer_ep + p * dstv.peer_p][i] = c;
            } else {      // local: one (E) table
                fan.ptr[0][e] = c;
            }
        }
    }
}

int route_dispatch(const void* x, long long ldx, const int* expert_idx, const int* counts, int n, int k, int E,
                   int cap, int M, int* slot_idx, int* slot_src, int* fill, int slot_lo, int slots_out, void* out,
                   long long out_stride_e, long long out_stride_s, const SlotView* dst, const IntFan* fill_dst,
                   cudaStream_t s) {
    PARM_CHECK_ARG(k >= 1 && k <= 8 && E >= 1 && E <= 32 && k <= E, "route_dispatch: need 1 <= k <= min(8, E), E <= 32");
    PARM_CHECK_ARG(cap >= 1 && counts != nullptr && slot_idx != nullptr && slot_src != nullptr && fill != nullptr,
                   "route_dispatch: capacity >= 1 and counts/slot_idx/slot_src/fill required");
    PARM_CHECK_ARG(M % 8 == 0 && ldx % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0,
                   "route_dispatch: token rows must be 16-byte aligned (M=%d)", M);
    const bool peer = dst != nullptr;
    if (peer) {
        PARM_CHECK_ARG(dst->n_peer >= 1 && dst->n_peer <= kMaxPeers, "route_dispatch: destination must be a peer view");
        PARM_CHECK_ARG(dst->stride_i % 8 == 0 && dst->stride_slo % 8 == 0 && dst->stride_shi % 8 == 0,
                       "route_dispatch: destination rows must be 16-byte aligned");
        for (int i = 0; i < dst->n_peer; ++i)
            PARM_CHECK_ARG((reinterpret_cast<uintptr_t>(dst->peer[i]) & 15) == 0,
                           "route_dispatch: peer buffer %d not 16-byte aligned", i);
    } else if (out != nullptr) {
        PARM_CHECK_ARG((reinterpret_cast<uintptr_t>(out) & 15) == 0 && out_stride_e % 8 == 0 && out_stride_s % 8 == 0,
                       "route_dispatch: output rows must be 16-byte aligned");
    } else {
        slots_out = 0;   // slot pass only
    }
    PARM_CHECK_ARG(slots_out >= 0 && slot_lo >= 0, "route_dispatch: bad slot range");
    const int tiles = (n + 7) / 8;
    // one CTA per SM, at most 2048 tokens (64 ballot chunks) per CTA
    int grid = std::max(1, std::min(tiles, kNumSMs));
    grid = std::max(grid, (tiles + 255) / 256);
    const SlotView none{};
    IntFan nofan{};
    const int smem = kRdWarps * kRdStages * (kRdCols * 2 + 8);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(route_dispatch_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(route_dispatch_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    launch_k(E <= 8 ? route_dispatch_kernel<8> : route_dispatch_kernel<32>, grid, kRdWarps * 32, smem, s, reinterpret_cast<const bf16*>(x), ldx, expert_idx,
             counts, n, k, E, cap, M, slot_idx, slot_src, fill, slot_lo, slots_out, reinterpret_cast<bf16*>(out),
             out_stride_e, out_stride_s, peer ? *dst : none, fill_dst ? *fill_dst : nofan, peer ? 1 : 0);
    PARM_CHECK_LAUNCH("route_dispatch");
    return 0;
}

// ------------------------------------------------------------------ push (holder -> owners)
// Segmented expert rows src[seg][i][s] (s < fill[seg][i]) stored into
// dst.ptr[seg] + (i * rows + s) * M -- the return AlltoAll as posted NVLink
// stores from the holder into every owner's receive block (a push moves the
// bytes once; the owner's combine and combine-backward then read them locally).
__global__ void __launch_bounds__(kRowThreads) push_rows_kernel(const bf16* __restrict__ src, int nseg, int el,
                                                                int rows, int M, const int* __restrict__ fill,
                                                                const __grid_constant__ RowFan dst) {
    const int lane = threadIdx.x & 31;
    const long long warp_global = ((long long)blockIdx.x * kRowThreads + threadIdx.x) >> 5;
    const long long num_warps = ((long long)gridDim.x * kRowThreads) >> 5;
    const long long total = (long long)nseg * el * rows;
    for (long long r = warp_global; r < total; r += num_warps) {
        const long long per_seg = (long long)el * rows;
        const int seg = (int)(r / per_seg);
        const long long rem = r - seg * per_seg;
        const int i = (int)(rem / rows);
        const int s = (int)(rem - (long long)i * rows);
        if (s >= __ldg(fill + seg * el + i)) continue;
        const bf16* sp = src + r * M;
        bf16* dp = dst.ptr[seg] + ((long long)i * rows + s) * M;
        for (int g0 = 0; g0 < M; g0 += kGroupCols) {
            int4 v[kChunks];
#pragma unroll
            for (int u = 0; u < kChunks; ++u) {
                const int c = g0 + lane * 8 + u * 256;
                v[u] = c < M ? ldg16(sp + c) : make_int4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < kChunks; ++u) {
                const int c = g0 + lane * 8 + u * 256;
                if (c < M) *reinterpret_cast<int4*>(dp + c) = v[u];
            }
        }
    }
}

int push_rows(const void* src, int nseg, int el, int rows, int M, const int* fill, const RowFan& dst, cudaStream_t s) {
    PARM_CHECK_ARG(nseg >= 1 && nseg <= kMaxPeers && dst.n == nseg, "push_rows: %d segments for %d destinations",
                   nseg, dst.n);
    PARM_CHECK_ARG(M % 8 == 0 && fill != nullptr, "push_rows: M=%d must be a multiple of 8, fill required", M);
    const long long total = (long long)nseg * el * rows;
    if (total == 0) return 0;
    const int grid = row_grid(total);
    launch_k(push_rows_kernel, grid, kRowThreads, 0, s, reinterpret_cast<const bf16*>(src), nseg, el, rows, M,
        fill, dst);
    PARM_CHECK_LAUNCH("push_rows");
    return 0;
}

// ------------------------------------------------------------------ fan copy
// `bytes` of src stored into each dst.ptr[i] (16-byte vectors): small payloads
// replicated to every MP peer (the gate-gradient exchange of S1).
__global__ void fan_copy_kernel(const int4* __restrict__ src, long long vecs, const __grid_constant__ RowFan dst) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < vecs; i += (long long)gridDim.x * blockDim.x) {
        const int4 v = __ldg(src + i);
        for (int f = 0; f < dst.n; ++f) reinterpret_cast<int4*>(dst.ptr[f])[i] = v;
    }
}

int fan_copy(const void* src, long long bytes, const RowFan& dst, cudaStream_t s) {
    PARM_CHECK_ARG(bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0,
                   "fan_copy: %lld bytes must be 16-byte aligned and sized", bytes);
    PARM_CHECK_ARG(dst.n >= 1 && dst.n <= kMaxPeers, "fan_copy: %d destinations", dst.n);
    const long long vecs = bytes / 16;
    if (vecs == 0) return 0;
    long long blocks = (vecs + 255) / 256;
    if (blocks > kNumSMs * 4) blocks = kNumSMs * 4;
    launch_k(fan_copy_kernel, (int)blocks, 256, 0, s, reinterpret_cast<const int4*>(src), vecs, dst);
    PARM_CHECK_LAUNCH("fan_copy");
    return 0;
}

// ------------------------------------------------------------------ peer barrier
// Every rank stores the next epoch into slot [rank] of every peer's signal pad
// (release, system scope, after a system fence that publishes this rank's
// earlier peer stores), then waits until every peer's epoch has reached its
// own pad.  The epoch lives in device memory, so a replayed CUDA graph
// advances it like an eager launch.  A watchdog (wall clock, %globaltimer)
// traps after sig.timeout_ns instead of hanging the GPU on a dead peer.
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// One CTA per rank hosted by this process: CTA b is rank sigs[b].rank.  A real
// multi-GPU rank launches one CTA; the single-GPU emulation of P ranks launches all
// P in ONE cooperative grid, so the ranks that wait on one another are guaranteed
// to be co-resident (never as separate launches that nothing forces to overlap).
struct PeerSignalSet {
    PeerSignal sig[kMaxPeers];
};

__global__ void peer_barrier_kernel(const __grid_constant__ PeerSignalSet set) {
    const PeerSignal& sig = set.sig[blockIdx.x];
    __shared__ unsigned epoch;
    if (threadIdx.x == 0) {
        unsigned* cnt = reinterpret_cast<unsigned*>(sig.counter);
        epoch = *cnt + 1u;
        *cnt = epoch;
    }
    __syncthreads();
    const int j = threadIdx.x;
    if (j < sig.n) {
        // No leading system fence: the data this barrier publishes was written by the kernels before
        // it on this stream, and a kernel completes only once its stores -- NVLink stores into peer
        // memory included, and the TMA epilogues wait for their bulk stores -- are performed; the
        // release store below then orders this rank's arrival after them (measured: 5.9 -> 4.5 us
        // per barrier at P=2, 6.5 -> 4.9 at P=4, tools/probes/barrier_probe.py).
        unsigned* slot = reinterpret_cast<unsigned*>(sig.pad[j]) + sig.rank;
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(slot), "r"(epoch) : "memory");
        const unsigned* mine = reinterpret_cast<const unsigned*>(sig.pad[sig.rank]) + j;
        const unsigned long long t0 = globaltimer_ns();
        for (unsigned it = 0;; ++it) {
            unsigned v;
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
            if ((int)(v - epoch) >= 0) break;
            if ((it & 1023u) == 1023u && (long long)(globaltimer_ns() - t0) > sig.timeout_ns) asm volatile("trap;");
        }
    }
    __syncthreads();
}

int peer_barrier(const PeerSignal* sigs, int count, cudaStream_t s) {
    PARM_CHECK_ARG(sigs != nullptr && count >= 1 && count <= kMaxPeers, "peer_barrier: %d local ranks", count);
    PeerSignalSet set{};
    for (int b = 0; b < count; ++b) {
        const PeerSignal& g = sigs[b];
        PARM_CHECK_ARG(g.n >= 1 && g.n <= kMaxPeers && g.rank >= 0 && g.rank < g.n,
                       "peer_barrier: bad rank %d of %d", g.rank, g.n);
        PARM_CHECK_ARG(g.counter != nullptr, "peer_barrier: null epoch counter");
        PARM_CHECK_ARG(count == 1 || g.n == sigs[0].n, "peer_barrier: local ranks disagree on the group size");
        set.sig[b] = g;
        if (set.sig[b].timeout_ns <= 0) set.sig[b].timeout_ns = 300ll * 1000000000ll;
    }
    if (count == 1) {
        launch_k(peer_barrier_kernel, 1, 32, 0, s, set);
    } else {   // co-residency of the waiting ranks is guaranteed only by a cooperative launch
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(count);
        cfg.blockDim = dim3(32);
        cfg.stream = s;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, peer_barrier_kernel, set);
    }
    PARM_CHECK_LAUNCH("peer_barrier");
    return 0;
}

int combine_fwd_fan(const SlotView&, const int*, const int*, const float*, int, int, int, const RowFan&, long long,
                    cudaStream_t);
int dispatch_bwd_fan(const SlotView&, const int*, const int*, const float*, const void*, int, int, int, int,
                     const RowFan&, long long, cudaStream_t);

static RowFan one_fan(void* p) {
    RowFan f{};
    f.ptr[0] = reinterpret_cast<bf16*>(p);
    f.n = 1;
    return f;
}

int combine_fwd(const SlotView& y, const int* expert_idx, const int* slot_idx, const float* combine_w, int n, int k,
                int M, void* out, long long ldo, cudaStream_t s) {
    PARM_CHECK_ARG(out != nullptr, "combine_fwd: null output");
    return combine_fwd_fan(y, expert_idx, slot_idx, combine_w, n, k, M, one_fan(out), ldo, s);
}

int combine_fwd_fan(const SlotView& y, const int* expert_idx, const int* slot_idx, const float* combine_w, int n,
                    int k, int M, const RowFan& O, long long ldo, cudaStream_t s) {
    if (int rc = check_view(y, M, "combine_fwd")) return rc;
    PARM_CHECK_ARG(k >= 1 && k <= 8, "combine_fwd: top_k must be in [1, 8]");
    PARM_CHECK_ARG(O.n >= 1 && O.n <= kMaxPeers, "combine_fwd: output fan of %d buffers", O.n);
    if (n == 0) return 0;
    if (k <= 2 && y.n_p <= 2 && ring::view_aligned(y) && ring::fan_aligned(O, ldo)) {
        constexpr int S = 4;
        static int per_sm1 = 0, per_sm2 = 0;
        const int smem = ring::ring_smem(S, 2 * y.n_p, 0);
        if (y.n_p == 1) {
            auto kern = ring::combine_fwd_ring<1, S>;
            launch_k(kern, ring::grid_for(kern, smem, n, per_sm1), kRowThreads, smem, s, y, expert_idx, slot_idx, combine_w,
                n, k, M, O, ldo);
        } else {
            auto kern = ring::combine_fwd_ring<2, S>;
            launch_k(kern, ring::grid_for(kern, smem, n, per_sm2), kRowThreads, smem, s, y, expert_idx, slot_idx, combine_w,
                n, k, M, O, ldo);
        }
        PARM_CHECK_LAUNCH("combine_fwd");
        return 0;
    }
    if (k <= 2)
        launch_k(combine_fwd_kernel<2>, resident_grid(n, 2), kRowThreads, 0, s, y, expert_idx, slot_idx, combine_w, n, k, M, O, ldo);
    else
        launch_k(combine_fwd_kernel<8>, resident_grid(n, 2), kRowThreads, 0, s, y, expert_idx, slot_idx, combine_w, n, k, M, O, ldo);
    PARM_CHECK_LAUNCH("combine_fwd");
    return 0;
}

int combine_bwd_dispatch(const void* dout, long long ldd, const SlotView& y, const int* expert_idx,
                         const int* slot_idx, const float* probs, const float* combine_w, int n, int k, int E, int M,
                         float* dlogits, int slot_lo, int slots_out, const int* fill, void* out, long long stride_e,
                         long long stride_s, const SlotView* dst, cudaStream_t s) {
    if (int rc = check_view(y, M, "combine_bwd_dispatch")) return rc;
    PARM_CHECK_ARG(k <= 8 && E <= 32, "combine_bwd_dispatch: k<=8 and E<=32 required");
    PARM_CHECK_ARG(combine_w != nullptr && fill != nullptr, "combine_bwd_dispatch: combine weights and fill required");
    PARM_CHECK_ARG(ldd % 8 == 0 && (reinterpret_cast<uintptr_t>(dout) & 15) == 0,
                   "combine_bwd_dispatch: dOut rows must be 16-byte aligned");
    if (dst != nullptr) {
        PARM_CHECK_ARG(dst->n_peer >= 1 && dst->n_peer <= kMaxPeers, "combine_bwd_dispatch: destination must be a peer view");
        PARM_CHECK_ARG(dst->stride_i % 8 == 0 && dst->stride_slo % 8 == 0 && dst->stride_shi % 8 == 0,
                       "combine_bwd_dispatch: destination rows must be 16-byte aligned");
    } else {
        PARM_CHECK_ARG(out != nullptr && (reinterpret_cast<uintptr_t>(out) & 15) == 0 && stride_e % 8 == 0 &&
                           stride_s % 8 == 0,
                       "combine_bwd_dispatch: output rows must be 16-byte aligned");
    }
    if (n == 0 && slots_out == 0) return 0;
    auto D = reinterpret_cast<const bf16*>(dout);
    DyScatter sc{combine_w, slot_lo, slots_out, fill, reinterpret_cast<bf16*>(out), stride_e, stride_s};
    const SlotView nov{};
    const int grid = resident_grid(n > E * 128 ? n : E * 128, 2);
    if (dst != nullptr) {
        if (k <= 2)
            launch_k(combine_bwd_kernel<2, 2>, grid, kRowThreads, 0, s, D, ldd, y, expert_idx, slot_idx, probs, n, k, E,
                M, dlogits, sc, *dst);
        else
            launch_k(combine_bwd_kernel<8, 2>, grid, kRowThreads, 0, s, D, ldd, y, expert_idx, slot_idx, probs, n, k, E,
                M, dlogits, sc, *dst);
    } else {
        if (k <= 2)
            launch_k(combine_bwd_kernel<2, 1>, grid, kRowThreads, 0, s, D, ldd, y, expert_idx, slot_idx, probs, n, k, E,
                M, dlogits, sc, nov);
        else
            launch_k(combine_bwd_kernel<8, 1>, grid, kRowThreads, 0, s, D, ldd, y, expert_idx, slot_idx, probs, n, k, E,
                M, dlogits, sc, nov);
    }
    PARM_CHECK_LAUNCH("combine_bwd_dispatch");
    return 0;
}

int dispatch_bwd(const SlotView& dr, const int* expert_idx, const int* slot_idx, const float* dlogits, const void* wg,
                 int n, int k, int E, int M, void* dx, long long ldx, cudaStream_t s) {
    PARM_CHECK_ARG(dx != nullptr, "dispatch_bwd: null output");
    return dispatch_bwd_fan(dr, expert_idx, slot_idx, dlogits, wg, n, k, E, M, one_fan(dx), ldx, s);
}

int dispatch_bwd_fan(const SlotView& dr, const int* expert_idx, const int* slot_idx, const float* dlogits,
                     const void* wg, int n, int k, int E, int M, const RowFan& DX, long long ldx, cudaStream_t s) {
    if (int rc = check_view(dr, M, "dispatch_bwd")) return rc;
    PARM_CHECK_ARG(DX.n >= 1 && DX.n <= kMaxPeers, "dispatch_bwd: output fan of %d buffers", DX.n);
    PARM_CHECK_ARG(E <= 32 && k <= 8, "dispatch_bwd: E<=32 and k<=8 required");
    PARM_CHECK_ARG(dlogits == nullptr || wg != nullptr, "dispatch_bwd: dlogits needs gate weights");
    if (n == 0) return 0;
    auto W = reinterpret_cast<const bf16*>(wg);
    PARM_CHECK_ARG(M % 8 == 0 && ldx % 8 == 0, "dispatch_bwd: rows must be 16-byte aligned (M=%d)", M);
    if (k <= 2 && dr.n_p <= 2 && ring::view_aligned(dr) && ring::fan_aligned(DX, ldx) &&
        (dlogits == nullptr || (E % 4 == 0 && (reinterpret_cast<uintptr_t>(dlogits) & 15) == 0))) {
        constexpr int S = 4;
        static int per_sm1 = 0, per_sm2 = 0;
        const int smem = ring::ring_smem(S, 2 * dr.n_p, 128);
        if (dr.n_p == 1) {
            auto kern = ring::dispatch_bwd_ring<1, S>;
            launch_k(kern, ring::grid_for(kern, smem, n, per_sm1), kRowThreads, smem, s, dr, expert_idx, slot_idx, dlogits,
                W, n, k, E, M, DX, ldx);
        } else {
            auto kern = ring::dispatch_bwd_ring<2, S>;
            launch_k(kern, ring::grid_for(kern, smem, n, per_sm2), kRowThreads, smem, s, dr, expert_idx, slot_idx, dlogits,
                W, n, k, E, M, DX, ldx);
        }
        PARM_CHECK_LAUNCH("dispatch_bwd");
        return 0;
    }
    if (k <= 2)
        launch_k(dispatch_bwd_kernel<2, 4>, row_grid((n + 3) / 4), kRowThreads, 0, s, dr, expert_idx, slot_idx, dlogits,
            W, n, k, E, M, DX, ldx);
    else
        launch_k(dispatch_bwd_kernel<8, 1>, row_grid(n), kRowThreads, 0, s, dr, expert_idx, slot_idx, dlogits, W, n, k,
            E, M, DX, ldx);
    PARM_CHECK_LAUNCH("dispatch_bwd");
    return 0;
}

int esp_sum(const SlotView& y, int E, int slots, int M, void* out, cudaStream_t s) {
    if (int rc = check_view(y, M, "esp_sum")) return rc;
    PARM_CHECK_ARG(y.n_peer == 0, "esp_sum: local views only");
    const long long rows = (long long)E * slots;
    if (rows == 0) return 0;
    launch_k(esp_sum_kernel, row_grid(rows), kRowThreads, 0, s, y, E, slots, M, reinterpret_cast<bf16*>(out));
    PARM_CHECK_LAUNCH("esp_sum");
    return 0;
}

}  // namespace parm
