// Fused gate: logits -> softmax -> stable top-k -> token-major capacity slots,
// plus the gate's backward (softmax adjoint and the Wg weight gradient).
//
// Reference semantics (moesched dataplane.py:80-119):
//   scores  = softmax(X @ Wg)                       (f64)
//   ranked  = argsort(-scores, stable)[:, :k]       ties -> lower expert index
//   weights = scores[ranked]                        (raw probabilities, no renorm)
//   slots   : for t ascending, j ascending: e = ranked[t, j];
//             slot = fill[e]++ if fill[e] < capacity else dropped
//
// Routing (expert_index, slot_index) is integer work and must be bit-exact.
// Logits are therefore accumulated in f64 from the same bf16 inputs the oracle
// sees (every bf16 x bf16 product is exact in f64, so only the summation order
// differs from the oracle's BLAS f64 dot); softmax and ranking run in f64.
// The slot pass is an exact per-expert exclusive prefix count over tokens.
//
// Gate weights live on the device TRANSPOSED, wgT (E, M), so a lane's 8
// consecutive columns of one expert are one 16-byte load.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace parm {

constexpr int kGateThreads = 128;
constexpr int kGateChunks = 4;   // 16-B x chunks per lane per 1024-column group

// Warp-level reduce-scatter of 32 doubles: on return v[0] of lane L holds the
// warp-wide sum of input index L.  31 double shuffles instead of 5 x 32.
__device__ __forceinline__ double reduce_scatter32(double (&v)[32], int lane) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const double send = upper ? v[i] : v[i + o];
            const double keep = upper ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0];
}

// One warp handles TPW = 32 / EMAX tokens; every x load of a 1024-column group
// of all TPW tokens is issued before the f64 FMAs (memory-level parallelism),
// and each Wg^T vector is reused across the TPW tokens.  After the
// reduce-scatter lane L = q * EMAX + e owns (token t0 + q, expert e): softmax
// max/sum over the EMAX-lane group by shuffles, one exp and one divide per
// lane, stable rank against the group's other lanes.
template <int EMAX>
__global__ void __launch_bounds__(kGateThreads) gate_fwd_kernel(const bf16* __restrict__ x, long long ldx,
                                                                 const double* __restrict__ wgT, int n, int M, int E,
                                                                 int k, int* __restrict__ expert_idx,
                                                                 float* __restrict__ combine_w,
                                                                 float* __restrict__ probs) {
    pdl_entry();
    constexpr int TPW = 32 / EMAX;
    const int lane = threadIdx.x & 31;
    const int warp_global = (blockIdx.x * kGateThreads + threadIdx.x) >> 5;
    const int num_warps = (gridDim.x * kGateThreads) >> 5;
    for (int t0 = warp_global * TPW; t0 < n; t0 += num_warps * TPW) {
        double v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.0;
        for (int g0 = 0; g0 < M; g0 += kGateChunks * 256) {
            int4 xb[TPW][kGateChunks];
#pragma unroll
            for (int q = 0; q < TPW; ++q)
#pragma unroll
                for (int i = 0; i < kGateChunks; ++i) {
                    const int c = g0 + lane * 8 + i * 256;
                    xb[q][i] = (t0 + q < n && c < M)
                                   ? __ldg(reinterpret_cast<const int4*>(x + (long long)(t0 + q) * ldx + c))
                                   : make_int4(0, 0, 0, 0);
                }
#pragma unroll
            for (int i = 0; i < kGateChunks; ++i) {
                const int c = g0 + lane * 8 + i * 256;
                if (c >= M) break;
                float xv[TPW][8];
#pragma unroll
                for (int q = 0; q < TPW; ++q) {
                    Vec8 t8;
                    *reinterpret_cast<int4*>(&t8) = xb[q][i];
                    vec8_to_f32(t8, xv[q]);
                }
#pragma unroll
                for (int u = 0; u < 8; u += 2) {
                    double xd[TPW][2];
#pragma unroll
                    for (int q = 0; q < TPW; ++q) {
                        xd[q][0] = (double)xv[q][u];
                        xd[q][1] = (double)xv[q][u + 1];
                    }
#pragma unroll
                    for (int e = 0; e < EMAX; ++e) {
                        if (e < E) {   // Wg^T held as exact f64 upcasts: no per-element conversion here
                            const double2 w = __ldg(reinterpret_cast<const double2*>(wgT + (long long)e * M + c + u));
#pragma unroll
                            for (int q = 0; q < TPW; ++q) {
                                v[q * EMAX + e] = fma(xd[q][0], w.x, v[q * EMAX + e]);
                                v[q * EMAX + e] = fma(xd[q][1], w.y, v[q * EMAX + e]);
                            }
                        }
                    }
                }
            }
        }
        const double logit = reduce_scatter32(v, lane);
        const int q = lane / EMAX;
        const int e = lane - q * EMAX;
        const int t = t0 + q;
        const bool valid = (e < E);
        double mx = valid ? logit : -INFINITY;
#pragma unroll
        for (int o = 1; o < EMAX; o <<= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const double ex = valid ? exp(logit - mx) : 0.0;
        double sum = ex;
#pragma unroll
        for (int o = 1; o < EMAX; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        const double score = ex / sum;
        int rank = 0;
        const int base = q * EMAX;
#pragma unroll
        for (int i = 0; i < EMAX; ++i) {
            const double other = __shfl_sync(0xffffffffu, score, base + i);
            rank += (i < E) && ((other > score) || (other == score && i < e));
        }
        if (valid && t < n) {
            if (rank < k) {
                expert_idx[(long long)t * k + rank] = e;
                combine_w[(long long)t * k + rank] = (float)score;
            }
            if (probs) probs[(long long)t * E + e] = (float)score;
        }
    }
}

// FP64 tensor-core gate (DMMA, mma.m8n8k4.f64) for M % 128 == 0.  A block of
// four warps owns 8 tokens; warp w and quad lane q own the contiguous column
// range [(4w + q) * M/16, ...) of all 8 tokens, so every lane streams its own
// x and Wg^T segments with 16-byte loads.  The MMA's k index is the quad lane,
// mapped to a lane-dependent column -- the same mapping for the A (x) and B
// (Wg^T) fragments, which is all a dot product needs.  One DMMA = 8 tokens x 8
// experts x 4 columns of exact-product f64 FMAs; the four warps' partial
// logits are summed in a fixed order in shared memory, then warp 0 runs the
// softmax and the stable top-k for its 8 tokens (token g on quad g).
constexpr int kDmmaWarps = 4;

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Softmax + stable top-k of one token's logits held by a lane quad: lane
// (g, q) owns experts nt * 8 + 2q + h of token t (the DMMA C-fragment layout).
template <int NT>
__device__ __forceinline__ void gate_topk_epilogue(double (&lg)[NT][2], int g, int q, int t, bool tok, int E, int k,
                                                   int* __restrict__ expert_idx, float* __restrict__ combine_w,
                                                   float* __restrict__ probs) {
    double sc[NT][2];
    double mx = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            sc[nt][h] = lg[nt][h];
            if (nt * 8 + 2 * q + h < E) mx = fmax(mx, sc[nt][h]);
        }
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    double sum = 0.0;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            sc[nt][h] = (nt * 8 + 2 * q + h < E) ? exp(sc[nt][h] - mx) : 0.0;
            sum += sc[nt][h];
        }
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    int rank[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            sc[nt][h] = sc[nt][h] / sum;
            rank[nt][h] = 0;
        }
#pragma unroll
    for (int qq = 0; qq < 4; ++qq)
#pragma unroll
        for (int nt2 = 0; nt2 < NT; ++nt2)
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                const double other = __shfl_sync(0xffffffffu, sc[nt2][h2], (g << 2) | qq);
                const int e2 = nt2 * 8 + 2 * qq + h2;
                if (e2 >= E) continue;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int e = nt * 8 + 2 * q + h;
                        rank[nt][h] += (other > sc[nt][h]) || (other == sc[nt][h] && e2 < e);
                    }
            }
    if (tok) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int e = nt * 8 + 2 * q + h;
                if (e >= E) continue;
                if (rank[nt][h] < k) {
                    expert_idx[(long long)t * k + rank[nt][h]] = e;
                    combine_w[(long long)t * k + rank[nt][h]] = (float)sc[nt][h];
                }
                if (probs) probs[(long long)t * E + e] = (float)sc[nt][h];
            }
    }
}

template <int NT>   // n-tiles of 8 experts (E <= 8 NT)
__global__ void __launch_bounds__(kDmmaWarps * 32) gate_fwd_dmma_kernel(
    const bf16* __restrict__ x, long long ldx, const double* __restrict__ wgT, int n, int M, int E, int k,
    int* __restrict__ expert_idx, float* __restrict__ combine_w, float* __restrict__ probs) {
    pdl_entry();
    __shared__ double red[kDmmaWarps][NT][64];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, q = lane & 3;
    const int span = M / (4 * kDmmaWarps);
    const int col0 = (warp * 4 + q) * span;
    const double* wr[NT];
    bool wok[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        const int e = nt * 8 + g;
        wok[nt] = e < E;
        wr[nt] = wgT + (long long)(wok[nt] ? e : 0) * M + col0;
    }
    for (int t0 = blockIdx.x * 8; t0 < n; t0 += gridDim.x * 8) {
        const int t = t0 + g;
        const bool tok = t < n;
        const bf16* xr = x + (long long)(tok ? t : 0) * ldx + col0;
        double acc[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
        for (int j = 0; j < span; j += 8) {
            const int4 xv = tok ? __ldg(reinterpret_cast<const int4*>(xr + j)) : make_int4(0, 0, 0, 0);
            double2 wv[NT][4];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    wv[nt][i] = wok[nt] ? __ldg(reinterpret_cast<const double2*>(wr[nt] + j) + i) : make_double2(0, 0);
            Vec8 x8;
            *reinterpret_cast<int4*>(&x8) = xv;
            float xf[8];
            vec8_to_f32(x8, xf);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const double a = (double)xf[u];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
                    dmma884(acc[nt][0], acc[nt][1], a, (u & 1) ? wv[nt][u >> 1].y : wv[nt][u >> 1].x);
            }
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            red[warp][nt][g * 8 + 2 * q] = acc[nt][0];
            red[warp][nt][g * 8 + 2 * q + 1] = acc[nt][1];
        }
        __syncthreads();
        if (warp == 0) {
            double lg[NT][2];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int idx = g * 8 + 2 * q + h;
                    double s = red[0][nt][idx];
#pragma unroll
                    for (int w = 1; w < kDmmaWarps; ++w) s += red[w][nt][idx];
                    lg[nt][h] = s;
                }
            gate_topk_epilogue<NT>(lg, g, q, t, tok, E, k, expert_idx, combine_w, probs);
        }
        __syncthreads();
    }
}

// Same DMMA formulation with Wg^T staged once per CTA in shared memory (f64,
// E x M padded so the 32 lanes' B-fragment reads hit distinct bank pairs) and
// one 8-token tile per warp: lane quad q owns the column quarter [qM/4, ...),
// so a tile's whole reduction stays inside one warp (no cross-warp sum) and the
// only global traffic is the x rows.  Used when the padded Wg^T fits in shared
// memory; x chunks of 64 columns are loaded together ahead of their DMMAs.
__device__ __forceinline__ int4 ldg_v4_ordered(const void* p) {
    int4 r;
    asm volatile("ld.global.nc.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

constexpr int kGateSmemWarps = 8;


__host__ __device__ constexpr long long gate_smem_stride(int M) { return M + 33; }   // doubles per expert row

template <int NT>
__global__ void __launch_bounds__(kGateSmemWarps * 32) gate_fwd_dmma_smem_kernel(
    const bf16* __restrict__ x, long long ldx, const double* __restrict__ wgT, int n, int M, int E, int k,
    int* __restrict__ expert_idx, float* __restrict__ combine_w, float* __restrict__ probs) {
    pdl_entry();
    extern __shared__ double sw[];
    const int Q = M / 4;
    const long long stride = gate_smem_stride(M);
    // stage Wg^T: 8 double2 loads in flight per thread per batch (M even: a pair never straddles rows/quarters)
    const int pairs = NT * 8 * M / 2;
    for (int b0 = 0; b0 < pairs; b0 += 8 * blockDim.x) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = b0 + u * blockDim.x + threadIdx.x;
            const int e = (2 * i) / M;
            v[u] = (i < pairs && e < E) ? __ldg(reinterpret_cast<const double2*>(wgT) + i) : make_double2(0, 0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = b0 + u * blockDim.x + threadIdx.x;
            if (i >= pairs) break;
            const int e = (2 * i) / M, c = 2 * i - e * M;
            double* d = sw + e * stride + c + (c / Q) * 8;
            d[0] = v[u].x;
            d[1] = v[u].y;
        }
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, q = lane & 3;
    const double* wrow[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) wrow[nt] = sw + (nt * 8 + g) * stride + (long long)q * (Q + 8);
    const int tiles = (n + 7) / 8;
    const int wpc = blockDim.x >> 5;   // warps per CTA (host-chosen so the CTAs cover the SMs evenly)
    for (int tile = blockIdx.x * wpc + warp; tile < tiles; tile += gridDim.x * wpc) {
        const int t = tile * 8 + g;
        const bool tok = t < n;
        const bf16* xr = x + (long long)(tok ? t : 0) * ldx + (long long)q * Q;
        double acc[2][NT][2];
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) acc[c][nt][0] = acc[c][nt][1] = 0.0;
        int4 nxt[8];                            // chunk j0 + 64 is in flight while chunk j0 is consumed
#pragma unroll
        for (int i = 0; i < 8; ++i) nxt[i] = ldg_v4_ordered(xr + (8 * i < Q ? 8 * i : 0));
        for (int j0 = 0; j0 < Q; j0 += 64) {
            int4 xv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) xv[i] = nxt[i];
            if (j0 + 64 < Q) {
#pragma unroll
                for (int i = 0; i < 8; ++i) nxt[i] = ldg_v4_ordered(xr + (j0 + 64 + 8 * i < Q ? j0 + 64 + 8 * i : 0));
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (j0 + 8 * i >= Q) break;
                Vec8 x8;
                *reinterpret_cast<int4*>(&x8) = tok ? xv[i] : make_int4(0, 0, 0, 0);
                float xf[8];
                vec8_to_f32(x8, xf);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int c = j0 + 8 * i + u;
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt)
                        dmma884(acc[u & 1][nt][0], acc[u & 1][nt][1], (double)xf[u], wrow[nt][c]);
                }
            }
        }
        double lg[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            lg[nt][0] = acc[0][nt][0] + acc[1][nt][0];
            lg[nt][1] = acc[0][nt][1] + acc[1][nt][1];
        }
        gate_topk_epilogue<NT>(lg, g, q, t, tok, E, k, expert_idx, combine_w, probs);
    }
}

// Exclusive per-expert prefix count over tokens -> slots, exact, in two
// parallel passes over 256-token chunks (one CTA each):
//   slot_count  per-chunk per-expert pick counts (+ slot_src := -1)
//   slot_assign chunk base = sum of earlier chunks' counts, then ballot
//               prefixes within the chunk in token order.
constexpr int kSlotChunk = 256;
constexpr int kSlotWarps = kSlotChunk / 32;

__device__ __forceinline__ unsigned pick_mask(const int* __restrict__ expert_idx, int t, int n, int k, int (&ex)[8]) {
    unsigned m = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        ex[j] = (t < n && j < k) ? __ldg(expert_idx + (long long)t * k + j) : -1;
        if (ex[j] >= 0) m |= 1u << ex[j];
    }
    return m;
}

template <int EMAX>
__global__ void __launch_bounds__(kSlotChunk) slot_count_kernel(const int* __restrict__ expert_idx, int n, int k,
                                                                 int E, int cap, int* __restrict__ chunk_cnt,
                                                                 int* __restrict__ slot_src) {
    pdl_entry();
    __shared__ int wc[kSlotWarps][EMAX];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long tot = (long long)E * cap;
    for (long long i = (long long)blockIdx.x * kSlotChunk + threadIdx.x; i < tot; i += (long long)gridDim.x * kSlotChunk)
        slot_src[i] = -1;
    int ex[8];
    const unsigned m = pick_mask(expert_idx, blockIdx.x * kSlotChunk + threadIdx.x, n, k, ex);
#pragma unroll
    for (int e = 0; e < EMAX; ++e) {
        const int c = __popc(__ballot_sync(0xffffffffu, (m >> e) & 1u));
        if (lane == 0) wc[warp][e] = c;
    }
    __syncthreads();
    if (threadIdx.x < E) {
        int s = 0;
#pragma unroll
        for (int w = 0; w < kSlotWarps; ++w) s += wc[w][threadIdx.x];
        chunk_cnt[blockIdx.x * E + threadIdx.x] = s;
    }
}

template <int EMAX>
__global__ void __launch_bounds__(kSlotChunk) slot_assign_kernel(const int* __restrict__ expert_idx, int n, int k,
                                                                  int E, int cap, const int* __restrict__ chunk_cnt,
                                                                  int* __restrict__ slot_idx,
                                                                  int* __restrict__ slot_src, int* __restrict__ fill) {
    pdl_entry();
    __shared__ int base[EMAX];
    __shared__ int wc[kSlotWarps][EMAX];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c = blockIdx.x;
    if (threadIdx.x < E) {
        int s = 0;
        for (int cc = 0; cc < c; ++cc) s += __ldg(chunk_cnt + cc * E + threadIdx.x);
        base[threadIdx.x] = s;
        if (c == gridDim.x - 1) {
            const int total = s + __ldg(chunk_cnt + c * E + threadIdx.x);
            fill[threadIdx.x] = total < cap ? total : cap;
        }
    }
    const int t = c * kSlotChunk + threadIdx.x;
    int ex[8];
    const unsigned m = pick_mask(expert_idx, t, n, k, ex);
    const unsigned lt = (1u << lane) - 1u;
    int pre[EMAX];
#pragma unroll
    for (int e = 0; e < EMAX; ++e) {
        const unsigned b = __ballot_sync(0xffffffffu, (m >> e) & 1u);
        pre[e] = __popc(b & lt);
        if (lane == 0) wc[warp][e] = __popc(b);
    }
    __syncthreads();
    if (threadIdx.x < E) {   // exclusive scan over warps, per expert
        int s = base[threadIdx.x];
#pragma unroll
        for (int w = 0; w < kSlotWarps; ++w) {
            const int v = wc[w][threadIdx.x];
            wc[w][threadIdx.x] = s;
            s += v;
        }
    }
    __syncthreads();
    if (t < n) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (j >= k) break;
            const int e = ex[j];
            int p = 0;
#pragma unroll
            for (int ee = 0; ee < EMAX; ++ee)
                if (ee == e) p = pre[ee];
            const int slot = wc[warp][e] + p;
            if (slot < cap) {
                slot_idx[(long long)t * k + j] = slot;
                slot_src[(long long)e * cap + slot] = t * k + j;
            } else {
                slot_idx[(long long)t * k + j] = -1;
            }
        }
    }
}

// dWg^T partials: part[c][e][m] = sum_{t in chunk c} dlogits[t][e] * x[t][m].
// 512 threads = 4 token sub-groups x 128 lanes of 8 columns; 16-B loads, four
// tokens in flight per thread; sub-groups reduced through shared memory.
constexpr int kWgCols = 256;             // 32 column lanes x 8 columns per CTA
constexpr int kWgSub = 4;
constexpr int kWgChunks = 64;
constexpr int kWgThreads = kWgCols / 8 * kWgSub;

template <int EMAX>
__global__ void __launch_bounds__(kWgCols / 8 * kWgSub) gate_wgrad_partial_kernel(const bf16* __restrict__ x, long long ldx,
                                                                  const float* __restrict__ dlogits, int n, int M,
                                                                  int E, int chunk, float* __restrict__ part) {
    pdl_entry();
    __shared__ float red[8][kWgCols / 8][8 + 1];     // one 8-expert block of one sub-group at a time
    const int col_lane = threadIdx.x % (kWgCols / 8);
    const int sub = threadIdx.x / (kWgCols / 8);
    const int c = blockIdx.x * kWgCols + col_lane * 8;
    const int t_begin = blockIdx.y * chunk;
    const int t_end = min(n, t_begin + chunk);
    float acc[EMAX][8];
#pragma unroll
    for (int e = 0; e < EMAX; ++e)
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[e][u] = 0.0f;
    if (c < M) {
        for (int t = t_begin + sub; t < t_end; t += 4 * kWgSub) {
            int4 xv[4];
            float dl[4][EMAX];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int tt = t + q * kWgSub;
                xv[q] = tt < t_end ? __ldg(reinterpret_cast<const int4*>(x + (long long)tt * ldx + c))
                                   : make_int4(0, 0, 0, 0);
#pragma unroll
                for (int e = 0; e < EMAX; ++e) dl[q][e] = (tt < t_end && e < E) ? __ldg(dlogits + (long long)tt * E + e) : 0.f;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                Vec8 t8;
                *reinterpret_cast<int4*>(&t8) = xv[q];
                float f[8];
                vec8_to_f32(t8, f);
#pragma unroll
                for (int e = 0; e < EMAX; ++e)
#pragma unroll
                    for (int u = 0; u < 8; ++u) acc[e][u] = fmaf(dl[q][e], f[u], acc[e][u]);
            }
        }
    }
    // Sub-groups fold into shared memory one after another (deterministic order), 8 experts at a time.
#pragma unroll
    for (int eb = 0; eb < EMAX; eb += 8) {
        for (int g = 0; g < kWgSub; ++g) {
            if (sub == g) {
#pragma unroll
                for (int e = 0; e < 8; ++e)
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        red[e][col_lane][u] = (g == 0 ? 0.0f : red[e][col_lane][u]) + acc[eb + e][u];
            }
            __syncthreads();
        }
        if (sub == 0 && c < M) {
            for (int e = 0; e < 8 && eb + e < E; ++e) {
                float* dst = part + ((long long)blockIdx.y * E + eb + e) * M + c;
                reinterpret_cast<float4*>(dst)[0] =
                    make_float4(red[e][col_lane][0], red[e][col_lane][1], red[e][col_lane][2], red[e][col_lane][3]);
                reinterpret_cast<float4*>(dst)[1] =
                    make_float4(red[e][col_lane][4], red[e][col_lane][5], red[e][col_lane][6], red[e][col_lane][7]);
            }
        }
        __syncthreads();
    }
}

// out[i] (+)= sum_c part[c][i]: a CTA owns 32 consecutive outputs; warp w sums
// chunks w, w + 8, ... with all its loads in flight, then the eight warp sums
// are added in a fixed order (deterministic).
__global__ void __launch_bounds__(256) sum_partials_kernel(const float* __restrict__ part, int chunks, long long len,
                                                           float* __restrict__ out, int accumulate) {
    pdl_entry();
    __shared__ float ws[8][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long i = (long long)blockIdx.x * 32 + lane;
    float s = 0.0f;
    if (i < len) {
        float v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int c = warp + 8 * r;
            v[r] = c < chunks ? __ldg(part + (long long)c * len + i) : 0.0f;
        }
        for (int c = warp + 64; c < chunks; c += 8) s += __ldg(part + (long long)c * len + i);
#pragma unroll
        for (int r = 0; r < 8; ++r) s += v[r];
    }
    ws[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && i < len) {
        float tot = ws[0][lane];
#pragma unroll
        for (int w = 1; w < 8; ++w) tot += ws[w][lane];
        out[i] = accumulate ? out[i] + tot : tot;
    }
}

// ------------------------------------------------------------------ host
template <int EMAX>
static void launch_gate_fwd(const bf16* x, long long ldx, const double* wgT, int n, int M, int E, int k, int* ei,
                            float* cw, float* probs, cudaStream_t s) {
    constexpr int TPW = 32 / EMAX;
    const int warps_needed = (n + TPW - 1) / TPW;
    int blocks = (warps_needed * 32 + kGateThreads - 1) / kGateThreads;
    const int max_blocks = kNumSMs * 16;
    if (blocks > max_blocks) blocks = max_blocks;
    if (blocks < 1) blocks = 1;
    launch_k(gate_fwd_kernel<EMAX>, blocks, kGateThreads, 0, s, x, ldx, wgT, n, M, E, k, ei, cw, probs);
}

// PARM_GATE_DMMA=0 selects the FP64-FMA gate kernel (A/B comparisons).
static bool gate_dmma_enabled() {
    static int mode = -1;
    if (mode < 0) {
        const char* e = getenv("PARM_GATE_DMMA");
        mode = (e && e[0] == '0') ? 0 : 1;
    }
    return mode == 1;
}

int gate_fwd(const void* x, long long ldx, const void* wgT, int n, int M, int E, int k, int* expert_idx,
             float* combine_w, float* probs, cudaStream_t s) {
    PARM_CHECK_ARG(k >= 1 && k <= E, "top_k (%d) exceeds number of experts (%d)", k, E);
    PARM_CHECK_ARG(E <= 32, "gate: at most 32 experts supported (got %d)", E);
    PARM_CHECK_ARG(M % 8 == 0 && ldx % 8 == 0, "gate: embed (%d) and row stride must be multiples of 8", M);
    if (n == 0) return 0;
    auto X = reinterpret_cast<const bf16*>(x);
    auto W = reinterpret_cast<const double*>(wgT);
    const int nt_need = (E + 7) / 8;
    const size_t smem_bytes = (size_t)(nt_need <= 2 ? nt_need : 4) * 8 * gate_smem_stride(M) * sizeof(double);
    if (M % 64 == 0 && nt_need <= 2 && smem_bytes <= 200 * 1024 && gate_dmma_enabled()) {
        const int tiles = (n + 7) / 8;
        // warps per CTA (one 8-token tile each): the fewest tiles on the busiest SM, e.g. 7 warps x 147
        // CTAs for 8192 tokens instead of 8 x 128 (20 SMs idle); one CTA per SM holds the Wg^T copy
        int wpc = kGateSmemWarps;
        long long best = -1;
        for (int w = kGateSmemWarps; w >= 4; --w) {
            const long long ctas = (tiles + w - 1) / w;
            const long long load = (ctas + kNumSMs - 1) / kNumSMs * w;
            if (best < 0 || load < best) {
                best = load;
                wpc = w;
            }
        }
        const int blocks = (int)std::min<long long>((tiles + wpc - 1) / wpc, kNumSMs * 2);
        if (nt_need == 1) {
            cudaFuncSetAttribute(gate_fwd_dmma_smem_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem_bytes);
            launch_k(gate_fwd_dmma_smem_kernel<1>, blocks, wpc * 32, smem_bytes, s, X, ldx, W, n, M, E, k,
                expert_idx, combine_w, probs);
        } else {
            cudaFuncSetAttribute(gate_fwd_dmma_smem_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem_bytes);
            launch_k(gate_fwd_dmma_smem_kernel<2>, blocks, wpc * 32, smem_bytes, s, X, ldx, W, n, M, E, k,
                expert_idx, combine_w, probs);
        }
    } else if (M % (16 * kDmmaWarps * 2) == 0 && gate_dmma_enabled()) {   // span per lane a multiple of 8
        const int blocks = (int)std::min<long long>((n + 7) / 8, (long long)kNumSMs * 64);
        if (E <= 8)
            launch_k(gate_fwd_dmma_kernel<1>, blocks, kDmmaWarps * 32, 0, s, X, ldx, W, n, M, E, k, expert_idx, combine_w,
                probs);
        else if (E <= 16)
            launch_k(gate_fwd_dmma_kernel<2>, blocks, kDmmaWarps * 32, 0, s, X, ldx, W, n, M, E, k, expert_idx, combine_w,
                probs);
        else
            launch_k(gate_fwd_dmma_kernel<4>, blocks, kDmmaWarps * 32, 0, s, X, ldx, W, n, M, E, k, expert_idx, combine_w,
                probs);
    } else if (E <= 2)
        launch_gate_fwd<2>(X, ldx, W, n, M, E, k, expert_idx, combine_w, probs, s);
    else if (E <= 4)
        launch_gate_fwd<4>(X, ldx, W, n, M, E, k, expert_idx, combine_w, probs, s);
    else if (E <= 8)
        launch_gate_fwd<8>(X, ldx, W, n, M, E, k, expert_idx, combine_w, probs, s);
    else if (E <= 16)
        launch_gate_fwd<16>(X, ldx, W, n, M, E, k, expert_idx, combine_w, probs, s);
    else
        launch_gate_fwd<32>(X, ldx, W, n, M, E, k, expert_idx, combine_w, probs, s);
    PARM_CHECK_LAUNCH("gate_fwd");
    return 0;
}

size_t gate_slots_workspace(int n, int E) {
    return (size_t)((n + kSlotChunk - 1) / kSlotChunk) * E * sizeof(int);
}

int gate_slots(const int* expert_idx, int n, int k, int E, int cap, int* slot_idx, int* slot_src, int* fill,
               int* ws, size_t ws_bytes, cudaStream_t s) {
    PARM_CHECK_ARG(k >= 1 && k <= 8, "gate_slots: top_k must be in [1, 8] (got %d)", k);
    PARM_CHECK_ARG(E >= 1 && E <= 32, "gate_slots: experts must be in [1, 32]");
    PARM_CHECK_ARG(cap >= 1, "gate_slots: capacity must be >= 1");
    PARM_CHECK_ARG(ws_bytes >= gate_slots_workspace(n, E), "gate_slots: workspace too small");
    const int chunks = n > 0 ? (n + kSlotChunk - 1) / kSlotChunk : 1;
    if (E <= 8) {
        launch_k(slot_count_kernel<8>, chunks, kSlotChunk, 0, s, expert_idx, n, k, E, cap, ws, slot_src);
        launch_k(slot_assign_kernel<8>, chunks, kSlotChunk, 0, s, expert_idx, n, k, E, cap, ws, slot_idx, slot_src, fill);
    } else {
        launch_k(slot_count_kernel<32>, chunks, kSlotChunk, 0, s, expert_idx, n, k, E, cap, ws, slot_src);
        launch_k(slot_assign_kernel<32>, chunks, kSlotChunk, 0, s, expert_idx, n, k, E, cap, ws, slot_idx, slot_src, fill);
    }
    PARM_CHECK_LAUNCH("gate_slots");
    return 0;
}

size_t gate_wgrad_workspace(int n, int M, int E) {
    return (size_t)kWgChunks * M * E * sizeof(float);
}

int gate_wgrad(const void* x, long long ldx, const float* dlogits, int n, int M, int E, float* ws, size_t ws_bytes,
               float* dwgT, int accumulate, cudaStream_t s) {
    PARM_CHECK_ARG(E <= 32, "gate_wgrad: at most 32 experts supported");
    PARM_CHECK_ARG(M % 8 == 0 && ldx % 8 == 0, "gate_wgrad: embed must be a multiple of 8");
    PARM_CHECK_ARG(ws_bytes >= gate_wgrad_workspace(n, M, E), "gate_wgrad: workspace too small");
    const int chunk = (n + kWgChunks - 1) / kWgChunks;
    dim3 grid((M + kWgCols - 1) / kWgCols, kWgChunks);
    auto X = reinterpret_cast<const bf16*>(x);
    if (E <= 8)
        launch_k(gate_wgrad_partial_kernel<8>, grid, kWgThreads, 0, s, X, ldx, dlogits, n, M, E, chunk, ws);
    else if (E <= 16)
        launch_k(gate_wgrad_partial_kernel<16>, grid, kWgThreads, 0, s, X, ldx, dlogits, n, M, E, chunk, ws);
    else
        launch_k(gate_wgrad_partial_kernel<32>, grid, kWgThreads, 0, s, X, ldx, dlogits, n, M, E, chunk, ws);
    PARM_CHECK_LAUNCH("gate_wgrad_partial");
    const long long len = (long long)M * E;
    launch_k(sum_partials_kernel, (int)((len + 31) / 32), 256, 0, s, ws, kWgChunks, len, dwgT, accumulate);
    PARM_CHECK_LAUNCH("gate_wgrad_sum");
    return 0;
}

}  // namespace parm
